"""Multi-rank row-band partition (config 4's 2/4/8-GPU layout) on CPU: gloo,
world_size 2 and 3.

The orchestration in paper_1710_07745_b200.bands.distributed_band_canny --
halo exchange with batch_isend_irecv, band-edge export, all_gather of edge
rows, the host seam union-find (ef_band_merge from the C-ABI library), and
finalisation -- runs for real; only the per-band pixel compute is an
oracle-backed stand-in for the CUDA band backend (there is no GPU here).  The
assembled result must equal the oracle on the whole frame.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleBandBackend:
    """Band compute with the oracle: labels from the haloed buffer, band-local
    8-connected components (scipy), component ids exported for the edge rows."""

    def __init__(self, rows, width):
        self.rows, self.width = rows, width

    def classify_trace(self, buf, row0, full_height, weights, low, high):
        from scipy import ndimage

        r = (len(weights) - 1) // 2
        halo = r + 2
        ht = min(halo, row0)
        lab_buf, _ = O.canny(buf.numpy(), weights, low, high)
        lab = lab_buf[ht:ht + self.rows]
        self.labels = torch.from_numpy(np.ascontiguousarray(lab))
        comp, n = ndimage.label(lab != 0, structure=np.ones((3, 3), int))
        strong = np.zeros(n + 1, np.uint8)
        strong[np.unique(comp[lab == 2])] = 1
        strong[0] = 0
        self.comp, self.cstrong = comp, strong

    def edges(self):
        ids = np.concatenate([self.comp[0], self.comp[-1]]).astype(np.int64) - 1  # background -> -1
        st = self.cstrong[ids + 1]
        st[ids < 0] = 0
        return torch.from_numpy(ids), torch.from_numpy(st)

    def finalize(self, strong_edges):
        se = strong_edges.numpy()
        ids = np.concatenate([self.comp[0], self.comp[-1]])
        merged = self.cstrong.copy()
        merged[ids[se.astype(bool)]] = 1
        merged[0] = 0
        return torch.from_numpy(merged[self.comp])


class OracleBandBackendWithMerge(OracleBandBackend):
    """Takes distributed_band_canny's device-path branch (gather band-local
    edge rows, backend.merge) with the host union-find standing in for
    ef_band_merge_device."""

    def merge(self, ids_all, strong_all):
        from paper_1710_07745_b200 import bands

        nb = ids_all.shape[0]
        gids = np.stack([bands.globalize_ids(ids_all[k].numpy(), k) for k in range(nb)])
        return torch.from_numpy(bands.merge_edges(gids, strong_all.numpy(), self.width))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, frame, weights, low, high, out, with_merge=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_07745_b200 import bands

        plan = bands.band_plan(frame.shape[0], world)
        s, e = plan[rank]
        staged = None
        if with_merge:  # the in-place halo buffer (bench.py's layout)
            staged, band = bands.band_buffer(e - s, frame.shape[1], s, frame.shape[0], (len(weights) - 1) // 2)
            band.copy_(torch.from_numpy(np.ascontiguousarray(frame[s:e])))
        else:
            band = torch.from_numpy(np.ascontiguousarray(frame[s:e]))
        lab, fin = bands.distributed_band_canny(band, s, frame.shape[0], weights, low, high, staged=staged,
                                                backend=(OracleBandBackendWithMerge if with_merge else
                                                         OracleBandBackend)(e - s, frame.shape[1]))
        out[rank] = (s, e, lab.numpy().copy(), fin.numpy().astype(np.uint8).copy())
    finally:
        dist.destroy_process_group()


def _snake_frame(h, w):
    """A bright zig-zag stroke crossing every band seam many times."""
    img = np.full((h, w), 40, np.uint8)
    for y in range(4, h - 4, 10):
        img[y:y + 3, 4:w - 4] = 200
        x = (w - 8) if (y // 10) % 2 == 0 else 4
        img[y:y + 13, x:x + 3] = 200
    return img


@pytest.mark.parametrize("world,with_merge", [(2, False), (3, False), (3, True)])
def test_distributed_band_canny_gloo(world, with_merge):
    from paper_1710_07745_b200 import synth

    frames = [synth.config4(256, tile=64), _snake_frame(97, 80)]
    weights = O.gaussian_weights(1.4, radius=2)
    for frame in frames:
        manager = mp.Manager()
        out = manager.dict()
        port = _free_port()
        mp.spawn(_worker, args=(world, port, frame, weights, 20.0, 50.0, out, with_merge), nprocs=world, join=True)
        el, ef_ = O.canny(frame, weights, 20.0, 50.0)
        lab = np.zeros_like(el)
        fin = np.zeros_like(el)
        for rank in range(world):
            s, e, l, f = out[rank]
            lab[s:e], fin[s:e] = l, f
        assert np.array_equal(lab, el)
        assert np.array_equal(fin.astype(bool), ef_)
