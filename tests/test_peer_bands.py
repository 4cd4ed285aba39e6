"""Row bands with the halo rows read in place from the neighbours' HBM
(ef_band_canny_u8_peer + CUDA IPC mappings), the multi-GPU C4 path without a
halo exchange step.

The ranks are separate processes that share one GPU here (gpurun gives one
B200): each maps its neighbours' band buffers over CUDA IPC exactly as it would
map another GPU's (where the loads then travel over NVLink), and the group is
gloo (NCCL refuses two ranks on one device).  No rank's kernel waits on another
rank's kernel: bands are written, the group synchronises, then every rank reads.
The assembled result must equal the whole-frame call bit for bit.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, frame, plan, weights, low, high, steps, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_07745_b200 import bands

        s, e = plan[rank]
        band = torch.from_numpy(np.ascontiguousarray(frame[s:e])).cuda()
        be = bands.CudaBandBackend(e - s, frame.shape[1])
        for _ in range(steps):  # repeated calls reuse the mappings
            lab, fin = bands.distributed_band_canny(band, s, frame.shape[0], weights, low, high, backend=be,
                                                    peer=True)
        torch.cuda.synchronize()
        out[rank] = (lab.cpu().numpy().copy(), fin.cpu().numpy().copy())
        dist.barrier()  # nobody unmaps a band another rank may still be reading
        be.close_peers()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,radius", [(2, 2), (3, 2), (3, 5)])
def test_peer_halo_bands_match_whole_frame(world, radius):
    import torch.multiprocessing as mp

    from paper_1710_07745_b200 import bands, canny, synth
    from paper_1710_07745_b200.filtering import build_gaussian_kernel

    frame = synth.config4(1024, tile=256)
    w = build_gaussian_kernel(1.4, radius=radius).weights
    plan = bands.band_plan(frame.shape[0], world) if world != 3 else [(0, 300), (300, 701), (701, 1024)]
    lab, fin = canny.canny_u8(torch.from_numpy(frame).cuda(), w, 20.0, 50.0)
    lab, fin = lab.cpu().numpy()[0], fin.cpu().numpy()[0]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), frame, plan, w, 20.0, 50.0, 2, out), nprocs=world, join=True)
    for rank, (s, e) in enumerate(plan):
        bl, bf = out[rank]
        assert np.array_equal(bl, lab[s:e]), rank
        assert np.array_equal(bf, fin[s:e]), rank


def test_peer_abi_validation():
    from paper_1710_07745_b200 import _lib, canny

    canny.require_cuda()
    lib = _lib.load()
    band = torch.zeros((64, 128), dtype=torch.uint8, device="cuda")
    lab, fin = torch.empty_like(band), torch.empty_like(band)
    ws = canny.new_workspace(1, 64, 128)
    _, wp, r = canny.host_weights(np.array([0.25, 0.5, 0.25]))
    # band rows 100..163 of a 300-row frame need 3 halo rows each side: none given
    rc = lib.ef_band_canny_u8_peer(band.data_ptr(), None, 0, None, 0, 100, 64, 300, 128, wp, r, 20.0, 50.0,
                                   lab.data_ptr(), fin.data_ptr(), ws.data_ptr(), ws.numel(), None)
    assert rc == _lib.EF_EINVAL
    assert b"halo" in _lib.load().ef_last_error()
