"""Row bands with the halo rows read in place from the neighbours' HBM
(ef_band_canny_u8_peer + CUDA IPC mappings), the multi-GPU C4 path without a
halo exchange step.

The ranks are separate processes that share one GPU here (gpurun gives one
B200): each maps its neighbours' band buffers over CUDA IPC exactly as it would
map another GPU's (where the loads then travel over NVLink), and the group is
gloo (NCCL refuses two ranks on one device).  The steps are ordered on the
device by interprocess CUDA events (bands.distributed_band_canny): a rank's
stream waits for its neighbours' "band written" events before its classifier
reads their rows, and for their "halo rows read" events before its next work;
the host never synchronises a stream (no kernel spins on another's progress).
The assembled result must equal the whole-frame call bit for bit, also when
every rank enqueues a new frame into its band right after each call returns
(the write-after-read hazard), and when one rank's stream runs far behind the
others.  Negative control: with EF_TEST_PEER_NO_WAIT=1 (the event waits
dropped) the delayed cases must fail (tools/gpu_peer.sh runs it).
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


def _worker(rank, world, port, frames, plan, weights, low, high, steps, out, delay_rank=-1):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if os.environ.get("EF_TEST_PEER_NO_WAIT"):  # negative control only: drop the event waits (must then fail)
        torch.cuda.Stream.wait_event = lambda self, event: None
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_07745_b200 import bands

        s, e = plan[rank]
        h, w = frames[0].shape
        src = torch.from_numpy(np.ascontiguousarray(np.stack([f[s:e] for f in frames]))).cuda()
        band = torch.empty((e - s, w), dtype=torch.uint8, device="cuda")
        be = bands.CudaBandBackend(e - s, w)
        res = []
        for step in range(steps):  # a new frame every call, written on this rank's stream
            if rank == delay_rank:  # this rank's stream runs ~20 ms behind its neighbours' every step
                torch.cuda._sleep(40_000_000)
            band.copy_(src[step % len(frames)])
            lab, fin = bands.distributed_band_canny(band, s, h, weights, low, high, backend=be, peer=True)
            res.append((lab.clone(), fin.clone()))  # stream-ordered snapshot, no host sync
        torch.cuda.synchronize()
        out[rank] = [(a.cpu().numpy().copy(), b.cpu().numpy().copy()) for a, b in res]
        dist.barrier()  # nobody unmaps a band another rank may still be reading
        be.close_peers()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,radius,delay_rank", [(2, 2, -1), (3, 2, -1), (3, 5, -1), (2, 2, 0), (2, 2, 1),
                                                     (3, 2, 1)])
def test_peer_halo_bands_match_whole_frame(world, radius, delay_rank):
    """delay_rank: that rank's stream sleeps before each write, so without the
    event ordering its neighbours would read its rows before they are written
    (delay 0) or write their next frame while it still reads theirs (delay 1)."""
    import torch.multiprocessing as mp

    from paper_1710_07745_b200 import bands, canny, synth
    from paper_1710_07745_b200.filtering import build_gaussian_kernel

    frames = [synth.config4(1024, seed=4 + k, tile=256) for k in range(3)]
    w = build_gaussian_kernel(1.4, radius=radius).weights
    plan = bands.band_plan(1024, world) if world != 3 else [(0, 300), (300, 701), (701, 1024)]
    want = []
    for f in frames:
        lab, fin = canny.canny_u8(torch.from_numpy(f).cuda(), w, 20.0, 50.0)
        want.append((lab.cpu().numpy()[0], fin.cpu().numpy()[0]))
    manager = mp.Manager()
    out = manager.dict()
    steps = 5
    mp.spawn(_worker, args=(world, _free_port(), frames, plan, w, 20.0, 50.0, steps, out, delay_rank), nprocs=world,
             join=True)
    for rank, (s, e) in enumerate(plan):
        for step in range(steps):
            bl, bf = out[rank][step]
            lab, fin = want[step % len(frames)]
            assert np.array_equal(bl, lab[s:e]), (rank, step)
            assert np.array_equal(bf, fin[s:e]), (rank, step)


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
