"""bench.py's multi-GPU batch path on CPU: the fixed C1/C3 batch is sharded
N ways by frame index (BASELINE configs[3] "sharded evenly over 1/2/4/8
GPUs"; engine.py:46-95 / SPEC.md:133 determinism: any partition gives the
same output).  gloo, world_size 2; the per-frame compute is the oracle (the
CUDA kernel's CPU checker) since there is no GPU here.  Also checks that
`bench.py --gpus 2` re-launches itself as 2 ranks."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_partition_the_batch():
    for n in (1, 7, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            parts = [bench.shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def _rank(rank, world, port, nframes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames, name, low, high, total = bench.workload(3, nframes, rank, world)
        w = O.gaussian_weights(1.4, radius=2)
        lab, fin = O.canny(frames, w, low, high, threads=2)
        lo, hi = bench.shard(total, rank, world)
        assert frames.shape[0] == hi - lo
        pad = -(-total // world)
        buf = np.zeros((pad, *frames.shape[1:]), np.uint8)
        buf[: len(frames)] = lab + fin.astype(np.uint8) * 4
        got = [torch.empty(buf.shape, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(got, torch.from_numpy(buf))
        cnt = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(cnt, torch.tensor([len(frames)]))
        if rank == 0:
            q.put(np.concatenate([g.numpy()[: int(c)] for g, c in zip(got, cnt)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_c3_batch_equals_whole_batch(world):
    nframes = 5  # uneven split: 2 + 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, nframes, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1710_07745_b200 import synth

    full = synth.config3(nframes)
    lab, fin = O.canny(full, O.gaussian_weights(1.4, radius=2), 20.0, 50.0, threads=4)
    assert np.array_equal(merged, lab + fin.astype(np.uint8) * 4)


def test_bench_gpus_flag_relaunches_ranks():
    """`python bench.py --gpus 2` without torchrun becomes 2 ranks; rank 0 alone
    prints the line (here the CPU reference arm, which needs no GPU)."""
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--frames", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [json.loads(x) for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    assert lines[0]["config"]["workload"].startswith("C3: 2 x")
