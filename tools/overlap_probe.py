"""Probe: does running sub-batches of the fused pipeline on concurrent streams
beat one call over the whole batch?  (Latency-bound hysteresis kernels of one
sub-batch could fill the SMs beside the compute-bound classifier of another.)

    python tools/overlap_probe.py [--frames 64] [--splits 1 2 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1710_07745_b200 import _lib, canny, synth
from paper_1710_07745_b200.filtering import build_gaussian_kernel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--splits", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    frames = synth.config1(a.frames)
    dev = torch.device("cuda", 0)
    low, high = synth.CONFIG_THRESHOLDS[1]
    w = build_gaussian_kernel(1.4, radius=2).weights
    _, wp, r = canny.host_weights(w)
    lib = _lib.load()
    b, h, wd = frames.shape
    srcs = [torch.from_numpy(np.roll(frames, k, axis=0).copy()).to(dev) for k in range(3)]
    labels = torch.empty_like(srcs[0])
    final = torch.empty_like(srcs[0])
    for n in a.splits:
        sub = b // n
        streams = [torch.cuda.Stream() for _ in range(n)]
        wss = [canny.new_workspace(sub, h, wd, device=dev) for _ in range(n)]

        def step(i, concurrent):
            src = srcs[i % 3]
            main = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(main)
            for k in range(n):
                s = streams[k] if concurrent else main
                if concurrent:
                    s.wait_event(ev)
                sl = slice(k * sub, (k + 1) * sub)
                rc = lib.ef_canny_u8(src[sl].data_ptr(), sub, h, wd, wp, r, float(low), float(high),
                                     labels[sl].data_ptr(), final[sl].data_ptr(), wss[k].data_ptr(),
                                     wss[k].numel(), int(s.cuda_stream))
                _lib.check(rc, "canny")
            if concurrent:
                for s in streams:
                    e = torch.cuda.Event()
                    e.record(s)
                    main.wait_event(e)

        for concurrent in ([False, True] if n > 1 else [False]):
            for i in range(5):
                step(i, concurrent)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for i in range(a.reps):
                step(i, concurrent)
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / a.reps
            print(f"splits={n} concurrent={concurrent}: {ms:.4f} ms/step  {b * h * wd / ms / 1e3:.0f} MP/s", flush=True)


if __name__ == "__main__":
    main()
