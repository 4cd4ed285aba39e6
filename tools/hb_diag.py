"""Whole-frame hysteresis A/B (bit sweeps vs tile union-find) on the configs:
device time per fused ef_canny_u8 call (CUDA events), walks, fix-ups."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1710_07745_b200 import canny, synth  # noqa: E402
from paper_1710_07745_b200.filtering import build_gaussian_kernel  # noqa: E402

w = build_gaussian_kernel(1.4, radius=2).weights
cases = {"C0": synth.make_config(0), "C1": synth.config1(64), "C3x256": synth.config3(256)}
for name, arr in cases.items():
    frames = torch.from_numpy(arr).cuda()
    low, high = (15.0, 45.0) if name == "C2" else (20.0, 50.0)
    ws = canny.new_workspace(*frames.shape)
    lab = torch.empty_like(frames)
    fin = torch.empty_like(frames)
    for mode in ("sweep", "unionfind"):
        canny.set_hysteresis_mode(mode)
        for _ in range(3):
            canny.canny_u8(frames, w, low, high, lab, fin, ws=ws)
        torch.cuda.synchronize()
        canny.reset_stats(ws)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            canny.canny_u8(frames, w, low, high, lab, fin, ws=ws)
        b.record()
        torch.cuda.synchronize()
        st = canny.read_stats(ws)
        print(f"{name:7s} {mode:9s} {a.elapsed_time(b) / 10:.4f} ms/call  walks={canny.read_paths(ws)['hb_rounds']} "
              f"fixups/call={st['fixups'] // 10}", flush=True)
canny.set_hysteresis_mode("sweep")
