"""Tail of the host-buffer entry's call times on C3 (1 GiB per call): N calls, the
slowest five and how many exceed 1.5x the median.   python tools/e2e_outliers.py [N]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_07745_b200 import canny, synth
from paper_1710_07745_b200.filtering import build_gaussian_kernel

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
frames = synth.config_range(3, 0, 1024)
b, h, wd = frames.shape
w = build_gaussian_kernel(1.4, radius=2).weights
hsrc = torch.from_numpy(frames).pin_memory()
hlab = torch.empty_like(hsrc).pin_memory(); hfin = torch.empty_like(hsrc).pin_memory()
t = []
for i in range(n + 3):
    t0 = time.perf_counter()
    canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, 20.0, 50.0, hlab.data_ptr(), hfin.data_ptr(), 0)
    if i >= 3:
        t.append((time.perf_counter() - t0) * 1e3)
t = np.array(t); med = float(np.median(t))
print(json.dumps({"lib": os.environ.get("EF_LIB_OVERRIDE", "in-tree"), "calls": n, "median_ms": round(med, 2), "mean_ms": round(float(t.mean()), 2),
                  "slowest_ms": [round(float(v), 1) for v in np.sort(t)[-5:]], "over_1.5x_median": int((t > 1.5 * med).sum())}))
