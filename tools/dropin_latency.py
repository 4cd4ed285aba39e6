"""Latency of the drop-in run_pipeline on one 1080p frame (float64 GrayImage in,
host EdgeMap out), default radius (ceil(3 sigma) = 5) and the configs' 5x5."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1710_07745_b200 as ef
from paper_1710_07745_b200 import synth

frame = synth.make_config(1)[0].astype(np.float64)
img = ef.GrayImage.from_array(frame) if hasattr(ef.GrayImage, "from_array") else ef.GrayImage(frame.shape[1], frame.shape[0], frame)
for radius in (None, 2):
    cfg = ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0), radius=radius)
    for _ in range(3):
        ef.run_pipeline(img, cfg)
    t0 = time.perf_counter()
    n = 20
    for _ in range(n):
        res = ef.run_pipeline(img, cfg)
    dt = (time.perf_counter() - t0) / n
    print(f"radius {radius}: {dt * 1e3:.2f} ms per 1080p frame ({frame.size / dt / 1e6:.0f} MP/s)")

# breakdown
from paper_1710_07745_b200 import canny
from paper_1710_07745_b200.filtering import build_gaussian_kernel
w = build_gaussian_kernel(1.4).weights
t0 = time.perf_counter()
for _ in range(20):
    u8 = img.as_u8()
t1 = time.perf_counter()
for _ in range(20):
    canny.canny_u8_host(u8, w, 20.0, 50.0)
t2 = time.perf_counter()
print(f"as_u8 {(t1 - t0) / 20 * 1e3:.2f} ms, canny_u8_host {(t2 - t1) / 20 * 1e3:.2f} ms")
