"""Time the host-buffer entry point and its pieces (debug probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1710_07745_b200 import canny, synth
from paper_1710_07745_b200.filtering import build_gaussian_kernel

frames = synth.make_config(1)
b, h, wd = frames.shape
w = build_gaussian_kernel(1.4, radius=2).weights
hsrc = torch.from_numpy(frames).pin_memory()
hlab = torch.empty_like(hsrc).pin_memory(); hfin = torch.empty_like(hsrc).pin_memory()
plab = np.empty(frames.shape, np.uint8); pfin = np.empty(frames.shape, np.uint8)
d = torch.empty_like(hsrc, device="cuda")
def t(f, n=8):
    f(); f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / n
print("H2D only      %.3f ms" % t(lambda: d.copy_(hsrc, non_blocking=True)))
print("host pinned   %.3f ms" % t(lambda: canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, 20., 50., hlab.data_ptr(), hfin.data_ptr())))
print("host pageable-out %.3f ms" % t(lambda: canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, 20., 50., plab.ctypes.data, pfin.ctypes.data)))
print("host pageable-in  %.3f ms" % t(lambda: canny.canny_u8_host_ptr(frames.ctypes.data, b, h, wd, w, 20., 50., plab.ctypes.data, pfin.ctypes.data)))
