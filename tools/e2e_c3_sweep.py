"""e2e (host buffers through ef_canny_u8_host) on C3, 1024 frames: the host
pipeline tunables swept in subprocesses (EF_HOST_UNPACK_THREADS, EF_HOST_CHUNK_MB).
Run on the GPU box: python tools/e2e_c3_sweep.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time
sys.path.insert(0, %r)
import numpy as np, torch
from paper_1710_07745_b200 import canny, synth
from paper_1710_07745_b200.filtering import build_gaussian_kernel
frames = np.load("/tmp/c3.npy", mmap_mode="r")
b, h, wd = frames.shape
w = build_gaussian_kernel(1.4, radius=2).weights
hsrc = torch.from_numpy(np.ascontiguousarray(frames)).pin_memory()
hlab = torch.empty_like(hsrc).pin_memory(); hfin = torch.empty_like(hsrc).pin_memory()
f = lambda: canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, 20., 50., hlab.data_ptr(), hfin.data_ptr())
f(); f()
ts = []
for _ in range(8):
    t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
print("%%.2f" %% (1e3 * sorted(ts)[len(ts) // 2]))
''' % ROOT

def main():
    sys.path.insert(0, ROOT)
    if not os.path.exists("/tmp/c3.npy"):
        from paper_1710_07745_b200 import synth
        import numpy as np
        np.save("/tmp/c3.npy", synth.config_range(3, 0, 1024))
    sets = [(4, 8), (4, 16), (4, 32), (4, 64), (3, 32), (5, 32)] if "--focus" in sys.argv else \
        [(t, c) for t in (2, 4, 6, 8) for c in (4, 8, 16, 32)]
    reps = 3 if "--focus" in sys.argv else 1
    for _ in range(reps):
      for t, c in sets:
        if True:
            env = dict(os.environ, EF_HOST_UNPACK_THREADS=str(t), EF_HOST_CHUNK_MB=str(c))
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True).stdout.strip()
            print(f"threads={t} chunkMB={c} ms={out}", flush=True)

if __name__ == "__main__":
    main()
