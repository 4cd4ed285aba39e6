"""K1 (classify only) on 1024 flat 1024^2 frames (no candidates: phases 1-2 only), warm, CUDA events."""
import json, os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_07745_b200 import canny
from paper_1710_07745_b200.filtering import build_gaussian_kernel
w = build_gaussian_kernel(1.4, radius=2).weights
src = torch.full((1024, 1024, 1024), 100, dtype=torch.uint8, device="cuda")
lab = torch.empty_like(src)
ws = canny.new_workspace(1024, 1024, 1024)
for _ in range(3):
    canny.classify_u8(src, w, 20.0, 50.0, labels=lab, ws=ws)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    canny.classify_u8(src, w, 20.0, 50.0, labels=lab, ws=ws)
e.record(); torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("EF_LIB_OVERRIDE", "in-tree"), "flat_c3_classify_ms": round(s.elapsed_time(e) / 10, 4)}))
