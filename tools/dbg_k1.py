import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import os, numpy as np, torch
from paper_1710_07745_b200 import canny, synth
from oracle import oracle as O
w = O.gaussian_weights(1.4, radius=2)
for name, frames in [("c0", synth.make_config(0)), ("c1r", synth.make_config(1, reduced=True)), ("c4r", synth.make_config(4, reduced=True))]:
    low, high = 20.0, 50.0
    lab, fin = canny.canny_u8(torch.from_numpy(frames).cuda(), w, low, high)
    el, ef_ = O.canny(frames, w, low, high)
    L = lab.cpu().numpy()
    bad = np.argwhere(L != el)
    print(name, frames.shape, "mismatch", len(bad), "of", L.size)
    if len(bad):
        f, y, x = bad[:, 0], bad[:, 1], bad[:, 2]
        print("  rows (mod 104):", np.bincount(y % 104, minlength=104).nonzero()[0][:40])
        print("  rows:", np.unique(y)[:40])
        print("  cols mod 120:", np.unique(x % 120)[:40])
        print("  got/expected samples:", [(int(a), int(b)) for a, b in zip(L[f[:10], y[:10], x[:10]], el[f[:10], y[:10], x[:10]])])
