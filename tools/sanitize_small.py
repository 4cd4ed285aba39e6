"""Small-shape run of every kernel family for compute-sanitizer (racecheck /
memcheck / synccheck): fused path (TMA and load staging, edge tiles, several
radii, batch), fix-up overflow, hysteresis from labels (union-find, both H1
variants), bands + device seam merge, exact float64 path, stage kernels, host
buffer entry.  Every result is checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1710_07745_b200 import bands, canny, synth  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(lab, fin, frames, w, lo, hi):
    el, ef_ = O.canny(frames, w, lo, hi)
    lab, fin = lab.reshape(el.shape), fin.reshape(el.shape)
    assert np.array_equal(lab.cpu().numpy(), el) and np.array_equal(fin.cpu().numpy().astype(bool), ef_)


rng = np.random.default_rng(0)
for r in (1, 2, 5, 7):
    w = O.gaussian_weights(max(0.5, r / 3), radius=r)
    for shape in [(2, 70, 144), (1, 33, 100), (1, 130, 260)]:
        f = synth.config1(*shape)
        f[0, :20, :20] = rng.integers(0, 256, (20, 20))
        lab, fin = canny.canny_u8(dev(f), w, 20.0, 50.0)
        check(lab, fin, f, w, 20.0, 50.0)
print("fused ok", flush=True)
for thr in (0, 32):
    canny.set_block_tile_threshold(thr)
    lab = rng.choice([0, 1, 2], size=(200, 300), p=[0.5, 0.4, 0.1]).astype(np.uint8)
    fin = canny.trace_edges_u8(dev(lab))
    assert np.array_equal(fin.cpu().numpy()[0].astype(bool), O.trace(lab))
canny.set_block_tile_threshold(8)
print("trace ok", flush=True)
blk = rng.choice(np.array([0, 16], np.uint8), size=(64, 64))
f = np.kron(blk, np.ones((4, 4), np.uint8))[None]
wd = np.array([0.25, 0.5, 0.25])
lab, fin = canny.canny_u8(dev(f), wd, 48.0, 48.0)
check(lab, fin, f, wd, 48.0, 48.0)
print("fix overflow ok", flush=True)
frame = synth.config4(512, tile=128)
w = O.gaussian_weights(1.4, radius=2)
lab, fin = canny.canny_u8(dev(frame), w, 20.0, 50.0)
bl, bf = bands.canny_bands_local(dev(frame), 3, w, 20.0, 50.0)
assert torch.equal(bl, lab[0]) and torch.equal(bf, fin[0])
print("bands ok", flush=True)
img = rng.random((40, 50)) * 255.0
lab, fin = canny.canny_f64(dev(img), w, 20.0, 50.0)
check(lab, fin, img, w, 20.0, 50.0)
st = canny.stages_f64(dev(img), w, 20.0, 50.0)
ref = O.stages(img, w, 20.0, 50.0)
for k in ("blurred", "gx", "gy", "magnitude", "thinned", "labels"):
    assert np.array_equal(st[k].cpu().numpy(), ref[k]), k
print("exact ok", flush=True)
f = synth.config3(3, 128)
hl, hf = canny.canny_u8_host(f, w, 20.0, 50.0)
el, ef_ = O.canny(f, w, 20.0, 50.0)
assert np.array_equal(hl, el) and np.array_equal(hf.astype(bool), ef_)
print("host ok", flush=True)
print("SANITIZE-SMALL OK")
