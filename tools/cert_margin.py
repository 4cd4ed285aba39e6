"""How much of the certification bands do the fp32 errors actually use?

Runs K1 from a debug build (-DEF_DEBUG_DUMP: K1 stores the fp32 squared
magnitude, gx and gy of every output pixel) and compares them with the exact
float64 values (ef_stages_f64, bit-identical to the reference).  For each input
it reports the largest error as a fraction of the analytic bound that
make_fast() (csrc/ef_abi.cu) certifies with -- before its safety factor S:

    gradient:  |g32 - g64| / E_g
    magnitude: (|sqrt(m2_32) - m64| + 2^-22 m64) / Em(m64)
               (2^-22 m64: the worst case of sqrt.approx, which the dump does
               not include; Em(M) = sqrt(2) E_g + rel M)

    EF_LIB_OVERRIDE=_variants/dump/libedgeforge_b200.so python tools/cert_margin.py

Test infrastructure: the exact path is the product's own float64 kernel.
"""
import ctypes
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402  (weights only)
from paper_1710_07745_b200 import _lib, canny, synth  # noqa: E402


def bounds(r):
    u, u64 = 2.0 ** -24, 2.0 ** -53
    eh = (r + 2) * u * 255.0
    eb = eh + (r + 3) * u * 255.0 + (4 * r + 6) * u64 * 255.0
    eg = 8.0 * eb + 4080.0 * u + 12.0 * u64 * 1020.0 + 1e-9
    rel = 2.0 ** -20 + 3.0 * u
    return eg, rel


def study(name, frames, r, sigma, low, high):
    lib = _lib.load()
    lib.ef_debug_dump.argtypes = [ctypes.c_void_p] * 3
    lib.ef_debug_dump.restype = ctypes.c_int
    w = O.gaussian_weights(sigma, radius=r)
    eg, rel = bounds(r)
    b, h, wd = frames.shape
    dev = torch.device("cuda", 0)
    m2 = torch.full((b, h, wd), float("nan"), dtype=torch.float32, device=dev)
    gx = torch.full_like(m2, float("nan"))
    gy = torch.full_like(m2, float("nan"))
    assert lib.ef_debug_dump(m2.data_ptr(), gx.data_ptr(), gy.data_ptr()) == 0
    src = torch.from_numpy(frames).to(dev)
    canny.canny_u8(src, w, low, high)
    torch.cuda.synchronize()
    assert lib.ef_debug_dump(None, None, None) == 0
    worst_g = worst_m = 0.0
    covered = 0
    for f in range(b):
        ex = canny.stages_f64(src[f], w, low, high)
        g64x, g64y, m64 = ex["gx"], ex["gy"], ex["magnitude"]
        ok = ~torch.isnan(m2[f])
        covered += int(ok.sum())
        eg_x = ((gx[f].double() - g64x).abs()[ok]).max().item() / eg
        eg_y = ((gy[f].double() - g64y).abs()[ok]).max().item() / eg
        mag32 = m2[f].double().clamp_min(0).sqrt()
        em = math.sqrt(2.0) * eg + rel * m64 + 1e-9
        ratio = ((mag32 - m64).abs() + 2.0 ** -22 * m64) / em
        worst_g = max(worst_g, eg_x, eg_y)
        worst_m = max(worst_m, ratio[ok].max().item())
    row = {"input": name, "radius": r, "frames": b, "pixels_checked": covered, "pixels": b * h * wd,
           "max_grad_err_over_Eg": round(worst_g, 4), "max_mag_err_over_Em": round(worst_m, 4)}
    print(json.dumps(row), flush=True)
    return row


def main():
    rng = np.random.default_rng(7)
    rows = []
    rows.append(study("C3 frames 0-31", synth.config_range(3, 0, 32), 2, 1.4, 20.0, 50.0))
    rows.append(study("C1 frames 0-3", synth.config_range(1, 0, 4), 2, 1.4, 20.0, 50.0))
    rows.append(study("C2", np.asarray(synth.make_config(2)).reshape(1, 4096, 4096), 2, 1.4, 15.0, 45.0))
    noise = rng.integers(0, 256, size=(4, 512, 512), dtype=np.uint8)
    blocks = (np.kron(rng.integers(0, 2, (4, 64, 64)), np.ones((1, 8, 8))) * 255).astype(np.uint8)
    for r in (1, 2, 3, 5, 6):
        sigma = max(0.3, r / 3.0)
        rows.append(study(f"uniform noise r={r}", noise, r, sigma, 20.0, 50.0))
        rows.append(study(f"0/255 blocks r={r}", blocks, r, sigma, 20.0, 50.0))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
