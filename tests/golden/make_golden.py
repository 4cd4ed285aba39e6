"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports edgeforge read-only from /root/reference/pkg/src and writes small
compressed fixtures next to this file.  The fixtures travel with the repo; the
reference does not (nothing at test time reads /root/reference).

Fixtures:
  stages.npz    every intermediate (blurred, gx, gy, magnitude, orientation,
                thinned, labels, final) for small hand-made cases, float64 and
                integer inputs, default radius ceil(3*sigma) and explicit radii.
  pipeline.npz  run_pipeline(img, PipelineConfig(...)) labels/final for a
                fixture set (steps, ramps, checkers, noise, constants, 1x1 ...)
                under explicit, degenerate and auto thresholds.
  configs.npz   labels/final for the seeded config generators (reduced sizes;
                C0 at full size) under the configs' 5x5 kernel (radius 2) and
                the reference default radius 5; inputs are pinned by sha256.
  quantize.npz  quantize_orientation on axis, diagonal and near-boundary
                gradient pairs.
  pgm.npz       load_pgm on a seeded corpus of valid and malformed P5/P2 files
                (pixels, or PgmFormatError message + offset), save_pgm bytes,
                and the CLI detect path's output bytes
                save_pgm(edges_to_image(run_pipeline(load_pgm(f), cfg).edges)).
  laplacian.npz run_pipeline(operator="laplacian", keep_intermediates=True)
                response + blurred for the fixture set (sigma 1.4 and 0.6), and
                gaussian_blur -> laplacian with the configs' radius-2 kernel.

    python tests/golden/make_golden.py [stages pipeline configs quantize laplacian pgm]
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import edgeforge as ef  # noqa: E402
from edgeforge.filtering import GaussianKernel  # noqa: E402

from paper_1710_07745_b200 import synth  # noqa: E402

W1 = ef.WorkerConfig(workers=1)


def kernel(sigma, radius=None):
    if radius is None:
        return ef.build_gaussian_kernel(sigma)
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    w /= w.sum()
    return GaussianKernel(sigma=sigma, radius=radius, weights=w)


def staged(arr, k, low, high, workers=W1):
    img = ef.GrayImage.from_array(arr)
    blurred = ef.gaussian_blur(img, k, workers)
    grad = ef.sobel(blurred, workers)
    thin = ef.non_max_suppress(grad, workers)
    labeled = ef.double_threshold(thin, ef.Thresholds(low=low, high=high))
    traced = ef.trace_edges(labeled)
    return dict(blurred=blurred.pixels, gx=grad.gx, gy=grad.gy, magnitude=grad.magnitude,
                orientation=grad.orientation, thinned=thin.magnitude, labels=traced.labels,
                final=traced.final)


def fixture_set():
    """Own fixture shapes (not the reference suite's list): edge cases by size,
    content and value type."""
    rng = np.random.default_rng(5150)
    yy = lambda h, w: np.mgrid[0:h, 0:w]  # noqa: E731
    cases = []

    def add(name, arr):
        cases.append((name, np.asarray(arr, dtype=np.float64)))

    add("zero_1x1", np.zeros((1, 1)))
    add("white_1x1", np.full((1, 1), 255.0))
    add("row_1x9", rng.integers(0, 256, (1, 9)))
    add("col_11x1", rng.integers(0, 256, (11, 1)))
    add("noise_2x3", rng.integers(0, 256, (2, 3)))
    add("vstep_5x4", np.where(yy(5, 4)[1] >= 2, 255.0, 0.0))
    add("hstep_16x16", np.where(yy(16, 16)[0] >= 8, 255.0, 0.0))
    add("vstep_16x16", np.where(yy(16, 16)[1] >= 8, 255.0, 0.0))
    y, x = yy(6, 9)
    add("ramp_frac_6x9", (2 * x + y) * 255.0 / 21.0)
    y, x = yy(10, 10)
    add("checker_10x10", ((x + y) % 2) * 255.0)
    y, x = yy(40, 40)
    add("diag_40x40", np.where(x > y, 255.0, 0.0))
    add("antidiag_33x47", np.where(yy(33, 47)[1] + yy(33, 47)[0] > 38, 200.0, 20.0))
    y, x = yy(64, 64)
    add("disk_64", np.where((y - 31.5) ** 2 + (x - 30.25) ** 2 < 400, 180.0, 40.0))
    add("noise_31x29", rng.integers(0, 256, (31, 29)))
    add("noise_96x80", rng.integers(0, 256, (96, 80)))
    add("float_noise_24x36", rng.random((24, 36)) * 255.0)
    add("const_50x70", np.full((50, 70), 87.0))
    add("clipped_blocks_48x48", np.kron(rng.integers(0, 2, (6, 6)) * 255.0, np.ones((8, 8))))
    add("c0_crop_128", synth.config0()[:128, :128])
    add("c2_crop_160", synth.config2(512)[100:260, 150:310])
    return cases


def pack(b):
    return np.packbits(np.asarray(b, dtype=bool).ravel())


def make_laplacian():
    out = {}
    names = []
    cases = [c for c in fixture_set() if not c[0].startswith(("c0_", "c2_"))]
    rng = np.random.default_rng(4242)
    cases.append(("u8_40x50", rng.integers(0, 256, (40, 50)).astype(np.float64)))
    cases.append(("c3_crop_48", synth.config3_image(0)[200:248, 300:348].astype(np.float64)))
    for name, arr in cases:
        img = ef.GrayImage.from_array(arr)
        names.append(name)
        out[f"{name}/input"] = arr
        for sigma in (1.4, 0.6):
            res = ef.run_pipeline(img, ef.PipelineConfig(sigma=sigma, operator="laplacian"), keep_intermediates=True)
            out[f"{name}/s{sigma}/response"] = res.response.pixels
            out[f"{name}/s{sigma}/blurred"] = res.blurred.pixels
            out[f"{name}/s{sigma}/weights"] = ef.build_gaussian_kernel(sigma).weights.copy()
        k = kernel(1.4, 2)
        blurred = ef.gaussian_blur(img, k, W1)
        out[f"{name}/r2/response"] = ef.gradient.laplacian(blurred, W1).pixels
        out[f"{name}/r2/weights"] = k.weights.copy()
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "laplacian.npz"), **out)
    print("laplacian.npz", os.path.getsize(os.path.join(HERE, "laplacian.npz")))


def pgm_corpus():
    """Seeded PGM byte strings: valid files with comments, odd whitespace,
    small maxval, trailing bytes; and malformed ones (own corpus)."""
    rng = np.random.default_rng(1710)
    out = []

    def p5(w, h, px, maxval=255, sep=b"\n", pre=b""):
        return pre + b"P5" + sep + f"{w} {h}".encode() + sep + str(maxval).encode() + b"\n" + bytes(px)

    def p2(w, h, px, maxval=255, sep=b" "):
        return b"P2\n" + f"{w} {h}".encode() + b"\n" + str(maxval).encode() + b"\n" + sep.join(
            str(int(v)).encode() for v in px)

    for (w, h) in [(1, 1), (3, 2), (17, 5), (64, 48), (33, 33)]:
        px = rng.integers(0, 256, w * h)
        out.append(p5(w, h, px))
        out.append(p5(w, h, px, sep=b" # a comment\n\t"))
        out.append(p5(w, h, px, pre=b"# leading comment\n") + b"trailing bytes")
        out.append(p2(w, h, px))
        out.append(p2(w, h, px, sep=b"\n#c\n"))
        small = rng.integers(0, 8, w * h)
        out.append(p5(w, h, small, maxval=7))
        out.append(p2(w, h, small, maxval=7))
    base = p5(6, 4, rng.integers(0, 256, 24))
    bad = [b"", b"   ", b"# only a comment", b"P6\n1 1\n255\n\x00", b"P5", b"P5 3", b"P5 3 2", b"P5 3 2 255",
           b"P5 3 2 255\x01\x02", b"P5\n3 2\n255\n\x00\x01", b"P5 0 2 255 ", b"P5 2 0 255 ", b"P5 2 2 0 ",
           b"P5 2 2 256 ", b"P5 2 2 1000 ", b"P5 -2 2 255 ", b"P5 2x 2 255 ", b"P5 2 2 2.5 ", b"P5 2 2 255#c\n1234",
           b"p5 2 2 255 1234", b"P2 2 2 255 1 2 3", b"P2 2 2 255 1 2 3 x", b"P2 2 2 9 1 2 3 10", b"P2 1 1 255 +5",
           b"P2 2 1 3 3 4", b"P5 2 2 7 \x00\x01\x08\x02", b"\xffP5 1 1 255 \x00", b"P5 b'q' 1 255 ",
           b'P5 a"b 1 255 ', b"P5 a'b 1 255 ", b"P5 \\x 1 255 ", b"P5 1 1 255\t\x07", b"P5 2 2 255 \x01",
           b"P25 2 2 255 ", b"P2 3 1 255 1 2#3\n4", base[:-1], base + b"\x00"]
    for i in range(40):  # truncations and single-byte corruptions of a valid file
        b = bytearray(base)
        if i % 2:
            b = b[: int(rng.integers(0, len(b)))]
        else:
            b[int(rng.integers(0, 16))] = int(rng.integers(0, 256))
        bad.append(bytes(b))
    return out + bad


def make_pgm():
    from edgeforge.bench import edges_to_image, run_pipeline

    out = {}
    corpus = pgm_corpus()
    for i, data in enumerate(corpus):
        out[f"in/{i}"] = np.frombuffer(data, np.uint8)
        try:
            img = ef.load_pgm(data)
        except ef.PgmFormatError as err:
            out[f"err/{i}"] = np.array(str(err))
            out[f"off/{i}"] = np.array(err.offset)
            continue
        out[f"px/{i}"] = img.pixels.astype(np.uint8)
        out[f"save/{i}"] = np.frombuffer(ef.save_pgm(img), np.uint8)
    out["n"] = np.array(len(corpus))
    # the CLI detect path on P5 inputs: edges -> 0/255 P5 bytes
    rng = np.random.default_rng(77)
    det = []
    for k, arr in enumerate([synth.config0()[:160, :200], synth.config3_image(7)[:128, :256],
                             rng.integers(0, 256, (45, 67)).astype(np.uint8)]):
        data = b"P5\n%d %d\n255\n" % (arr.shape[1], arr.shape[0]) + arr.tobytes()
        for tag, cfg in (("t2050", ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0))),
                         ("auto", ef.PipelineConfig(sigma=1.4)),
                         ("s2_par", ef.PipelineConfig(sigma=2.0, thresholds=ef.Thresholds(10.0, 30.0),
                                                      hysteresis_mode="parallel"))):
            res = run_pipeline(ef.load_pgm(data), cfg)
            out[f"det/{k}/{tag}/in"] = np.frombuffer(data, np.uint8)
            out[f"det/{k}/{tag}/out"] = np.frombuffer(ef.save_pgm(edges_to_image(res.edges)), np.uint8)
            det.append(f"{k}/{tag}")
    out["det"] = np.array(det)
    np.savez_compressed(os.path.join(HERE, "pgm.npz"), **out)
    print("pgm.npz", os.path.getsize(os.path.join(HERE, "pgm.npz")), len(corpus), "files")


def main():
    which = set(sys.argv[1:]) or {"stages", "pipeline", "configs", "quantize", "laplacian", "pgm"}
    if "laplacian" in which:
        make_laplacian()
    if "pgm" in which:
        make_pgm()
    if which <= {"laplacian", "pgm"}:
        return
    out = {}
    # ---------------- stages ----------------
    rng = np.random.default_rng(77)
    stage_cases = [
        ("u8_37x41_s14", rng.integers(0, 256, (37, 41)).astype(float), 1.4, None, 20.0, 50.0),
        ("u8_37x41_s14_r2", rng.integers(0, 256, (37, 41)).astype(float), 1.4, 2, 20.0, 50.0),
        ("f64_23x17_s10", rng.random((23, 17)) * 255.0, 1.0, None, 30.0, 90.0),
        ("u8_9x13_s05", rng.integers(0, 256, (9, 13)).astype(float), 0.5, None, 100.0, 400.0),
        ("u8_1x1", np.array([[42.0]]), 1.4, None, 20.0, 50.0),
        ("u8_3x2", rng.integers(0, 256, (3, 2)).astype(float), 2.0, None, 5.0, 10.0),
        ("u8_7x1", rng.integers(0, 256, (7, 1)).astype(float), 1.4, 2, 1.0, 2.0),
        ("step_4x4", np.array([[0.0, 0.0, 255.0, 255.0]] * 4), 1.4, None, 20.0, 50.0),
        ("f64_ramp_12x20", (np.mgrid[0:12, 0:20][1] * 3.3 + np.mgrid[0:12, 0:20][0] * 1.7),
         1.4, 2, 0.5, 1.0),
        ("u8_60x44_zero_thr", rng.integers(0, 256, (60, 44)).astype(float), 1.4, 2, 0.0, 0.0),
    ]
    names = []
    for name, arr, sigma, radius, low, high in stage_cases:
        k = kernel(sigma, radius)
        res = staged(arr, k, low, high)
        names.append(name)
        out[f"{name}/input"] = arr
        out[f"{name}/weights"] = k.weights.copy()
        out[f"{name}/thresholds"] = np.array([low, high])
        for key, val in res.items():
            out[f"{name}/{key}"] = val
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "stages.npz"), **out)

    # ---------------- pipeline ----------------
    out = {}
    names = []
    for name, arr in fixture_set():
        img = ef.GrayImage.from_array(arr)
        names.append(name)
        out[f"{name}/input"] = arr
        out[f"{name}/weights"] = ef.build_gaussian_kernel(1.4).weights.copy()
        for tag, thr in (("t2050", ef.Thresholds(20.0, 50.0)), ("auto", None),
                         ("t00", ef.Thresholds(0.0, 0.0)), ("t0_30", ef.Thresholds(0.0, 30.0)),
                         ("tbig", ef.Thresholds(1e9, 1e9))):
            res = ef.run_pipeline(img, ef.PipelineConfig(sigma=1.4, thresholds=thr))
            out[f"{name}/{tag}/labels"] = res.edges.labels
            out[f"{name}/{tag}/final"] = pack(res.edges.final)
            out[f"{name}/{tag}/thresholds"] = np.array([res.thresholds.low, res.thresholds.high])
        # sigma variants through run_pipeline (radius ceil(3 sigma))
        for sigma in (0.6, 2.2):
            res = ef.run_pipeline(img, ef.PipelineConfig(sigma=sigma, thresholds=ef.Thresholds(10.0, 40.0)))
            out[f"{name}/s{sigma}/labels"] = res.edges.labels
            out[f"{name}/s{sigma}/final"] = pack(res.edges.final)
            out[f"{name}/s{sigma}/weights"] = ef.build_gaussian_kernel(sigma).weights.copy()
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "pipeline.npz"), **out)

    # ---------------- configs ----------------
    out = {}
    for cfg in range(5):
        frames = synth.make_config(cfg, reduced=True)
        low, high = synth.CONFIG_THRESHOLDS[cfg]
        out[f"c{cfg}/sha256"] = np.array(synth.sha256_u8(frames))
        out[f"c{cfg}/shape"] = np.array(frames.shape)
        for radius in (2, None):
            k = kernel(1.4, radius)
            tag = f"c{cfg}/r{k.radius}"
            out[f"{tag}/weights"] = k.weights.copy()
            labs, fins = [], []
            for f in frames:
                img = ef.GrayImage.from_array(f.astype(np.float64))
                if radius is None:
                    res = ef.run_pipeline(img, ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(low, high)))
                    labs.append(res.edges.labels)
                    fins.append(res.edges.final)
                else:
                    res = staged(f.astype(np.float64), k, low, high, ef.WorkerConfig(workers=8))
                    labs.append(res["labels"])
                    fins.append(res["final"])
            out[f"{tag}/labels"] = np.stack(labs)
            out[f"{tag}/final"] = pack(np.stack(fins))
            print(f"config {cfg} r={k.radius}: strong={int((np.stack(labs) == 2).sum())} "
                  f"weak={int((np.stack(labs) == 1).sum())} final={int(np.stack(fins).sum())}")
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **out)

    # ---------------- quantize ----------------
    t = np.sqrt(2.0) - 1.0
    pairs = [(1, 0), (1, 1), (0, 1), (-1, 1), (0, 0), (-1, 0), (0, -1), (-1, -1), (1, -1),
             (1.0, t), (1.0, t * (1 + 1e-15)), (1.0, t * (1 - 1e-15)), (t, 1.0), (-t, 1.0),
             (-1.0, t), (1e-300, 1.0), (-5.0, 1e-300), (1020.0, 0.0), (0.0, 1020.0)]
    rng = np.random.default_rng(8)
    for _ in range(2000):
        pairs.append(tuple(rng.normal(size=2) * 300))
    gx = np.array([p[0] for p in pairs], dtype=np.float64)
    gy = np.array([p[1] for p in pairs], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "quantize.npz"), gx=gx, gy=gy,
                        ori=ef.gradient.quantize_orientation_array(gx, gy))
    for f in ("stages.npz", "pipeline.npz", "configs.npz", "quantize.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
