"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/ef_oracle.c) is the checker for every GPU parity test, so
before it is trusted it must reproduce the reference bit-for-bit on every
committed fixture: all float64 intermediates, orientation bins, labels, and
the traced edge set.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_1710_07745_b200 import synth

from golden_data import load, unpack

STAGES = load("stages.npz")
PIPE = load("pipeline.npz")
CONFIGS = load("configs.npz")


@pytest.mark.parametrize("name", [str(n) for n in STAGES["names"]])
def test_oracle_stages_bit_exact(name):
    g = {k.split("/", 1)[1]: STAGES[k] for k in STAGES.files if k.startswith(name + "/")}
    low, high = g["thresholds"]
    res = O.stages(g["input"], g["weights"], low, high)
    for key in ("blurred", "gx", "gy", "magnitude", "orientation", "thinned", "labels"):
        assert np.array_equal(res[key], g[key]), f"{name}: {key} differs"
    assert np.array_equal(res["final"], g["final"])


@pytest.mark.parametrize("name", [str(n) for n in PIPE["names"]])
def test_oracle_pipeline_fixtures(name):
    arr = PIPE[f"{name}/input"]
    w = PIPE[f"{name}/weights"]
    for tag in ("t2050", "t00", "t0_30", "tbig", "auto"):
        low, high = PIPE[f"{name}/{tag}/thresholds"]
        labels, final = O.canny(arr, w, low, high)
        assert np.array_equal(labels, PIPE[f"{name}/{tag}/labels"]), (name, tag)
        assert np.array_equal(final, unpack(PIPE[f"{name}/{tag}/final"], arr.shape)), (name, tag)
    for sigma in ("0.6", "2.2"):
        labels, final = O.canny(arr, PIPE[f"{name}/s{sigma}/weights"], 10.0, 40.0)
        assert np.array_equal(labels, PIPE[f"{name}/s{sigma}/labels"]), (name, sigma)
        assert np.array_equal(final, unpack(PIPE[f"{name}/s{sigma}/final"], arr.shape))


@pytest.mark.parametrize("cfg", range(5))
def test_oracle_configs(cfg):
    frames = synth.make_config(cfg, reduced=True)
    assert synth.sha256_u8(frames) == str(CONFIGS[f"c{cfg}/sha256"]), "generator drifted"
    low, high = synth.CONFIG_THRESHOLDS[cfg]
    for r in (2, 5):
        tag = f"c{cfg}/r{r}"
        labels, final = O.canny(frames, CONFIGS[f"{tag}/weights"], low, high, threads=4)
        assert np.array_equal(labels, CONFIGS[f"{tag}/labels"]), tag
        assert np.array_equal(final, unpack(CONFIGS[f"{tag}/final"], frames.shape)), tag


def test_oracle_quantize_matches_reference():
    q = load("quantize.npz")
    got = np.array([O.quantize(a, b) for a, b in zip(q["gx"], q["gy"])])
    assert np.array_equal(got, q["ori"])


def test_oracle_weights_restatement():
    # filtering.py:32-40 -- radius ceil(3 sigma); 1.4 -> 5 (11 taps)
    w = O.gaussian_weights(1.4)
    assert len(w) == 11 and np.array_equal(w, w[::-1]) and abs(w.sum() - 1) < 1e-12
    assert np.array_equal(w, PIPE[f"{PIPE['names'][0]}/weights"])
    assert len(O.gaussian_weights(1.4, radius=2)) == 5
    with pytest.raises(ValueError):
        O.gaussian_weights(0.0)


def test_oracle_trace_snake_and_chains():
    # hysteresis.py:63-69 semantics: 8-connected flood from strong seeds
    assert O.trace(np.array([[2, 1, 1, 0, 1]], np.uint8)).tolist() == [[True, True, True, False, False]]
    h, w = 16, 8
    lab = np.zeros((h, w), np.uint8)
    for y in range(h):
        if y % 2 == 0:
            lab[y, :] = 1
        else:
            lab[y, 0 if (y // 2) % 2 else w - 1] = 1
    lab[h - 1, 0] = 2
    assert O.trace(lab).sum() == (lab != 0).sum()


LAPL = load("laplacian.npz")


@pytest.mark.parametrize("name", [str(n) for n in LAPL["names"]])
def test_oracle_laplacian_matches_reference(name):
    """operator="laplacian" (bench.py:94-100): blur then the 5-point Laplacian
    (gradient.py:93-107), both bit-exact against the reference's own outputs."""
    arr = LAPL[f"{name}/input"]
    for tag in ("s1.4", "s0.6"):
        blurred = O.blur(arr, LAPL[f"{name}/{tag}/weights"])
        assert np.array_equal(blurred, LAPL[f"{name}/{tag}/blurred"]), (name, tag)
        assert np.array_equal(O.laplacian(blurred), LAPL[f"{name}/{tag}/response"]), (name, tag)
    got = O.laplacian(O.blur(arr, LAPL[f"{name}/r2/weights"]))
    assert np.array_equal(got, LAPL[f"{name}/r2/response"]), name
