"""GPU parity of the drop-in's Python API (the reference's stage-level seams,
keep_intermediates, the Laplacian operator, quantize_orientation) against the
golden vectors the reference itself produced (tests/golden/make_golden.py),
and the full C3 batch against the oracle.  Bar: bit-exact everywhere.
"""

import numpy as np
import pytest

from golden_data import load, unpack
from oracle import oracle as O
from paper_1710_07745_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ef():
    import paper_1710_07745_b200 as m
    from paper_1710_07745_b200 import canny

    canny.require_cuda()
    return m


def _sigma_for(ef, weights):
    """The sigma a stage fixture was made with (its weights pin it)."""
    r = (len(weights) - 1) // 2
    for s in (0.5, 1.0, 1.4, 2.0):
        k = ef.build_gaussian_kernel(s, radius=r)
        if np.array_equal(k.weights, weights):
            return s, r
    raise AssertionError("unknown fixture kernel")


def test_quantize_orientation_golden_on_gpu(ef):
    """gradient.py:37-44 on axis, diagonal, near-boundary (t*(1 +- 1e-15)),
    denormal-scale and random pairs: the GPU sector test (with its atan2
    fallback near the boundaries) against the reference's numpy arctan2."""
    from paper_1710_07745_b200 import canny, gradient

    q = load("quantize.npz")
    got = canny.quantize_f64(torch.from_numpy(q["gx"]).cuda(), torch.from_numpy(q["gy"]).cuda()).cpu().numpy()
    bad = np.nonzero(got != q["ori"])[0]
    assert bad.size == 0, [(q["gx"][i], q["gy"][i], got[i], q["ori"][i]) for i in bad[:10]]
    assert np.array_equal(gradient.quantize_orientation_array(q["gx"], q["gy"]), q["ori"])
    assert gradient.quantize_orientation(1.0, 0.0) == 0 and gradient.quantize_orientation(0.0, 1.0) == 90


def test_stage_functions_match_reference_golden(ef):
    """gaussian_blur -> sobel -> non_max_suppress -> double_threshold ->
    trace_edges / trace_edges_parallel through the Python mirrors
    (filtering.py:66-91, gradient.py:73-90, nms.py:36-55, hysteresis.py:54-69)."""
    g = load("stages.npz")
    wc = ef.WorkerConfig(workers=3, band_granularity=2)
    for name in [str(n) for n in g["names"]]:
        arr = g[f"{name}/input"]
        sigma, r = _sigma_for(ef, g[f"{name}/weights"])
        k = ef.build_gaussian_kernel(sigma, radius=r)
        low, high = (float(v) for v in g[f"{name}/thresholds"])
        img = ef.GrayImage.from_array(arr)
        blurred = ef.gaussian_blur(img, k, wc)
        assert np.array_equal(blurred.pixels, g[f"{name}/blurred"]), name
        grad = ef.sobel(blurred, wc)
        for key in ("gx", "gy", "magnitude", "orientation"):
            assert np.array_equal(getattr(grad, key), g[f"{name}/{key}"]), (name, key)
        thin = ef.non_max_suppress(grad, wc)
        assert np.array_equal(thin.magnitude, g[f"{name}/thinned"]), name
        em = ef.double_threshold(thin, ef.Thresholds(low, high))
        assert np.array_equal(em.labels, g[f"{name}/labels"]), name
        assert np.array_equal(ef.trace_edges(em).final, g[f"{name}/final"]), name
        assert np.array_equal(ef.trace_edges_parallel(em, wc).final, g[f"{name}/final"]), name
        # outputs are read-only like the reference's frozen dataclasses
        assert not grad.gx.flags.writeable and not thin.magnitude.flags.writeable
        assert not em.labels.flags.writeable


def test_run_pipeline_keep_intermediates_golden(ef):
    """run_pipeline(..., keep_intermediates=True) (bench.py:124-125): blurred,
    GradientField and ThinnedField in reference dtypes, bit-exact."""
    g = load("stages.npz")
    for name in [str(n) for n in g["names"]]:
        arr = g[f"{name}/input"]
        sigma, r = _sigma_for(ef, g[f"{name}/weights"])
        low, high = (float(v) for v in g[f"{name}/thresholds"])
        res = ef.run_pipeline(ef.GrayImage.from_array(arr),
                              ef.PipelineConfig(sigma=sigma, radius=r, thresholds=ef.Thresholds(low, high)),
                              keep_intermediates=True)
        assert np.array_equal(res.blurred.pixels, g[f"{name}/blurred"]), name
        for key in ("gx", "gy", "magnitude", "orientation"):
            got = getattr(res.grad, key)
            assert got.dtype == g[f"{name}/{key}"].dtype and np.array_equal(got, g[f"{name}/{key}"]), (name, key)
        assert np.array_equal(res.thinned.magnitude, g[f"{name}/thinned"]), name
        assert np.array_equal(res.edges.labels, g[f"{name}/labels"]), name
        assert np.array_equal(res.edges.final, g[f"{name}/final"]), name


def test_laplacian_operator_golden(ef):
    """operator="laplacian" (bench.py:94-100): blurred + 5-point Laplacian
    response (gradient.py:93-107) through run_pipeline, and the stage function
    with the configs' radius-2 kernel."""
    g = load("laplacian.npz")
    for name in [str(n) for n in g["names"]]:
        arr = g[f"{name}/input"]
        img = ef.GrayImage.from_array(arr)
        for sigma in (1.4, 0.6):
            res = ef.run_pipeline(img, ef.PipelineConfig(sigma=sigma, operator="laplacian"), keep_intermediates=True)
            assert np.array_equal(res.response.pixels, g[f"{name}/s{sigma}/response"]), (name, sigma)
            assert np.array_equal(res.blurred.pixels, g[f"{name}/s{sigma}/blurred"]), (name, sigma)
            assert res.edges is None
        k = ef.build_gaussian_kernel(1.4, radius=2)
        resp = ef.laplacian(ef.gaussian_blur(img, k))
        assert np.array_equal(resp.pixels, g[f"{name}/r2/response"]), name
        res = ef.run_pipeline(img, ef.PipelineConfig(sigma=1.4, radius=2, operator="laplacian"))
        assert np.array_equal(res.response.pixels, g[f"{name}/r2/response"]), name


def test_laplacian_random_vs_oracle(ef):
    from paper_1710_07745_b200 import canny

    rng = np.random.default_rng(17)
    for (h, w) in [(1, 1), (1, 300), (257, 1), (3, 5), (129, 130), (512, 700)]:
        arr = rng.integers(0, 256, (h, w)).astype(np.float64) if h * w > 9 else rng.random((h, w)) * 1e3
        wt = O.gaussian_weights(1.4)
        blurred = canny.blur_f64(torch.from_numpy(arr).cuda(), wt)
        assert np.array_equal(blurred.cpu().numpy(), O.blur(arr, wt)), (h, w)
        assert np.array_equal(canny.laplacian_f64(blurred).cpu().numpy(), O.laplacian(O.blur(arr, wt))), (h, w)


def test_full_config3_all_1024_frames_vs_oracle():
    """The headline workload, BASELINE.json configs[3], in full: 1024 seeded
    1024x1024 images through one fused call, every label and edge bit against
    the oracle (the oracle runs on every host core)."""
    from paper_1710_07745_b200 import canny

    canny.require_cuda()
    frames = synth.config3(1024)
    w = O.gaussian_weights(1.4, radius=2)
    ws = canny.new_workspace(*frames.shape)
    canny.reset_stats(ws)
    lab, fin = canny.canny_u8(torch.from_numpy(frames).cuda(), w, 20.0, 50.0, ws=ws)
    stats = canny.read_stats(ws)
    lab, fin = lab.cpu().numpy(), fin.cpu().numpy().view(np.bool_)
    el, ef_ = O.canny(frames, w, 20.0, 50.0, threads=0)
    bad = np.nonzero((lab != el).reshape(len(frames), -1).any(1) | (fin != ef_).reshape(len(frames), -1).any(1))[0]
    assert bad.size == 0, f"frames differing from the oracle: {bad[:20].tolist()}"
    print(f"C3 1024 frames: strong={int((el == 2).sum())} final={int(ef_.sum())} stats={stats}")


def test_detect_pgm_matches_reference_cli_bytes(ef):
    """The CLI detect path (cli.py:82-90): PGM bytes -> edge-map P5 bytes,
    decoded into pinned memory as u8, encoded 0/255 on the device -- byte for
    byte the reference's save_pgm(edges_to_image(run_pipeline(...).edges)),
    with explicit and auto thresholds and parallel hysteresis."""
    g = load("pgm.npz")
    cfgs = {"t2050": ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0)),
            "auto": ef.PipelineConfig(sigma=1.4),
            "s2_par": ef.PipelineConfig(sigma=2.0, thresholds=ef.Thresholds(10.0, 30.0), hysteresis_mode="parallel")}
    for key in [str(k) for k in g["det"]]:
        tag = key.split("/")[1]
        data = g[f"det/{key}/in"].tobytes()
        want = g[f"det/{key}/out"].tobytes()
        assert ef.detect_pgm(data, cfgs[tag]) == want, key
        # the same through the drop-in stage API
        res = ef.run_pipeline(ef.load_pgm(data), cfgs[tag])
        assert ef.save_pgm(ef.edges_to_image(res.edges)) == want, key
    with pytest.raises(ef.PgmFormatError):
        ef.detect_pgm(b"P5 2 2 255 \x00", cfgs["t2050"])


def test_run_pipeline_stage_timings(ef):
    """timings receives the reference's five stage records (bench.py:76-120)
    with device times; results are unchanged by timing."""
    g = load("pipeline.npz")
    name = [str(n) for n in g["names"]][-1]
    arr = g[f"{name}/input"]
    timings = []
    res = ef.run_pipeline(ef.GrayImage.from_array(arr), ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0)),
                          timings=timings)
    assert [t.stage_name for t in timings] == ["gaussian", "sobel", "nms", "threshold", "hysteresis"]
    assert timings[0].wall_ns > 0 and timings[4].wall_ns > 0 and all(t.rows_processed == arr.shape[0] for t in timings)
    assert np.array_equal(res.edges.labels, g[f"{name}/t2050/labels"])
    assert np.array_equal(res.edges.final, unpack(g[f"{name}/t2050/final"], arr.shape))
    t2 = []
    ef.run_pipeline(ef.GrayImage.from_array(arr), ef.PipelineConfig(operator="laplacian"), timings=t2)
    assert [t.stage_name for t in t2] == ["gaussian", "laplacian"]
