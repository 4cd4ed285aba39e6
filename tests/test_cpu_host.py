"""CPU-side tests: the C-ABI library loads and exports what include/*.h
declares, host-side logic (band plan, seam union-find, validation, PGM), and
that the product refuses to run without a CUDA device (no CPU fallback)."""

import os
import re

import numpy as np
import pytest

import paper_1710_07745_b200 as ef
from paper_1710_07745_b200 import _lib, bands

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _declared_symbols():
    names = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            text = open(os.path.join(inc, f)).read()
            names |= set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(ef_\w+)\(", text, re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.exported_symbols())
    assert lib.ef_abi_version() == 1


def test_workspace_sizes_are_positive_and_monotone():
    lib = _lib.load()
    a = lib.ef_workspace_bytes(1, 1080, 1920)
    b = lib.ef_workspace_bytes(64, 1080, 1920)
    assert 0 < a < b
    assert lib.ef_workspace_bytes(0, 10, 10) == 0
    assert lib.ef_band_halo_rows(2) == 4 and lib.ef_band_halo_rows(5) == 7


def _py_merge(ids_all, strong_all, width):
    parent = {}

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    strong = {}
    for ids, st in zip(ids_all, strong_all):
        for i, s in zip(ids, st):
            if i >= 0:
                parent.setdefault(i, i)
                strong[i] = strong.get(i, 0) | int(s)
    for k in range(len(ids_all) - 1):
        top, bot = ids_all[k][width:], ids_all[k + 1][:width]
        for x in range(width):
            for s in (-1, 0, 1):
                if 0 <= x + s < width and top[x] >= 0 and bot[x + s] >= 0:
                    a, b = find(top[x]), find(bot[x + s])
                    if a != b:
                        parent[b] = a
    root_strong = {}
    for i in parent:
        root_strong[find(i)] = root_strong.get(find(i), 0) | strong[i]
    return np.array([[root_strong[find(i)] if i >= 0 else 0 for i in ids] for ids in ids_all], np.uint8)


def test_band_merge_host_matches_python_union_find():
    rng = np.random.default_rng(0)
    for trial in range(30):
        nb, w = int(rng.integers(1, 6)), int(rng.integers(1, 40))
        ids_all = []
        for k in range(nb):
            local = rng.integers(-1, 6, size=2 * w)
            ids_all.append(bands.globalize_ids(local, k))
        ids_all = np.stack(ids_all)
        strong = (rng.random(ids_all.shape) < 0.15).astype(np.uint8)
        strong[ids_all < 0] = 0
        # a component's strong flag is per id: make it consistent
        for k in range(nb):
            for i in np.unique(ids_all[k]):
                if i >= 0:
                    strong[k][ids_all[k] == i] = strong[k][ids_all[k] == i].max()
        got = bands.merge_edges(ids_all, strong, w)
        assert np.array_equal(got, _py_merge(ids_all, strong, w)), trial


def test_band_plan_and_ids():
    assert bands.band_plan(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert bands.band_plan(16384, 8)[-1] == (14336, 16384)
    g = bands.globalize_ids(np.array([-1, 0, 5]), 3)
    assert g[0] == -1 and g[1] == 3 << 40 and g[2] == (3 << 40) | 5
    assert ef.plan_bands(10, ef.WorkerConfig(workers=4, band_granularity=1)) == [(0, 3), (3, 6), (6, 9), (9, 10)]


def test_reference_api_validation():
    with pytest.raises(ValueError):
        ef.Thresholds(low=5.0, high=2.0)
    with pytest.raises(ValueError):
        ef.Thresholds(low=-1.0, high=2.0)
    with pytest.raises(ValueError):
        ef.PipelineConfig(hysteresis_mode="bogus")
    with pytest.raises(ValueError):
        ef.PipelineConfig(operator="sobel")
    with pytest.raises(ValueError):
        ef.build_gaussian_kernel(0.0)
    with pytest.raises(ValueError):
        ef.GaussianKernel(sigma=1.0, radius=1, weights=np.array([0.2, 0.5, 0.3]))
    k = ef.build_gaussian_kernel(1.4)
    assert k.radius == 5 and len(k.weights) == 11  # ceil(3 * 1.4) = 5, filtering.py:36
    assert ef.build_gaussian_kernel(1.4, radius=2).weights.shape == (5,)
    assert ef.PipelineConfig().kernel().radius == 5
    with pytest.raises(ValueError):
        ef.GrayImage.from_array(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        ef.EdgeMap(width=2, height=2, labels=np.zeros((3, 3), np.uint8))


def test_grayimage_u8_detection():
    assert ef.GrayImage.from_array(np.array([[0.0, 255.0]])).as_u8() is not None
    assert ef.GrayImage.from_array(np.array([[0.5, 1.0]])).as_u8() is None
    assert ef.GrayImage.from_array(np.array([[256.0]])).as_u8() is None
    assert ef.GrayImage.from_array(np.array([[-1.0]])).as_u8() is None


def test_pgm_roundtrip_and_errors():
    rng = np.random.default_rng(1)
    arr = rng.integers(0, 256, (7, 9)).astype(np.float64)
    img = ef.GrayImage.from_array(arr)
    back = ef.load_pgm(ef.save_pgm(img))
    assert np.array_equal(back.pixels, arr)
    assert np.array_equal(ef.load_pgm(b"P2\n2 1\n255\n3 4\n").pixels, [[3.0, 4.0]])
    with pytest.raises(ef.PgmFormatError):
        ef.load_pgm(b"P6\n1 1\n255\n\x00")
    with pytest.raises(ef.PgmFormatError):
        ef.load_pgm(b"P5\n4 4\n255\n\x00\x00")


def test_edges_to_image_and_auto_thresholds():
    em = ef.EdgeMap(width=2, height=1, labels=np.array([[2, 0]], np.uint8), final=np.array([[True, False]]))
    assert ef.edges_to_image(em).pixels.tolist() == [[255.0, 0.0]]
    t = ef.auto_thresholds(ef.ThinnedField(width=3, height=1, magnitude=np.array([[0.0, 10.0, 5.0]])))
    assert (t.low, t.high) == (0.4 * (0.2 * 10.0), 0.2 * 10.0)
    assert ef.auto_thresholds(ef.ThinnedField(width=1, height=1, magnitude=np.zeros((1, 1)))).high == 1.0


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    img = ef.GrayImage.from_array(np.zeros((4, 4)))
    with pytest.raises(RuntimeError, match="CUDA"):
        ef.run_pipeline(img, ef.PipelineConfig(thresholds=ef.Thresholds(1.0, 2.0)))
    with pytest.raises(RuntimeError, match="CUDA"):
        ef.trace_edges(ef.EdgeMap(width=1, height=1, labels=np.zeros((1, 1), np.uint8)))


def test_unpack_codes_matches_scalar_decode(tmp_path):
    """The host unpack of the packed (labels, final) stream (SIMD and scalar
    paths, every alignment) -- compiled against the built library."""
    import shutil
    import subprocess
    from paper_1710_07745_b200 import build as B

    if shutil.which("g++") is None:
        pytest.skip("no g++")
    lib = B.build()
    exe = tmp_path / "unpack_check"
    src = os.path.join(os.path.dirname(__file__), "native", "unpack_check.cpp")
    subprocess.run(["g++", "-O2", "-o", str(exe), src, lib, f"-Wl,-rpath,{os.path.dirname(lib)}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "unpack ok" in out


def test_host_f64_to_u8_integer_test():
    """GrayImage.as_u8 (the drop-in's fast-path test) through the library's
    threaded float64 -> u8 pass: integers in [0,255] convert, anything else
    (fractions, out of range, negatives) routes to the float64 path."""
    rng = np.random.default_rng(7)
    a = rng.integers(0, 256, size=(517, 1031)).astype(np.float64)
    u8 = ef.GrayImage.from_array(a).as_u8()
    assert u8 is not None and u8.dtype == np.uint8 and np.array_equal(u8, a)
    for bad in (0.5, 255.5, 256.0, -1.0, 1e9):
        b = a.copy()
        b[rng.integers(0, 517), rng.integers(0, 1031)] = bad
        assert ef.GrayImage.from_array(b).as_u8() is None, bad
    assert ef.GrayImage.from_array(np.zeros((3, 5))).as_u8() is not None


def test_host_f64_to_u8_vector_body_and_tail():
    """ef_host_f64_to_u8 directly: the 8-wide vector body and the scalar tail agree
    with numpy for every length 0..40 and for a bad value at every position --
    NaN, +-inf, -0.0 (an integer: accepted), 2^31, 2^53, denormals, 255 + 1ulp."""
    lib = _lib.load()
    rng = np.random.default_rng(9)

    def call(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.full(a.size + 8, 0xAB, np.uint8)
        rc = lib.ef_host_f64_to_u8(a.ctypes.data, a.size, out.ctypes.data)
        assert (out[a.size:] == 0xAB).all()
        return rc, out[:a.size]

    for n in range(0, 41):
        a = rng.integers(0, 256, n).astype(np.float64)
        rc, out = call(a)
        assert rc == 1 and np.array_equal(out, a.astype(np.uint8)), n
    base = rng.integers(0, 256, 37).astype(np.float64)
    bads = [np.nan, np.inf, -np.inf, 2.0 ** 31, -2.0 ** 31, 2.0 ** 53, 5e-324, -5e-324, np.nextafter(255.0, 256.0),
            np.nextafter(0.0, -1.0), 0.5, -1.0, 256.0, 1e300]
    for pos in range(37):
        for bad in bads:
            b = base.copy()
            b[pos] = bad
            assert call(b)[0] == 0, (pos, bad)
        b = base.copy()
        b[pos] = -0.0
        rc, out = call(b)
        assert rc == 1 and out[pos] == 0


def _canny_u8_call(weights, ws_ptr=None, ws_bytes=1 << 30):
    """ef_canny_u8 with dummy device pointers: argument validation runs on the
    host before anything touches a device, so the status and message are
    observable without a GPU."""
    lib = _lib.load()
    w = np.ascontiguousarray(weights, dtype=np.float64)
    r = (len(w) - 1) // 2
    rc = lib.ef_canny_u8(0x1000, 1, 8, 8, w.ctypes.data, r, 20.0, 50.0, 0x2000, 0x3000, ws_ptr, ws_bytes, None)
    return rc, lib.ef_last_error().decode()


def test_abi_weight_sum_tolerance_matches_gaussian_kernel():
    """check_params mirrors GaussianKernel (filtering.py:25-26): |sum - 1| <= 1e-12
    with numpy's summation order; beyond it EF_EINVAL (ValueError)."""
    good = ef.build_gaussian_kernel(1.4, radius=5).weights
    rc, msg = _canny_u8_call(good)  # valid weights: fails later, on the NULL workspace
    assert rc == _lib.EF_EINVAL and "workspace" in msg
    for eps in (3e-12, 1e-10, 1e-9 / 2):
        bad = np.array(good, copy=True)
        bad[5] += eps
        rc, msg = _canny_u8_call(bad)
        assert rc == _lib.EF_EINVAL and "sum to 1" in msg, eps
        with pytest.raises(ValueError):
            ef.GaussianKernel(sigma=1.4, radius=5, weights=bad)
    # accepted / rejected exactly where the Python mirror (numpy sum) says so
    rng = np.random.default_rng(4)
    for _ in range(300):
        r = int(rng.integers(0, 16))
        half = rng.random(r + 1) + 0.1
        w = np.concatenate([half[:0:-1], half]) if r else half[:1]
        w = w / w.sum()
        w = w + (rng.integers(-3, 4) * 2e-13 if rng.random() < 0.5 else 0.0)
        w = (w + w[::-1]) / 2.0
        ok = abs(w.sum() - 1.0) <= 1e-12
        rc, msg = _canny_u8_call(w)
        assert ("sum to 1" not in msg) == ok, (r, w.sum() - 1.0)


def test_abi_rejects_misaligned_workspace():
    w = ef.build_gaussian_kernel(1.4, radius=2).weights
    rc, msg = _canny_u8_call(w, ws_ptr=0x100010)
    assert rc == _lib.EF_EINVAL and "256-byte aligned" in msg


def test_portable_host_build_compiles():
    """ef_host.cu builds without the x86 intrinsics (aarch64 / Grace hosts):
    the portable branch, forced with -DEF_PORTABLE_HOST."""
    import subprocess
    import tempfile

    from paper_1710_07745_b200 import build as B

    with tempfile.TemporaryDirectory() as d:
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, "-DEF_PORTABLE_HOST", "-c", os.path.join(B.CSRC, "ef_host.cu"), "-o",
               os.path.join(d, "h.o")]
        res = subprocess.run(cmd, capture_output=True, text=True)
        assert res.returncode == 0, res.stderr


def test_band_meta_must_be_contiguous_in_rank_order():
    bands.check_band_meta([(0, 10), (10, 5), (15, 1)], 16)
    for meta, h in (([(10, 6), (0, 10)], 16), ([(0, 10), (11, 5)], 16), ([(0, 10), (10, 5)], 16),
                    ([(0, 0), (0, 16)], 16)):
        with pytest.raises(ValueError):
            bands.check_band_meta(meta, h)


def test_pgm_codec_matches_reference_corpus():
    """load_pgm / save_pgm (image.py:87-135) against the reference's own results
    on a seeded corpus of valid and malformed files: pixels, PgmFormatError
    message and byte offset, save_pgm bytes.  Host parsing in the library."""
    from golden_data import load

    g = load("pgm.npz")
    n_ok = n_err = 0
    for i in range(int(g["n"])):
        data = g[f"in/{i}"].tobytes()
        if f"err/{i}" in g.files:
            with pytest.raises(ef.PgmFormatError) as ei:
                ef.load_pgm(data)
            assert str(ei.value) == str(g[f"err/{i}"]), (i, data[:40])
            assert ei.value.offset == int(g[f"off/{i}"]), (i, data[:40])
            n_err += 1
        else:
            img = ef.load_pgm(data)
            assert img.pixels.dtype == np.float64 and np.array_equal(img.pixels, g[f"px/{i}"]), i
            assert ef.save_pgm(img) == g[f"save/{i}"].tobytes(), i
            assert np.array_equal(ef.decode_pgm_u8(data), g[f"px/{i}"]), i
            n_ok += 1
    assert n_ok >= 30 and n_err >= 40
