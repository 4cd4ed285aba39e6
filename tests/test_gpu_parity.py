"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle
and the reference-generated golden fixtures.  Bar: bit-exact labels and final
edge sets (integer work); float64 intermediates bit-exact as well.
"""

import numpy as np
import pytest

from golden_data import load, unpack
from oracle import oracle as O
from paper_1710_07745_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def canny():
    from paper_1710_07745_b200 import canny as c

    c.require_cuda()
    return c


@pytest.fixture(params=[(0, True), (32, True), (0, False)],
                ids=["warp-per-tile", "block-per-tile-when-few", "warp-per-tile-no-reach"])
def h1_path(request, canny):
    """The hysteresis tile passes: threshold 0 = always one warp per tile (with
    the dense tile hand-over), 32 = one block per tile for launches with at
    most 32 tiles per SM (the default is 8); reach = the tile-local reach prefilter before
    the union-find (default on; off: union-find over every weak pixel)."""
    thr, reach = request.param
    canny.set_block_tile_threshold(thr)
    canny.set_tile_reach(reach)
    yield request.param
    canny.set_block_tile_threshold(8)
    canny.set_tile_reach(True)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _np(t):
    return t.cpu().numpy()


# ---------------------------------------------------------------- golden ----
@pytest.mark.parametrize("cfg", range(5))
@pytest.mark.parametrize("r", [2, 5])
def test_configs_match_reference_golden(canny, cfg, r, h1_path):
    g = load("configs.npz")
    frames = synth.make_config(cfg, reduced=True)
    assert synth.sha256_u8(frames) == str(g[f"c{cfg}/sha256"])
    low, high = synth.CONFIG_THRESHOLDS[cfg]
    w = g[f"c{cfg}/r{r}/weights"]
    lab, fin = canny.canny_u8(_dev(frames), w, low, high)
    assert np.array_equal(_np(lab), g[f"c{cfg}/r{r}/labels"])
    assert np.array_equal(_np(fin).astype(bool), unpack(g[f"c{cfg}/r{r}/final"], frames.shape))


def test_stages_match_reference_golden(canny):
    g = load("stages.npz")
    for name in [str(n) for n in g["names"]]:
        arr = g[f"{name}/input"]
        low, high = g[f"{name}/thresholds"]
        st = canny.stages_f64(_dev(arr), g[f"{name}/weights"], low, high)
        for key in ("blurred", "gx", "gy", "magnitude", "orientation", "thinned", "labels"):
            assert np.array_equal(_np(st[key]), g[f"{name}/{key}"]), (name, key)
        if np.array_equal(arr, np.floor(arr)) and arr.min() >= 0 and arr.max() <= 255:
            lab, fin = canny.canny_u8(_dev(arr.astype(np.uint8)), g[f"{name}/weights"], low, high)
            assert np.array_equal(_np(lab)[0], g[f"{name}/labels"]), name
            assert np.array_equal(_np(fin)[0].astype(bool), g[f"{name}/final"]), name
        lab, fin = canny.canny_f64(_dev(arr), g[f"{name}/weights"], low, high)
        assert np.array_equal(_np(lab)[0], g[f"{name}/labels"]), name
        assert np.array_equal(_np(fin)[0].astype(bool), g[f"{name}/final"]), name


def test_dropin_run_pipeline_matches_reference_golden():
    import paper_1710_07745_b200 as ef

    g = load("pipeline.npz")
    for name in [str(n) for n in g["names"]]:
        arr = g[f"{name}/input"]
        img = ef.GrayImage.from_array(arr)
        for tag, thr in (("t2050", ef.Thresholds(20.0, 50.0)), ("auto", None), ("t00", ef.Thresholds(0.0, 0.0)),
                         ("t0_30", ef.Thresholds(0.0, 30.0)), ("tbig", ef.Thresholds(1e9, 1e9))):
            res = ef.run_pipeline(img, ef.PipelineConfig(sigma=1.4, thresholds=thr))
            assert np.array_equal(res.edges.labels, g[f"{name}/{tag}/labels"]), (name, tag)
            assert np.array_equal(res.edges.final, unpack(g[f"{name}/{tag}/final"], arr.shape)), (name, tag)
            assert (res.thresholds.low, res.thresholds.high) == tuple(g[f"{name}/{tag}/thresholds"]), (name, tag)
        res = ef.run_pipeline(img, ef.PipelineConfig(thresholds=ef.Thresholds(20.0, 50.0), hysteresis_mode="parallel",
                                                     workers=ef.WorkerConfig(workers=3, band_granularity=2)))
        assert np.array_equal(res.edges.final, unpack(g[f"{name}/t2050/final"], arr.shape)), name


# ------------------------------------------------------- random vs oracle ----
def _random_image(rng, h, w, kind):
    if kind == "noise":
        return rng.integers(0, 256, (h, w)).astype(np.uint8)
    if kind == "blocks":
        blk = rng.integers(0, 2, (h // 8 + 1, w // 8 + 1)) * 255
        return np.kron(blk, np.ones((8, 8)))[:h, :w].astype(np.uint8)
    y, x = np.mgrid[0:h, 0:w]
    return ((x * 7 + y * 3) % 256).astype(np.uint8)


@pytest.mark.parametrize("r", [0, 1, 2, 3, 4, 5, 6, 7, 8, 15])
def test_fast_path_random_vs_oracle(canny, r, h1_path):
    rng = np.random.default_rng(100 + r)
    sigma = max(0.3, r / 3.0)
    w = O.gaussian_weights(sigma, radius=r)
    shapes = [(1, 1), (1, 37), (29, 1), (2, 3), (31, 65), (64, 64), (97, 130), (200, 333),
              (1, 4), (3, 8), (5, 128), (7, 120), (66, 124), (130, 244), (67, 500), (129, 1024)]
    for (h, wd) in shapes:
        for kind in ("noise", "blocks", "ramp"):
            img = _random_image(rng, h, wd, kind)
            low = float(rng.choice([0.0, 5.0, 20.0, 100.0]))
            high = low + float(rng.choice([0.0, 10.0, 40.0, 300.0]))
            lab, fin = canny.canny_u8(_dev(img), w, low, high)
            el, ef_ = O.canny(img, w, low, high)
            assert np.array_equal(_np(lab)[0], el), (r, h, wd, kind, low, high)
            assert np.array_equal(_np(fin)[0].astype(bool), ef_), (r, h, wd, kind, low, high)


@pytest.mark.parametrize("density", ["sparse", "mixed", "dense"])
def test_fused_foreground_lists_vs_two_call_path(canny, density):
    """ef_canny_u8 builds per-tile foreground lists in the classifier (final
    prefilled with the strong pixels); ef_classify_u8 + ef_trace_edges rescans
    the labels.  Both must equal the oracle -- including tiles whose list
    overflows (dense noise) and frames whose size is not a multiple of 64."""
    rng = np.random.default_rng({"sparse": 1, "mixed": 2, "dense": 3}[density])
    w = O.gaussian_weights(1.4, radius=2)
    for (b, h, wd) in [(2, 130, 200), (1, 64, 128), (3, 97, 252)]:
        if density == "sparse":
            frames = synth.config1(b, h, wd)
        elif density == "mixed":
            frames = synth.config1(b, h, wd)
            frames[:, : h // 2, : wd // 2] = rng.integers(0, 256, size=(b, h // 2, wd // 2), dtype=np.uint8)
        else:
            frames = rng.integers(0, 256, size=(b, h, wd), dtype=np.uint8)
        lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
        lab2 = canny.classify_u8(_dev(frames), w, 20.0, 50.0)
        fin2 = canny.trace_edges_u8(lab2)
        el, ef_ = O.canny(frames, w, 20.0, 50.0)
        assert np.array_equal(_np(lab), el) and np.array_equal(_np(lab2), el)
        assert np.array_equal(_np(fin).astype(bool), ef_), (density, b, h, wd)
        assert np.array_equal(_np(fin2).astype(bool), ef_), (density, b, h, wd)


def test_workspace_reuse_across_inputs_and_shapes(canny):
    """One workspace, dirtied by a dense noise batch, reused for smaller and
    differently shaped sparse batches (stale perimeter slots, bit planes and list
    counters must never leak into a later call), and by the two-call path."""
    import torch
    rng = np.random.default_rng(11)
    w = O.gaussian_weights(1.4, radius=2)
    big = (3, 256, 320)
    ws = torch.full((canny.new_workspace(*big).numel(),), 0xA5, dtype=torch.uint8, device="cuda")
    cases = [rng.integers(0, 256, size=big, dtype=np.uint8), synth.config1(2, 130, 200), synth.config1(3, 256, 320),
             synth.config1(1, 64, 64), rng.integers(0, 256, size=(2, 200, 96), dtype=np.uint8)]
    for frames in cases:
        el, ef_ = O.canny(frames, w, 20.0, 50.0)
        lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0, ws=ws)
        assert np.array_equal(_np(lab), el) and np.array_equal(_np(fin).astype(bool), ef_), frames.shape
        lab2 = canny.classify_u8(_dev(frames), w, 20.0, 50.0, ws=ws)
        fin2 = canny.trace_edges_u8(lab2, ws=ws)
        assert np.array_equal(_np(fin2).astype(bool), ef_), frames.shape


@pytest.mark.parametrize("low,high", [(5.0, 100.0), (2.0, 400.0)])
def test_dense_noise_overflow_paths(canny, low, high, h1_path):
    """Dense noise with low thresholds: tiles beyond the warp kernel's capacity
    (block-kernel path), node and pending-list stripes that overflow (perimeter
    scan / tile re-run fallbacks) -- all must still equal the oracle."""
    rng = np.random.default_rng(int(low * 10 + high))
    frames = rng.integers(0, 256, size=(1, 2048, 2048), dtype=np.uint8)
    w = O.gaussian_weights(0.6, radius=1)
    el, ef_ = O.canny(frames, w, low, high)
    ws = canny.new_workspace(*frames.shape)
    lab, fin = canny.canny_u8(_dev(frames), w, low, high, ws=ws)
    paths = canny.read_paths(ws)
    # the fallbacks this test is for ran at the lower threshold (a third of the
    # pixels weak): the pending-list overflow and (one warp per tile) the
    # hand-over of tiles with more than 512 weak pixels to the block kernel; at
    # 5 / 100 a third of the pixels are strong and only 0.3% weak
    assert paths["pending_overflow"] == (low < 5.0), paths
    thr, reach = h1_path
    if not reach:  # with the reach prefilter a tile's union-find input rarely exceeds the warp's lists
        assert (paths["dense_tiles"] > 0) == (thr == 0 and low < 5.0), paths
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)
    lab2 = canny.classify_u8(_dev(frames), w, low, high)
    assert np.array_equal(_np(canny.trace_edges_u8(lab2)).astype(bool), ef_)


@pytest.mark.parametrize("low,high", [(48.0, 48.0), (16.0, 48.0)])
def test_fix_list_overflow_on_threshold_ties(canny, low, high):
    """Binary blocks with a dyadic kernel make magnitudes exactly 16, 48, ...:
    thresholds on those values put ~13% of the pixels inside the certification
    bands (and NMS plateaus), far more than the fix list holds -- the full-scan
    fix-up must still reproduce the reference exactly."""
    rng = np.random.default_rng(3)
    blk = rng.choice(np.array([0, 16], np.uint8), size=(512, 512))
    frames = np.kron(blk, np.ones((4, 4), np.uint8))[None]
    w = np.array([0.25, 0.5, 0.25])
    el, ef_ = O.canny(frames, w, low, high)
    ws = canny.new_workspace(*frames.shape)
    lab, fin = canny.canny_u8(_dev(frames), w, low, high, ws=ws)
    assert canny.read_paths(ws)["fix_overflow"]  # the full-scan fix-up ran
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)


def test_node_list_overflow_large_noise(canny):
    """8192^2 noise with a third of the pixels weak: ~45 weak border components
    per 64x64 tile, beyond the node-list capacity (32 per tile), so the resolve
    pass falls back to scanning every perimeter slot."""
    rng = np.random.default_rng(8192)
    frames = rng.integers(0, 256, size=(1, 8192, 8192), dtype=np.uint8)
    w = O.gaussian_weights(0.6, radius=1)
    el, ef_ = O.canny(frames, w, 2.0, 400.0)
    ws = canny.new_workspace(*frames.shape)
    lab, fin = canny.canny_u8(_dev(frames), w, 2.0, 400.0, ws=ws)
    assert canny.read_paths(ws)["node_overflow"]  # H3's perimeter-scan fallback ran
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)


def test_signed_kernel_takes_exact_path(canny):
    """A kernel with negative taps (GaussianKernel accepts any weights) is not
    covered by the fp32 certification: the exact float64 kernel runs, followed by
    the same hysteresis -- through the fused entry and through run_pipeline."""
    rng = np.random.default_rng(21)
    w = np.array([-0.05, 0.3, 0.5, 0.3, -0.05])
    for _ in range(2):  # twice: the second call must not see the first one's counters
        frames = synth.config1(2, 130, 200)
        frames[1] = rng.integers(0, 256, size=frames.shape[1:], dtype=np.uint8)
        el, ef_ = O.canny(frames, w, 20.0, 50.0)
        lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
        assert np.array_equal(_np(lab), el) and np.array_equal(_np(fin).astype(bool), ef_)


def test_float_path_random_vs_oracle(canny):
    rng = np.random.default_rng(5)
    for (h, wd) in [(1, 1), (7, 5), (33, 47), (128, 96)]:
        img = rng.random((h, wd)) * 300.0 - 20.0
        w = O.gaussian_weights(1.4)
        lab, fin = canny.canny_f64(_dev(img), w, 10.0, 40.0)
        el, ef_ = O.canny(img, w, 10.0, 40.0)
        assert np.array_equal(_np(lab)[0], el)
        assert np.array_equal(_np(fin)[0].astype(bool), ef_)


def test_batch_of_frames_vs_oracle(canny):
    frames = synth.config1(3, 135, 241)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    el, ef_ = O.canny(frames, w, 20.0, 50.0, threads=8)
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)
    for i in range(3):  # batch invariance
        l1, f1 = canny.canny_u8(_dev(frames[i]), w, 20.0, 50.0)
        assert np.array_equal(_np(l1)[0], _np(lab)[i])
        assert np.array_equal(_np(f1)[0], _np(fin)[i])


def test_concurrent_calls_from_host_threads(canny):
    """Distinct runs may run concurrently (one orchestrating thread per run):
    four host threads, each with its own stream and workspace, issue fused calls
    on different frame sizes at once; every result equals the oracle."""
    import threading

    w = O.gaussian_weights(1.4, radius=2)
    shapes = [(2, 135, 241), (1, 300, 512), (3, 97, 160), (1, 512, 128)]
    inputs = [synth.config1(*sh) for sh in shapes]
    want = [O.canny(f, w, 20.0, 50.0, threads=4) for f in inputs]
    got, errors = [None] * len(shapes), []

    def run(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                x = _dev(inputs[k])
                ws = canny.new_workspace(*inputs[k].shape)
                for _ in range(5):  # overlap several calls per thread
                    lab, fin = canny.canny_u8(x, w, 20.0, 50.0, ws=ws, stream=st)
                st.synchronize()
                got[k] = (_np(lab), _np(fin))
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(len(shapes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (lab, fin), (el, ef_) in zip(got, want):
        assert np.array_equal(lab, el)
        assert np.array_equal(fin.astype(bool), ef_)


# ----------------------------------------------------------- hysteresis -----
def _snake(h, w):
    lab = np.zeros((h, w), np.uint8)
    for y in range(0, h, 2):
        lab[y, :] = 1
        if y + 1 < h:
            lab[y + 1, (w - 1) if (y // 2) % 2 == 0 else 0] = 1
    lab[h - 1 - ((h - 1) % 2), 0] = 2
    return lab


def _spiral_labels(n):
    lab = np.zeros((n, n), np.uint8)
    y, x, dy, dx = 0, 0, 0, 1
    seen = np.zeros((n, n), bool)
    for _ in range(n * n):
        lab[y, x] = 1
        seen[y, x] = True
        ny, nx = y + 2 * dy, x + 2 * dx
        if not (0 <= ny < n and 0 <= nx < n) or seen[ny, nx]:
            dy, dx = dx, -dy
            ny, nx = y + 2 * dy, x + 2 * dx
            if not (0 <= ny < n and 0 <= nx < n) or seen[ny, nx]:
                break
        lab[y + dy, x + dx] = 1
        seen[y + dy, x + dx] = True
        y, x = ny, nx
    lab[y, x] = 2
    return lab


def test_hysteresis_vs_oracle(canny, h1_path):
    rng = np.random.default_rng(3)
    cases = [_snake(300, 257), _spiral_labels(333), _snake(64, 64), _snake(65, 129)]
    for p in ([0.55, 0.35, 0.10], [0.3, 0.65, 0.05], [0.9, 0.09, 0.01]):
        for (h, w) in [(1, 1), (1, 200), (200, 1), (63, 65), (128, 128), (517, 389)]:
            cases.append(rng.choice([0, 1, 2], size=(h, w), p=p).astype(np.uint8))
    for lab in cases:
        fin = canny.trace_edges_u8(_dev(lab))
        assert np.array_equal(_np(fin)[0].astype(bool), O.trace(lab)), lab.shape
    # the snake and the spiral are single components reaching every tile
    assert _np(canny.trace_edges_u8(_dev(_spiral_labels(333))))[0].sum() == (_spiral_labels(333) != 0).sum()


def _maze(h, w, rng):
    """A random spanning-tree maze of 1-pixel corridors (one component), weak
    everywhere: paths wind up, down, left and right across many tiles."""
    ch, cw = (h - 1) // 2, (w - 1) // 2
    lab = np.zeros((h, w), np.uint8)
    seen = np.zeros((ch, cw), bool)
    stack = [(0, 0)]
    seen[0, 0] = True
    lab[1, 1] = 1
    while stack:
        y, x = stack[-1]
        nb = [(y + dy, x + dx) for dy, dx in ((0, 1), (1, 0), (0, -1), (-1, 0))
              if 0 <= y + dy < ch and 0 <= x + dx < cw and not seen[y + dy, x + dx]]
        if not nb:
            stack.pop()
            continue
        ny, nx = nb[rng.integers(len(nb))]
        seen[ny, nx] = True
        lab[2 * ny + 1, 2 * nx + 1] = 1
        lab[y + ny + 1, x + nx + 1] = 1
        stack.append((ny, nx))
    return lab


@pytest.mark.parametrize("shape", [(257, 129), (301, 1999), (1025, 2048), (67, 64 * 33 + 5)])
def test_hysteresis_mazes_vs_oracle(canny, shape, h1_path):
    """Long winding weak paths: a maze whose one strong cell makes the whole
    maze an edge, mazes cut into many components with a few strong cells, and
    a snake -- against the oracle."""
    rng = np.random.default_rng(sum(shape))
    h, w = shape
    full = _maze(h, w, rng)
    ys, xs = np.nonzero(full)
    full[ys[-1], xs[-1]] = 2
    cut = _maze(h, w, rng)
    cut[rng.random(cut.shape) < 0.02] = 0
    ys, xs = np.nonzero(cut)
    cut[ys[:3], xs[:3]] = 2
    for lab in (full, cut, _snake(h, w)):
        fin = canny.trace_edges_u8(_dev(lab))
        assert np.array_equal(_np(fin)[0].astype(bool), O.trace(lab)), shape
    assert _np(canny.trace_edges_u8(_dev(full)))[0].sum() == (full != 0).sum()


def test_band_paths_match_whole_frame(canny):
    from paper_1710_07745_b200 import bands

    frame = synth.config4(1024, tile=256)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frame), w, 20.0, 50.0)
    for nb in (2, 3, 8):
        bl, bf = bands.canny_bands_local(_dev(frame), nb, w, 20.0, 50.0)
        assert np.array_equal(_np(bl), _np(lab)[0]), nb
        assert np.array_equal(_np(bf), _np(fin)[0]), nb
    snake = _snake(300, 257)
    ref = O.trace(snake)
    for plan in ([(0, 100), (100, 300)], [(0, 7), (7, 8), (8, 150), (150, 300)]):
        got = bands.trace_bands_local(_dev(snake), plan)
        assert np.array_equal(_np(got).astype(bool), ref), plan


def test_device_band_merge_matches_host_merge(canny):
    """ef_band_merge_device (band-local ids, union-find on the GPU) against the
    host ef_band_merge on globalised ids: random edge rows with heavy id reuse
    (components spanning many columns), empty bands, one band, width 1, and a
    chain crossing every seam."""
    from paper_1710_07745_b200 import bands

    rng = np.random.default_rng(11)
    cases = []
    for nb, w, nid, p_bg in [(2, 64, 5, 0.3), (8, 1000, 40, 0.5), (5, 1, 2, 0.2), (1, 77, 9, 0.1),
                             (16, 4096, 3000, 0.6), (3, 50, 50, 1.0), (8, 16384, 200, 0.9)]:
        ids = rng.integers(0, nid, size=(nb, 2 * w)).astype(np.int64) * 7 + 3  # sparse, large local ids
        ids[rng.random((nb, 2 * w)) < p_bg] = -1
        strong = (rng.random((nb, 2 * w)) < 0.05).astype(np.uint8)
        strong[ids < 0] = 0
        cases.append((ids, strong))
    # one component snaking through every seam, strong only in the last band
    nb, w = 6, 32
    ids = np.full((nb, 2 * w), -1, np.int64)
    strong = np.zeros((nb, 2 * w), np.uint8)
    for k in range(nb):
        ids[k, 5] = ids[k, w + 6] = 100 + k  # top x=5 and bottom x=6 are one band-local component
    strong[nb - 1, 5] = 1
    cases.append((ids, strong))
    for ids, strong in cases:
        nb, w = ids.shape[0], ids.shape[1] // 2
        gids = np.stack([bands.globalize_ids(ids[k], k) for k in range(nb)])
        want = bands.merge_edges(gids, strong, w)
        got = _np(bands.merge_edges_device(_dev(ids), _dev(strong), w))
        assert np.array_equal(got, want), (nb, w)
    assert want[0, 5] == 1  # the snake's strong pixel reached the first band


def test_host_buffer_entry_matches_device(canny):
    frames = synth.config3(3, 256)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    hl, hf = canny.canny_u8_host(frames, w, 20.0, 50.0)
    assert np.array_equal(hl, _np(lab)) and np.array_equal(hf, _np(fin))


@pytest.mark.parametrize("shape", [(5, 67, 131), (7, 33, 64), (1, 1, 3), (9, 120, 160)])
def test_host_entry_packed_transfer_shapes(canny, shape):
    """Host path ships (labels, final) packed to 2 bits/px and unpacks on the host:
    odd pixel counts, chunk tails and single pixels must round-trip exactly."""
    rng = np.random.default_rng(sum(shape))
    frames = rng.integers(0, 256, size=shape, dtype=np.uint8)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    hl, hf = canny.canny_u8_host(frames, w, 20.0, 50.0)
    assert np.array_equal(hl, _np(lab)) and np.array_equal(hf, _np(fin))


def test_host_entry_pinned_pageable_and_misaligned_outputs(canny):
    import torch
    frames = synth.config3(6, 128)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    lab, fin = _np(lab), _np(fin)
    # pinned input
    pin = torch.from_numpy(frames).pin_memory()
    hl = np.empty(frames.shape, np.uint8)
    hf = np.empty(frames.shape, np.uint8)
    canny.canny_u8_host_ptr(pin.data_ptr(), *frames.shape, w, 20.0, 50.0, hl.ctypes.data, hf.ctypes.data)
    assert np.array_equal(hl, lab) and np.array_equal(hf, fin)
    # pageable input, outputs at different 16-byte phases
    big_l = np.full(frames.size + 64, 7, np.uint8)
    big_f = np.full(frames.size + 64, 7, np.uint8)
    ol = big_l[3:3 + frames.size].reshape(frames.shape)
    of = big_f[8:8 + frames.size].reshape(frames.shape)
    canny.canny_u8_host_ptr(frames.ctypes.data, *frames.shape, w, 20.0, 50.0, ol.ctypes.data, of.ctypes.data)
    assert np.array_equal(ol, lab) and np.array_equal(of, fin)
    assert (big_l[:3] == 7).all() and (big_l[3 + frames.size:] == 7).all()
    assert (big_f[:8] == 7).all() and (big_f[8 + frames.size:] == 7).all()
    # device-resident "host" pointer (cudaMemcpyDefault path)
    d = _dev(frames)
    canny.canny_u8_host_ptr(d.data_ptr(), *frames.shape, w, 20.0, 50.0, hl.ctypes.data, hf.ctypes.data)
    assert np.array_equal(hl, lab) and np.array_equal(hf, fin)


@pytest.mark.parametrize("shape", [(5, 67, 131), (7, 33, 64), (1, 1, 3), (1, 1, 9), (9, 120, 160), (3, 256, 256)])
def test_host_entry_edges_only(canny, shape):
    """h_labels == NULL: the edge map alone crosses PCIe at 1 bit/px; the bytes
    written equal the oracle's final map (odd pixel counts, chunk tails, outputs at
    odd addresses with guard bytes around them)."""
    rng = np.random.default_rng(sum(shape) + 1)
    frames = synth.config3(shape[0], 256)[:, :shape[1], :shape[2]].copy() if shape[1] > 8 else \
        rng.integers(0, 256, size=shape, dtype=np.uint8)
    w = O.gaussian_weights(1.4, radius=2)
    _, want = O.canny(frames, w, 20.0, 50.0)
    none, hf = canny.canny_u8_host(frames, w, 20.0, 50.0, edges_only=True)
    assert none is None and np.array_equal(hf.astype(bool), want)
    assert set(np.unique(hf)) <= {0, 1}
    for phase in (1, 8, 32):
        big = np.full(frames.size + 96, 7, np.uint8)
        out = big[phase:phase + frames.size].reshape(frames.shape)
        canny.canny_u8_host_ptr(frames.ctypes.data, *frames.shape, w, 20.0, 50.0, 0, out.ctypes.data)
        assert np.array_equal(out.astype(bool), want)
        assert (big[:phase] == 7).all() and (big[phase + frames.size:] == 7).all()


def test_host_entry_many_chunks_pageable_input(canny):
    """A pageable input of many chunks: every chunk is staged through a pinned buffer
    that an earlier chunk's copy may still be reading, so the call waits on copy events
    (polling) between its kernel launches.  Results equal the device-resident call."""
    frames = np.tile(synth.config3(4, 512), (24, 1, 1))  # 96 frames x 512^2 = 25 MB: 8 MB chunks with ramps
    frames[::7] = frames[::7][:, ::-1].copy()
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    for _ in range(3):  # the waits depend on timing: a few calls
        hl, hf = canny.canny_u8_host(frames, w, 20.0, 50.0)
        assert np.array_equal(hl, _np(lab)) and np.array_equal(hf, _np(fin))
        _, of = canny.canny_u8_host(frames, w, 20.0, 50.0, edges_only=True)
        assert np.array_equal(of, _np(fin))
    el, ef_ = O.canny(frames[:4], w, 20.0, 50.0)
    assert np.array_equal(hl[:4], el) and np.array_equal(hf[:4].astype(bool), ef_)


def test_invalid_arguments_raise_valueerror(canny):
    w = O.gaussian_weights(1.4)
    img = _dev(np.zeros((8, 8), np.uint8))
    with pytest.raises(ValueError):
        canny.canny_u8(img, w, 50.0, 20.0)
    with pytest.raises(ValueError):
        canny.canny_u8(img, np.array([0.2, 0.5, 0.3]), 1.0, 2.0)
    with pytest.raises(ValueError):
        canny.canny_u8(img, np.ones(33) / 33, 1.0, 2.0)


# --------------------------------------------------- full-size configs ------
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_full_size_configs_vs_oracle(canny, cfg):
    frames = synth.make_config(cfg)
    low, high = synth.CONFIG_THRESHOLDS[cfg]
    w = O.gaussian_weights(1.4, radius=2)
    ws = canny.new_workspace(*frames.shape)
    canny.reset_stats(ws)
    lab, fin = canny.canny_u8(_dev(frames), w, low, high, ws=ws)
    stats = canny.read_stats(ws)
    el, ef_ = O.canny(frames, w, low, high, threads=0)
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)
    print(f"config {cfg}: {frames.size} px, stats {stats}")


def test_full_size_config4_band_invariance(canny):
    from paper_1710_07745_b200 import bands

    frame = synth.config4()
    w = O.gaussian_weights(1.4, radius=2)
    d = _dev(frame)
    lab, fin = canny.canny_u8(d, w, 20.0, 50.0)
    el, ef_ = O.canny(frame, w, 20.0, 50.0, threads=0)
    assert np.array_equal(_np(lab)[0], el)
    assert np.array_equal(_np(fin)[0].astype(bool), ef_)
    bl, bf = bands.canny_bands_local(d, 8, w, 20.0, 50.0)
    assert torch.equal(bl, lab[0]) and torch.equal(bf, fin[0])


def test_full_size_config3_subset_and_properties(canny):
    frames = synth.config3(48)
    w = O.gaussian_weights(1.4, radius=2)
    lab, fin = canny.canny_u8(_dev(frames), w, 20.0, 50.0)
    el, ef_ = O.canny(frames, w, 20.0, 50.0, threads=0)
    assert np.array_equal(_np(lab), el)
    assert np.array_equal(_np(fin).astype(bool), ef_)
    # properties: strong pixels are final, final pixels are labelled, and a
    # stricter high threshold never adds edges
    L, F = _np(lab), _np(fin).astype(bool)
    assert F[L == 2].all() and not F[L == 0].any()
    _, fin2 = canny.canny_u8(_dev(frames), w, 20.0, 80.0)
    assert not (_np(fin2).astype(bool) & ~F).any()
