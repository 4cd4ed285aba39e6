"""Seeded synthetic inputs for BASELINE.json's five configs.

There is no public dataset behind the reference's configs: every image is
generated here from a recorded seed.  Generators use only integer math,
IEEE-exact numpy ops (+, -, *, /, sqrt, floor) and ``numpy.random.Generator``
draws -- no transcendental ufuncs, whose SIMD dispatch differs between hosts --
so the same seed gives the same bytes on this container and on the GPU box.
(Golden fixtures store a sha256 of each generated input to prove it.)

Config map (BASELINE.json ``configs``):
  C0  512x512, seed 0: background 64, 20 rectangles + 20 disks with U(0..255)
      intensities, additive N(0, 8^2) noise, clipped and rounded.
  C1  64 frames of 1920x1080, seed 1000+i: linear ramp + 50 polygons
      (3-8 vertices, uniform intensities) + N(0, 5^2).
  C2  4096x4096, seed 2: concentric rings + an Archimedean spiral, 2 px wide,
      contrast 40 over a N(0, 10^2) background.  Thresholds 15/45.
  C3  1024 images of 1024x1024, seed 3000+i: octave-4 value noise (amplitude
      60) + 30 rectangles/disks + N(0, 8^2).
  C4  16384x16384, seed 4: tiles mixing C0-style shapes and C2-style spirals
      whose strokes cross tile (and therefore row-band) boundaries, N(0, 8^2).
"""

from __future__ import annotations

import hashlib

import numpy as np

CONFIG_THRESHOLDS = {0: (20.0, 50.0), 1: (20.0, 50.0), 2: (15.0, 45.0), 3: (20.0, 50.0), 4: (20.0, 50.0)}
CONFIG_SHAPES = {0: (1, 512, 512), 1: (64, 1080, 1920), 2: (1, 4096, 4096), 3: (1024, 1024, 1024), 4: (1, 16384, 16384)}
CONFIG_SIGMA = 1.4
CONFIG_RADIUS = 2  # the configs' "Gaussian 5x5"; the reference default is ceil(3*sigma) = 5


def sha256_u8(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.uint8).tobytes()).hexdigest()


def _finish(canvas: np.ndarray, rng: np.random.Generator, noise_sigma: float) -> np.ndarray:
    noisy = canvas + rng.normal(0.0, noise_sigma, size=canvas.shape)
    return np.clip(np.floor(noisy + 0.5), 0, 255).astype(np.uint8)


def _rect(canvas, rng, h, w, value):
    y0, y1 = np.sort(rng.integers(0, h, size=2))
    x0, x1 = np.sort(rng.integers(0, w, size=2))
    canvas[y0 : y1 + 1, x0 : x1 + 1] = value


def _disk(canvas, rng, h, w, value, rmax):
    cy, cx = int(rng.integers(0, h)), int(rng.integers(0, w))
    rad = int(rng.integers(2, max(3, rmax)))
    y0, y1 = max(0, cy - rad), min(h, cy + rad + 1)
    x0, x1 = max(0, cx - rad), min(w, cx + rad + 1)
    yy, xx = np.mgrid[y0:y1, x0:x1]
    inside = (yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad
    canvas[y0:y1, x0:x1][inside] = value


def _pseudo_angle(dx: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """Monotone in the true angle, exact arithmetic only (no atan2)."""
    p = dy / (np.abs(dx) + np.abs(dy) + 1e-300)
    return np.where(dx >= 0, 1.0 - p, 3.0 + p)


def _polygon(canvas, rng, h, w, value, size):
    n = int(rng.integers(3, 9))
    cy, cx = rng.uniform(0, h), rng.uniform(0, w)
    px = cx + rng.uniform(-size, size, n)
    py = cy + rng.uniform(-size, size, n)
    order = np.argsort(_pseudo_angle(px - px.mean(), py - py.mean()), kind="stable")
    px, py = px[order], py[order]
    x0, x1 = max(0, int(np.floor(px.min()))), min(w, int(np.floor(px.max())) + 1)
    y0, y1 = max(0, int(np.floor(py.min()))), min(h, int(np.floor(py.max())) + 1)
    if x0 >= x1 or y0 >= y1:
        return
    yy, xx = np.mgrid[y0:y1, x0:x1].astype(np.float64)
    yy += 0.5
    xx += 0.5
    inside = np.zeros(yy.shape, dtype=bool)
    for i in range(n):
        ax, ay, bx, by = px[i], py[i], px[(i + 1) % n], py[(i + 1) % n]
        crosses = (ay > yy) != (by > yy)
        with np.errstate(divide="ignore", invalid="ignore"):
            xint = ax + (yy - ay) * (bx - ax) / (by - ay)
        inside ^= crosses & (xx < xint)
    canvas[y0:y1, x0:x1][inside] = value


def _stroke(mask, xs, ys):
    """Mark a 2-px-wide stroke: the 2x2 pixel block around every sample."""
    h, w = mask.shape
    bx = np.floor(xs - 0.5).astype(np.int64)
    by = np.floor(ys - 0.5).astype(np.int64)
    for oy in (0, 1):
        for ox in (0, 1):
            yy, xx = by + oy, bx + ox
            ok = (yy >= 0) & (yy < h) & (xx >= 0) & (xx < w)
            mask[yy[ok], xx[ok]] = True


def _spiral_samples(cx, cy, a, b, turns, step=0.25):
    """Archimedean spiral r = a + b*theta sampled ~every `step` px.  cos/sin come
    from an exact-arithmetic rotation recurrence in Python floats."""
    xs, ys = [], []
    c, s, theta = 1.0, 0.0, 0.0
    total = 2.0 * 3.141592653589793 * turns
    while theta < total:
        rad = a + b * theta
        xs.append(cx + rad * c)
        ys.append(cy + rad * s)
        dth = step / max(rad, 1.0)
        # rotation by dth with 4th-order series for cos/sin (exact ops only)
        d2 = dth * dth
        cd = 1.0 - d2 / 2.0 + d2 * d2 / 24.0
        sd = dth - dth * d2 / 6.0 + dth * d2 * d2 / 120.0
        c, s = c * cd - s * sd, s * cd + c * sd
        norm = np.sqrt(c * c + s * s)
        c, s = c / norm, s / norm
        theta += dth
    return np.array(xs), np.array(ys)


def _rings_and_spiral(h, w, rng, cy, cx, extent, bg, contrast):
    mask = np.zeros((h, w), dtype=bool)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    dist = np.sqrt((yy - cy) ** 2 + (xx - cx) ** 2)
    spacing = max(8.0, extent / 24.0)
    k = np.floor(dist / spacing + 0.5)
    mask |= (np.abs(dist - k * spacing) < 1.0) & (k >= 1) & (dist < extent * 0.45)
    sx, sy = _spiral_samples(cx + extent * 0.5 * rng.uniform(-0.1, 0.1), cy, 2.0,
                             extent / 120.0, turns=10)
    _stroke(mask, sx, sy)
    canvas = np.full((h, w), float(bg))
    canvas[mask] = bg + contrast
    return canvas


def config0(seed: int = 0, size: int = 512) -> np.ndarray:
    rng = np.random.default_rng(seed)
    canvas = np.full((size, size), 64.0)
    for _ in range(20):
        _rect(canvas, rng, size, size, float(rng.integers(0, 256)))
    for _ in range(20):
        _disk(canvas, rng, size, size, float(rng.integers(0, 256)), size // 8)
    return _finish(canvas, rng, 8.0)


def config1_frame(index: int, height: int = 1080, width: int = 1920, base_seed: int = 1000) -> np.ndarray:
    rng = np.random.default_rng(base_seed + index)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    gx, gy = rng.uniform(-1, 1, 2)
    ramp = 128.0 + 100.0 * (gx * (xx / width - 0.5) + gy * (yy / height - 0.5))
    canvas = ramp
    for _ in range(50):
        _polygon(canvas, rng, height, width, float(rng.integers(0, 256)), min(height, width) / 6)
    return _finish(canvas, rng, 5.0)


def config1(frames: int = 64, height: int = 1080, width: int = 1920, workers: int | None = None) -> np.ndarray:
    out = np.empty((frames, height, width), dtype=np.uint8)
    return _fill_parallel(out, lambda i: config1_frame(i, height, width), workers)


def config2(size: int = 4096, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    canvas = _rings_and_spiral(size, size, rng, size / 2.0, size / 2.0, float(size), 100, 40)
    return _finish(canvas, rng, 10.0)


def _value_noise(rng, h, w, octaves=4, amplitude=60.0):
    out = np.zeros((h, w))
    amp, total = 1.0, 0.0
    for o in range(octaves):
        cells = 4 << o
        lat = rng.uniform(-1.0, 1.0, size=(cells + 1, cells + 1))
        fy = np.arange(h, dtype=np.float64) * cells / h
        fx = np.arange(w, dtype=np.float64) * cells / w
        iy, ix = np.floor(fy).astype(np.int64), np.floor(fx).astype(np.int64)
        ty, tx = fy - iy, fx - ix
        ty = ty * ty * (3.0 - 2.0 * ty)
        tx = tx * tx * (3.0 - 2.0 * tx)
        # x-interpolate each lattice row once, then pick rows per image row: the
        # same operations on the same operands as a per-pixel 2-D gather
        la, lb = lat[:, ix], lat[:, ix + 1]
        rows = la + (lb - la) * tx[None, :]
        top = rows[iy]
        bot = rows[iy + 1]
        out += amp * (top + (bot - top) * ty[:, None])
        total += amp
        amp *= 0.5
    return out * (amplitude / total)


def config3_image(index: int, size: int = 1024, base_seed: int = 3000) -> np.ndarray:
    rng = np.random.default_rng(base_seed + index)
    canvas = 128.0 + _value_noise(rng, size, size)
    for _ in range(15):
        _rect(canvas, rng, size, size, float(rng.integers(0, 256)))
    for _ in range(15):
        _disk(canvas, rng, size, size, float(rng.integers(0, 256)), size // 10)
    return _finish(canvas, rng, 8.0)


def _fill_parallel(out: np.ndarray, make, workers: int | None = None) -> np.ndarray:
    """out[i] = make(i) for every i, in forked worker processes writing into a
    shared anonymous mapping (each image depends only on its own seed, so the
    bytes equal the serial loop's)."""
    import mmap
    import multiprocessing as mp
    import os

    n = len(out)
    workers = workers or min(n, len(os.sched_getaffinity(0)))
    if workers <= 1 or n < 8 or "fork" not in mp.get_all_start_methods():
        for i in range(n):
            out[i] = make(i)
        return out
    buf = mmap.mmap(-1, out.nbytes)
    shared = np.frombuffer(buf, dtype=out.dtype).reshape(out.shape)
    chunks = [range(k, n, workers) for k in range(workers)]
    pids = []
    for ch in chunks:
        pid = os.fork()
        if pid == 0:  # child: numpy only, no CUDA
            code = 0
            try:
                for i in ch:
                    shared[i] = make(i)
            except BaseException:  # noqa: BLE001
                code = 1
            os._exit(code)
        pids.append(pid)
    bad = [pid for pid in pids if os.waitpid(pid, 0)[1] != 0]
    if bad:
        raise RuntimeError(f"synthetic image workers failed: {bad}")
    out[...] = shared
    del shared
    buf.close()
    return out


def config3(images: int = 1024, size: int = 1024, workers: int | None = None) -> np.ndarray:
    out = np.empty((images, size, size), dtype=np.uint8)
    return _fill_parallel(out, lambda i: config3_image(i, size), workers)


def config4(size: int = 16384, seed: int = 4, tile: int = 2048) -> np.ndarray:
    """Tiles alternate between C0-style shapes and C2-style spirals; spirals are
    centred on tile corners so their strokes cross tile/band boundaries."""
    rng = np.random.default_rng(seed)
    canvas = np.full((size, size), 64.0)
    nt = max(1, size // tile)
    for ty in range(nt):
        for tx in range(nt):
            y0, x0 = ty * tile, tx * tile
            sub = canvas[y0 : y0 + tile, x0 : x0 + tile]
            th, tw = sub.shape
            if (ty + tx) % 2 == 0:
                for _ in range(20):
                    _rect(sub, rng, th, tw, float(rng.integers(0, 256)))
                for _ in range(20):
                    _disk(sub, rng, th, tw, float(rng.integers(0, 256)), max(3, tile // 8))
    # spirals centred on interior tile corners, drawn on the full canvas
    mask = np.zeros((size, size), dtype=bool)
    for ty in range(1, nt + 1):
        for tx in range(1, nt + 1):
            if (ty + tx) % 2:
                continue
            cy, cx = min(ty * tile, size - 1), min(tx * tile, size - 1)
            sx, sy = _spiral_samples(cx, cy, 2.0, tile / 80.0, turns=8)
            _stroke(mask, sx, sy)
    canvas[mask] = 200.0
    return _finish(canvas, rng, 8.0)


def make_config(cfg: int, reduced: bool = False) -> np.ndarray:
    """Return a (batch, H, W) uint8 array for config `cfg`.

    reduced=True gives the small variants used for oracle-checked parity tests
    (the full sizes are exercised through size-independent properties)."""
    if cfg == 0:
        return config0()[None]
    if cfg == 1:
        return config1(2, 270, 480) if reduced else config1()
    if cfg == 2:
        return config2(512 if reduced else 4096)[None]
    if cfg == 3:
        return config3(2, 256) if reduced else config3()
    if cfg == 4:
        return config4(1024, tile=256)[None] if reduced else config4()[None]
    raise ValueError(f"unknown config {cfg}")


def config_range(cfg: int, lo: int, hi: int, workers: int | None = None) -> np.ndarray:
    """Frames [lo, hi) of batched config 1 or 3 (a rank's shard): equal to
    make_config(cfg)[lo:hi], generated without the other frames."""
    if cfg == 1:
        out = np.empty((hi - lo, 1080, 1920), dtype=np.uint8)
        return _fill_parallel(out, lambda i: config1_frame(lo + i), workers)
    if cfg == 3:
        out = np.empty((hi - lo, 1024, 1024), dtype=np.uint8)
        return _fill_parallel(out, lambda i: config3_image(lo + i), workers)
    raise ValueError(f"config {cfg} is not a batch")
