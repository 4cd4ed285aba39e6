"""K1 (classify only) on one 4096^2 frame by content and row pitch: is C2's K1 time
(2x C3's per pixel) the content (classifier rounds), the 4096-byte pitch, or the
launch's size?  CUDA events, 30 timed launches after 5 warm-ups, inputs > L2 rotated."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1710_07745_b200 import canny, synth  # noqa: E402

canny.require_cuda()
w = np.asarray(canny.host_weights(__import__("paper_1710_07745_b200.filtering", fromlist=["x"]).build_gaussian_kernel(1.4, 2).weights)[0])


def timeit(frames, tag):
    b, h, wd = frames.shape
    nbuf = max(1, int(np.ceil(3 * 126e6 / frames.size)))
    srcs = [torch.from_numpy(frames).cuda() for _ in range(nbuf)]
    lab = torch.empty_like(srcs[0])
    ws = canny.new_workspace(b, h, wd)
    for i in range(5):
        canny.classify_u8(srcs[i % nbuf], w, 20.0, 50.0, labels=lab, ws=ws)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    s.record()
    for i in range(n):
        canny.classify_u8(srcs[i % nbuf], w, 20.0, 50.0, labels=lab, ws=ws)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / n * 1e3
    fg = float((lab != 0).float().mean())
    print(json.dumps({"case": tag, "shape": list(frames.shape), "us": round(us, 2),
                      "gpx_s": round(frames.size / us / 1e3, 1), "foreground": round(fg, 5)}), flush=True)


c2 = synth.make_config(2)
timeit(c2, "C2 4096^2")
c3 = synth.config_range(3, 0, 16)
mosaic = c3.reshape(4, 4, 1024, 1024).transpose(0, 2, 1, 3).reshape(1, 4096, 4096).copy()
timeit(mosaic, "C3 mosaic 4096^2")
timeit(c3, "C3 16 x 1024^2")
rng = np.random.default_rng(1)
timeit(np.full((1, 4096, 4096), 100, np.uint8), "flat 4096^2")
timeit(np.ascontiguousarray(c2[:, :, :4096 - 128]), "C2 4096 x 3968")
timeit(np.concatenate([c2, c2, c2, c2]), "C2 x 4 frames")
timeit(np.concatenate([c2] * 16), "C2 x 16 frames")
