"""Latency of the drop-in run_pipeline (float64 GrayImage in, host EdgeMap out)
against the reference's own run_pipeline on the same host, for one 512x512
frame (config 0) and one 1080p frame (a config-1 frame): the reference's
default kernel (radius ceil(3 sigma) = 5), thresholds 20 / 50.  The results
are compared for equality (labels and final).  Run on the GPU box:

    python tools/dropin_latency.py [--json out.json]

The reference is imported from baseline/_ref (its unmodified install); without
it only this package is timed.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1710_07745_b200 as ef  # noqa: E402
from paper_1710_07745_b200 import synth  # noqa: E402


def timed(fn, reps, warm=2):
    for _ in range(warm):
        out = fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t.append(time.perf_counter() - t0)
    return float(np.median(t)), out


def main():
    ref = None
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "edgeforge")):
        sys.path.insert(0, ref_dir)
        import edgeforge as ref  # the reference, unmodified
    cores = len(os.sched_getaffinity(0))
    frames = {"C0 512x512": np.asarray(synth.make_config(0)).reshape(512, 512),
              "C1 frame 0 (1080p)": np.asarray(synth.config1_frame(0)).reshape(1080, 1920)}
    rows = []
    for name, f in frames.items():
        f64 = np.ascontiguousarray(f, dtype=np.float64)
        img = ef.GrayImage.from_array(f64)
        cfg = ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0))
        ours_s, res = timed(lambda: ef.run_pipeline(img, cfg), 20)
        row = {"frame": name, "pixels": int(f.size), "ours_ms": round(ours_s * 1e3, 3)}
        if ref is not None:
            rimg = ref.GrayImage.from_array(f64)
            rcfg = ref.PipelineConfig(sigma=1.4, thresholds=ref.Thresholds(20.0, 50.0),
                                      workers=ref.WorkerConfig(workers=cores))
            ref_s, rres = timed(lambda: ref.run_pipeline(rimg, rcfg), 3, warm=1)
            row.update({"reference_ms": round(ref_s * 1e3, 3), "reference_workers": cores,
                        "speedup": round(ref_s / ours_s, 1),
                        "labels_equal": bool(np.array_equal(np.asarray(res.edges.labels),
                                                            np.asarray(rres.edges.labels))),
                        "final_equal": bool(np.array_equal(np.asarray(res.edges.final),
                                                           np.asarray(rres.edges.final)))})
        rows.append(row)
        print(json.dumps(row))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
