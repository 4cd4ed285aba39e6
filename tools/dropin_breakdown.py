"""Where the drop-in run_pipeline's single-image latency goes (host side)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1710_07745_b200 as ef
from paper_1710_07745_b200 import synth, canny

def med(fn, n=50):
    for _ in range(5): fn()
    t = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); t.append(time.perf_counter() - t0)
    return np.median(t) * 1e3

for name, f in (("512^2", np.asarray(synth.make_config(0)).reshape(512, 512)), ("1080p", np.asarray(synth.config1_frame(0)).reshape(1080, 1920))):
    f64 = np.ascontiguousarray(f, dtype=np.float64)
    img = ef.GrayImage.from_array(f64)
    cfg = ef.PipelineConfig(sigma=1.4, thresholds=ef.Thresholds(20.0, 50.0))
    w = cfg.kernel().weights
    u8 = img.as_u8()
    print(name, "run_pipeline        %.3f ms" % med(lambda: ef.run_pipeline(img, cfg)))
    print(name, "  as_u8             %.3f ms" % med(lambda: img.as_u8()))
    print(name, "  cfg.kernel()      %.3f ms" % med(lambda: cfg.kernel()))
    print(name, "  canny_u8_host     %.3f ms" % med(lambda: canny.canny_u8_host(u8, w, 20.0, 50.0)))
    lab, fin = canny.canny_u8_host(u8, w, 20.0, 50.0)
    print(name, "  EdgeMap           %.3f ms" % med(lambda: ef.EdgeMap(width=img.width, height=img.height, labels=np.ascontiguousarray(lab), final=np.ascontiguousarray(fin).view(np.bool_))))
    d = torch.from_numpy(u8).cuda()
    def dev():
        canny.canny_u8(d, w, 20.0, 50.0); torch.cuda.synchronize()
    print(name, "  device canny+sync %.3f ms" % med(dev))
    pin = torch.from_numpy(u8).pin_memory(); hl = torch.empty_like(pin).pin_memory(); hf = torch.empty_like(pin).pin_memory()
    print(name, "  host_ptr pinned   %.3f ms" % med(lambda: canny.canny_u8_host_ptr(pin.data_ptr(), 1, *u8.shape, w, 20.0, 50.0, hl.data_ptr(), hf.data_ptr())))
    print(name, "  np.empty x2       %.3f ms" % med(lambda: (np.empty(u8.shape, np.uint8), np.empty(u8.shape, np.uint8))))
