"""Per-stage device timing of one fused ef_canny_u8 step (debug probe):
times ef_classify_u8 (ws_begin + K1 + FX) and ef_trace_edges (H1..H4, label
path) separately and the fused call, with CUDA events, 64 x 1080p."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1710_07745_b200 import canny, synth, _lib
from paper_1710_07745_b200.filtering import build_gaussian_kernel

frames = torch.from_numpy(synth.make_config(1)).cuda()
b, h, w = frames.shape
wt = build_gaussian_kernel(1.4, radius=2).weights
lab = torch.empty_like(frames); fin = torch.empty_like(frames)
ws = canny.new_workspace(b, h, w, device=frames.device)
lib = _lib.load(); _, wp, r = canny.host_weights(wt)
st = torch.cuda.current_stream(); sp = int(st.cuda_stream)
def fused():
    _lib.check(lib.ef_canny_u8(frames.data_ptr(), b, h, w, wp, r, 20.0, 50.0, lab.data_ptr(), fin.data_ptr(),
                               ws.data_ptr(), ws.numel(), sp), "canny")
def classify():
    _lib.check(lib.ef_classify_u8(frames.data_ptr(), b, h, w, wp, r, 20.0, 50.0, lab.data_ptr(),
                                  ws.data_ptr(), ws.numel(), sp), "classify")
def trace():
    _lib.check(lib.ef_trace_edges(lab.data_ptr(), b, h, w, fin.data_ptr(), ws.data_ptr(), ws.numel(), sp), "trace")
def timeit(f, n=20):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    for _ in range(n): f()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print("fused ef_canny_u8   %.1f us" % timeit(fused))
print("ef_classify_u8      %.1f us" % timeit(classify))
print("ef_trace_edges      %.1f us (label path)" % timeit(trace))
