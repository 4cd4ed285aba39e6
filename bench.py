"""Benchmark: Canny megapixels/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--radius 2]
    python bench.py --impl reference ...     # the reference path on the host CPU

Workload (N=1): BASELINE.json configs[1] -- a batch of 64 seeded synthetic
1920x1080 u8 frames, Gaussian sigma 1.4 "5x5" (radius 2), Sobel 3x3,
thresholds 20/50.  A step is the whole Canny path over the batch: fused
classify kernel (+ exact fix-ups) and hysteresis, labels and final edges
written to HBM.  Under torchrun each rank processes its own 64-frame batch
(weak scaling, no data-path collective: frames are independent units).

value  device-timed (CUDA events, max over ranks), inputs resident in HBM,
       rotating over 3 input batches (3 x 133 MB > 126 MB L2).
e2e    the same work through the host-buffer C-ABI entry (ef_canny_u8_host):
       pinned host frames in, pinned host labels + final out, copies timed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Canny megapixels/sec (1/2/4/8 B200) and fused-kernel HBM GB/s as % of roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    p.add_argument("--radius", type=int, default=2, help="Gaussian radius (configs' 5x5 = 2; reference default 5)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--frames", type=int, default=None, help="override batch size (configs 1 and 3)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--bands", action="store_true", help="config 4: row-band partition across ranks")
    p.add_argument("--peer", action="store_true",
                   help="with --bands: halo rows read in place from the neighbours' HBM (CUDA IPC / NVLink), "
                        "no halo exchange step")
    return p.parse_args()


def workload(args):
    from paper_1710_07745_b200 import synth

    cfg = args.config
    if cfg == 1:
        n = args.frames or 64
        frames = synth.config1(n)
        name = f"C1: {n} x 1920x1080 u8 frames (seeded ramp + 50 polygons + N(0,5^2))"
    elif cfg == 3:
        n = args.frames or 1024
        frames = synth.config3(n)
        name = f"C3: {n} x 1024x1024 u8 images (value noise + 30 shapes + N(0,8^2))"
    else:
        frames = synth.make_config(cfg)
        name = {0: "C0: 512x512 u8 (rects + disks + N(0,8^2))", 2: "C2: 4096x4096 u8 rings + spiral",
                4: "C4: 16384x16384 u8 tiled shapes + spirals"}[cfg]
    low, high = synth.CONFIG_THRESHOLDS[cfg]
    return frames, name, low, high


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clock and throttle reasons polled through NVML (every ~2 ms) while
    the timed region runs; falls back to one nvidia-smi query if NVML fails."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index: int):
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self.stop_evt = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.nv = None
        return self

    def _poll(self):
        nv = self.nv
        masks = {k: getattr(nv, v, 0) for k, v in self.REASONS.items()}
        i = 0
        while not self.stop_evt.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                if i % 4 == 0:  # throttle reasons: every 4th poll (the slower query)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    self.reasons |= {k for k, m in masks.items() if m and (r & m)}
            except Exception:  # noqa: BLE001
                break
            i += 1
            time.sleep(0.0005)

    def __exit__(self, *exc):
        self.stop_evt.set()
        if self.nv is not None:
            self.t.join(timeout=1)
            try:  # the region's last reasons, read once after it
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons |= {k for k, v in self.REASONS.items()
                                 if getattr(self.nv, v, 0) and (r & getattr(self.nv, v, 0))}
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(kernel_prefix="void k1v3_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the roofline
    kernel, from the committed ncu capture of this bench command
    (profiles/r01_k1v3_dram_64frames.csv: `ncu --metrics ...dram__bytes_*...
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu`)."""
    import csv

    path = os.path.join(ROOT, "profiles", "r01_k1v3_dram_64frames.csv")
    try:
        rows = list(csv.reader(open(path)))
    except OSError:
        return None
    hdr, by = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Kernel Name"].startswith(kernel_prefix) and d["Metric Name"].startswith("dram__bytes_"):
                by.setdefault(d["ID"], 0.0)
                by[d["ID"]] += float(d["Metric Value"].replace(",", ""))
    return round(sum(by.values()) / len(by)) if by else None


def cpu_baseline(frames, weights, low, high):
    """Oracle port (oracle/ef_oracle.c: the reference's float64 algorithm in
    C) on the host cores, bounded sample."""
    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    n = min(len(frames), 16)
    O.canny(frames[:2], weights, low, high, threads=cores)  # warm-up
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.canny(frames[:n], weights, low, high, threads=cores)
        reps += 1
        if time.perf_counter() - t0 > 5.0 or reps >= 20:
            break
    dt = time.perf_counter() - t0
    mp = reps * frames[:n].size / 1e6
    return {"value": round(mp / dt, 3), "unit": "MP/s", "cores": cores, "kind": "port",
            "sample": f"{reps} x {n} frames ({mp:.1f} MP) of the same workload, C float64 oracle port, "
                      f"{cores} threads"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as O

    frames, name, low, high = workload(args)
    w = O.gaussian_weights(1.4, radius=args.radius)
    cores = len(os.sched_getaffinity(0))
    # bounded sample per step so the whole run stays within minutes
    per_step = frames if frames.size <= 140e6 else frames[: max(1, int(140e6 // frames[0].size))]
    for _ in range(args.warmup):
        O.canny(per_step[:1], w, low, high, threads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.canny(per_step, w, low, high, threads=cores)
        times.append(time.perf_counter() - t0)
    ms = statistics.median(times) * 1e3
    value = per_step.size / 1e6 / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "MP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, see synth.py)",
        "config": {"workload": name, "radius": args.radius, "thresholds": [low, high],
                   "sample_frames_per_step": int(len(per_step))},
        "cpu_baseline": {"value": round(value, 3), "unit": "MP/s", "cores": cores, "kind": "port",
                         "sample": f"{len(per_step)} frames per step, C float64 oracle port "
                                   f"(reference is pure Python; no compiled reference exists)"},
        "e2e": {"value": round(value, 3), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_bands(args):
    """Config 4 across ranks: one 16384^2 frame, row bands (one per GPU), halo
    rows and band-edge component ids exchanged over NCCL (bands.py).  Total
    work is fixed as N grows: "scaling": "strong"."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1710_07745_b200 import bands, synth
    from paper_1710_07745_b200.filtering import build_gaussian_kernel

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev) if world > 1 else dist.init_process_group(
        "nccl", rank=0, world_size=1, init_method="tcp://127.0.0.1:29533", device_id=dev)
    frame = synth.config4() if not args.frames else synth.config4(args.frames * 1024, tile=256)
    H, W = frame.shape
    low, high = synth.CONFIG_THRESHOLDS[4]
    w = build_gaussian_kernel(1.4, radius=args.radius).weights
    s0, s1 = bands.band_plan(H, world)[rank]
    staged, band = bands.band_buffer(s1 - s0, W, s0, H, args.radius, device=dev)
    band.copy_(torch.from_numpy(np.ascontiguousarray(frame[s0:s1])))  # halo rows arrive in place each step
    st = torch.cuda.current_stream()
    be = bands.CudaBandBackend(s1 - s0, W)  # workspace and band metadata reused across steps
    for _ in range(args.warmup):
        bands.distributed_band_canny(band, s0, H, w, low, high, backend=be, staged=None if args.peer else staged,
                                     peer=args.peer)
    torch.cuda.synchronize()
    dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(st)
    for _ in range(args.steps):
        bands.distributed_band_canny(band, s0, H, w, low, high, backend=be, staged=None if args.peer else staged,
                                     peer=args.peer)
    stop.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([start.elapsed_time(stop) / args.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        line = {"metric": METRIC, "value": round(H * W / 1e6 / (ms / 1e3), 3), "unit": "MP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "dtype_note": "certified f32 decisions, f64 fix-up of uncertified pixels; u8 in, u8 out",
                "data": "synthetic (seeded generators, paper_1710_07745_b200/synth.py)",
                "config": {"workload": f"C4: one {H}x{W} frame, row bands over {world} GPU(s)",
                           "radius": args.radius, "thresholds": [low, high],
                           "parallelism": f"{world} row bands, " + ("halo rows read in place from peer HBM (CUDA IPC)"
                                                                      if args.peer else "NCCL P2P halo exchange")
                                          + ", all_gather of edge ids, device seam merge"},
                "e2e": None, "gpu_launches": None}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch

    from paper_1710_07745_b200 import _lib, canny

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    frames, name, low, high = workload(args)
    from paper_1710_07745_b200.filtering import build_gaussian_kernel

    w = build_gaussian_kernel(1.4, radius=args.radius).weights
    b, h, wd = frames.shape
    px = frames.size
    nbuf = 3
    srcs = [torch.from_numpy(np.roll(frames, k, axis=0).copy()).to(dev) for k in range(nbuf)]
    labels = torch.empty_like(srcs[0])
    final = torch.empty_like(srcs[0])
    ws = canny.new_workspace(b, h, wd, device=dev)
    st = torch.cuda.current_stream()
    lib = _lib.load()
    _, wp, r = canny.host_weights(w)
    sptr = int(st.cuda_stream)

    def step(i, ev=None):
        # one fused ef_canny_u8 call; the library records `ev` right before the
        # classifier kernel and right after its fix-up launches (same stream)
        src = srcs[i % nbuf]
        if ev is not None:
            _lib.check(lib.ef_set_classify_events(ev[0].cuda_event, ev[1].cuda_event), "events")
        rc = lib.ef_canny_u8(src.data_ptr(), b, h, wd, wp, r, float(low), float(high), labels.data_ptr(),
                             final.data_ptr(), ws.data_ptr(), ws.numel(), sptr)
        _lib.check(rc, "canny")
        if ev is not None:
            _lib.check(lib.ef_set_classify_events(None, None), "events")

    for i in range(args.warmup):
        step(i)
    canny.reset_stats(ws)
    # K1's own duration is sampled on every EV_EVERY-th timed step: an event
    # recorded between two kernels of the PDL chain stops the classifier from
    # launching early, which cost 2.4% of the step when every step carried them
    EV_EVERY = 5
    sampled = [i for i in range(args.steps) if i % EV_EVERY == 0]
    evs = {i: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for i in sampled}
    for a, c in evs.values():  # torch creates the CUDA event on first record
        a.record(st)
        c.record(st)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        start.record(st)
        for i in range(args.steps):
            step(i, evs.get(i))
        stop.record(st)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    total_ms = start.elapsed_time(stop)
    k1_ms = statistics.mean(a.elapsed_time(c) for a, c in evs.values())
    stats = canny.read_stats(ws)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(t.item())
    ms = total_ms / args.steps
    value = world * px / 1e6 / (ms / 1e3)

    # e2e: host buffers through the C ABI (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hsrc = torch.from_numpy(frames).pin_memory()
        hlab = torch.empty_like(hsrc).pin_memory()
        hfin = torch.empty_like(hsrc).pin_memory()
        for _ in range(2):
            canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, low, high, hlab.data_ptr(), hfin.data_ptr(),
                                    dev.index)
        if world > 1:
            torch.distributed.barrier()
        e_steps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            canny.canny_u8_host_ptr(hsrc.data_ptr(), b, h, wd, w, low, high, hlab.data_ptr(), hfin.data_ptr(),
                                    dev.index)
        e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        et = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(et.item())
        e2e = {"value": round(world * px / 1e6 / (e_ms / 1e3), 3), "unit": "MP/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": int(px), "d2h_bytes_per_step": int(-(-px // 4)),
               "path": "ef_canny_u8_host (pinned input; 3-stream chunked copy/compute overlap; labels+final "
                       "cross PCIe packed to 2 bits/px and are expanded into the host arrays by a host thread pool)"}

    peak, peak_kind = peaks()
    # algorithmic bytes of the roofline kernel: u8 in + label byte out (SURVEY 8d's
    # 2 B/px) + the final byte the fused K1 also writes (final = strong; the
    # hysteresis only adds the weak pixels that join an edge) = 3 B/px
    alg_bytes = 3 * px
    achieved = alg_bytes / (k1_ms / 1e3) / 1e9
    if rank == 0:
        # the CPU baseline is timed on rank 0 at N=1 only (a reported baseline, not per-rank work)
        cpu = None if (args.no_cpu or world > 1) else cpu_baseline(frames, w, low, high)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "MP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "dtype_note": "certified f32 decisions, f64 fix-up of uncertified pixels; u8 in, u8 out",
            "data": "synthetic (seeded generators, paper_1710_07745_b200/synth.py)",
            "config": {"workload": name, "frames_per_gpu": int(b), "height": int(h), "width": int(wd),
                       "radius": args.radius, "sigma": 1.4, "thresholds": [low, high],
                       "parallelism": f"{world} independent batches (one per GPU)",
                       "l2": f"rotating {nbuf} resident input batches ({nbuf * px / 1e6:.0f} MB > 126 MB L2)"},
            "roofline": {"bound": "hbm", "kernel": "k1v3_kernel (+fix-up launches)",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": ncu_traffic() if (args.config == 1 and b == 64 and args.radius == 2) else None,
                         "traffic_source": "profiles/r01_k1v3_dram_64frames.csv (ncu dram__bytes_read+write per launch)",
                         "peak_kind": peak_kind,
                         "alg_bytes_per_launch": int(alg_bytes),
                         "alg_bytes_note": "3 B/px: u8 in, label out, final out (K1 writes final = strong in the "
                                           "fused path); SURVEY 8d's classify-only figure is 2 B/px",
                         "frac_at_2bpx": round(achieved * 2 / 3 / peak, 4),
                         "avg_launch_ms": round(k1_ms, 4),
                         "timing": f"CUDA events the library records on the launching stream around K1 + fix-ups, "
                                   f"on {len(evs)} of the {args.steps} timed steps (every {EV_EVERY}th)",
                         "share_of_step": round(k1_ms / ms, 3)},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": 8 * args.steps,  # ws_begin, K1, fix-up, H1, dense H1, merge, resolve, finalize
            "stats": {k: int(v) for k, v in stats.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.bands:
        run_bands(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
