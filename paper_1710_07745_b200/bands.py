"""Row-band partition of one frame: within a GPU (trace_edges_parallel) and
across GPUs (config 4: one 16384^2 image over 2/4/8 B200s).

The reference's template is trace_edges_parallel (hysteresis.py:90-131):
label each band independently, renumber into one id space, union the
components that touch across each band seam (shifts -1/0/+1), then keep
components that reach a strong pixel.  Here:

  band compute   ef_band_canny_u8 (classify + band-local tile union-find) or
                 ef_band_trace (labels given); components touching the band's
                 top/bottom row stay undecided.
  edge export    ef_band_edges: per column of the top and bottom row, the
                 band-local component root and whether it already holds a
                 strong pixel.  ids are made global as (band << 40) | root.
  seam merge     ef_band_merge_device (union-find over the nbands*2*W edge
                 entries on the GPU, four stream-ordered launches), identical on
                 every rank; ef_band_merge is the same merge on the host (used
                 by backends without a device, and as the GPU tests' check).
  finalize       ef_band_finalize: mark merged-strong roots, re-finalise the
                 tiles that had undecided components.

Multi-GPU (one process per GPU, torch.distributed):
  halo exchange  each rank owns rows [row0, row0+rows) in HBM and needs
                 radius+2 rows from each neighbour: batch_isend_irecv over NCCL
                 (NVLink P2P); frame edges are clamped instead.
  edge exchange  all_gather of the 2*W edge ids/flags (NCCL), device to
                 device: no host round trip on the band path.
The compute steps go through a backend object so that the orchestration runs
under gloo on CPU in the tests with an oracle-backed backend.
"""

from __future__ import annotations

import numpy as np

from . import _lib

ID_SHIFT = 40


def band_plan(height: int, nbands: int) -> list[tuple[int, int]]:
    """Near-equal contiguous bands (engine.plan_bands with granularity 1)."""
    size = -(-height // nbands)
    return [(s, min(s + size, height)) for s in range(0, height, size)]


def check_band_meta(meta: list[tuple[int, int]], full_height: int) -> None:
    """The seam merge joins gathered block k's bottom row to block k+1's top
    row, so rank k must hold the k-th band from the top: bands sorted by row0 in
    rank order, contiguous, covering [0, full_height)."""
    row = 0
    for rank, (r0, rows) in enumerate(meta):
        if r0 != row or rows < 1:
            raise ValueError(f"row bands must be contiguous, non-empty and in rank order from row 0: rank {rank} "
                             f"holds rows [{r0}, {r0 + rows}), expected to start at row {row}")
        row = r0 + rows
    if row != full_height:
        raise ValueError(f"row bands cover rows [0, {row}) of a {full_height}-row frame")


def halo_rows(radius: int) -> int:
    return radius + 2  # blur radius + Sobel 1 + NMS 1 (ef_band_halo_rows)


def globalize_ids(ids: np.ndarray, band: int) -> np.ndarray:
    out = ids.astype(np.int64, copy=True)
    m = out >= 0
    out[m] = (np.int64(band) << ID_SHIFT) | out[m]
    return out


def merge_edges(ids_all: np.ndarray, strong_all: np.ndarray, width: int) -> np.ndarray:
    """Host union-find over every band's edge rows (ef_band_merge).
    ids_all/strong_all: (nbands, 2*width) int64/uint8, ids already global."""
    nb = ids_all.shape[0]
    ids = np.ascontiguousarray(ids_all, dtype=np.int64)
    strong = np.ascontiguousarray(strong_all, dtype=np.uint8)
    out = np.empty_like(strong)
    _lib.check(_lib.load().ef_band_merge(nb, width, ids.ctypes.data, strong.ctypes.data, out.ctypes.data),
               "ef_band_merge")
    return out


def merge_edges_device(ids_local, strong, width: int):
    """Device seam merge (ef_band_merge_device).  ids_local/strong: (nbands,
    2*width) int64/uint8 CUDA tensors, ids band-local as ef_band_edges writes
    them.  Returns the merged strong flags, same shape, on the device."""
    from . import canny

    torch = canny.require_cuda()
    nb = ids_local.shape[0]
    ids_local = ids_local.contiguous()
    strong = strong.contiguous()
    lib = _lib.load()
    need = lib.ef_band_merge_scratch_bytes(nb, width)
    if need == 0:
        raise ValueError(f"bad band merge dimensions: {nb} bands x {width}")
    scratch = torch.empty(need, dtype=torch.uint8, device=ids_local.device)
    out = torch.empty_like(strong)
    st = int(torch.cuda.current_stream(ids_local.device).cuda_stream)
    _lib.check(lib.ef_band_merge_device(nb, width, ids_local.data_ptr(), strong.data_ptr(), out.data_ptr(),
                                        scratch.data_ptr(), need, st), "ef_band_merge_device")
    return out


class CudaBandBackend:
    """Band compute on the local CUDA device through the C ABI."""

    def __init__(self, rows: int, width: int):
        from . import canny

        self.torch = canny.require_cuda()
        self.canny = canny
        self.rows, self.width = rows, width
        self.ws = canny.new_workspace(1, rows, width)
        self.labels = None
        self.final = None

    def _stream(self):
        return int(self.torch.cuda.current_stream().cuda_stream)

    def classify_trace(self, buf, row0: int, full_height: int, weights, low: float, high: float):
        """buf: u8 CUDA tensor holding rows [row0-ht, row0+rows+hb) of the frame."""
        t = self.torch
        self.labels = t.empty((self.rows, self.width), dtype=t.uint8, device=buf.device)
        self.final = t.empty_like(self.labels)
        _, wp, r = self.canny.host_weights(weights)
        rc = _lib.load().ef_band_canny_u8(buf.data_ptr(), row0, self.rows, full_height, self.width, wp, r,
                                          float(low), float(high), self.labels.data_ptr(), self.final.data_ptr(),
                                          self.ws.data_ptr(), self.ws.numel(), self._stream())
        _lib.check(rc, "ef_band_canny_u8")

    def classify_trace_peer(self, band, top_ptr: int, top_rows: int, bot_ptr: int, bot_rows: int, row0: int,
                            full_height: int, weights, low: float, high: float):
        """band: this rank's rows only; the halo rows are read in place through
        top_ptr / bot_ptr (neighbour bands, e.g. IPC-mapped peer HBM)."""
        t = self.torch
        self.labels = t.empty((self.rows, self.width), dtype=t.uint8, device=band.device)
        self.final = t.empty_like(self.labels)
        _, wp, r = self.canny.host_weights(weights)
        rc = _lib.load().ef_band_canny_u8_peer(band.data_ptr(), top_ptr or None, top_rows, bot_ptr or None, bot_rows,
                                               row0, self.rows, full_height, self.width, wp, r, float(low),
                                               float(high), self.labels.data_ptr(), self.final.data_ptr(),
                                               self.ws.data_ptr(), self.ws.numel(), self._stream())
        _lib.check(rc, "ef_band_canny_u8_peer")

    def close_peers(self):
        for base in getattr(self, "peer_bases", []):
            _lib.check(_lib.load().ef_ipc_close(base), "ef_ipc_close")
        self.peer_bases = []
        self.peer_ptrs = None

    def trace(self, labels):
        t = self.torch
        self.labels = labels
        self.final = t.empty_like(labels)
        rc = _lib.load().ef_band_trace(labels.data_ptr(), self.rows, self.width, self.final.data_ptr(),
                                       self.ws.data_ptr(), self.ws.numel(), self._stream())
        _lib.check(rc, "ef_band_trace")

    def edges(self):
        t = self.torch
        ids = t.empty(2 * self.width, dtype=t.int64, device=self.labels.device)
        strong = t.empty(2 * self.width, dtype=t.uint8, device=self.labels.device)
        rc = _lib.load().ef_band_edges(self.ws.data_ptr(), self.ws.numel(), self.rows, self.width,
                                       ids.data_ptr(), strong.data_ptr(), self._stream())
        _lib.check(rc, "ef_band_edges")
        return ids, strong

    def merge(self, ids_all, strong_all):
        """Seam merge of every band's gathered edge rows, on the device."""
        return merge_edges_device(ids_all, strong_all, self.width)

    def finalize(self, strong_edges):
        rc = _lib.load().ef_band_finalize(strong_edges.data_ptr(), self.rows, self.width, self.labels.data_ptr(),
                                          self.final.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                          self._stream())
        _lib.check(rc, "ef_band_finalize")
        return self.final


def trace_bands_local(labels, plan: list[tuple[int, int]]):
    """trace_edges_parallel on one GPU: band-local tracing + device seam merge."""
    from . import canny

    torch = canny.require_cuda()
    h, w = labels.shape
    final = torch.empty_like(labels)
    backends, ids_all, strong_all = [], [], []
    for k, (s, e) in enumerate(plan):
        be = CudaBandBackend(e - s, w)
        be.trace(labels[s:e])
        ids, strong = be.edges()
        backends.append(be)
        ids_all.append(ids)
        strong_all.append(strong)
    merged = merge_edges_device(torch.stack(ids_all), torch.stack(strong_all), w)
    for k, ((s, e), be) in enumerate(zip(plan, backends)):
        final[s:e].copy_(be.finalize(merged[k]))
    return final


def canny_bands_local(frame_u8, nbands: int, weights, low: float, high: float):
    """Whole-frame Canny through the band path on one GPU (each band reads its
    halo from the resident frame) -- the single-device emulation of the
    multi-GPU partition, used to test the band kernels against ef_canny_u8."""
    from . import canny

    torch = canny.require_cuda()
    h, w = frame_u8.shape
    r = (len(weights) - 1) // 2
    halo = halo_rows(r)
    labels = torch.empty_like(frame_u8)
    final = torch.empty_like(frame_u8)
    plan = band_plan(h, nbands)
    backends, ids_all, strong_all = [], [], []
    for k, (s, e) in enumerate(plan):
        lo, hi = max(0, s - halo), min(h, e + halo)
        be = CudaBandBackend(e - s, w)
        be.classify_trace(frame_u8[lo:hi].contiguous(), s, h, weights, low, high)
        ids, strong = be.edges()
        backends.append(be)
        ids_all.append(ids)
        strong_all.append(strong)
    merged = merge_edges_device(torch.stack(ids_all), torch.stack(strong_all), w)
    for k, ((s, e), be) in enumerate(zip(plan, backends)):
        final[s:e].copy_(be.finalize(merged[k]))
        labels[s:e].copy_(be.labels)
    return labels, final


def band_buffer(rows: int, width: int, row0: int, full_height: int, radius: int, device=None):
    """A band's HBM buffer with room for its halo rows: returns (buf, band),
    band = buf[ht:ht+rows], the view the caller fills with its own rows once.
    Passing buf as `staged` to distributed_band_canny then receives the halos
    in place (no per-step copy of the band)."""
    import torch

    halo = halo_rows(radius)
    ht, hb = min(halo, row0), min(halo, full_height - row0 - rows)
    buf = torch.empty((ht + rows + hb, width), dtype=torch.uint8, device=device)
    return buf, buf[ht:ht + rows]


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    import ctypes

    h = (ctypes.c_ubyte * 64)()
    off = ctypes.c_uint64()
    _lib.check(_lib.load().ef_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "ef_ipc_export")
    return bytes(h), int(off.value)


def ipc_open(handle: bytes, offset: int) -> tuple[int, int]:
    """Map another process's buffer: (device pointer, mapping base to close)."""
    import ctypes

    h = (ctypes.c_ubyte * 64).from_buffer_copy(handle)
    ptr, base = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(_lib.load().ef_ipc_open(h, offset, ctypes.byref(ptr), ctypes.byref(base)), "ef_ipc_open")
    return int(ptr.value), int(base.value)


def _gather_stacked(tensor, world, group):
    """Every rank's `tensor` stacked along a new first axis: one band needs no
    collective; NCCL gathers straight into the stacked buffer (no per-rank
    list, no stacking copy); gloo goes through _gather."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return tensor.unsqueeze(0)
    if tensor.is_cuda and dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(tensor.shape), dtype=tensor.dtype, device=tensor.device)
        dist.all_gather_into_tensor(out, tensor.contiguous(), group=group)
        return out
    return torch.stack(_gather(tensor, world, group))


def _gather(tensor, world, group):
    """all_gather that also works for CUDA tensors under gloo (host staging)."""
    import torch
    import torch.distributed as dist

    host = tensor.is_cuda and dist.get_backend(group) == "gloo"
    src = tensor.cpu() if host else tensor
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src, group=group)
    return [o.to(tensor.device) for o in out] if host else out


def _peer_halos(be, band_u8, row0, rows, full_height, halo, meta, rank, world, group):
    """Device pointers to the halo rows inside the neighbour bands (opened once
    per backend and band buffer over CUDA IPC: NVLink peer memory when the
    neighbour is another GPU), plus the step handshake: this rank's two
    interprocess CUDA events ("band written", "halo rows read"), the
    neighbours' events opened from their IPC handles, and a host-only (gloo)
    group for the per-step barriers.  Set up collectively, once."""
    import torch
    import torch.distributed as dist

    w = band_u8.shape[1]
    key = (band_u8.data_ptr(), row0, rows, full_height, world)
    if getattr(be, "peer_ptrs", None) is not None and be.peer_ptrs[0] == key:
        return be.peer_ptrs[1:]
    if getattr(be, "peer_ptrs", None) is not None:
        be.close_peers()
    dev = band_u8.device
    if getattr(be, "ev_written", None) is None:
        with torch.cuda.device(dev):
            be.ev_written = torch.cuda.Event(interprocess=True)  # my band is written (this step)
            be.ev_read = torch.cuda.Event(interprocess=True)  # I have read my neighbours' rows (this step)
            be.ev_written.record()  # materialised on this device before its handle is exported
            be.ev_read.record()
        # host-only barriers: a barrier of an NCCL group would wait for this rank's stream
        be.host_group = group if dist.get_backend(group) == "gloo" else dist.new_group(
            dist.get_process_group_ranks(group) if group is not None else None, backend="gloo")
    objs = [None] * world
    dist.all_gather_object(objs, (ipc_export(band_u8), bytes(be.ev_written.ipc_handle()),
                                  bytes(be.ev_read.ipc_handle())), group=group)
    ht, hb = min(halo, row0), min(halo, full_height - row0 - rows)
    top = bot = 0
    be.peer_bases = []
    be.peer_events = []  # (written, read) of every neighbour whose rows I read or who reads mine
    for peer, (p0, pr) in enumerate(meta):
        if peer == rank:
            continue
        above, below = p0 + pr == row0, p0 == row0 + rows
        if ht and above:  # the band just above: its last ht rows
            if pr < ht:
                raise ValueError("peer halos need neighbour bands of at least radius+2 rows")
            ptr, base = ipc_open(*objs[peer][0])
            be.peer_bases.append(base)
            top = ptr + (pr - ht) * w
        if hb and below:  # the band just below: its first hb rows
            if pr < hb:
                raise ValueError("peer halos need neighbour bands of at least radius+2 rows")
            ptr, base = ipc_open(*objs[peer][0])
            be.peer_bases.append(base)
            bot = ptr
        if above or below:
            be.peer_events.append((torch.cuda.Event.from_ipc_handle(dev, objs[peer][1]),
                                   torch.cuda.Event.from_ipc_handle(dev, objs[peer][2])))
    be.peer_ptrs = (key, top, ht, bot, hb)
    return be.peer_ptrs[1:]


def distributed_band_canny(band_u8, row0: int, full_height: int, weights, low: float, high: float,
                           backend=None, group=None, staged=None, peer: bool = False):
    """One rank's share of a row-band-partitioned frame.

    band_u8: this rank's rows [row0, row0+rows) as a (rows, W) u8 tensor on the
    rank's device (CUDA under NCCL, CPU under gloo with a test backend).
    staged: optional buffer from band_buffer() whose middle rows are band_u8;
    the halos are received into it in place (otherwise the band is copied
    into a fresh haloed buffer every call).
    peer: no halo exchange -- the classifier reads the neighbours' halo rows in
    place from their HBM (CUDA IPC mappings of their band buffers, opened once;
    NVLink loads between GPUs).  Every rank's band must stay at the same address
    across calls and be written on the current stream before the call; the
    classifier reads the neighbours' rows only after every band's write (an
    interprocess-event wait on the stream), and work the caller enqueues on
    the stream after the call runs only after every neighbour has finished
    reading, so the caller may enqueue its next write into its band right
    away.  The host never waits for the GPU; it takes two host barriers per
    call.
    Returns (labels, final) for those rows, equal to the rows of the
    whole-frame result."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rows, w = band_u8.shape
    r = (len(weights) - 1) // 2
    halo = halo_rows(r)
    be = backend if backend is not None else CudaBandBackend(rows, w)
    # every rank's (row0, rows): how many halo rows each neighbour can give.
    # Exchanged once per backend (a reused backend keeps it: no collective and
    # no host sync per step)
    key = (row0, rows, full_height, world)
    cached = getattr(be, "band_meta", None)
    if cached is not None and cached[0] == key:
        meta = cached[1]
    else:
        counts = _gather(torch.tensor([row0, rows], dtype=torch.int64, device=band_u8.device), world, group)
        meta = [(int(c[0]), int(c[1])) for c in counts]
        check_band_meta(meta, full_height)
        be.band_meta = (key, meta)
    ht = min(halo, row0)
    hb = min(halo, full_height - row0 - rows)
    if peer:
        top, ht_, bot, hb_ = _peer_halos(be, band_u8, row0, rows, full_height, halo, meta, rank, world, group)
        # Two-phase handshake, ordered on the devices by interprocess CUDA
        # events (no stream synchronisation: the host never waits for a GPU):
        # (1) every rank records "band written" behind its write of this step;
        # once every rank has ENQUEUED that record (host barrier), each stream
        # waits on its neighbours' records before the classifier reads their
        # rows; (2) likewise "halo rows read" after the classifier, which every
        # stream waits on before its next work -- so a caller's next write into
        # its band cannot overtake a neighbour still reading it.  The barrier
        # is what makes a wait see THIS step's record (a wait issued before the
        # record would see the previous one).  (A barrier-free handshake --
        # cuStreamWaitValue32 on IPC-mapped flags -- was measured: a stream
        # waiting on a flag written by another context on the same GPU never
        # resumed, so it is not used.)
        stream = torch.cuda.current_stream(band_u8.device)
        be.ev_written.record(stream)
        dist.barrier(group=be.host_group)
        for written, _ in be.peer_events:
            stream.wait_event(written)
        be.classify_trace_peer(band_u8, top, ht_, bot, hb_, row0, full_height, weights, low, high)
        be.ev_read.record(stream)
        dist.barrier(group=be.host_group)
        for _, read in be.peer_events:
            stream.wait_event(read)
        return _merge_and_finalize(be, band_u8, rank, world, group)
    if staged is not None:
        if staged.shape != (ht + rows + hb, w) or staged[ht:ht + rows].data_ptr() != band_u8.data_ptr():
            raise ValueError("staged must be band_buffer()'s buffer holding band_u8 as its middle rows")
        buf = staged
    else:
        buf = torch.empty((ht + rows + hb, w), dtype=torch.uint8, device=band_u8.device)
        buf[ht:ht + rows].copy_(band_u8)
    # halo exchange (a halo may span several thin neighbour bands)
    ops = []
    for peer in range(world):
        if peer == rank:
            continue
        p0, pr = meta[peer]
        # rows of mine that the peer needs: its halo window intersected with my rows
        need0, need1 = max(0, p0 - halo), min(full_height, p0 + pr + halo)
        s0, s1 = max(need0, row0), min(need1, row0 + rows)
        if s0 < s1 and not (p0 <= s0 and s1 <= p0 + pr):
            ops.append(dist.P2POp(dist.isend, band_u8[s0 - row0:s1 - row0].contiguous(), peer, group))
        # rows of the peer that I need
        g0, g1 = max(p0, row0 - ht), min(p0 + pr, row0 + rows + hb)
        if g0 < g1 and not (row0 <= g0 and g1 <= row0 + rows):
            dst = buf[g0 - (row0 - ht):g1 - (row0 - ht)]
            ops.append(dist.P2POp(dist.irecv, dst, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    be.classify_trace(buf, row0, full_height, weights, low, high)
    return _merge_and_finalize(be, band_u8, rank, world, group)


def _merge_and_finalize(be, band_u8, rank, world, group):
    import torch
    import torch.distributed as dist

    w = band_u8.shape[1]
    ids, strong = be.edges()
    if world == 1:  # one band: no seams; every edge entry keeps its own component's flag
        return be.labels, be.finalize(strong)
    if hasattr(be, "merge"):
        # device path: gather the edge rows device to device, merge on the device
        merged = be.merge(_gather_stacked(ids, world, group), _gather_stacked(strong, world, group))
        return be.labels, be.finalize(merged[rank])
    # host path (backends without a device merge): globalised ids, host union-find
    gids = torch.from_numpy(globalize_ids(ids.cpu().numpy(), rank)).to(band_u8.device)
    ids_l = [torch.empty_like(gids) for _ in range(world)]
    st_l = [torch.empty_like(strong) for _ in range(world)]
    dist.all_gather(ids_l, gids, group=group)
    dist.all_gather(st_l, strong, group=group)
    ids_all = np.stack([t.cpu().numpy() for t in ids_l])
    st_all = np.stack([t.cpu().numpy() for t in st_l])
    merged = merge_edges(ids_all, st_all, w)
    fin = be.finalize(torch.from_numpy(merged[rank]).to(band_u8.device))
    return be.labels, fin
