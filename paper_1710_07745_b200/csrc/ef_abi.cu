// ef_abi.cu -- the extern "C" surface of libedgeforge_b200.so (include/edgeforge_b200.h).
//
// Host responsibilities: argument validation with the reference's error
// semantics (ValueError -> EF_EINVAL), the certified fp32 error bounds for the
// fast path, workspace layout, kernel sequencing, the host-buffer pipeline and
// the cross-band union-find.
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost a function-pointer check when no tool is attached

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_host.h"
#include "ef_launch.cuh"

using namespace ef;

namespace {

thread_local std::string g_err;

// NVTX range over a host-side section (kernel enqueue sequences, host-buffer chunks):
// shows the library's phases in Nsight Systems timelines
struct Range {
    explicit Range(const char* name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return EF_ECUDA;
}

#define EF_CHECK(call, what)                          \
    do {                                              \
        cudaError_t _e = (call);                      \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

int sm_count_current() {
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n;
    return n;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct WsLayout {
    size_t hdr, fix, perim, gpar, gstrong, pending, border, plist_idx, plist_node, plist_count, node_list, node_count,
        pend_tiles, dense, fgbits, stbits, plane_bytes, total;
    unsigned long long fix_cap, plist_scap, node_scap;
    HystLayout hl;
};

WsLayout ws_layout(int64_t batch, int H, int W) {
    WsLayout L;
    L.hl = hyst_layout(batch, H, W);
    unsigned long long npx = (unsigned long long)batch * H * W;
    L.fix_cap = std::max<unsigned long long>(1ull << 16, npx / 64);
    size_t off = 0;
    L.hdr = off;
    off = align_up(off + sizeof(WsHeader));
    L.fix = off;
    off = align_up(off + L.fix_cap * sizeof(unsigned long long));
    L.perim = off;
    off = align_up(off + (size_t)L.hl.slots * sizeof(int));
    L.gpar = off;
    off = align_up(off + (size_t)L.hl.slots * sizeof(int));
    L.gstrong = off;
    off = align_up(off + (size_t)L.hl.slots);
    L.pending = off;
    off = align_up(off + (size_t)L.hl.tiles);
    L.border = off;
    off = align_up(off + (size_t)L.hl.tiles);
    L.plist_scap = std::max<unsigned long long>(1ull << 10, npx / 64 / PL_STRIPES);
    L.plist_idx = off;
    off = align_up(off + L.plist_scap * PL_STRIPES * sizeof(unsigned long long));
    L.plist_node = off;
    off = align_up(off + L.plist_scap * PL_STRIPES * sizeof(int));
    L.plist_count = off;
    off = align_up(off + PL_STRIPES * sizeof(unsigned long long));
    L.node_scap = std::max<unsigned long long>(1ull << 10, (unsigned long long)L.hl.slots / 8 / PL_STRIPES);
    L.node_list = off;
    off = align_up(off + L.node_scap * PL_STRIPES * sizeof(int));
    L.node_count = off;
    off = align_up(off + PL_STRIPES * sizeof(unsigned long long));
    L.pend_tiles = off;
    off = align_up(off + PL_STRIPES * sizeof(unsigned long long));
    L.dense = off;
    off = align_up(off + (size_t)L.hl.tiles * sizeof(int));
    L.plane_bytes = (size_t)batch * H * ((W + 63) / 64) * sizeof(unsigned long long);
    L.fgbits = off;
    off = align_up(off + L.plane_bytes);
    L.stbits = off;
    off = align_up(off + L.plane_bytes);
    L.total = off;
    return L;
}

struct Ws {
    WsHeader* hdr;
    unsigned long long* fix;
    HystBufs hb;
    unsigned long long* fgbits;
    unsigned long long* stbits;
};

Ws ws_bind(void* base, const WsLayout& L) {
    char* p = static_cast<char*>(base);
    Ws w;
    w.hdr = reinterpret_cast<WsHeader*>(p + L.hdr);
    w.fix = reinterpret_cast<unsigned long long*>(p + L.fix);
    w.hb.perim = reinterpret_cast<int*>(p + L.perim);
    w.hb.gpar = reinterpret_cast<int*>(p + L.gpar);
    w.hb.gstrong = reinterpret_cast<uint8_t*>(p + L.gstrong);
    w.hb.pending = reinterpret_cast<uint8_t*>(p + L.pending);
    w.hb.border = reinterpret_cast<uint8_t*>(p + L.border);
    w.hb.plist_idx = reinterpret_cast<unsigned long long*>(p + L.plist_idx);
    w.hb.plist_node = reinterpret_cast<int*>(p + L.plist_node);
    w.hb.plist_count = reinterpret_cast<unsigned long long*>(p + L.plist_count);
    w.hb.plist_scap = L.plist_scap;
    w.hb.node_list = reinterpret_cast<int*>(p + L.node_list);
    w.hb.node_count = reinterpret_cast<unsigned long long*>(p + L.node_count);
    w.hb.node_scap = L.node_scap;
    w.hb.pend_tiles = reinterpret_cast<unsigned long long*>(p + L.pend_tiles);
    w.hb.dense = reinterpret_cast<int*>(p + L.dense);
    w.fgbits = reinterpret_cast<unsigned long long*>(p + L.fgbits);
    w.stbits = reinterpret_cast<unsigned long long*>(p + L.stbits);
    return w;
}

// Resets the per-call workspace state; with `planes` (the fused path) also
// zeroes the two foreground bit planes (2 * nwords words).
__global__ void ws_begin_kernel(WsHeader* hdr, unsigned long long cap, HystBufs hb, unsigned long long* planes,
                                unsigned long long nwords) {
    pdl_wait();  // the previous call's kernels on this stream read the same workspace
    pdl_trigger();
    // 16-byte stores (the planes start 256-byte aligned), then the odd last word
    const unsigned long long n16 = nwords / 2;
    uint4* p16 = reinterpret_cast<uint4*>(planes);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (unsigned long long)gridDim.x * blockDim.x)
        p16[i] = make_uint4(0u, 0u, 0u, 0u);
    if ((nwords & 1ull) && blockIdx.x == 0 && threadIdx.x == 0) planes[nwords - 1] = 0ull;
    if (blockIdx.x != 0) return;
    if (threadIdx.x == 0) {
        hdr->fix_count = 0;
        hdr->fix_cap = cap;
        hdr->overflow = 0;
        hdr->plist_overflow = 0;
        hdr->dense_count = 0;
        hdr->node_overflow = 0;
    }
    if (threadIdx.x < PL_STRIPES) {
        hb.plist_count[threadIdx.x] = 0;
        hb.node_count[threadIdx.x] = 0;
        hb.pend_tiles[threadIdx.x] = 0;
    }
}

cudaError_t launch_ws_begin(const Ws& ws, const WsLayout& L, unsigned long long nwords, int sms, cudaStream_t st) {
    const unsigned long long want = (nwords / 2 + 255) / 256;
    const unsigned blocks = (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(want, 4ull * sms));
    return launch_pdl(ws_begin_kernel, dim3(blocks), dim3(256), 0, st, ws.hdr, L.fix_cap, ws.hb, ws.fgbits, nwords);
}

__global__ void ws_reset_stats_kernel(WsHeader* hdr) {
    hdr->stats.fixups = 0;
    hdr->stats.ambiguous = 0;
    hdr->stats.border_nodes = 0;
    hdr->stats.pending_tiles = 0;
}

int check_dims(int64_t batch, int32_t H, int32_t W) {
    if (batch < 1 || H < 1 || W < 1)
        return fail(EF_EINVAL, "image dimensions must be >= 1, got batch=" + std::to_string(batch) + " " +
                                   std::to_string(W) + "x" + std::to_string(H));
    if ((unsigned long long)batch * H * W > (1ull << 40)) return fail(EF_EINVAL, "image too large");
    if (batch > 65535) return fail(EF_EINVAL, "batch > 65535 frames per call (grid z limit); split the batch");
    if (H > (1 << 22) || W > (1 << 22)) return fail(EF_EINVAL, "frame dimension above 4194304");
    if ((long long)((W + 63) / 64) * ((H + 63) / 64) * batch * 256 >= (1ll << 31))
        return fail(EF_EINVAL, "too many tiles for 32-bit node ids; split the batch");
    return EF_OK;
}

// numpy's float64 add.reduce of a short contiguous vector (its pairwise
// summation below the 128-element block: eight interleaved partial sums, a
// fixed combine tree, then the tail), so weights on the 1e-12 edge are
// accepted or rejected exactly as GaussianKernel's w.sum() does.
double numpy_sum(const double* a, int n) {
    if (n < 8) {
        double s = -0.0;
        for (int i = 0; i < n; ++i) s += a[i];
        return s;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) s += a[i];
    return s;
}

// GaussianKernel validation (filtering.py:20-29) plus the threshold validation
// (hysteresis.py:31-33).
int check_params(const double* w, int32_t r, double low, double high) {
    if (!w) return fail(EF_EINVAL, "weights pointer is NULL");
    if (r < 0 || r > EF_MAX_RADIUS)
        return fail(EF_EINVAL, "radius must be in [0, " + std::to_string(EF_MAX_RADIUS) + "], got " +
                                   std::to_string(r));
    for (int i = 0; i <= 2 * r; ++i) {
        if (!std::isfinite(w[i])) return fail(EF_EINVAL, "kernel weights must be finite");
        if (w[i] != w[2 * r - i]) return fail(EF_EINVAL, "kernel weights must be symmetric");
    }
    const double sum = numpy_sum(w, 2 * r + 1);
    // GaussianKernel's own check (filtering.py:25-26): |sum - 1| <= 1e-12
    if (!(std::fabs(sum - 1.0) <= 1e-12)) return fail(EF_EINVAL, "kernel weights must sum to 1");
    if (!(0.0 <= low && low <= high))
        return fail(EF_EINVAL, "need 0 <= low <= high, got low=" + std::to_string(low) +
                                   ", high=" + std::to_string(high));
    return EF_OK;
}

ExactParams make_exact(const double* w, int r, double low, double high) {
    ExactParams P;
    std::memset(&P, 0, sizeof P);
    for (int i = 0; i <= 2 * r; ++i) P.w[i] = w[i];
    P.r = r;
    P.low = low;
    P.high = high;
    return P;
}

// Certified bounds of the fp32 fast path.  u8
// inputs: |b| <= 255, |gx|,|gy| <= 1020, magnitude <= 1442.5.
FastParams make_fast(const double* w, int r, double low, double high) {
    FastParams P;
    std::memset(&P, 0, sizeof P);
    P.r = r;
    for (int k = 0; k <= r; ++k) P.wf[k] = (float)w[r + k];
    const double u = std::ldexp(1.0, -24), u64 = std::ldexp(1.0, -53);
    const double eh = (r + 2) * u * 255.0;                                  // horizontal pass
    const double eb = eh + (r + 3) * u * 255.0 + (4 * r + 6) * u64 * 255.0;  // vertical pass (+f64 side)
    const double eg = 8.0 * eb + 4080.0 * u + 12.0 * u64 * 1020.0 + 1e-9;   // Sobel
    const double rel = std::ldexp(1.0, -20) + 3.0 * u;                      // m^2 rounding + sqrt.approx
    // safety factor on the analytic bounds: the largest errors observed against
    // the exact float64 path use at most 18% of E_g and 14% of Em (32 C3 frames,
    // 4 C1 frames, C2, noise and 0/255 blocks at radius 1-6, every pixel:
    // tools/cert_margin.py, profiles/r02_cert_margin.json), so the bounds carry
    // a 5.5x margin on their own; round 1 used S = 2 on top
    const double S = 1.0;
    auto Em = [&](double M) { return std::sqrt(2.0) * eg + rel * M + 1e-9; };
    auto band = [&](double T, float& lo, float& hi) {
        if (!(T > 0.0)) {  // every magnitude is >= 0 >= T
            lo = hi = -1.0f;
            return;
        }
        double e = S * Em(T + 1.0);
        lo = std::nextafter((float)(T - e), -INFINITY);
        hi = std::nextafter((float)(T + e), INFINITY);
    };
    band(low, P.lo_lo, P.lo_hi);
    band(high, P.hi_lo, P.hi_hi);
    P.e_nms = (float)(S * 2.0 * Em(1443.0 * 1.01));
    // the same bound relative to the two magnitudes compared: |c - n| must
    // exceed Em(c) + Em(n) = 2 sqrt(2) eg + rel (c + n) (+ the true-vs-computed
    // magnitude slack in the rel term: 2^-10), so ties between small
    // magnitudes are not flagged with the band of the largest possible one
    P.e_nms0 = std::nextafter((float)(S * (2.0 * std::sqrt(2.0) * eg + 1e-8)), INFINITY);
    P.e_nms_rel = std::nextafter((float)(S * rel * (1.0 + std::ldexp(1.0, -10))), INFINITY);
    P.e_sec = (float)(S * ((1.0 + 0.41421356237309503) * eg + 3000.0 * u));
    P.cls0 = high <= 0.0 ? 2 : (low <= 0.0 ? 1 : 0);
    return P;
}

FrameGeom frame_geom(int H, int W) { return FrameGeom{H, W, 0, H, 0, H}; }

// ef_set_classify_events: events this thread's classify launches record around
// the classifier + fix-up kernels (bench.py's roofline timing).
struct Timing {
    cudaEvent_t start = nullptr, stop = nullptr;
};
Timing& timing() {
    thread_local Timing t;
    return t;
}

bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) == 0; }

bool has_negative(const double* w, int r) {
    for (int i = 0; i <= 2 * r; ++i)
        if (w[i] < 0.0) return true;
    return false;
}

// fin != nullptr (fused pipeline): where the production classifier runs, it
// also fills the workspace's foreground bit planes and *bits describes them
// (bits->fg == nullptr otherwise).
int run_classify_u8(const uint8_t* src, int64_t batch, const FrameGeom& g, const double* w, int r,
                    double low, double high, uint8_t* labels, const Ws& ws, const WsLayout& L,
                    cudaStream_t st, uint8_t* fin = nullptr, FgBits* bits = nullptr) {
    Range nvtx("edgeforge classify (ws_begin, K1, fix-ups)");
    int sms = sm_count_current();
    if (bits) *bits = FgBits{};
    if (has_negative(w, r)) {
        // the certified bounds assume a convex (non-negative) kernel; a signed
        // kernel takes the exact float64 kernel instead
        if (g.g0 != 0 || g.full_H != g.H || g.rows != g.H) return fail(EF_EINVAL, "signed kernel on a band");
        EF_CHECK(launch_ws_begin(ws, L, 0, sms, st), "ws_begin");  // the trace that follows reuses the counters
        ExactParams XP = make_exact(w, r, low, high);
        EF_CHECK(launch_exact<uint8_t>(src, batch, g.H, g.W, XP, labels, nullptr, nullptr, nullptr, nullptr,
                                       nullptr, nullptr, nullptr, ws.hdr, st),
                 "exact kernel");
        return EF_OK;
    }
    FastParams FP = make_fast(w, r, low, high);
    // the production classifier moves 32-bit words: misaligned caller buffers
    // take the byte-wise generic classifier (g.top/g.bot peer rows are checked
    // by the peer entry point)
    FP.no_v2 = !aligned4(src) || !aligned4(labels) || (fin && !aligned4(fin));
    FgBits B{};
    unsigned long long nwords = 0;  // bit-plane words ws_begin zeroes (both planes and the gap between)
    static const bool no_bits = getenv("EF_NO_FG_BITS") != nullptr;  // A/B switch for profiling
    if (fin && bits && !no_bits && k1_emits_bits(FP, g)) {
        const int words = (g.W + 63) / 64;
        nwords = (unsigned long long)(ws.stbits - ws.fgbits) + (unsigned long long)batch * g.rows * words;
        B = FgBits{ws.fgbits, ws.stbits, words, (unsigned long long)g.rows * words,
                   (long long)(reinterpret_cast<intptr_t>(fin) - reinterpret_cast<intptr_t>(labels))};
        *bits = B;
    }
    EF_CHECK(launch_ws_begin(ws, L, nwords, sms, st), "ws_begin");
    const Timing& T = timing();
    if (T.start) EF_CHECK(cudaEventRecord(T.start, st), "timing event");
    EF_CHECK(launch_k1(src, batch, g, FP, labels, ws.fix, ws.hdr, B, st), "classify kernel");
    ExactParams XP = make_exact(w, r, low, high);
    EF_CHECK(launch_fix(src, batch, g, XP, labels, ws.fix, ws.hdr, B, sms, st), "fix-up kernel");
    if (T.stop) EF_CHECK(cudaEventRecord(T.stop, st), "timing event");
    return EF_OK;
}

// The workspace's foreground bit planes for frames of H rows x W columns.
FgBits ws_planes(const Ws& ws, int H, int W) {
    const int words = (W + 63) / 64;
    return FgBits{ws.fgbits, ws.stbits, words, (unsigned long long)H * words, 0};
}

// Hysteresis over the bit planes: the classifier's (bits, with final = strong
// already written) or, without them, planes packed from the label bytes plus
// final = strong.  reset: the workspace header has not been initialised by a
// classify launch of this call (standalone tracing).
int run_trace(const uint8_t* labels, int64_t batch, int H, int W, uint8_t* fin, const Ws& ws, const WsLayout& L,
              cudaStream_t st, bool finalize, bool reset, const FgBits* bits = nullptr) {
    Range nvtx("edgeforge trace (H1-H4)");
    const int sms = sm_count_current();
    if (reset) EF_CHECK(launch_ws_begin(ws, L, 0, sms, st), "ws_begin");
    FgBits B;
    if (bits && bits->fg) {
        B = *bits;
    } else {
        B = ws_planes(ws, H, W);
        EF_CHECK(launch_hyst_pack(labels, batch, H, W, B, sms, st), "bit-plane pack");
        EF_CHECK(launch_strong_final(labels, (long long)batch * H * W, fin, sms, st), "final = strong");
    }
    EF_CHECK(launch_hyst_local(B, batch, H, W, fin, ws.hb, ws.hdr, sms, st), "hysteresis");
    if (finalize) EF_CHECK(launch_hyst_final(B, batch, H, W, fin, ws.hb, ws.hdr, sms, st), "hysteresis finalize");
    return EF_OK;
}

int check_ws(void* ws, size_t bytes, const WsLayout& L) {
    if (!ws) return fail(EF_EINVAL, "workspace pointer is NULL");
    if (reinterpret_cast<uintptr_t>(ws) % kAlign)
        return fail(EF_EINVAL, "workspace must be 256-byte aligned (cudaMalloc / torch allocations are)");
    if (bytes < L.total)
        return fail(EF_ENOMEM, "workspace too small: need " + std::to_string(L.total) + " bytes, got " +
                                   std::to_string(bytes));
    return EF_OK;
}

}  // namespace

extern "C" {

int ef_abi_version(void) { return EF_ABI_VERSION; }

const char* ef_last_error(void) { return g_err.c_str(); }

size_t ef_workspace_bytes(int64_t batch, int32_t height, int32_t width) {
    if (batch < 1 || height < 1 || width < 1) return 0;
    return ws_layout(batch, height, width).total;
}

int ef_reset_stats(void* d_workspace, size_t workspace_bytes, void* stream) {
    if (!d_workspace || workspace_bytes < sizeof(WsHeader)) return fail(EF_EINVAL, "bad workspace");
    ws_reset_stats_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<WsHeader*>(d_workspace));
    EF_CHECK(cudaGetLastError(), "reset stats");
    return EF_OK;
}

int ef_read_stats(const void* d_workspace, size_t workspace_bytes, void* stream, ef_stats* h_out) {
    if (!d_workspace || workspace_bytes < sizeof(WsHeader) || !h_out) return fail(EF_EINVAL, "bad arguments");
    EF_CHECK(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
    EF_CHECK(cudaMemcpy(h_out, d_workspace, sizeof(ef_stats), cudaMemcpyDeviceToHost), "stats copy");
    return EF_OK;
}

int ef_set_block_tile_threshold(int32_t tiles_per_sm) {
    if (tiles_per_sm < 0) return fail(EF_EINVAL, "tiles_per_sm must be >= 0");
    set_block_tile_threshold(tiles_per_sm);
    return EF_OK;
}

int ef_set_tile_reach(int32_t on) {
    if (on != 0 && on != 1) return fail(EF_EINVAL, "on must be 0 or 1");
    set_tile_reach(on);
    return EF_OK;
}

int ef_read_paths(const void* d_workspace, size_t workspace_bytes, void* stream, uint32_t* h_out) {
    if (!d_workspace || workspace_bytes < sizeof(WsHeader) || !h_out) return fail(EF_EINVAL, "bad arguments");
    EF_CHECK(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
    WsHeader h;
    EF_CHECK(cudaMemcpy(&h, d_workspace, sizeof h, cudaMemcpyDeviceToHost), "header copy");
    h_out[0] = h.overflow;
    h_out[1] = h.plist_overflow;
    h_out[2] = h.dense_count;
    h_out[3] = h.node_overflow;
    return EF_OK;
}

int ef_classify_u8(const uint8_t* d_src, int64_t batch, int32_t height, int32_t width,
                   const double* h_weights, int32_t radius, double low, double high, uint8_t* d_labels,
                   void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(batch, height, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (!d_src || !d_labels) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(batch, height, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    return run_classify_u8(d_src, batch, frame_geom(height, width), h_weights, radius, low, high, d_labels, ws,
                           L, (cudaStream_t)stream);
}

int ef_canny_u8(const uint8_t* d_src, int64_t batch, int32_t height, int32_t width, const double* h_weights,
                int32_t radius, double low, double high, uint8_t* d_labels, uint8_t* d_final,
                void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(batch, height, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (!d_src || !d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(batch, height, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    cudaStream_t st = (cudaStream_t)stream;
    FgBits bits;
    if ((rc = run_classify_u8(d_src, batch, frame_geom(height, width), h_weights, radius, low, high, d_labels,
                              ws, L, st, d_final, &bits)))
        return rc;
    return run_trace(d_labels, batch, height, width, d_final, ws, L, st, true, false, &bits);
}

int ef_set_classify_events(void* start_event, void* stop_event) {
    timing().start = static_cast<cudaEvent_t>(start_event);
    timing().stop = static_cast<cudaEvent_t>(stop_event);
    return EF_OK;
}

int ef_canny_f64(const double* d_src, int64_t batch, int32_t height, int32_t width, const double* h_weights,
                 int32_t radius, double low, double high, uint8_t* d_labels, uint8_t* d_final,
                 void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(batch, height, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (!d_src || !d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(batch, height, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    cudaStream_t st = (cudaStream_t)stream;
    ExactParams XP = make_exact(h_weights, radius, low, high);
    EF_CHECK(launch_exact<double>(d_src, batch, height, width, XP, d_labels, nullptr, nullptr, nullptr, nullptr,
                                  nullptr, nullptr, nullptr, ws.hdr, st),
             "exact kernel");
    return run_trace(d_labels, batch, height, width, d_final, ws, L, st, true, true);
}

int ef_trace_edges(const uint8_t* d_labels, int64_t batch, int32_t height, int32_t width, uint8_t* d_final,
                   void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(batch, height, width))) return rc;
    if (!d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(batch, height, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    return run_trace(d_labels, batch, height, width, d_final, ws, L, (cudaStream_t)stream, true, true);
}

int ef_stages_f64(const uint8_t* d_src8, const double* d_src64, int32_t height, int32_t width,
                  const double* h_weights, int32_t radius, double low, double high, double* d_blurred,
                  double* d_gx, double* d_gy, double* d_magnitude, int64_t* d_orientation, double* d_thinned,
                  uint8_t* d_labels, void* stream) {
    int rc;
    if ((rc = check_dims(1, height, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if ((d_src8 == nullptr) == (d_src64 == nullptr)) return fail(EF_EINVAL, "exactly one source pointer");
    ExactParams XP = make_exact(h_weights, radius, low, high);
    cudaStream_t st = (cudaStream_t)stream;
    if (d_src8)
        EF_CHECK(launch_exact<uint8_t>(d_src8, 1, height, width, XP, d_labels, d_blurred, d_gx, d_gy, d_magnitude,
                                       d_orientation, d_thinned, nullptr, nullptr, st),
                 "exact kernel");
    else
        EF_CHECK(launch_exact<double>(d_src64, 1, height, width, XP, d_labels, d_blurred, d_gx, d_gy, d_magnitude,
                                      d_orientation, d_thinned, nullptr, nullptr, st),
                 "exact kernel");
    return EF_OK;
}

int ef_thinned_max(const uint8_t* d_src8, const double* d_src64, int32_t height, int32_t width,
                   const double* h_weights, int32_t radius, double* d_max, void* stream) {
    int rc;
    if ((rc = check_dims(1, height, width)) || (rc = check_params(h_weights, radius, 0.0, 0.0))) return rc;
    if ((d_src8 == nullptr) == (d_src64 == nullptr) || !d_max) return fail(EF_EINVAL, "bad buffers");
    ExactParams XP = make_exact(h_weights, radius, 0.0, 0.0);
    cudaStream_t st = (cudaStream_t)stream;
    EF_CHECK(cudaMemsetAsync(d_max, 0, sizeof(double), st), "memset");
    auto* bits = reinterpret_cast<unsigned long long*>(d_max);
    if (d_src8)
        EF_CHECK(launch_exact<uint8_t>(d_src8, 1, height, width, XP, nullptr, nullptr, nullptr, nullptr, nullptr,
                                       nullptr, nullptr, bits, nullptr, st),
                 "exact kernel");
    else
        EF_CHECK(launch_exact<double>(d_src64, 1, height, width, XP, nullptr, nullptr, nullptr, nullptr, nullptr,
                                      nullptr, nullptr, bits, nullptr, st),
                 "exact kernel");
    return EF_OK;
}

int ef_nms_f64(const double* d_magnitude, const int64_t* d_orientation, int32_t height, int32_t width,
               double* d_thinned, void* stream) {
    int rc;
    if ((rc = check_dims(1, height, width))) return rc;
    if (!d_magnitude || !d_orientation || !d_thinned) return fail(EF_EINVAL, "NULL buffer");
    EF_CHECK(launch_nms(d_magnitude, d_orientation, height, width, d_thinned, nullptr, (cudaStream_t)stream),
             "nms kernel");
    return EF_OK;
}

int ef_double_threshold_f64(const double* d_thinned, int64_t n, double low, double high, uint8_t* d_labels,
                            void* stream) {
    if (n < 0 || (n && (!d_thinned || !d_labels))) return fail(EF_EINVAL, "bad buffers");
    if (!(0.0 <= low && low <= high)) return fail(EF_EINVAL, "need 0 <= low <= high");
    if (n) EF_CHECK(launch_threshold(d_thinned, n, low, high, d_labels, (cudaStream_t)stream), "threshold kernel");
    return EF_OK;
}

int ef_quantize_f64(const double* d_gx, const double* d_gy, int64_t n, int64_t* d_orientation, void* stream) {
    if (n < 0 || (n && (!d_gx || !d_gy || !d_orientation))) return fail(EF_EINVAL, "bad buffers");
    if (n) EF_CHECK(launch_quantize(d_gx, d_gy, n, d_orientation, (cudaStream_t)stream), "quantize kernel");
    return EF_OK;
}

int ef_laplacian_f64(const double* d_src, int32_t height, int32_t width, double* d_out, void* stream) {
    int rc;
    if ((rc = check_dims(1, height, width))) return rc;
    if (!d_src || !d_out) return fail(EF_EINVAL, "NULL buffer");
    EF_CHECK(launch_laplacian(d_src, height, width, d_out, (cudaStream_t)stream), "laplacian kernel");
    return EF_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline (the drop-in's path: run_pipeline returns host arrays).
// Chunks of frames round-robin over three streams so the H2D copy of chunk
// i+1, the kernels of chunk i and the D2H of chunk i-1 overlap.  The output
// crosses PCIe packed to 2 bits per pixel and is expanded into the caller's
// labels/final arrays by a host thread pool (ef_host.cu); pageable inputs are
// staged into pinned memory by the same pool.
//
// Measured on the B200 box (16-core VM, tools/host_bw.cu, tools/e2e_probe.py):
//  * host DRAM bandwidth is what binds -- the DMA reading the input and the
//    unpack writing 2 B/px share it, so the unpack of a chunk that overlaps
//    copies uses 4 threads (more only slows the DMA), the last chunk all;
//  * the packed staging lines are flushed from the CPU caches after the unpack:
//    DMA writes into CPU-cached pinned lines ran ~3x slower and dragged the
//    concurrent H2D down with them;
//  * chunks ramp up to 8-32 MB (1/32 of the input) and back down, so the pipeline fills and drains
//    quickly while the middle chunks are large enough for the kernels to keep
//    up with the copy engine.
// ---------------------------------------------------------------------------
namespace {
constexpr int kHostStreams = 3;
constexpr int kPackSlots = 2 * kHostStreams;  // packed chunks in flight (D2H or unpack)
// tunables (env overrides for measurement runs: EF_HOST_UNPACK_THREADS, EF_HOST_CHUNK_MB)
int overlap_unpack_threads() {
    static const int n = getenv("EF_HOST_UNPACK_THREADS") ? std::max(1, atoi(getenv("EF_HOST_UNPACK_THREADS"))) : 4;
    return n;
}
// largest chunk: 1/32 of the call's input, between 8 and 32 MB (C1's 132 MB:
// 8 MB, 3.68 vs 3.91 ms at 32 MB; C3's 1 GiB: 32 MB, 24.4 vs 25.7 ms at 8 MB --
// fewer, larger copies once the batch can keep the pipeline full)
size_t max_chunk_bytes(size_t total_bytes) {
    static const size_t env = getenv("EF_HOST_CHUNK_MB") ? std::max<size_t>(1, atoi(getenv("EF_HOST_CHUNK_MB"))) << 20
                                                         : 0;
    if (env) return env;
    return std::min<size_t>((size_t)32 << 20, std::max<size_t>((size_t)8 << 20, total_bytes / 32));
}

struct PackSlot {
    uint8_t* packed = nullptr;   // pinned
    cudaEvent_t done = nullptr;  // recorded after the packed D2H
    Latch latch;
    bool failed = false;
    bool last = false;  // last chunk of the call: unpack with every pool thread
    size_t nbytes = 0, npx = 0;
    uint8_t* labels = nullptr;
    uint8_t* final_map = nullptr;
    bool used = false;
};

struct HostCtx {
    std::mutex mu;
    int dev = -1;
    cudaStream_t st[kHostStreams] = {};
    uint8_t* buf[kHostStreams] = {};  // src | labels | final | packed per stream
    void* ws[kHostStreams] = {};
    uint8_t* stage[kHostStreams] = {};  // pinned staging for pageable inputs
    cudaEvent_t h2d[kHostStreams] = {};
    bool h2d_pending[kHostStreams] = {};
    size_t buf_px = 0, ws_bytes = 0, stage_bytes = 0, slot_bytes = 0;
    PackSlot slot[kPackSlots];
};

HostCtx& host_ctx(int dev) {
    static std::mutex mu;
    static std::unordered_map<int, HostCtx*> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    auto& p = ctxs[dev];
    if (!p) p = new HostCtx();
    return *p;
}

void unpack_part(PackSlot* s, size_t b0, size_t b1) {
    Range nvtx("edgeforge host unpack");
    if (s->labels) unpack_codes(s->packed, b0, b1, s->npx, s->labels, s->final_map);
    else unpack_bits(s->packed, b0, b1, s->npx, s->final_map);  // edges-only call
    flush_lines(s->packed + b0, b1 - b0);
}

// Pool task: wait for the chunk's packed D2H, then fan the unpack out over the
// pool.  (An event wait, not cudaLaunchHostFunc: a host callback would stall
// the stream -- and the next chunk's H2D behind it -- until it returns.)
void fan_out_unpack(PackSlot* s);

#ifndef EF_HOST_POLL
#define EF_HOST_POLL 1
#endif
#ifndef EF_HOST_POLL_US
#define EF_HOST_POLL_US 20
#endif

// Wait for a chunk's event without holding a core and without depending on an
// interrupt: poll with short sleeps.  (Blocking-sync events slept through a lost
// wake-up about once in 25 one-GiB calls on the measured host: one call of 80 ms
// among 24 ms ones, always ~56 ms late.)
cudaError_t wait_event(cudaEvent_t ev) {
#if EF_HOST_POLL
    bool polled = false;
    for (;;) {
        const cudaError_t q = cudaEventQuery(ev);
        if (q != cudaErrorNotReady) {
            // cudaErrorNotReady is left behind as the thread's "last error": a later
            // cudaGetLastError() after a kernel launch (launch_pack) would report it
            if (polled) cudaGetLastError();
            return q;
        }
        polled = true;
        std::this_thread::sleep_for(std::chrono::microseconds(EF_HOST_POLL_US));
    }
#else
    return cudaEventSynchronize(ev);
#endif
}

void wait_and_unpack(PackSlot* s, int device) {
    cudaSetDevice(device);
    if (wait_event(s->done) != cudaSuccess) {
        s->failed = true;
        s->latch.done();
        return;
    }
    fan_out_unpack(s);
}

// The chunk's packed bytes are on the host: expand them with the calling thread
// plus pool threads, then count the chunk done.
void fan_out_unpack(PackSlot* s) {
    HostPool& P = host_pool();
    const size_t threads = s->last ? (size_t)P.size() : (size_t)std::min(P.size(), overlap_unpack_threads());
    const size_t parts = std::max<size_t>(1, std::min<size_t>(threads, s->nbytes / 16384));
    const size_t per = ((s->nbytes + parts - 1) / parts + 63) & ~size_t(63);
    const int n = (int)((s->nbytes + per - 1) / per);
    s->latch.add(n - 1);
    for (size_t b0 = per; b0 < s->nbytes; b0 += per) {
        const size_t b1 = std::min(s->nbytes, b0 + per);
        P.submit([s, b0, b1] {
            unpack_part(s, b0, b1);
            s->latch.done();
        }, true);
    }
    unpack_part(s, 0, std::min(s->nbytes, per));
    s->latch.done();
}

// 0: pinned host (DMA directly), 1: pageable (stage), 2: device/managed
int host_kind(const void* p, size_t bytes) {
    cudaPointerAttributes a;
    auto kind = [&](const void* q) {
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return 1;
        }
        if (a.type == cudaMemoryTypeHost) return 0;
        if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return 2;
        return 1;
    };
    const int k0 = kind(p);
    if (k0 == 1 || bytes <= 1) return k0;
    return kind(static_cast<const uint8_t*>(p) + bytes - 1) == k0 ? k0 : 1;
}

// wait until every queued chunk has landed in the caller's arrays
bool drain(HostCtx& C) {
    for (int i = 0; i < kHostStreams; ++i)
        if (C.st[i]) cudaStreamSynchronize(C.st[i]);
    bool failed = false;
    for (auto& s : C.slot) {
        if (!s.used) continue;
        s.latch.wait();
        failed |= s.failed;
        s.used = false;
    }
    for (int i = 0; i < kHostStreams; ++i) C.h2d_pending[i] = false;
    return failed;
}

// frames per chunk: ramp up from max/8 to the max chunk, hold, ramp back down
std::vector<int64_t> chunk_plan(int64_t batch, size_t fpx) {
    const size_t cbytes = max_chunk_bytes((size_t)batch * fpx);
    const int64_t cmax = std::max<int64_t>(1, (int64_t)(cbytes / fpx));
    const int64_t c0 = std::max<int64_t>(1, std::min<int64_t>(cmax, (int64_t)((cbytes / 8) / fpx)));
    std::vector<int64_t> ramp;
    for (int64_t c = c0; c < cmax; c *= 2) ramp.push_back(c);
    int64_t ramp_sum = 0;
    for (int64_t c : ramp) ramp_sum += c;
    std::vector<int64_t> plan;
    if (2 * ramp_sum + cmax > batch) {  // short batch: up to three near-equal chunks of <= cmax
        const int64_t n = std::max<int64_t>(std::min<int64_t>(batch, kHostStreams), (batch + cmax - 1) / cmax);
        for (int64_t i = 0; i < n; ++i) plan.push_back(batch / n + (i < batch % n ? 1 : 0));
        return plan;
    }
    plan = ramp;
    int64_t mid = batch - 2 * ramp_sum;
    while (mid > 0) {
        const int64_t c = std::min(mid, cmax);
        plan.push_back(c);
        mid -= c;
    }
    plan.insert(plan.end(), ramp.rbegin(), ramp.rend());
    return plan;
}
}  // namespace

int ef_host_f64_to_u8(const double* src, int64_t n, uint8_t* dst) {
    if (n < 0 || (n > 0 && (!src || !dst))) return fail(EF_EINVAL, "bad buffers");
    return parallel_f64_to_u8(src, (size_t)n, dst) ? 1 : 0;
}

int ef_canny_u8_host(const uint8_t* h_src, int64_t batch, int32_t height, int32_t width, const double* h_weights,
                     int32_t radius, double low, double high, uint8_t* h_labels, uint8_t* h_final,
                     int32_t device) {
    int rc;
    if ((rc = check_dims(batch, height, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (!h_src || !h_final) return fail(EF_EINVAL, "NULL buffer");  // h_labels == NULL: edges only
    Range nvtx("edgeforge canny_u8_host");
    EF_CHECK(cudaSetDevice(device), "cudaSetDevice");
    HostCtx& C = host_ctx(device);
    std::lock_guard<std::mutex> lk(C.mu);
    const size_t fpx = (size_t)height * width;
    const std::vector<int64_t> plan = chunk_plan(batch, fpx);
    const int64_t chunk = *std::max_element(plan.begin(), plan.end());
    const size_t need_px = align_up((size_t)chunk * fpx);
    const size_t need_packed = align_up(need_px / 4 + 1);
    const size_t need_ws = ef_workspace_bytes(chunk, height, width);
    const int src_kind = host_kind(h_src, (size_t)batch * fpx);
    if (C.dev != device) {
        C.dev = device;
        // a pool thread waiting on a chunk must not spin on a core the unpack needs:
        // wait_event polls with short sleeps (EF_HOST_POLL=0: blocking-sync events)
        const unsigned evflags = cudaEventDisableTiming | (EF_HOST_POLL ? 0u : (unsigned)cudaEventBlockingSync);
        for (int i = 0; i < kHostStreams; ++i) {
            EF_CHECK(cudaStreamCreateWithFlags(&C.st[i], cudaStreamNonBlocking), "stream");
            EF_CHECK(cudaEventCreateWithFlags(&C.h2d[i], evflags), "event");
        }
        for (auto& s : C.slot) EF_CHECK(cudaEventCreateWithFlags(&s.done, evflags), "event");
    }
    if (C.buf_px < need_px || C.ws_bytes < need_ws) {
        for (int i = 0; i < kHostStreams; ++i) {
            if (C.buf[i]) cudaFree(C.buf[i]);
            if (C.ws[i]) cudaFree(C.ws[i]);
            C.buf[i] = nullptr;
            C.ws[i] = nullptr;
        }
        C.buf_px = C.ws_bytes = 0;
        for (int i = 0; i < kHostStreams; ++i) {
            EF_CHECK(cudaMalloc(&C.buf[i], 3 * need_px + need_packed), "cudaMalloc");
            EF_CHECK(cudaMalloc(&C.ws[i], need_ws), "cudaMalloc");
        }
        C.buf_px = need_px;
        C.ws_bytes = need_ws;
    }
    if (C.slot_bytes < need_packed) {
        for (auto& s : C.slot) {
            if (s.packed) cudaFreeHost(s.packed);
            s.packed = nullptr;
        }
        C.slot_bytes = 0;
        for (auto& s : C.slot) EF_CHECK(cudaMallocHost(&s.packed, need_packed), "cudaMallocHost");
        C.slot_bytes = need_packed;
    }
    if (src_kind == 1 && C.stage_bytes < need_px) {
        for (int i = 0; i < kHostStreams; ++i) {
            if (C.stage[i]) cudaFreeHost(C.stage[i]);
            C.stage[i] = nullptr;
        }
        C.stage_bytes = 0;
        for (int i = 0; i < kHostStreams; ++i) EF_CHECK(cudaMallocHost(&C.stage[i], need_px), "cudaMallocHost");
        C.stage_bytes = need_px;
    }
    const int sms = sm_count_current();
    int64_t f0 = 0;
    for (size_t i = 0; i < plan.size(); f0 += plan[i], ++i) {
        Range nvtx_chunk("edgeforge host chunk (H2D, kernels, packed D2H)");
        const int k = (int)(i % kHostStreams);
        PackSlot& s = C.slot[i % kPackSlots];
        const int64_t n = plan[i];
        const size_t bytes = (size_t)n * fpx;
        cudaStream_t st = C.st[k];
        uint8_t* d_src = C.buf[k];
        uint8_t* d_lab = d_src + C.buf_px;
        uint8_t* d_fin = d_lab + C.buf_px;
        uint8_t* d_packed = d_fin + C.buf_px;
        cudaError_t e = cudaSuccess;
        if (s.used) {  // the slot's previous chunk must be unpacked before its D2H is overwritten
            s.latch.wait();
            s.used = false;
            if (s.failed) e = cudaErrorUnknown;
        }
        const uint8_t* src = h_src + f0 * fpx;
        if (e == cudaSuccess && src_kind == 1) {
            if (C.h2d_pending[k]) e = wait_event(C.h2d[k]);
            if (e == cudaSuccess) parallel_copy(C.stage[k], src, bytes);
            src = C.stage[k];
        }
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_src, src, bytes, src_kind == 2 ? cudaMemcpyDefault : cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess && src_kind == 1) {
            e = cudaEventRecord(C.h2d[k], st);
            C.h2d_pending[k] = true;
        }
        if (e != cudaSuccess) {
            drain(C);
            return cuda_fail(e, "H2D");
        }
        if ((rc = ef_canny_u8(d_src, n, height, width, h_weights, radius, low, high, d_lab, d_fin, C.ws[k],
                              C.ws_bytes, st))) {
            drain(C);
            return rc;
        }
        const size_t pbytes = h_labels ? (bytes + 3) / 4 : (bytes + 7) / 8;
        e = h_labels ? launch_pack(d_lab, d_fin, (long long)bytes, d_packed, sms, st)
                     : launch_pack_final(d_fin, (long long)bytes, d_packed, sms, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(s.packed, d_packed, pbytes, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) {
            s.nbytes = pbytes;
            s.npx = bytes;
            s.labels = h_labels ? h_labels + f0 * fpx : nullptr;
            s.final_map = h_final + f0 * fpx;
            s.last = i + 1 == plan.size();
            e = cudaEventRecord(s.done, st);
        }
        if (e != cudaSuccess) {
            drain(C);
            return cuda_fail(e, "D2H");
        }
        s.used = true;
        s.failed = false;
        s.latch.add(1);
        PackSlot* sp = &s;
        if (plan.size() == 1) {
            // one chunk (a single frame, a small batch): nothing to overlap, so the calling
            // thread waits on the stream itself and unpacks -- a pool hand-off and a
            // blocking-sync event wake-up cost ~0.1 ms of a 0.27 ms call on one 512x512 frame
            if (cudaStreamSynchronize(st) != cudaSuccess) {
                s.failed = true;
                s.latch.done();
            } else {
                fan_out_unpack(sp);
            }
        } else {
            host_pool().submit([sp, device] { wait_and_unpack(sp, device); });
        }
    }
    cudaError_t first = cudaSuccess;
    for (int k = 0; k < kHostStreams; ++k) {
        cudaError_t e = cudaStreamSynchronize(C.st[k]);
        if (first == cudaSuccess) first = e;
    }
    const bool failed = drain(C);
    if (first != cudaSuccess) return cuda_fail(first, "sync");
    if (failed) return fail(EF_ECUDA, "D2H of packed edges failed");
    return EF_OK;
}

// ---------------------------------------------------------------------------
// Row bands (multi-GPU partition of one frame).
// ---------------------------------------------------------------------------
int ef_band_halo_rows(int32_t radius) { return radius + 2; }

int ef_band_canny_u8(const uint8_t* d_src, int32_t row0, int32_t rows, int32_t full_height, int32_t width,
                     const double* h_weights, int32_t radius, double low, double high, uint8_t* d_labels,
                     uint8_t* d_final, void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(1, rows, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (row0 < 0 || row0 + rows > full_height) return fail(EF_EINVAL, "band outside the frame");
    if (!d_src || !d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(1, rows, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    const int halo = radius + 2;
    const int ht = std::min(row0, halo), hb = std::min(full_height - row0 - rows, halo);
    FrameGeom g{ht + rows + hb, width, row0 - ht, full_height, row0, rows};
    cudaStream_t st = (cudaStream_t)stream;
    FgBits bits;
    if ((rc = run_classify_u8(d_src, 1, g, h_weights, radius, low, high, d_labels, ws, L, st, d_final, &bits)))
        return rc;
    return run_trace(d_labels, 1, rows, width, d_final, ws, L, st, false, false, &bits);
}

int ef_band_canny_u8_peer(const uint8_t* d_band, const uint8_t* d_top, int32_t top_rows, const uint8_t* d_bot,
                          int32_t bot_rows, int32_t row0, int32_t rows, int32_t full_height, int32_t width,
                          const double* h_weights, int32_t radius, double low, double high, uint8_t* d_labels,
                          uint8_t* d_final, void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(1, rows, width)) || (rc = check_params(h_weights, radius, low, high))) return rc;
    if (row0 < 0 || row0 + rows > full_height) return fail(EF_EINVAL, "band outside the frame");
    if (!d_band || !d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    const int halo = radius + 2;
    const int ht = std::min(row0, halo), hb = std::min(full_height - row0 - rows, halo);
    if (top_rows != ht || bot_rows != hb || (ht > 0 && !d_top) || (hb > 0 && !d_bot))
        return fail(EF_EINVAL, "peer halos must hold min(row0, radius+2) rows above and "
                               "min(full_height-row0-rows, radius+2) rows below the band");
    FastParams FP = make_fast(h_weights, radius, low, high);
    if (has_negative(h_weights, radius)) return fail(EF_EINVAL, "signed kernel on a band");
    if (!aligned4(d_band) || !aligned4(d_labels) || !aligned4(d_final) || (ht && !aligned4(d_top)) ||
        (hb && !aligned4(d_bot)))
        return fail(EF_EINVAL, "peer halos need 4-byte aligned band, halo, labels and final buffers");
    FrameGeom g{ht + rows + hb, width, row0 - ht, full_height, row0, rows};
    g.top = ht > 0 ? d_top : nullptr;
    g.bot = hb > 0 ? d_bot : nullptr;
    // the halo rows are read in place by the classifier kernel (needs W % 4 == 0
    // and radius <= 6 -- the production kernel; without peers the buffer is contiguous)
    if ((g.top || g.bot) && !k1v2_supported(FP, g))
        return fail(EF_EINVAL, "peer halos need width % 4 == 0 and radius <= 6");
    WsLayout L = ws_layout(1, rows, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    cudaStream_t st = (cudaStream_t)stream;
    FgBits bits;
    if ((rc = run_classify_u8(d_band, 1, g, h_weights, radius, low, high, d_labels, ws, L, st, d_final, &bits)))
        return rc;
    return run_trace(d_labels, 1, rows, width, d_final, ws, L, st, false, false, &bits);
}

// CUDA IPC of a device buffer (any pointer inside an allocation): the handle of
// its allocation plus the offset, so another process can read it in place.
int ef_ipc_export(const void* d_ptr, void* h_handle64, uint64_t* h_offset) {
    if (!d_ptr || !h_handle64 || !h_offset) return fail(EF_EINVAL, "bad arguments");
    static const auto range_fn = []() -> CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(p);
        return nullptr;
    }();
    if (!range_fn) return fail(EF_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return fail(EF_EINVAL, "pointer is not inside a device allocation");
    cudaIpcMemHandle_t h;
    EF_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(h_handle64, &h, sizeof h);
    *h_offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return EF_OK;
}

int ef_ipc_open(const void* h_handle64, uint64_t offset, void** d_ptr_out, void** d_base_out) {
    if (!h_handle64 || !d_ptr_out || !d_base_out) return fail(EF_EINVAL, "bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h_handle64, sizeof h);
    void* base = nullptr;
    EF_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    *d_base_out = base;
    *d_ptr_out = static_cast<char*>(base) + offset;
    return EF_OK;
}

int ef_ipc_close(void* d_base) {
    if (!d_base) return fail(EF_EINVAL, "bad arguments");
    EF_CHECK(cudaIpcCloseMemHandle(d_base), "cudaIpcCloseMemHandle");
    return EF_OK;
}

int ef_band_trace(const uint8_t* d_labels, int32_t rows, int32_t width, uint8_t* d_final, void* d_workspace,
                  size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(1, rows, width))) return rc;
    if (!d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    WsLayout L = ws_layout(1, rows, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    Ws ws = ws_bind(d_workspace, L);
    return run_trace(d_labels, 1, rows, width, d_final, ws, L, (cudaStream_t)stream, false, true);
}

int ef_band_edges(const void* d_workspace, size_t workspace_bytes, int32_t rows, int32_t width, int64_t* d_ids,
                  uint8_t* d_strong, void* stream) {
    int rc;
    if ((rc = check_dims(1, rows, width))) return rc;
    WsLayout L = ws_layout(1, rows, width);
    if ((rc = check_ws(const_cast<void*>(d_workspace), workspace_bytes, L))) return rc;
    if (!d_ids || !d_strong) return fail(EF_EINVAL, "NULL buffer");
    Ws ws = ws_bind(const_cast<void*>(d_workspace), L);
    EF_CHECK(launch_band_edges(rows, width, ws.hb, ws_planes(ws, rows, width), d_ids, d_strong, (cudaStream_t)stream),
             "band edges");
    return EF_OK;
}

size_t ef_band_merge_scratch_bytes(int32_t nbands, int32_t width) {
    if (nbands < 1 || width < 1 || (long long)nbands * 2 * width > (1ll << 30)) return 0;
    return band_merge_scratch_bytes(nbands, width);
}

int ef_band_merge_device(int32_t nbands, int32_t width, const int64_t* d_ids, const uint8_t* d_strong,
                         uint8_t* d_strong_out, void* d_scratch, size_t scratch_bytes, void* stream) {
    const size_t need = ef_band_merge_scratch_bytes(nbands, width);
    if (!need) return fail(EF_EINVAL, "bad band merge dimensions");
    if (!d_ids || !d_strong || !d_strong_out || !d_scratch) return fail(EF_EINVAL, "NULL buffer");
    if (scratch_bytes < need) return fail(EF_EINVAL, "band merge scratch too small");
    EF_CHECK(launch_band_merge(nbands, width, d_ids, d_strong, d_strong_out, d_scratch, (cudaStream_t)stream),
             "band merge");
    return EF_OK;
}

int ef_band_finalize(const uint8_t* d_strong_edges, int32_t rows, int32_t width, const uint8_t* d_labels,
                     uint8_t* d_final, void* d_workspace, size_t workspace_bytes, void* stream) {
    int rc;
    if ((rc = check_dims(1, rows, width))) return rc;
    WsLayout L = ws_layout(1, rows, width);
    if ((rc = check_ws(d_workspace, workspace_bytes, L))) return rc;
    if (!d_strong_edges || !d_labels || !d_final) return fail(EF_EINVAL, "NULL buffer");
    Ws ws = ws_bind(d_workspace, L);
    cudaStream_t st = (cudaStream_t)stream;
    EF_CHECK(launch_band_apply(rows, width, ws.hb, d_strong_edges, st), "band apply");
    EF_CHECK(launch_hyst_final(ws_planes(ws, rows, width), 1, rows, width, d_final, ws.hb, ws.hdr, sm_count_current(),
                               st),
             "hysteresis finalize");
    return EF_OK;
}

// Serial union-find over the band-edge components, the analogue of
// hysteresis.py:112-130 (pairs at shifts -1/0/+1 across each band seam).
int ef_band_merge(int32_t nbands, int32_t width, const int64_t* h_ids, const uint8_t* h_strong,
                  uint8_t* h_strong_out) {
    if (nbands < 1 || width < 1 || !h_ids || !h_strong || !h_strong_out) return fail(EF_EINVAL, "bad arguments");
    const size_t n = (size_t)nbands * 2 * width;
    std::unordered_map<int64_t, int> index;
    index.reserve(n);
    std::vector<int> parent;
    std::vector<uint8_t> strong;
    std::vector<int> slot(n, -1);
    for (size_t i = 0; i < n; ++i) {
        if (h_ids[i] < 0) continue;
        auto it = index.find(h_ids[i]);
        int id;
        if (it == index.end()) {
            id = (int)parent.size();
            index.emplace(h_ids[i], id);
            parent.push_back(id);
            strong.push_back(0);
        } else {
            id = it->second;
        }
        slot[i] = id;
        if (h_strong[i]) strong[id] = 1;
    }
    auto find = [&](int a) {
        while (parent[a] != a) {
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        return a;
    };
    for (int b = 0; b + 1 < nbands; ++b) {
        const int* top = &slot[(size_t)b * 2 * width + width];   // bottom row of band b
        const int* bot = &slot[(size_t)(b + 1) * 2 * width];     // top row of band b+1
        for (int x = 0; x < width; ++x) {
            if (top[x] < 0) continue;
            for (int s = -1; s <= 1; ++s) {
                int x2 = x + s;
                if (x2 < 0 || x2 >= width || bot[x2] < 0) continue;
                int ra = find(top[x]), rb = find(bot[x2]);
                if (ra != rb) {
                    parent[rb] = ra;
                    strong[ra] = strong[ra] | strong[rb];
                }
            }
        }
    }
    for (size_t i = 0; i < n; ++i) h_strong_out[i] = slot[i] < 0 ? 0 : strong[find(slot[i])];
    return EF_OK;
}

}  // extern "C"
