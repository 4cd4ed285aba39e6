// ef_hystb.cu -- hysteresis by bit-parallel row sweeps (trace_edges,
// hysteresis.py:63-69) over the classifier's foreground bit planes: the fused
// path of ef_canny_u8.
//
// The reference keeps every 8-connected component of labels != 0 that holds a
// strong pixel.  Equivalently: the final set F is the smallest set with
// strong ⊆ F ⊆ fg that is closed under 8-adjacency inside fg.  Here F is grown
// by word-parallel operations on the 1-bit-per-pixel planes:
//
//   * a warp owns a block of 32 rows x S words (lane = one 64-bit word of a
//     row; frames up to 32 words = 2048 columns wide, S = words rounded up to
//     a power of two, a warp holds 32 / S blocks side by side);
//   * row fill: the runs of fg that contain a seed, found with one 64-bit add
//     per word -- f + s carries from every seed through its run (bits up to
//     the run's top), the same on the bit-reversed word gives the bits down to
//     the run's start; a carry that leaves a word enters the next lane's
//     word, resolved for the whole warp with two ballots and one 32-bit add
//     (carry-lookahead over lanes) only when some carry crossed a word;
//   * vertical growth: row r's seeds include the 8-neighbour dilation of row
//     r-1 (down sweep) or r+1 (up sweep); sweeps alternate until an up sweep
//     changes nothing (then every row is closed against both neighbours);
//   * pass 1 closes every block from its own strong pixels and exports its
//     first and last rows (final bits, undecided bits); pass 2 walks each
//     frame's blocks down and up with one warp per frame group, re-closing a
//     block when a neighbour's final border row touches its undecided border
//     pixels -- the block-level analogue of the row sweeps, so a chain through
//     many blocks costs one walk per change of direction, not one grid-wide
//     round per block.
//
// Only weak pixels that join an edge are written (K1 already wrote final =
// strong).  The result is the unique closure, the same set the reference's
// labelling keeps.  Wider frames (C2, C4) use the tile union-find (ef_hyst.cu).
#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_launch.cuh"

#include <algorithm>
#include <atomic>

namespace ef {

namespace {

constexpr int HB_R = 32;       // rows per block
constexpr int HB_WARPS = 4;    // warps per CTA
constexpr unsigned FULL = 0xffffffffu;
typedef unsigned long long u64;

__device__ __forceinline__ u64 brev64(u64 x) {
    return ((u64)__brev((unsigned)x) << 32) | (u64)__brev((unsigned)(x >> 32));
}

// a + b with the carry out of bit 63
__device__ __forceinline__ u64 add_co(u64 a, u64 b, unsigned& co) {
    unsigned lo, hi, c;
    asm("add.cc.u32 %0, %3, %5;\n\t"
        "addc.cc.u32 %1, %4, %6;\n\t"
        "addc.u32 %2, 0, 0;"
        : "=r"(lo), "=r"(hi), "=r"(c)
        : "r"((unsigned)a), "r"((unsigned)(a >> 32)), "r"((unsigned)b), "r"((unsigned)(b >> 32)));
    co = c;
    return ((u64)hi << 32) | lo;
}

// Carry into every lane (bit i = lane i) given each lane's generate G and
// propagate P (exclusive); carries flow from bit i to bit i+1 and die at the
// bits in `cut` (the last lane of every block).  X + G adds g+g (generate) or
// p+0 (propagate) at every position, so its carries are exactly the lanes'.
__device__ __forceinline__ unsigned carries(unsigned G, unsigned P, unsigned cut) {
    G &= ~cut;
    P &= ~cut;
    const unsigned X = G | P;
    return (X + G) ^ P;  // (X + G) ^ X ^ G, and X ^ G == P
}

struct Seg {
    int lane, sl;        // lane, lane inside the block (word of the row)
    unsigned last_cut;   // lanes that are the last word of their block
    unsigned first_cut;  // the same for the reversed lane order
    int S;
};

// The runs of f (a row of the block, one word per lane) that contain a bit of
// s (s within f): bits from each run's start to its end, across words.
__device__ __forceinline__ u64 fill_row(u64 f, u64 s, const Seg& q) {
    unsigned co;
    u64 a = add_co(f, s, co);
    const unsigned G = __ballot_sync(FULL, co) & ~q.last_cut;
    if (G) {  // a carry left some word inside a block (warp-uniform branch)
        const unsigned P = __ballot_sync(FULL, a == ~0ull);
        a += (carries(G, P, q.last_cut) >> q.lane) & 1u;
    }
    const u64 up = ((a ^ f) & f) | s;  // from each seeded run's lowest seed to its top
    // the same towards lower columns: bit-reversed words, carries to lower lanes
    const u64 rf = brev64(f), ru = brev64(up);
    u64 b = add_co(rf, ru, co);
    const unsigned G2 = __brev(__ballot_sync(FULL, co)) & ~q.first_cut;
    if (G2) {
        const unsigned P2 = __brev(__ballot_sync(FULL, b == ~0ull));
        b += (carries(G2, P2, q.first_cut) >> (31 - q.lane)) & 1u;
    }
    return brev64(((b ^ rf) & rf) | ru);
}

// 8-neighbour dilation of a row inside its block: x | x << 1 | x >> 1 across words
__device__ __forceinline__ u64 dil_row(u64 x, const Seg& q) {
    const unsigned from_left = __shfl_up_sync(FULL, (unsigned)(x >> 32), 1, q.S);  // word to the left: bit 63
    const unsigned from_right = __shfl_down_sync(FULL, (unsigned)x, 1, q.S);      // word to the right: bit 0
    u64 d = x | (x << 1) | (x >> 1);
    if (q.sl > 0) d |= (u64)(from_left >> 31);
    if (q.sl < q.S - 1) d |= (u64)(from_right & 1u) << 63;
    return d;
}

struct HbGeom {
    int H, W, words;  // output rows per frame, columns, 64-bit words per row (<= 32)
    int S, lg_s;      // words (lanes) per block, a power of two; blocks per warp = 32 / S
    int RB;           // row blocks per frame
    long long frames, nblocks, nwb, nfg;  // frames, blocks, warp-blocks, frame groups (32 / S frames)
};

struct HbBufs {
    u64* ftop;  // [block * S + word]: final bits of the block's first row
    u64* utop;  //   foreground bits of that row that are not final
    u64* fbot;  //   the same for the block's last row
    u64* ubot;
};

__device__ __forceinline__ u64 ldcg64(const u64* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned seg_mask(const Seg& q) {
    return (q.S == 32 ? FULL : ((1u << q.S) - 1u)) << (q.lane & ~(q.S - 1));
}

// Close block b (this lane's segment; b < 0: the segment is idle) from its
// strong pixels plus the seed rows etop / ebot (already dilated from the
// neighbours' borders) and export its border rows.  Writes final = 1 for the
// weak pixels that joined an edge.  Every lane of the warp must call this.
__device__ void hb_close(const HbGeom& G, const FgBits& B, uint8_t* __restrict__ final_out, const HbBufs& hb,
                         long long b, u64 etop, u64 ebot, const Seg& q, u64 (*sfg)[32]) {
    const bool run = b >= 0;
    long long f = 0;
    int by = 0;
    if (run) {
        f = b / G.RB;
        by = (int)(b - f * G.RB);
    }
    const int y0 = by * HB_R;
    const bool lane_ok = run && q.sl < G.words;
    const u64* fgp = B.fg + (u64)f * B.frame_words + (u64)y0 * G.words + q.sl;
    const u64* stp = B.st + (u64)f * B.frame_words + (u64)y0 * G.words + q.sl;
    u64 F[HB_R];
#pragma unroll
    for (int r = 0; r < HB_R; ++r) {
        const bool ok = lane_ok && y0 + r < G.H;
        sfg[r][q.lane] = ok ? __ldg(fgp + (size_t)r * G.words) : 0ull;
        F[r] = ok ? __ldg(stp + (size_t)r * G.words) : 0ull;
    }
    F[0] |= etop & sfg[0][q.lane];
    F[HB_R - 1] |= ebot & sfg[HB_R - 1][q.lane];
    __syncwarp();
    // nothing to grow: no weak pixel, or no seed at all
    bool weak = false, seed = false;
#pragma unroll
    for (int r = 0; r < HB_R; ++r) {
        weak |= (sfg[r][q.lane] & ~F[r]) != 0ull;
        seed |= F[r] != 0ull;
    }
    if (__any_sync(FULL, weak && seed)) {
        // first down sweep: every row is filled (the seeds are not yet closed along rows)
        u64 prev = 0ull;
#pragma unroll
        for (int r = 0; r < HB_R; ++r) {
            const u64 fr = sfg[r][q.lane];
            F[r] = fill_row(fr, r ? (F[r] | (dil_row(prev, q) & fr)) : F[r], q);
            prev = F[r];
        }
        bool first = true;
        while (true) {
            if (!first) {  // down sweep over closed rows: fill only where the row above adds seeds
                prev = 0ull;
#pragma unroll
                for (int r = 0; r < HB_R; ++r) {
                    const u64 fr = sfg[r][q.lane];
                    const u64 add = r ? (dil_row(prev, q) & fr & ~F[r]) : 0ull;
                    if (__any_sync(FULL, add != 0ull)) F[r] = fill_row(fr, F[r] | add, q);
                    prev = F[r];
                }
            }
            first = false;
            bool changed = false;
            prev = 0ull;
#pragma unroll
            for (int r = HB_R - 1; r >= 0; --r) {
                const u64 fr = sfg[r][q.lane];
                const u64 add = r < HB_R - 1 ? (dil_row(prev, q) & fr & ~F[r]) : 0ull;
                if (__any_sync(FULL, add != 0ull)) {
                    F[r] = fill_row(fr, F[r] | add, q);
                    changed = true;
                }
                prev = F[r];
            }
            if (!__any_sync(FULL, changed)) break;
        }
    }
    // ---- weak pixels that joined an edge: final = 1 (strong ones are written by K1)
    if (lane_ok) {
        uint8_t* fbase = final_out + (size_t)f * G.H * G.W + (size_t)y0 * G.W + (size_t)q.sl * 64;
#pragma unroll
        for (int r = 0; r < HB_R; ++r) {
            u64 wf = y0 + r < G.H ? F[r] & ~__ldg(stp + (size_t)r * G.words) : 0ull;
            while (wf) {
                const int bit = __ffsll((long long)wf) - 1;
                wf &= wf - 1;
                fbase[(size_t)r * G.W + bit] = 1;
            }
        }
    }
    // ---- export the border rows
    if (run) {
        const long long bS = b * G.S + q.sl;
        hb.ftop[bS] = F[0];
        hb.utop[bS] = sfg[0][q.lane] & ~F[0];
        hb.fbot[bS] = F[HB_R - 1];
        hb.ubot[bS] = sfg[HB_R - 1][q.lane] & ~F[HB_R - 1];
    }
    __syncwarp();  // sfg is reused by the warp's next block
}

__device__ __forceinline__ Seg make_seg(int S) {
    Seg q;
    q.lane = threadIdx.x & 31;
    q.S = S;
    q.sl = q.lane & (S - 1);
    unsigned last = 0;
    for (int l = S - 1; l < 32; l += S) last |= 1u << l;
    q.last_cut = last;
    q.first_cut = __brev(last >> (S - 1));  // first lanes, in reversed lane order
    return q;
}

// Pass 1: every block closed from its own strong pixels (32 / S consecutive
// blocks per warp).
__global__ void __launch_bounds__(32 * HB_WARPS, 3)
hb_pass1_kernel(FgBits B, HbGeom G, uint8_t* __restrict__ final_out, HbBufs hb) {
    __shared__ u64 sfg[HB_WARPS][HB_R][32];
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5;
    const Seg q = make_seg(G.S);
    const long long gw = (long long)blockIdx.x * HB_WARPS + warp, nw = (long long)gridDim.x * HB_WARPS;
    for (long long wb = gw; wb < G.nwb; wb += nw) {
        const long long b = wb * (32 >> G.lg_s) + (q.lane >> G.lg_s);
        hb_close(G, B, final_out, hb, b < G.nblocks ? b : -1, 0ull, 0ull, q, sfg[warp]);
    }
}

// Pass 2: one warp per group of 32 / S frames walks each frame's blocks down
// and up (the block-level analogue of the row sweeps): a block whose
// neighbour's final border row touches one of its undecided border pixels is
// closed again with that row as extra seeds.  A chain through many blocks
// moves with the walk (one pass per change of vertical direction), and the
// walks repeat until an up walk re-closes nothing.
__global__ void __launch_bounds__(32 * HB_WARPS, 3)
hb_pass2_kernel(FgBits B, HbGeom G, uint8_t* __restrict__ final_out, HbBufs hb, WsHeader* hdr) {
    __shared__ u64 sfg[HB_WARPS][HB_R][32];
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5;
    const Seg q = make_seg(G.S);
    const long long fg_id = (long long)blockIdx.x * HB_WARPS + warp;
    if (fg_id >= G.nfg) return;
    const long long f = fg_id * (32 >> G.lg_s) + (q.lane >> G.lg_s);
    const bool fok = f < G.frames;
    const int S = G.S;
    unsigned walks = 0;
    auto visit = [&](int by) -> bool {  // re-close block by of this lane's frame if a neighbour reaches it
        const long long b = f * G.RB + by;
        u64 xt = 0, xb = 0;
        if (fok && by > 0) xt = ldcg64(hb.fbot + (b - 1) * S + q.sl);
        if (fok && by < G.RB - 1) xb = ldcg64(hb.ftop + (b + 1) * S + q.sl);
        const u64 dt = dil_row(xt, q), db = dil_row(xb, q);
        bool contact = false;
        if (fok) contact = ((dt & ldcg64(hb.utop + b * S + q.sl)) | (db & ldcg64(hb.ubot + b * S + q.sl))) != 0ull;
        const unsigned cm = __ballot_sync(FULL, contact);
        if (!cm) return false;
        const bool mine = (cm & seg_mask(q)) != 0u;
        hb_close(G, B, final_out, hb, mine ? b : -1, dt, db, q, sfg[warp]);
        return true;
    };
    while (true) {
        for (int by = 1; by < G.RB; ++by) visit(by);
        bool any = false;
        for (int by = G.RB - 2; by >= 0; --by) any |= visit(by);
        walks += 2;
        if (!any) break;
    }
    if (q.lane == 0) atomicMax(&hdr->pad[2], walks);
}

// labels (u8 0/1/2) -> foreground / strong bit planes, one thread per 64-bit
// word (standalone tracing, ef_trace_edges)
__global__ void hb_pack_kernel(const uint8_t* __restrict__ labels, long long rows, int W, int words,
                               u64* __restrict__ fg, u64* __restrict__ st) {
    pdl_wait();
    pdl_trigger();
    const long long n = rows * words;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / words;
        const int j = (int)(i - row * words);
        const uint8_t* p = labels + row * W + 64 * j;
        const int n8 = min(64, W - 64 * j);
        u64 f = 0, s = 0;
        if (n8 == 64 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
                const unsigned w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const unsigned nz = (w4[t] | (w4[t] >> 1)) & 0x01010101u, sg = (w4[t] >> 1) & 0x01010101u;
                    f |= (u64)((nz * 0x10204080u) >> 28) << (16 * q + 4 * t);
                    s |= (u64)((sg * 0x10204080u) >> 28) << (16 * q + 4 * t);
                }
            }
        } else {
            for (int b = 0; b < n8; ++b) {
                const unsigned v = p[b];
                f |= (u64)(v != 0u) << b;
                s |= (u64)(v >= 2u) << b;
            }
        }
        fg[i] = f;
        st[i] = s;
    }
}

// final = strong for every pixel (the fused classifier writes this itself)
__global__ void strong_final_kernel(const uint8_t* __restrict__ labels, long long n, uint8_t* __restrict__ fin) {
    pdl_wait();
    pdl_trigger();
    const bool vec = ((reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(fin)) & 15) == 0;
    const long long nv = vec ? n / 16 : 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(labels) + i);
        reinterpret_cast<uint4*>(fin)[i] =
            make_uint4((v.x >> 1) & 0x01010101u, (v.y >> 1) & 0x01010101u, (v.z >> 1) & 0x01010101u,
                       (v.w >> 1) & 0x01010101u);
    }
    for (long long i = nv * 16 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        fin[i] = labels[i] >= 2 ? 1 : 0;
}

int pow2_at_least(int v) {
    int s = 1;
    while (s < v) s <<= 1;
    return s;
}

HbGeom hb_geom(int64_t batch, int H, int W) {
    HbGeom G;
    G.H = H;
    G.W = W;
    G.words = (W + 63) / 64;
    G.S = pow2_at_least(G.words);
    G.lg_s = 0;
    while ((1 << G.lg_s) < G.S) ++G.lg_s;
    G.RB = (H + HB_R - 1) / HB_R;
    G.frames = batch;
    G.nblocks = batch * (long long)G.RB;
    const int per = 32 / G.S;
    G.nwb = (G.nblocks + per - 1) / per;
    G.nfg = (batch + per - 1) / per;
    return G;
}

}  // namespace

bool hb_supported(int W) { return W >= 1 && W <= 64 * 32; }

size_t hb_bytes(int64_t batch, int H, int W) {
    if (!hb_supported(W)) return 0;
    const HbGeom G = hb_geom(batch, H, W);
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    return 4 * al((size_t)G.nblocks * G.S * 8);
}

cudaError_t launch_hb_pack(const uint8_t* labels, int64_t batch, int H, int W, unsigned long long* fg,
                           unsigned long long* st, int sm_count, cudaStream_t st_) {
    const int words = (W + 63) / 64;
    const long long n = batch * (long long)H * words;
    const long long want = (n + 255) / 256;
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(want, 8ll * sm_count));
    return launch_pdl(hb_pack_kernel, dim3(grid), dim3(256), 0, st_, labels, batch * (long long)H, W, words, fg, st);
}

cudaError_t launch_strong_final(const uint8_t* labels, long long n, uint8_t* fin, int sm_count, cudaStream_t st) {
    const long long want = (n / 16 + 255) / 256;
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(want, 8ll * sm_count));
    return launch_pdl(strong_final_kernel, dim3(grid), dim3(256), 0, st, labels, n, fin);
}

cudaError_t launch_hystb(const FgBits& B, int64_t batch, int H, int W, uint8_t* final_out, void* buf, size_t bytes,
                         WsHeader* hdr, int sm_count, cudaStream_t st) {
    if (!hb_supported(W)) return cudaErrorInvalidValue;
    const HbGeom G = hb_geom(batch, H, W);
    if (bytes < hb_bytes(batch, H, W)) return cudaErrorInvalidValue;
    auto al = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t arr = al((size_t)G.nblocks * G.S * 8);
    char* p = static_cast<char*>(buf);
    HbBufs hb;
    hb.ftop = reinterpret_cast<u64*>(p);
    hb.utop = reinterpret_cast<u64*>(p + arr);
    hb.fbot = reinterpret_cast<u64*>(p + 2 * arr);
    hb.ubot = reinterpret_cast<u64*>(p + 3 * arr);
    static std::atomic<int> per_sm{0};
    int occ = per_sm.load();
    if (occ == 0) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, hb_pass1_kernel, 32 * HB_WARPS, 0);
        if (e != cudaSuccess) return e;
        per_sm.store(std::max(occ, 1));
        occ = std::max(occ, 1);
    }
    const long long want1 = (G.nwb + HB_WARPS - 1) / HB_WARPS;
    const unsigned grid1 = (unsigned)std::max<long long>(1, std::min<long long>(want1, (long long)occ * sm_count));
    cudaError_t e = launch_pdl(hb_pass1_kernel, dim3(grid1), dim3(32 * HB_WARPS), 0, st, B, G, final_out, hb);
    if (e != cudaSuccess) return e;
    const unsigned grid2 = (unsigned)std::max<long long>(1, (G.nfg + HB_WARPS - 1) / HB_WARPS);
    return launch_pdl(hb_pass2_kernel, dim3(grid2), dim3(32 * HB_WARPS), 0, st, B, G, final_out, hb, hdr);
}

}  // namespace ef
