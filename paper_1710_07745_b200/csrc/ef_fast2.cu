// ef_fast2.cu -- K1: the fused classify kernel (production path for
// radius 1..6 and W % 4 == 0; ef_fast.cu's v1 covers the rest).
//
// Certified fp32 decisions with kFlag + fix list for the rest (the contract of
// ef_fast.cu).  One CTA = 4 warps = a tile of 128 computed columns (32 lanes x
// 4 adjacent columns) x TH = 32 output rows; OW = 128 - 2*HXA output columns
// (HXA column halo each side: 4 for radius <= 2, 8 for radius <= 6).
//
//  staging   interior tiles: the u8 tile + halo arrives by one TMA box
//            (cp.async.bulk.tensor.3d + mbarrier); other tiles load rows
//            directly with clamping.
//  phase 1   each warp streams a quarter of the tile's 36 blurred rows: u8 ->
//            fp32 by byte-permute + one FADD2, vertical blur from a register
//            ring of the last 2R+1 rows (f32x2 FFMA2 on column pairs),
//            horizontal blur with neighbour lanes' columns from 64-bit
//            shuffles; the blurred rows land in shared memory (b tile).
//  phase 2   the 4 warps split the tile's 34 magnitude rows once:
//            Sobel from the b tile, squared magnitude into a shared m tile;
//            4-pixel groups certainly below `low` are written as background
//            right away, the others set a bit in their row's candidate word.
//  phase 3   after one barrier each warp compacts the non-empty candidate
//            words of its rows and classifies 32 groups at a time with every
//            lane busy (sector, NMS, thresholds, certification); the fused
//            pipeline's foreground bit planes are ORed in here.
//  (v2 -- per-warp magnitude rings recomputing 4 halo rows per 8, queues
//  flushed on a timer, branchy classifier -- needed 20% more instructions.)
//
// Border policy (np.pad edge at every stage): input rows/columns clamped on
// load; blurred and magnitude values at out-of-frame columns are replaced by
// the edge column's value (warp shuffle); magnitude rows -1 and H copy rows 0
// and H-1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstddef>
#include <cstdlib>
#include <cstring>

#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_launch.cuh"

namespace ef {

#ifdef EF_DEBUG_DUMP
struct DbgDump {
    float *m2, *gx, *gy;
};
__device__ DbgDump g_dbg = {nullptr, nullptr, nullptr};
#endif

#ifndef EF_K1_WARPS
#define EF_K1_WARPS 4
#endif
constexpr int V2_WARPS = EF_K1_WARPS;
constexpr int V2_THREADS = 32 * V2_WARPS;
constexpr int V2_COLS = 128;
#ifndef EF_K1_TH
#define EF_K1_TH 32
#endif
#ifndef EF_K1_MSPLIT
#define EF_K1_MSPLIT 0  // 1: magnitude rows split 9/9/8/8 (no recomputed rows; measured 3% slower on C3)
#endif
#ifndef EF_K1_POOL
#define EF_K1_POOL 1  // phase 3 pools the four warps' candidates (0: each warp classifies its own rows)
#endif
#ifndef EF_K1_HODD
#define EF_K1_HODD 0  // 1: odd horizontal taps as one FFMA2 over two scalar sums; 0: four scalar ops (same
                      // arithmetic; since the classifier's predicated loads 0 measures 0.45% faster on C3)
#endif
#ifndef EF_K1_EDGEPRED
#define EF_K1_EDGEPRED 2  // classifier: a group's edge columns are loaded only for edge pixels that can be
                          // foreground (1), the magnitude tile's only in the row the pixel's sector picks (2)
#endif
#ifndef EF_K1_MINB
#define EF_K1_MINB 6  // CTAs per SM the register budget is sized for (shared memory allows 6 at TH = 32)
#endif
constexpr int V2_TH = EF_K1_TH;  // output rows per tile
constexpr int V2_BROWS = V2_TH + 4;

constexpr int V2_MAXR = 6;
constexpr int V2_IN_ROWS = V2_BROWS + 2 * V2_MAXR;  // staged u8 input rows (TMA box height <= this)
// TMA box starts must be 16-byte aligned in the innermost (column) dimension
// (an unaligned start faults with "illegal instruction" on sm_100a), so the
// staged box starts at xv0 & ~15 and is 16 columns wider than the tile.
constexpr int V2_IN_COLS = V2_COLS + 16;

struct V2Out {
    uint8_t* labels;
    unsigned long long out_base;
    unsigned long long* fix_list;
    WsHeader* hdr;
#ifdef EF_DEBUG_CHECKS
    unsigned long long npx;  // pixels of the label buffer (bounds checks)
#endif
};

template <int R>
struct V2Cfg {
    static constexpr int HXA = R <= 2 ? 4 : 8;  // R <= 6: one- and two-hop shuffles stay inside the warp
    static constexpr int OW = V2_COLS - 2 * HXA;
    static constexpr int NR = 2 * R + 1;
};

__device__ __forceinline__ float u8f(uint32_t w, int k) {
    // byte k of w placed in the mantissa of 2^23: exact integer -> float
    return __int_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | (unsigned)k)) - 8388608.0f;
}

__device__ __forceinline__ float sqrt_apx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// The blurred (b) and magnitude (m) tiles have a padded row stride of 132
// floats (528 bytes): quad q of row r starts in bank group (r + q) mod 8, so
// the classifier's lanes -- 32 groups from different rows, often one above the
// other along an edge -- do not collide on the banks of 512-byte rows.  (An
// XOR swizzle does the same but costs address instructions in every phase.)
constexpr int V2_CS = V2_COLS + 4;

// ---------------------------------------------------------------- phase 1 --
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// Rows of b computed per warp in phase 1: the tile's 36 b rows split 4 ways.
constexpr int V2_P1_ROWS = (V2_BROWS + V2_WARPS - 1) / V2_WARPS;  // 9
static_assert(V2_P1_ROWS * V2_WARPS == V2_BROWS, "phase 1 rows split evenly");

// Phase 1 over the staged input tile (all rows and columns present: edge
// tiles have replicated their margins).  Warp w computes blurred rows
// ys .. ys + V2_P1_ROWS - 1 (frame rows), ys = y0 - 2 + w * V2_P1_ROWS.
template <int R, class Smem>
__device__ __forceinline__ void v2_phase1(int xv0, int y0, const FastParams& P, Smem& S, int warp, int lane) {
    constexpr int NR = V2Cfg<R>::NR;
    const int ys = y0 - 2 + warp * V2_P1_ROWS;
    auto fetch = [&](int Y) -> uint32_t {  // 4 staged input bytes of frame row Y
        EF_DCHECK(Y - (y0 - 2 - R) >= 0 && Y - (y0 - 2 - R) < V2_BROWS + 2 * R);
        EF_DCHECK((xv0 & 15) + 4 * lane + 3 < V2_IN_COLS);
        return *reinterpret_cast<const uint32_t*>(&S.in[Y - (y0 - 2 - R)][(xv0 & 15) + 4 * lane]);
    };
    float2 wf2[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wf2[k] = f2(P.wf[k], P.wf[k]);
    const float2 magic = f2(8388608.0f, 8388608.0f);
    auto cvt = [&](uint32_t w, float2& lo, float2& hi) {
        lo = add2(f2(__int_as_float(__byte_perm(w, 0x4B000000u, 0x7540u)),
                     __int_as_float(__byte_perm(w, 0x4B000000u, 0x7541u))), f2(-magic.x, -magic.y));
        hi = add2(f2(__int_as_float(__byte_perm(w, 0x4B000000u, 0x7542u)),
                     __int_as_float(__byte_perm(w, 0x4B000000u, 0x7543u))), f2(-magic.x, -magic.y));
    };

    float2 p[NR][2];  // converted input rows: columns (c, c+1), (c+2, c+3)
    uint32_t raw[NR];
    // input row ii is global row ys - R + ii
#pragma unroll
    for (int ii = 0; ii < 2 * R; ++ii) cvt(fetch(ys - R + ii), p[ii][0], p[ii][1]);
#pragma unroll
    for (int ii = 2 * R; ii < 4 * R; ++ii)  // look-ahead rows this warp will use (R > 4: fewer than 2R)
        if (ii - 2 * R < V2_P1_ROWS) raw[ii % NR] = fetch(ys - R + ii);
    const int rb = ys - (y0 - 2);  // first b row of this warp

#pragma unroll
    for (int u = 0; u < V2_P1_ROWS; ++u) {
        const int s = u % NR;
        cvt(raw[(s + 2 * R) % NR], p[(s + 2 * R) % NR][0], p[(s + 2 * R) % NR][1]);
        if (u + 2 * R < V2_P1_ROWS) raw[(s + 4 * R) % NR] = fetch(ys - R + u + 4 * R);
        // vertical pass on column pairs
        float2 v01 = mul2(wf2[0], p[(s + R) % NR][0]);
        float2 v23 = mul2(wf2[0], p[(s + R) % NR][1]);
#pragma unroll
        for (int o = 1; o <= R; ++o) {
            v01 = fma2(wf2[o], add2(p[(s + R - o) % NR][0], p[(s + R + o) % NR][0]), v01);
            v23 = fma2(wf2[o], add2(p[(s + R - o) % NR][1], p[(s + R + o) % NR][1]), v23);
        }
        // horizontal pass: neighbours' pairs by 64-bit shuffles
        // e[j] = column c - 8 + j, j = 0..19 (lanes -2..+2; lane +-2 only for R > 4)
        float e[20];
        {
            const double d01 = __hiloint2double(__float_as_int(v01.y), __float_as_int(v01.x));
            const double d23 = __hiloint2double(__float_as_int(v23.y), __float_as_int(v23.x));
            const double l23 = __shfl_up_sync(0xffffffffu, d23, 1);
            const double r01 = __shfl_down_sync(0xffffffffu, d01, 1);
            const double l01 = R > 2 ? __shfl_up_sync(0xffffffffu, d01, 1) : 0.0;
            const double r23 = R > 2 ? __shfl_down_sync(0xffffffffu, d23, 1) : 0.0;
            const double ll23 = R > 4 ? __shfl_up_sync(0xffffffffu, d23, 2) : 0.0;
            const double rr01 = R > 4 ? __shfl_down_sync(0xffffffffu, d01, 2) : 0.0;
            e[2] = __int_as_float(__double2loint(ll23)); e[3] = __int_as_float(__double2hiint(ll23));
            e[4] = __int_as_float(__double2loint(l01)); e[5] = __int_as_float(__double2hiint(l01));
            e[6] = __int_as_float(__double2loint(l23)); e[7] = __int_as_float(__double2hiint(l23));
            e[8] = v01.x; e[9] = v01.y; e[10] = v23.x; e[11] = v23.y;
            e[12] = __int_as_float(__double2loint(r01)); e[13] = __int_as_float(__double2hiint(r01));
            e[14] = __int_as_float(__double2loint(r23)); e[15] = __int_as_float(__double2hiint(r23));
            e[16] = __int_as_float(__double2loint(rr01)); e[17] = __int_as_float(__double2hiint(rr01));
            e[0] = e[1] = e[18] = e[19] = 0.f;
        }
        // b(k) = w0 e[8+k] + sum_o w_o (e[8+k-o] + e[8+k+o]); even o on aligned pairs
        float2 b01 = mul2(wf2[0], f2(e[8], e[9]));
        float2 b23 = mul2(wf2[0], f2(e[10], e[11]));
#pragma unroll
        for (int o = 1; o <= R; ++o) {
            if ((o & 1) == 0) {
                b01 = fma2(wf2[o], add2(f2(e[8 - o], e[9 - o]), f2(e[8 + o], e[9 + o])), b01);
                b23 = fma2(wf2[o], add2(f2(e[10 - o], e[11 - o]), f2(e[10 + o], e[11 + o])), b23);
            } else if (EF_K1_HODD) {
                // odd taps: the two sums land in a register pair, one FFMA2
                b01 = fma2(wf2[o], f2(e[8 - o] + e[8 + o], e[9 - o] + e[9 + o]), b01);
                b23 = fma2(wf2[o], f2(e[10 - o] + e[10 + o], e[11 - o] + e[11 + o]), b23);
            } else {
                b01.x = fmaf(wf2[o].x, e[8 - o] + e[8 + o], b01.x);
                b01.y = fmaf(wf2[o].x, e[9 - o] + e[9 + o], b01.y);
                b23.x = fmaf(wf2[o].x, e[10 - o] + e[10 + o], b23.x);
                b23.y = fmaf(wf2[o].x, e[11 - o] + e[11 + o], b23.y);
            }
        }
        EF_DCHECK(rb + u >= 0 && rb + u < V2_BROWS);
        *reinterpret_cast<float4*>(&S.b[rb + u][4 * lane]) = make_float4(b01.x, b01.y, b23.x, b23.y);
    }
}

// ---------------------------------------------------------------- phase 2 --
// The few scalars the classifier needs (kept in registers).
struct V2Cls {
    float lo_lo, lo_hi, hi_lo, hi_hi, e_nms0, e_nms_rel, e_sec;
    float cand_sq;  // squared magnitudes below this are certainly below `low` (phase 2's candidate test)
    int cls0;
    int W, FH, out0;
};



// Classify the 4 pixels of one candidate group (certified; kFlag otherwise),
// branch-free: the group's 6 columns (cc0-1 .. cc0+4) of
// the three magnitude and three blurred rows are loaded once (one 16-byte and
// two scalar loads per row), and every pixel's class, sector and NMS decision
// is computed with selects -- lanes of a warp classify different groups, so
// branches would serialise every path.
__device__ __forceinline__ void load6(const float* row, int cc0, float (&v)[6]) {
    const float4 mid = *reinterpret_cast<const float4*>(row + cc0);
    v[0] = row[cc0 - 1];
    v[1] = mid.x; v[2] = mid.y; v[3] = mid.z; v[4] = mid.w;
    v[5] = row[cc0 + 4];
}

// The column left of the group is read only by its pixel 0 and the column right of it
// only by pixel 3 (neighbours and Sobel taps of those pixels).  A pixel certainly below
// `low` gets the background class whatever its neighbours are, so its edge column is
// not loaded: the scalar edge loads are 4-way bank-conflicted by construction
// (elements 3 / 0 of a quad live in 8 of the 32 banks) and a third of the groups' edge
// pixels are below `low` -- fewer lanes per load, fewer wavefronts on the LSU pipe.
__device__ __forceinline__ void load6_edges(const float* row, int cc0, bool left, bool right, float (&v)[6]) {
    const float4 mid = *reinterpret_cast<const float4*>(row + cc0);
    v[0] = left ? row[cc0 - 1] : 0.f;
    v[1] = mid.x; v[2] = mid.y; v[3] = mid.z; v[4] = mid.w;
    v[5] = right ? row[cc0 + 4] : 0.f;
}

// The tile's output addresses, formed once per thread before the classifier's
// rounds (per group: 32-bit row / column offsets from these bases; forming the
// 64-bit label, final and bit-plane addresses from the frame geometry in every
// round cost ~30 instructions of ~330).
struct V2Dst {
    unsigned long long lab0;  // label index of (tile row 0, column xv0)
    uint8_t* lab;             // labels + lab0
    long long fin_off;        // final map - label map (bytes)
    unsigned long long* fg;   // bit-plane words of tile row 0
    unsigned long long* st;
    int words;                // words per output row
};

template <bool FUSED>
__device__ __forceinline__ void classify_group_bf(const V2Cls& P, int xv0, int j, int cl, const float* mu,
                                                  const float* mc, const float* md, const float* bu,
                                                  const float* bm, const float* bd, const V2Dst& D,
                                                  const V2Out& O) {
    const float t1 = 0.41421356237309503f;
    const int cc0 = 4 * cl;
    float Mu[6], Mc[6], Md[6], Bu[6], Bm[6], Bd[6];
    bool left = true, right = true;  // the group's pixel 0 / 3 can be foreground
    (void)left;
    (void)right;
#if EF_K1_EDGEPRED
    {
        const float4 mid = *reinterpret_cast<const float4*>(mc + cc0);
        Mc[1] = mid.x; Mc[2] = mid.y; Mc[3] = mid.z; Mc[4] = mid.w;
        left = Mc[1] >= P.cand_sq;
        right = Mc[4] >= P.cand_sq;
#if EF_K1_EDGEPRED >= 2
        // the magnitude tile's edge columns: one value per edge pixel, loaded once its
        // sector is known (below); only the blurred tile's edges are needed up front
        Mc[0] = Mc[5] = 0.f;
        load6_edges(mu, cc0, false, false, Mu);
        load6_edges(md, cc0, false, false, Md);
#else
        Mc[0] = left ? mc[cc0 - 1] : 0.f;
        Mc[5] = right ? mc[cc0 + 4] : 0.f;
        load6_edges(mu, cc0, left, right, Mu);
        load6_edges(md, cc0, left, right, Md);
#endif
        load6_edges(bu, cc0, left, right, Bu);
        load6_edges(bm, cc0, left, right, Bm);
        load6_edges(bd, cc0, left, right, Bd);
    }
#else
    load6(mu, cc0, Mu);
    load6(mc, cc0, Mc);
    load6(md, cc0, Md);
    load6(bu, cc0, Bu);
    load6(bm, cc0, Bm);
    load6(bd, cc0, Bd);
#endif
    uint32_t packed = 0;
    bool any_flag = false;
    const uint32_t cls0 = (uint32_t)P.cls0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float c = sqrt_apx(Mc[k + 1]);
        const float gx = fmaf(2.f, Bm[k + 2] - Bm[k], (Bu[k + 2] - Bu[k]) + (Bd[k + 2] - Bd[k]));
        const float gy = fmaf(2.f, Bd[k + 1], Bd[k] + Bd[k + 2]) - fmaf(2.f, Bu[k + 1], Bu[k] + Bu[k + 2]);
        const float a = fabsf(gx), b = fabsf(gy);
        const float uu = fmaf(t1, a, -b), vv = fmaf(t1, b, -a);
        // neighbours along the sector: 0 (W/E), 90 (N/S), 45 (NE/SW), 135 (NW/SE)
        const float n0 = fmaxf(Mc[k], Mc[k + 2]);
        const float n90 = fmaxf(Mu[k + 1], Md[k + 1]);
        const float n45 = fmaxf(Mu[k + 2], Md[k]);
        const float n135 = fmaxf(Mu[k], Md[k + 2]);
        const float ndiag = ((gx > 0.f) == (gy > 0.f)) ? n45 : n135;
        float nmax = uu > 0.f ? n0 : (vv > 0.f ? n90 : ndiag);
#if EF_K1_EDGEPRED >= 2
        if (k == 0 || k == 3) {
            // the edge pixel's neighbour in the column outside the group sits in the row
            // its sector picks (0: this row, 45 / 135: the row below or above; 90: none):
            // one load, by the lanes whose edge pixel can be foreground and is not 90 --
            // instead of three edge loads per side up front (Mu / Mc / Md[0] and [5] hold 0)
            const bool s0 = uu > 0.f, s90 = !s0 && vv > 0.f, same = (gx > 0.f) == (gy > 0.f);
            const int up = k == 0 ? (same ? V2_CS : -V2_CS) : (same ? -V2_CS : V2_CS);
            const bool need = (k == 0 ? left : right) && !s90;
            const float e = need ? mc[cc0 + (k == 0 ? -1 : 4) + (s0 ? 0 : up)] : 0.f;
            nmax = fmaxf(nmax, e);
        }
#endif
        const float nv = sqrt_apx(nmax);
        const float d = c - nv;
        const float e_nms = fmaf(P.e_nms_rel, c + nv, P.e_nms0);  // magnitude-relative certification band
        const bool amb = fabsf(uu) <= P.e_sec || fabsf(vv) <= P.e_sec;
        // threshold class: 2 / 1 / 0, or -1 inside a certification band
        // (as c > hi_hi ? 2 : c >= hi_lo ? -1 : c > lo_hi ? 1 : c >= lo_lo ? -1 : 0,
        // with lo_lo <= lo_hi and hi_lo <= hi_hi; written as two selects over
        // four compares so no lane branches on its pixel's class)
        const int lo_cls = c >= P.lo_lo ? (c > P.lo_hi ? 1 : -1) : 0;
        const int cls = c >= P.hi_lo ? (c > P.hi_hi ? 2 : -1) : lo_cls;
        const bool need_nms = cls >= 0 && (uint32_t)cls != cls0;
        const bool flag = cls < 0 || (need_nms && (amb || fabsf(d) <= e_nms));
        const uint32_t lab = flag ? (uint32_t)kFlag : ((need_nms && d > e_nms) ? (uint32_t)cls : cls0);
        any_flag |= flag;
        packed |= lab << (8 * k);
    }
    const unsigned off = (unsigned)j * (unsigned)P.W + (unsigned)cc0;  // from (tile row 0, column xv0)
    if (any_flag) {
        // one list append per group (global-space ops: see fg_bits_or)
        unsigned fm = 0, cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (((packed >> (8 * k)) & 0xffu) == kFlag) fm |= 1u << k;
        cnt = __popc(fm);
        unsigned long long slot, cap;
        asm volatile("atom.global.add.u64 %0, [%1], %2;" : "=l"(slot) : "l"(&O.hdr->fix_count), "l"((unsigned long long)cnt)
                     : "memory");
        asm volatile("ld.global.u64 %0, [%1];" : "=l"(cap) : "l"(&O.hdr->fix_cap) : "memory");
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!((fm >> k) & 1u)) continue;
            if (slot < cap)
                asm volatile("st.global.u64 [%0], %1;" ::"l"(O.fix_list + slot),
                             "l"(D.lab0 + off + (unsigned long long)k) : "memory");
            else
                st_global_u32(&O.hdr->overflow, 1u);
            ++slot;
        }
    }
    EF_DCHECK(cc0 >= 4 && cc0 + 4 < V2_CS && xv0 + cc0 >= 0 && xv0 + cc0 + 4 <= P.W);
#ifdef EF_DEBUG_CHECKS
    EF_DCHECK(D.lab0 + off + 4 <= O.npx);
#endif
    uint8_t* const lp = D.lab + off;
    st_global_u32(lp, packed);
    if (FUSED) {
        // final = strong (kFlag bytes give 0: the fix-up writes them)
        st_global_u32(lp + D.fin_off, (packed >> 1) & 0x01010101u);
        // bytes are 0, 1, 2 or kFlag (0x80, resolved by the fix-up, which sets its own bits)
        const uint32_t lo = packed & 0x03030303u;
        const uint32_t fgn = (((lo | (lo >> 1)) & 0x01010101u) * 0x10204080u) >> 28;
        const uint32_t stn = (((packed >> 1) & 0x01010101u) * 0x10204080u) >> 28;
        const int x = xv0 + cc0;
        const unsigned w = (unsigned)j * (unsigned)D.words + (unsigned)(x >> 6);
        EF_DCHECK((x & 3) == 0 && (unsigned)(x >> 6) < (unsigned)D.words);
        // global-space reductions (see fg_bits_or)
        if (fgn)
            asm volatile("red.global.or.b64 [%0], %1;" ::"l"(D.fg + w), "l"((unsigned long long)fgn << (x & 63)) : "memory");
        if (stn)
            asm volatile("red.global.or.b64 [%0], %1;" ::"l"(D.st + w), "l"((unsigned long long)stn << (x & 63)) : "memory");
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// TMA: the u8 tile + halo (144 columns x TH+4+2R rows of frame z) lands in
// shared memory in one bulk tensor copy; completion on an mbarrier.  Thread 0
// issues it first thing (tma_issue), so the CTA's prologue runs while the
// tile is in flight; everyone waits in tma_wait.
template <int R, bool PEER, class Smem>
__device__ __forceinline__ void tma_issue(Smem& S, const CUtensorMap& tmap, int xv0, int y0, const FrameGeom& g) {
    constexpr int rows = V2_BROWS + 2 * R;
    const uint32_t bar = smem_u32(&S.mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // init visible to the TMA unit
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rows * V2_IN_COLS)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(&S.in[0][0])), "l"(&tmap), "r"(xv0 & ~15), "r"(y0 - 2 - R - src_row0<PEER>(g)), "r"((int)blockIdx.z),
            "r"(bar)
        : "memory");
}

template <class Smem>
__device__ __forceinline__ void tma_wait(Smem& S) {
    __syncthreads();  // the mbarrier's initialisation is visible to every thread
    const uint32_t bar = smem_u32(&S.mbar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar)
            : "memory");
    }
}

// ---------------------------------------------------------------------------
// K1 v3: shared magnitude tile.  v2's warps each stream their own 8 output
// rows with a private magnitude ring, so every warp recomputes 4 halo rows of
// Sobel/magnitude (12 row steps per 8 rows).  Here the 4 warps split the 34
// magnitude rows of the tile once (y0-1 .. y0+TH), write them to a shared
// tile, record one candidate bit per 4-pixel group (the row's ballot), and
// after one barrier classify the candidates with every lane busy.
// ---------------------------------------------------------------------------
constexpr int V3_MROWS = V2_TH + 2;                                   // magnitude rows y0-1 .. y0+TH


struct V3Smem {
    union {  // first: the TMA destination must be 128-byte aligned
        float m[V3_MROWS][V2_CS];                   // squared magnitudes
        unsigned char in[V2_IN_ROWS][V2_IN_COLS];   // phase 1: TMA-staged input tile + halo
    };
    float b[V2_BROWS + 1][V2_CS];  // + 1: phase 2's one-row-ahead load of its last step (value unused)
    unsigned cmask[V2_TH];                          // candidate 4-pixel groups per output row (bit = lane)
    unsigned long long mbar;
    FgBits bits;
#ifdef EF_K1_SMEM_PAD
    unsigned char pad[EF_K1_SMEM_PAD];  // occupancy experiments only
#endif
};
static_assert(offsetof(V3Smem, in) % 128 == 0 && offsetof(V3Smem, b) % 16 == 0, "TMA / float4 alignment");
static_assert(EF_K1_MINB * (sizeof(V3Smem) + 1024) <= 233472, "CTAs per SM the register budget assumes fit in shared memory");


// d = b[x+1] - b[x-1] and s = b[x-1] + 2 b[x] + b[x+1] for this lane's 4 columns
__device__ __forceinline__ void sobel_vals(const float4 bb, float (&d)[4], float (&sm)[4]) {
    // neighbour lanes' edge columns (lanes 0 / 31 get wrapped values: only
    // columns no output depends on are affected)
    const float bl = __shfl_up_sync(0xffffffffu, bb.w, 1);
    const float br = __shfl_down_sync(0xffffffffu, bb.x, 1);
    d[0] = bb.y - bl;
    d[1] = bb.z - bb.x;
    d[2] = bb.w - bb.y;
    d[3] = br - bb.z;
    sm[0] = fmaf(2.f, bb.x, bl + bb.y);
    sm[1] = fmaf(2.f, bb.y, bb.x + bb.z);
    sm[2] = fmaf(2.f, bb.z, bb.y + bb.w);
    sm[3] = fmaf(2.f, bb.w, bb.z + br);
}

__device__ __forceinline__ float4 ldb(const float* brow) { return *reinterpret_cast<const float4*>(brow); }

__device__ __forceinline__ void sobel_row(const float* brow, float (&d)[4], float (&sm)[4]) {
    sobel_vals(ldb(brow), d, sm);
}

template <int R, bool FUSED>
__device__ __forceinline__ void v3_phase2a(const FrameGeom& g, int xv0, int y0, const FastParams& P, V3Smem& S,
                                           int warp, int lane, const V2Out& O) {
    constexpr int HXA = V2Cfg<R>::HXA;
    constexpr int OW = V2Cfg<R>::OW;
    const int W = g.W, FH = g.full_H;
    // this warp's magnitude rows j0 .. j0+nrows-1 (tile rows; Ym = y0 - 1 + j):
    // the 34 rows split 9 / 9 / 8 / 8 (the trip count is uniform inside each
    // warp, so no loop exit diverges around the shuffles and votes; an even
    // 9 / 9 / 9 / 9 split computed rows 25 and 26 twice)
#if EF_K1_MSPLIT
    constexpr int MBASE = V3_MROWS / V2_WARPS, MEXTRA = V3_MROWS % V2_WARPS;
    const int nrows = MBASE + (warp < MEXTRA ? 1 : 0);
    const int j0 = warp * MBASE + min(warp, MEXTRA);
#else
    // every warp runs ceil(34 / 4) = 9 rows; the last one starts at 25, so rows
    // 25 and 26 are computed twice (same values, labels and candidate words)
    constexpr int MPW = (V3_MROWS + V2_WARPS - 1) / V2_WARPS;
    constexpr int nrows = MPW;
    const int j0 = min(warp * MPW, V3_MROWS - MPW);
#endif
    const int ylim = min(g.out0 + g.rows, FH);  // rows at or past this are not classified here
    const int c = xv0 + 4 * lane;
    const bool out_lane = lane >= HXA / 4 && lane < (HXA + OW) / 4 && c < W;
    const uint32_t fill = (uint32_t)P.cls0 * 0x01010101u;
    const float cand_sq = P.lo_lo > 0.f ? P.lo_lo * P.lo_lo * (1.0f - 1.0f / 262144.0f) : -1.0f;
    const int Wq = W >> 2;
    auto brow = [&](int Y) -> const float* {
        EF_DCHECK(Y - (y0 - 2) >= 0 && Y - (y0 - 2) <= V2_BROWS);
        return &S.b[Y - (y0 - 2)][4 * lane];
    };
    uint32_t* lab = reinterpret_cast<uint32_t*>(O.labels + O.out_base + (long long)(y0 + j0 - 1 - g.out0) * W + c);
    const long long fin_off = FUSED ? S.bits.fin_off : 0;  // fused path: final = 0 off the candidates
    unsigned* const cmask = S.cmask;
    float d[3][4], sm[3][4];
    sobel_row(brow(y0 - 2 + j0), d[0], sm[0]);
    sobel_row(brow(y0 - 1 + j0), d[1], sm[1]);
    // one magnitude row; (pu, pm, pd) = ring slots of the b rows above, at and
    // below it (period 3)
    // the b row below each magnitude row is loaded one row step ahead (its
    // shared-memory latency overlaps the previous row's arithmetic: K1 -0.7%)
    float4 bnext = ldb(brow(y0 + j0));
    auto row_step = [&](int u, int pu, int pm, int pd) {
        const int j = j0 + u;
        const int Ym = y0 - 1 + j;
        const float4 bcur = bnext;
        bnext = ldb(brow(Ym + 2));  // the last warp's last step reads the spare row V2_BROWS
        sobel_vals(bcur, d[pd], sm[pd]);
        const float2 two = f2(2.f, 2.f);
        const float2 gx01 = fma2(two, f2(d[pm][0], d[pm][1]), add2(f2(d[pu][0], d[pu][1]), f2(d[pd][0], d[pd][1])));
        const float2 gx23 = fma2(two, f2(d[pm][2], d[pm][3]), add2(f2(d[pu][2], d[pu][3]), f2(d[pd][2], d[pd][3])));
        const float2 gy01 = add2(f2(sm[pd][0], sm[pd][1]), f2(-sm[pu][0], -sm[pu][1]));
        const float2 gy23 = add2(f2(sm[pd][2], sm[pd][3]), f2(-sm[pu][2], -sm[pu][3]));
        float2 m01 = fma2(gx01, gx01, mul2(gy01, gy01));
        float2 m23 = fma2(gx23, gx23, mul2(gy23, gy23));
#ifdef EF_DEBUG_DUMP
        // certification-margin study (tools/cert_margin.py): the fp32 squared
        // magnitude and gradient of every output pixel, as the classifier sees them
        if (g_dbg.m2 && j >= 1 && j <= V2_TH && out_lane && Ym < ylim) {
            const unsigned long long o = O.out_base + (unsigned long long)(Ym - g.out0) * W + c;
            *reinterpret_cast<float4*>(g_dbg.m2 + o) = make_float4(m01.x, m01.y, m23.x, m23.y);
            *reinterpret_cast<float4*>(g_dbg.gx + o) = make_float4(gx01.x, gx01.y, gx23.x, gx23.y);
            *reinterpret_cast<float4*>(g_dbg.gy + o) = make_float4(gy01.x, gy01.y, gy23.x, gy23.y);
        }
#endif
        EF_DCHECK(j >= 0 && j < V3_MROWS);
        *reinterpret_cast<float4*>(&S.m[j][4 * lane]) = make_float4(m01.x, m01.y, m23.x, m23.y);
        // output rows: groups certainly below `low` get the background class
        // now, the others are marked for the classifier
        // (straight-line: the vote runs on every row, the stores are predicated,
        // so no divergent region surrounds the vote)
        const bool outrow = j >= 1 && j <= V2_TH;
        const bool act = outrow && out_lane && Ym < ylim;
        const bool cand = act && fmaxf(fmaxf(m01.x, m01.y), fmaxf(m23.x, m23.y)) >= cand_sq;
        const unsigned b0 = __ballot_sync(0xffffffffu, cand);
        const bool bg = act && !cand;
        EF_DCHECK(!bg || (reinterpret_cast<const uint8_t*>(lab) >= O.labels &&
                          reinterpret_cast<const uint8_t*>(lab) + 4 <=
                              O.labels + (unsigned long long)gridDim.z * g.rows * g.W));
        if (bg) *lab = fill;
        if (FUSED && bg) *reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(lab) + fin_off) = 0u;
        EF_DCHECK(!(lane == 0 && outrow) || (j - 1 >= 0 && j - 1 < V2_TH));
        if (lane == 0 && outrow) cmask[j - 1] = b0;
        lab += Wq;
    };
    // period-3 register ring: whole periods, then the warp-uniform tail
    int u3 = 0;
#pragma unroll 1
    for (; u3 + 3 <= nrows; u3 += 3) {
        row_step(u3, 0, 1, 2);
        row_step(u3 + 1, 1, 2, 0);
        row_step(u3 + 2, 2, 0, 1);
    }
    if (u3 < nrows) row_step(u3, 0, 1, 2);
    if (u3 + 1 < nrows) row_step(u3 + 1, 1, 2, 0);
}

// position of the n-th (0-based) set bit of w
__device__ __forceinline__ int select32(unsigned w, int n) {
    int pos = 0;
    int c = __popc(w & 0xffffu);
    if (n >= c) { n -= c; w >>= 16; pos += 16; }
    c = __popc(w & 0xffu);
    if (n >= c) { n -= c; w >>= 8; pos += 8; }
    c = __popc(w & 0xfu);
    if (n >= c) { n -= c; w >>= 4; pos += 4; }
    c = __popc(w & 0x3u);
    if (n >= c) { n -= c; w >>= 2; pos += 2; }
    return pos + (n >= (int)(w & 1u) ? 1 : 0);
}

// Phase 3: this warp's candidate words (rows warp + 4 i) sit one per lane; a
// warp prefix count numbers their groups, and lane k takes group base + k --
// found by a binary search over the prefix counts and a bit select -- so every
// round classifies 32 groups with no queue in shared memory.
template <int R, bool FUSED>
__device__ __forceinline__ void v3_classify(const V2Cls P, int xv0, int y0, V3Smem& S, int warp, int lane,
                                         const V2Out O) {
#if EF_K1_POOL
    // pooled: every warp reads the whole tile's candidate words (one row per
    // lane) and takes rounds warp, warp + 4, ... of the tile's candidates, so
    // the lanes stay full across the warps' rows (per-warp pools left the last
    // round of every warp part-empty: 56% lane use on C3's dense content)
    constexpr int NW = V2_TH;
    static_assert(NW <= 32, "one word per lane");
    const int wrow = lane;
    const unsigned word = lane < NW ? S.cmask[lane] : 0u;
    const int first = 32 * warp, stride = 32 * V2_WARPS;
#else
    constexpr int NW = (V2_TH + V2_WARPS - 1) / V2_WARPS;  // candidate words per warp
    static_assert(NW <= 32, "one word per lane");
    const int wrow = warp + V2_WARPS * lane;
    const unsigned word = (lane < NW && wrow < V2_TH) ? S.cmask[wrow] : 0u;
    const int first = 0, stride = 32;
#endif
    (void)wrow;
    int incl = __popc(word);  // inclusive prefix over the lanes (lanes >= NW add 0)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    constexpr int NW2 = NW <= 1 ? 1 : (NW <= 2 ? 2 : (NW <= 4 ? 4 : (NW <= 8 ? 8 : (NW <= 16 ? 16 : 32))));
    if (first >= total) return;
    V2Dst D;
    D.lab0 = O.out_base + (unsigned long long)(y0 - P.out0) * (unsigned)P.W + (unsigned long long)xv0;
    D.lab = O.labels + D.lab0;
    D.fin_off = FUSED ? S.bits.fin_off : 0;
    D.words = FUSED ? S.bits.words : 0;
    D.fg = D.st = nullptr;
    if (FUSED) {
        const unsigned long long w0 = blockIdx.z * S.bits.frame_words + (unsigned long long)(y0 - P.out0) * S.bits.words;
        D.fg = S.bits.fg + w0;
        D.st = S.bits.st + w0;
    }
    for (int base = first; base < total; base += stride) {
        const int k = base + lane;
        int i = 0;  // first word whose inclusive count exceeds k
#pragma unroll
        for (int step = NW2 / 2; step >= 1; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, i + step - 1);
            if (v <= k) i += step;
        }
        const unsigned w = __shfl_sync(0xffffffffu, word, i);
        const int before = __shfl_sync(0xffffffffu, incl, i) - __popc(w);
        if (k < total) {
#if EF_K1_POOL
            const int j = i;  // output row y0 + j; m tile rows j..j+2, b rows j+1..j+3
#else
            const int j = warp + V2_WARPS * i;
#endif
            EF_DCHECK(j >= 0 && j + 2 < V3_MROWS && j + 3 < V2_BROWS && i >= 0 && i < NW);
            EF_DCHECK(select32(w, k - before) >= 0 && select32(w, k - before) < 32 && ((w >> select32(w, k - before)) & 1u));
            classify_group_bf<FUSED>(P, xv0, j, select32(w, k - before), S.m[j], S.m[j + 1], S.m[j + 2], S.b[j + 1],
                              S.b[j + 2], S.b[j + 3], D, O);
        }
    }
}

// Edge tiles on the TMA path: the box reads zeros outside the buffer, so the
// staged input, then the blurred tile, then the magnitude tile are completed
// in shared memory by replicating their edge rows / columns (np.pad edge at
// every stage, the reference's border policy) -- after which the interior code
// runs unchanged.  Columns first, then rows (corners = corner pixel).
// Only the margin the next stage reads is filled: `marg` columns / rows past
// the in-frame range [c_lo, c_hi] x [r_lo, r_hi] (R for the staged input, whose
// blurred values feed the in-frame columns; 1 for the blurred and magnitude
// tiles, read by the Sobel / NMS neighbours of the edge pixels), and never the
// staged box's alignment margin outside [c_use0, c_use1].  The out-of-frame
// rows copy the edge row at the CLAMPED column, so the column and row passes
// are independent: one barrier.
template <int NROWS, int NCOLS, int STRIDE, class T>
__device__ __forceinline__ void replicate_edges(T (*a)[STRIDE], int c_lo, int c_hi, int r_lo, int r_hi, int marg,
                                                int c_use0 = 0, int c_use1 = NCOLS - 1) {
    auto at = [&](int r, int c) -> T& { return a[r][c]; };  // (NCOLS logical columns of STRIDE)
    const int c0 = max(c_use0, c_lo - marg), c1 = min(c_use1, c_hi + marg);
    const int r0 = max(0, r_lo - marg), r1 = min(NROWS - 1, r_hi + marg);
    const bool cols = c0 < c_lo || c1 > c_hi, rows = r0 < r_lo || r1 > r_hi;  // block-uniform
    if (cols) {  // in-frame rows: one row per thread
        for (int r = r_lo + threadIdx.x; r <= r_hi; r += blockDim.x) {
            const T vl = at(r, c_lo), vr = at(r, c_hi);
            for (int c = c0; c < c_lo; ++c) at(r, c) = vl;
            for (int c = c_hi + 1; c <= c1; ++c) at(r, c) = vr;
        }
    }
    if (rows) {  // out-of-frame rows: one column per thread, the edge row at the clamped column
        for (int c = c0 + threadIdx.x; c <= c1; c += blockDim.x) {
            const int cs = min(max(c, c_lo), c_hi);
            const T vt = at(r_lo, cs), vb = at(r_hi, cs);
            for (int r = r0; r < r_lo; ++r) at(r, c) = vt;
            for (int r = r_hi + 1; r <= r1; ++r) at(r, c) = vb;
        }
    }
    if (cols || rows) __syncthreads();
}

template <int R, bool FUSED, bool PEER = false>
__global__ void __launch_bounds__(V2_THREADS, EF_K1_MINB)
k1v3_kernel(const uint8_t* __restrict__ src, FrameGeom g, FastParams P, uint8_t* __restrict__ labels,
            unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr,
            const __grid_constant__ CUtensorMap tmap, int use_tma, FgBits B) {
    extern __shared__ __align__(16) unsigned char smraw[];
    V3Smem& S = *reinterpret_cast<V3Smem*>(smraw);
    pdl_wait();  // workspace counters and bit planes are reset by the previous kernel
    pdl_trigger();
    const int x0 = blockIdx.x * V2Cfg<R>::OW;
    const int xv0 = x0 - V2Cfg<R>::HXA;
    const int y0 = g.out0 + blockIdx.y * V2_TH;
    // a tile whose input box reaches a peer band's rows stages them by loads
    // (the tensor map covers this band's own buffer only)
    const bool tma_tile = use_tma && !(PEER && g.top && y0 - 2 - R < g.out0) &&
                          !(PEER && g.bot && y0 + V2_TH + 2 + R > g.out0 + g.rows);
    if (tma_tile && threadIdx.x == 0) tma_issue<R, PEER>(S, tmap, xv0, y0, g);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* img = src + (size_t)blockIdx.z * g.H * g.W;
#ifdef EF_DEBUG_CHECKS
    const V2Out O{labels, (unsigned long long)blockIdx.z * g.rows * g.W, fix_list, hdr,
                  (unsigned long long)gridDim.z * g.rows * g.W};
#else
    const V2Out O{labels, (unsigned long long)blockIdx.z * g.rows * g.W, fix_list, hdr};
#endif
    if (threadIdx.x == 0) S.bits = B;
    const bool interior = xv0 >= 0 && xv0 + V2_COLS <= g.W && y0 - 2 - R >= max(g.g0, 0) &&
                          y0 + V2_TH + 2 + R <= min(g.full_H, g.g0 + g.H) && y0 + V2_TH <= g.out0 + g.rows;
    // one code path for every tile: the input tile + halo is staged in shared
    // memory (TMA when W % 16 == 0, else clamped loads); edge tiles complete
    // their halos there by replication, so phases 1-3 never clamp
    const int FH = g.full_H, W = g.W;
    {
        // staged input: row r <-> frame row yin + r, column c <-> x = xa + c
        constexpr int NIN = V2_BROWS + 2 * R;
        const int xa = xv0 & ~15, yin = y0 - 2 - R;
        const int ylo = max(0, g.g0), yhi = min(FH, g.g0 + g.H) - 1;  // frame rows present in the buffer
        if (tma_tile) {
            tma_wait(S);
            if (!interior) {  // the box read zeros outside the buffer: replicate the edges
                // (every thread has waited on the mbarrier itself: the box is visible, no barrier first)
                replicate_edges<NIN, V2_IN_COLS, V2_IN_COLS>(S.in, max(0, -xa), min(V2_IN_COLS - 1, W - 1 - xa),
                                                             max(0, ylo - yin), min(NIN - 1, yhi - yin), R,
                                                             xv0 - xa, xv0 - xa + V2_COLS - 1);
            }
        } else {
            // no TMA (W % 16 != 0 or an unaligned buffer): 4-byte loads (W % 4 == 0),
            // clamped bytes where a word crosses the frame edge
            constexpr int QW = V2_IN_COLS / 4;
            const bool al4 = ((reinterpret_cast<uintptr_t>(img) |
                               (PEER ? reinterpret_cast<uintptr_t>(g.top) | reinterpret_cast<uintptr_t>(g.bot) : 0)) &
                              3) == 0;
            for (int i = threadIdx.x; i < NIN * QW; i += V2_THREADS) {
                const int r = i / QW, c = 4 * (i - r * QW);
                const uint8_t* row = frame_row<PEER>(img, g, min(max(yin + r, ylo), yhi));
                const int X = xa + c;
                uint32_t v;
                if (al4 && X >= 0 && X + 3 < W) {
                    v = __ldg(reinterpret_cast<const unsigned int*>(row + X));
                } else {
                    v = 0;
                    for (int k = 0; k < 4; ++k) v |= (uint32_t)row[min(max(X + k, 0), W - 1)] << (8 * k);
                }
                *reinterpret_cast<uint32_t*>(&S.in[r][c]) = v;
            }
            __syncthreads();
        }
    }
    v2_phase1<R>(xv0, y0, P, S, warp, lane);
    __syncthreads();
    if (!interior)  // blurred: row i <-> frame row y0-2+i, column c <-> x = xv0 + c
        // blurred and magnitude values are read at most one column past the
        // frame (Sobel and NMS neighbours of the edge columns)
        replicate_edges<V2_BROWS, V2_COLS, V2_CS>(S.b, max(0, -xv0), min(V2_COLS - 1, W - 1 - xv0),
                                                  max(0, -(y0 - 2)), min(V2_BROWS - 1, FH - 1 - (y0 - 2)), 1);
    v3_phase2a<R, FUSED>(g, xv0, y0, P, S, warp, lane, O);
    __syncthreads();
    if (!interior)  // magnitudes: row j <-> frame row y0-1+j
        replicate_edges<V3_MROWS, V2_COLS, V2_CS>(S.m, max(0, -xv0), min(V2_COLS - 1, W - 1 - xv0),
                                                  max(0, -(y0 - 1)), min(V3_MROWS - 1, FH - 1 - (y0 - 1)), 1);
    const V2Cls CP{P.lo_lo, P.lo_hi, P.hi_lo, P.hi_hi, P.e_nms0, P.e_nms_rel, P.e_sec,
                   P.lo_lo > 0.f ? P.lo_lo * P.lo_lo * (1.0f - 1.0f / 262144.0f) : -1.0f,  // as phase 2's cand_sq
                   P.cls0, g.W, g.full_H, g.out0};
    v3_classify<R, FUSED>(CP, xv0, y0, S, warp, lane, O);
}

#ifdef EF_DEBUG_DUMP
// debug builds only (-DEF_DEBUG_DUMP): K1 stores its fp32 m^2 / gx / gy of every
// output pixel into these device buffers (one float per pixel, label layout;
// 16-byte aligned); nullptr turns it off
extern "C" int ef_debug_dump(float* m2, float* gx, float* gy) {
    DbgDump d{m2, gx, gy};
    return cudaMemcpyToSymbol(g_dbg, &d, sizeof d) == cudaSuccess ? 0 : -1;
}
#endif

// the production classifier reads the source and writes labels / final in
// 32-bit words: every caller buffer 4-byte aligned (P.no_v2 == 0), W % 4 == 0
bool k1v2_supported(const FastParams& P, const FrameGeom& g) {
    return !P.no_v2 && P.r >= 1 && P.r <= 6 && (g.W % 4) == 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    // thread-safe one-time lookup (function-local static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return nullptr;
    }();
    return fn;
}

// 3-D map (column, buffer row, frame) over the u8 source; box = 144 columns x
// (TH + 4 + 2R) rows.  TMA needs 16-byte aligned rows: W % 16 == 0.
static bool make_src_map(CUtensorMap& tm, const uint8_t* src, int64_t batch, const FrameGeom& g, int R) {
    auto enc = tensor_map_encoder();
    if (!enc || (g.W % 16) != 0 || (reinterpret_cast<uintptr_t>(src) & 15) != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.W, (cuuint64_t)src_rows(g), (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)g.W, (cuuint64_t)g.W * g.H};
    cuuint32_t box[3] = {(cuuint32_t)V2_IN_COLS, (cuuint32_t)(V2_BROWS + 2 * R), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(src), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int R>
static cudaError_t launch_r(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                            uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                            cudaStream_t st) {
    // FUSED (bit planes + final map) is a compile-time variant: the per-row
    // checks would otherwise sit in the hottest loop
    const bool peer = g.top || g.bot;
    auto kern = peer ? (B.fg ? k1v3_kernel<R, true, true> : k1v3_kernel<R, false, true>)
                     : (B.fg ? k1v3_kernel<R, true> : k1v3_kernel<R, false>);
    const int smem = (int)sizeof(V3Smem);
    static std::atomic<uint64_t> configured{0};
    cudaError_t e = once_per_device(configured, [&] {
        cudaError_t r = cudaSuccess;
        for (auto k : {k1v3_kernel<R, true>, k1v3_kernel<R, false>, k1v3_kernel<R, true, true>,
                       k1v3_kernel<R, false, true>}) {
            if (r == cudaSuccess) r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            // occupancy is shared-memory bound: ask for the largest carveout
            if (r == cudaSuccess)
                r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared);
        }
        return r;
    });
    if (e != cudaSuccess) return e;
    dim3 grid((g.W + V2Cfg<R>::OW - 1) / V2Cfg<R>::OW, (g.rows + V2_TH - 1) / V2_TH, (unsigned)batch);
    CUtensorMap tm;
    std::memset(&tm, 0, sizeof tm);
    const int use_tma = make_src_map(tm, src, batch, g, R) && !getenv("EF_NO_TMA");
    return launch_pdl(kern, grid, dim3(V2_THREADS), (size_t)smem, st, src, g, P, labels, fix_list, hdr, tm, use_tma, B);
}

cudaError_t launch_k1v2(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                        cudaStream_t st) {
    switch (P.r) {
        case 1: return launch_r<1>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 2: return launch_r<2>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 3: return launch_r<3>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 4: return launch_r<4>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 5: return launch_r<5>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 6: return launch_r<6>(src, batch, g, P, labels, fix_list, hdr, B, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ef
