// ef_k1s.cu -- K1s: the streaming classify kernel (blur + Sobel + magnitude +
// NMS + double threshold, certified fp32 decisions; the contract of
// ef_fast2.cu's k1v3, which it replaces on contiguous sources).
//
// One WARP owns one task: a strip of 128 computed columns (32 lanes x 4
// adjacent columns; 128 - 2*HXA output columns) over a segment of `seg`
// output rows of one frame, and streams down it on its own -- no block
// barriers, no TMA wait at a tile start, no shared blurred tile:
//
//   input     one coalesced 4-byte load per lane and row, issued LA rows
//             ahead into a register ring (rows clamped at the frame edge);
//   blur      u8 -> fp32 by byte-permute + FADD2, vertical pass from a
//             register window of the last 2R+1 converted rows (f32x2 on
//             column pairs), horizontal pass with the neighbour lanes'
//             columns from 64-bit shuffles -- the blurred row stays in
//             registers;
//   Sobel     d = b[x+1] - b[x-1], s = b[x-1] + 2 b[x] + b[x+1] per blurred
//             row; the magnitude row y needs rows y-1..y+1, carried as
//             P = d[y-1] + 2 d[y] and Q = s[y-1] (period-2 registers);
//   vote      the squared magnitude row goes to a per-warp ring in shared
//             memory (the NMS neighbourhoods); 4-pixel groups certainly below
//             `low` are written as background at once, the others are
//             candidates: their gx / gy (8 floats) and position are stashed;
//   classify  once 32 stashed candidates have their row below in the ring (or
//             the ring is about to drop a row they need, or the strip ends),
//             one round classifies them with every lane busy: sector from the
//             stashed gx / gy, NMS and thresholds from the magnitude ring.
//
// A segment recomputes only 4 blurred and 2 magnitude rows of halo (seg = 64:
// 6%; the tile kernel's 32-row tiles: 12.5%).  Border policy (np.pad edge at
// every stage): input rows and columns clamped; blurred and magnitude values
// of out-of-frame columns replaced by the edge column's (shuffle); blurred and
// magnitude rows above / below the frame repeat the edge row (the Sobel and
// NMS neighbours are clamped row indices).
#include <cuda.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_launch.cuh"

namespace ef {

constexpr int KS_COLS = 128;  // computed columns per task
constexpr int KS_CS = KS_COLS + 4;  // ring row stride (floats): quad q of row r in bank group (r + q) mod 8
#ifndef EF_K1S_MR
#define EF_K1S_MR 10
#endif
constexpr int KS_MR = EF_K1S_MR;  // magnitude ring rows
constexpr int KS_CAP = 128;       // stashed candidate groups (power of two; pending stays < 32 ready + two rows of <= 30)
#ifndef EF_K1S_MINW
#define EF_K1S_MINW 20  // resident warps per SM the register budget is sized for
#endif
#ifndef EF_K1S_LA
#define EF_K1S_LA 6  // input rows loaded ahead
#endif

struct KsWarp {
    float m[KS_MR][KS_CS];  // squared magnitudes, row Y in slot Y % KS_MR
    float4 cgx[KS_CAP];     // stashed candidates: gx of the 4 pixels
    float4 cgy[KS_CAP];     //   gy
    int cpos[KS_CAP];       //   (row << 5) | lane
};
static_assert(sizeof(KsWarp) % 16 == 0, "float4 alignment of the per-warp state");

template <int R>
struct KsCfg {
    static constexpr int HXA = R <= 2 ? 4 : 8;
    static constexpr int OW = KS_COLS - 2 * HXA;
    static constexpr int NR = 2 * R + 1;
    static constexpr int U = 2 * NR;  // unrolled rows: the window (NR) and the Sobel registers (2) repeat
    static constexpr int RAWN = NR;  // loaded-row ring (divides U)
    static constexpr int LA = EF_K1S_LA < RAWN - 1 ? EF_K1S_LA : RAWN - 1;
};

__device__ __forceinline__ float2 ks_f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 ks_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 ks_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 ks_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

__device__ __forceinline__ float ks_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct KsCls {
    float lo_lo, lo_hi, hi_lo, hi_hi, e_nms0, e_nms_rel, e_sec;
    int cls0;
};

// Classify one stashed group (4 pixels at columns cc0 .. cc0+3 of the strip,
// frame row Y): the three magnitude rows come from the ring, gx / gy from the
// stash.  Branch-free, as k1v3's classifier (lanes hold different groups).
template <bool FUSED>
__device__ __forceinline__ void ks_classify(const KsCls& P, const float* mu, const float* mc, const float* md,
                                            float4 gx4, float4 gy4, int cc0, uint8_t* __restrict__ labels,
                                            unsigned long long rowbase, int xcol, unsigned long long frame, int yo,
                                            unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr,
                                            const FgBits& B) {
    const float t1 = 0.41421356237309503f;
    float Mu[6], Mc[6], Md[6];
    auto load6 = [&](const float* row, float (&v)[6]) {
        const float4 mid = *reinterpret_cast<const float4*>(row + cc0);
        v[0] = row[cc0 - 1];
        v[1] = mid.x; v[2] = mid.y; v[3] = mid.z; v[4] = mid.w;
        v[5] = row[cc0 + 4];
    };
    load6(mu, Mu);
    load6(mc, Mc);
    load6(md, Md);
    const float GX[4] = {gx4.x, gx4.y, gx4.z, gx4.w};
    const float GY[4] = {gy4.x, gy4.y, gy4.z, gy4.w};
    uint32_t packed = 0;
    bool any_flag = false;
    const uint32_t cls0 = (uint32_t)P.cls0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float c = ks_sqrt(Mc[k + 1]);
        const float gx = GX[k], gy = GY[k];
        const float a = fabsf(gx), b = fabsf(gy);
        const float uu = fmaf(t1, a, -b), vv = fmaf(t1, b, -a);
        const float n0 = fmaxf(Mc[k], Mc[k + 2]);
        const float n90 = fmaxf(Mu[k + 1], Md[k + 1]);
        const float n45 = fmaxf(Mu[k + 2], Md[k]);
        const float n135 = fmaxf(Mu[k], Md[k + 2]);
        const float ndiag = ((gx > 0.f) == (gy > 0.f)) ? n45 : n135;
        const float nmax = uu > 0.f ? n0 : (vv > 0.f ? n90 : ndiag);
        const float nv = ks_sqrt(nmax);
        const float d = c - nv;
        const float e_nms = fmaf(P.e_nms_rel, c + nv, P.e_nms0);
        const bool amb = fabsf(uu) <= P.e_sec || fabsf(vv) <= P.e_sec;
        const int lo_cls = c >= P.lo_lo ? (c > P.lo_hi ? 1 : -1) : 0;
        const int cls = c >= P.hi_lo ? (c > P.hi_hi ? 2 : -1) : lo_cls;
        const bool need_nms = cls >= 0 && (uint32_t)cls != cls0;
        const bool flag = cls < 0 || (need_nms && (amb || fabsf(d) <= e_nms));
        const uint32_t lab = flag ? (uint32_t)kFlag : ((need_nms && d > e_nms) ? (uint32_t)cls : cls0);
        any_flag |= flag;
        packed |= lab << (8 * k);
    }
    if (any_flag) {
        unsigned fm = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (((packed >> (8 * k)) & 0xffu) == kFlag) fm |= 1u << k;
        const unsigned cnt = __popc(fm);
        unsigned long long slot, cap;
        asm volatile("atom.global.add.u64 %0, [%1], %2;" : "=l"(slot) : "l"(&hdr->fix_count), "l"((unsigned long long)cnt)
                     : "memory");
        asm volatile("ld.global.u64 %0, [%1];" : "=l"(cap) : "l"(&hdr->fix_cap) : "memory");
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!((fm >> k) & 1u)) continue;
            if (slot < cap)
                asm volatile("st.global.u64 [%0], %1;" ::"l"(fix_list + slot),
                             "l"(rowbase + (unsigned long long)(xcol + k)) : "memory");
            else
                st_global_u32(&hdr->overflow, 1u);
            ++slot;
        }
    }
    st_global_u32(labels + rowbase + xcol, packed);
    if (FUSED) {
        st_global_u32(labels + rowbase + xcol + B.fin_off, (packed >> 1) & 0x01010101u);
        const uint32_t lo = packed & 0x03030303u;
        const uint32_t fgn = (((lo | (lo >> 1)) & 0x01010101u) * 0x10204080u) >> 28;
        const uint32_t stn = (((packed >> 1) & 0x01010101u) * 0x10204080u) >> 28;
        if (fgn) fg_bits_or(B, frame, yo, xcol, fgn, stn);
    }
}

// Everything a classifier round needs besides the warp's ring and stash
// (built once per task; the round function is not inlined, so the stream's
// unrolled row loop carries one call site instead of a copy of the classifier
// per unrolled row -- the instruction cache holds the whole loop).
struct KsCtx {
    KsCls P;
    uint8_t* labels;
    unsigned long long* fix_list;
    WsHeader* hdr;
    FgBits B;
    unsigned long long out_base, frame;
    int W, FH, out0, xv0;
};

// Rounds of 32 over the stash entries [tail, ready) while 32 are ready, then
// the rest when `partial` (the ring is about to drop a row they need, or the
// strip ends).  Returns the new tail.
template <bool FUSED>
__device__ __noinline__ int ks_rounds(KsWarp& S, int tail, int ready, bool partial, const KsCtx& X) {
    const int lane = threadIdx.x & 31;
    while (ready - tail >= 32 || (partial && ready > tail)) {
        const int n = min(32, ready - tail);
        if (lane < n) {
            const int e = (tail + lane) % KS_CAP;
            const int pos = S.cpos[e];
            const int Y = pos >> 5, gl = pos & 31;
            const int Yu = max(Y - 1, 0), Yd = min(Y + 1, X.FH - 1);
            const unsigned long long rowbase = X.out_base + (unsigned long long)(Y - X.out0) * X.W;
            ks_classify<FUSED>(X.P, S.m[Yu % KS_MR], S.m[Y % KS_MR], S.m[Yd % KS_MR], S.cgx[e], S.cgy[e], 4 * gl,
                               X.labels, rowbase, X.xv0 + 4 * gl, X.frame, Y - X.out0, X.fix_list, X.hdr, X.B);
        }
        tail += n;
        __syncwarp();  // reads done before a later row overwrites their ring slot
    }
    return tail;
}

// One task: strip sx, segment sy of frame `frame`.  EDGE: the strip reaches
// past the frame's left or right edge (replicated columns); interior strips
// run code without any of that.
template <int R, bool FUSED, bool EDGE>
__device__ __forceinline__ void k1s_task(const uint8_t* __restrict__ src, const FrameGeom& g, const FastParams& P,
                                         uint8_t* __restrict__ labels, unsigned long long* __restrict__ fix_list,
                                         WsHeader* __restrict__ hdr, const FgBits& B, int seg, int sx, int sy,
                                         KsWarp& S) {
    constexpr int HXA = KsCfg<R>::HXA, OW = KsCfg<R>::OW, NR = KsCfg<R>::NR, U = KsCfg<R>::U, LA = KsCfg<R>::LA,
                  RAWN = KsCfg<R>::RAWN;
    const int lane = threadIdx.x;
    const int W = g.W, FH = g.full_H;
    const int xv0 = sx * OW - HXA;
    const int c = xv0 + 4 * lane;  // this lane's first computed column
    const int ya = g.out0 + sy * seg, yb = min(ya + seg, g.out0 + g.rows);
    const int ms = max(ya - 1, 0), me = min(yb, FH - 1);      // magnitude rows
    const int bs = max(ms - 1, 0), be = min(me + 1, FH - 1);  // blurred rows
    const int ylo = max(0, g.g0), yhi = min(FH, g.g0 + g.H) - 1;  // input rows held in the buffer
    const unsigned long long frame = blockIdx.y;
    const unsigned long long out_base = frame * (unsigned long long)g.rows * W;

    // ---- input: lane word at column clamp(c); edge lanes replicate the edge byte
    const int cl = EDGE ? min(max(c, 0), W - 4) : c;
    const uint8_t* const in0 = src + (size_t)frame * g.H * W + cl - (long long)g.g0 * W;  // + Y * W
    const uint32_t esel = c < 0 ? 0x0000u : 0x3333u;
    const bool eout = c < 0 || c >= W;
    auto fetch = [&](int j) -> uint32_t {  // input row bs - R + j (clamped)
        const int Y = min(max(bs - R + j, ylo), yhi);
        uint32_t w = __ldg(reinterpret_cast<const unsigned int*>(in0 + (long long)Y * W));
        if (EDGE && eout) w = __byte_perm(w, 0u, esel);
        return w;
    };
    // lanes holding the first / last in-frame column (edge strips)
    const int lfirst = max(0, (-xv0) >> 2), llast = min(31, ((W - 1) - xv0) >> 2);

    float2 wf2[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wf2[k] = ks_f2(P.wf[k], P.wf[k]);
    auto cvt = [&](uint32_t w, float2& lo, float2& hi) {
        lo = ks_add(ks_f2(__int_as_float(__byte_perm(w, 0x4B000000u, 0x7540u)),
                          __int_as_float(__byte_perm(w, 0x4B000000u, 0x7541u))), ks_f2(-8388608.0f, -8388608.0f));
        hi = ks_add(ks_f2(__int_as_float(__byte_perm(w, 0x4B000000u, 0x7542u)),
                          __int_as_float(__byte_perm(w, 0x4B000000u, 0x7543u))), ks_f2(-8388608.0f, -8388608.0f));
    };

    float2 p[NR][2];     // converted window: relative input row j in slot j % NR
    uint32_t raw[RAWN];  // loaded, not yet converted: relative row j in slot j % RAWN
    const int jmax = be - bs + 2 * R;  // last relative input row the strip needs
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) raw[j % RAWN] = fetch(j);  // 2R <= jmax
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) cvt(raw[j % RAWN], p[j % NR][0], p[j % NR][1]);
#pragma unroll
    for (int j = 2 * R; j < 2 * R + LA; ++j)  // after the conversions: rows j and j + RAWN share a slot
        if (j <= jmax) raw[j % RAWN] = fetch(j);

    // ---- Sobel carry: P = d[y-1] + 2 d[y], Q = s[y-1], Dp = d[y], Sp = s[y]
    float2 Pd[2] = {}, Qs[2] = {}, Dp[2] = {}, Sp[2] = {};
    // ---- magnitude ring / stash bookkeeping (warp-uniform)
    int mslot = (ms - 1 + KS_MR * 4) % KS_MR;  // slot of the last magnitude row written (ms - 1)
    int head = 0, tail = 0;                  // stash counters (monotonic)
    const float cand_sq = P.lo_lo > 0.f ? P.lo_lo * P.lo_lo * (1.0f - 1.0f / 262144.0f) : -1.0f;
    const uint32_t fill = (uint32_t)P.cls0 * 0x01010101u;
    const bool out_lane = lane >= HXA / 4 && lane < (HXA + OW) / 4 && c < W;
    // label word of this lane in magnitude row Ym = labp (advanced per row)
    uint8_t* labp = labels + out_base + (long long)(ms - g.out0) * W + c;
    const KsCtx X{{P.lo_lo, P.lo_hi, P.hi_lo, P.hi_hi, P.e_nms0, P.e_nms_rel, P.e_sec, P.cls0},
                  labels, fix_list, hdr, B, out_base, frame, W, FH, g.out0, xv0};

    // magnitude row Ym from the carry and the new blurred row's (dn, sn)
    auto emit = [&](int Ym, const float2 (&dn)[2], const float2 (&sn)[2]) {
        const float2 gx01 = ks_add(Pd[0], dn[0]), gx23 = ks_add(Pd[1], dn[1]);
        const float2 gy01 = ks_add(sn[0], ks_f2(-Qs[0].x, -Qs[0].y)), gy23 = ks_add(sn[1], ks_f2(-Qs[1].x, -Qs[1].y));
        float2 m01 = ks_fma(gx01, gx01, ks_mul(gy01, gy01));
        float2 m23 = ks_fma(gx23, gx23, ks_mul(gy23, gy23));
        if (EDGE) {  // out-of-frame columns take the edge column's magnitude
            const float vl = __shfl_sync(0xffffffffu, m01.x, lfirst), vr = __shfl_sync(0xffffffffu, m23.y, llast);
            if (c < 0) m01 = m23 = ks_f2(vl, vl);
            if (c >= W) m01 = m23 = ks_f2(vr, vr);
        }
        mslot = mslot + 1 == KS_MR ? 0 : mslot + 1;
        *reinterpret_cast<float4*>(&S.m[mslot][4 * lane]) = make_float4(m01.x, m01.y, m23.x, m23.y);
        if (Ym >= ya && Ym < yb) {  // an output row (warp-uniform)
            const bool cand = out_lane && fmaxf(fmaxf(m01.x, m01.y), fmaxf(m23.x, m23.y)) >= cand_sq;
            const unsigned bal = __ballot_sync(0xffffffffu, cand);
            if (out_lane && !cand) {
                st_global_u32(labp, fill);
                if (FUSED) st_global_u32(labp + B.fin_off, 0u);
            }
            if (cand) {
                const int e = (head + __popc(bal & ((1u << lane) - 1u))) & (KS_CAP - 1);
                S.cgx[e] = make_float4(gx01.x, gx01.y, gx23.x, gx23.y);
                S.cgy[e] = make_float4(gy01.x, gy01.y, gy23.x, gy23.y);
                S.cpos[e] = (Ym << 5) | lane;
            }
            head += __popc(bal);
        }
        labp += W;
        __syncwarp();  // the ring row and the stash are read by other lanes' rounds
    };

    // rounds over stash entries [tail, ready): full ones, then the rest if `partial`
    auto rounds = [&](int ready, bool partial) {
        while (ready - tail >= 32 || (partial && ready > tail)) {
            const int n = min(32, ready - tail);
            if (lane < n) {
                const int e = (tail + lane) & (KS_CAP - 1);
                const int pos = S.cpos[e];
                const int Y = pos >> 5, gl = pos & 31;
                const int Yu = max(Y - 1, 0), Yd = min(Y + 1, FH - 1);
                const unsigned long long rowbase = out_base + (unsigned long long)(Y - g.out0) * W;
                ks_classify<FUSED>(X.P, S.m[Yu % KS_MR], S.m[Y % KS_MR], S.m[Yd % KS_MR], S.cgx[e], S.cgy[e],
                                   4 * gl, labels, rowbase, xv0 + 4 * gl, frame, Y - g.out0, fix_list, hdr, B);
            }
            tail += n;
            __syncwarp();  // reads done before a later row overwrites their ring slot
        }
    };

    // ---- the stream: blurred rows bs .. be, magnitude rows ms .. me.  The
    // window (period NR) and the Sobel carry (period 2) index registers by
    // the row phase uu = u % U, a constant inside each unrolled step.  A step
    // that makes a classifier round due leaves the unrolled sequence for the
    // ONE round site below, which re-enters the sequence at the next phase
    // (a switch into the fall-through chain) -- the loop body holds U steps
    // and one copy of the classifier.
    const int nb = be - bs + 1;
    int u = 0;                    // next blurred row (relative to bs)
    int rd_ready = 0;             // the due round's ready count
    bool rd_partial = false;
    auto step = [&](auto KK) -> int {  // 0: next step, 1: a round is due, 2: the stream ended
        constexpr int uu = decltype(KK)::value;
        if (u >= nb) return 2;
        const int Yb = bs + u;
        // window: relative rows u .. u + 2R (the newest converted now); load ahead
        cvt(raw[(uu + 2 * R) % RAWN], p[(uu + 2 * R) % NR][0], p[(uu + 2 * R) % NR][1]);
        if (u + 2 * R + LA <= jmax) raw[(uu + 2 * R + LA) % RAWN] = fetch(u + 2 * R + LA);
        float2 v01 = ks_mul(wf2[0], p[(uu + R) % NR][0]);
        float2 v23 = ks_mul(wf2[0], p[(uu + R) % NR][1]);
#pragma unroll
        for (int o = 1; o <= R; ++o) {
            v01 = ks_fma(wf2[o], ks_add(p[(uu + R - o) % NR][0], p[(uu + R + o) % NR][0]), v01);
            v23 = ks_fma(wf2[o], ks_add(p[(uu + R - o) % NR][1], p[(uu + R + o) % NR][1]), v23);
        }
        // horizontal pass: e[j] = column c - 8 + j
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
        float2 b01 = ks_mul(wf2[0], ks_f2(e[8], e[9]));
        float2 b23 = ks_mul(wf2[0], ks_f2(e[10], e[11]));
#pragma unroll
        for (int o = 1; o <= R; ++o) {
            if ((o & 1) == 0) {
                b01 = ks_fma(wf2[o], ks_add(ks_f2(e[8 - o], e[9 - o]), ks_f2(e[8 + o], e[9 + o])), b01);
                b23 = ks_fma(wf2[o], ks_add(ks_f2(e[10 - o], e[11 - o]), ks_f2(e[10 + o], e[11 + o])), b23);
            } else {
                b01 = ks_fma(wf2[o], ks_f2(e[8 - o] + e[8 + o], e[9 - o] + e[9 + o]), b01);
                b23 = ks_fma(wf2[o], ks_f2(e[10 - o] + e[10 + o], e[11 - o] + e[11 + o]), b23);
            }
        }
        if (EDGE) {  // out-of-frame columns take the edge column's blurred value
            const float vl = __shfl_sync(0xffffffffu, b01.x, lfirst), vr = __shfl_sync(0xffffffffu, b23.y, llast);
            if (c < 0) b01 = b23 = ks_f2(vl, vl);
            if (c >= W) b01 = b23 = ks_f2(vr, vr);
        }
        // Sobel parts of this blurred row
        float2 dn[2], sn[2];
        {
            const float bl = __shfl_up_sync(0xffffffffu, b23.y, 1);
            const float br = __shfl_down_sync(0xffffffffu, b01.x, 1);
            dn[0] = ks_f2(b01.y - bl, b23.x - b01.x);
            dn[1] = ks_f2(b23.y - b01.y, br - b23.x);
            sn[0] = ks_f2(fmaf(2.f, b01.x, bl + b01.y), fmaf(2.f, b01.y, b01.x + b23.x));
            sn[1] = ks_f2(fmaf(2.f, b23.x, b01.y + b23.y), fmaf(2.f, b23.y, b23.x + br));
        }
        ++u;
        if (u == 1) {  // first blurred row: the row above repeats it (frame top; else replaced next row)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                Pd[h] = ks_fma(ks_f2(2.f, 2.f), dn[h], dn[h]);
                Qs[h] = sn[h];
                Dp[h] = dn[h];
                Sp[h] = sn[h];
            }
            return 0;
        }
        const int Ym = Yb - 1;
        int due = 0;
        if (Ym >= ms) {
            const int before = head;
            emit(Ym, dn, sn);
            // entries stashed before this row are classifiable (their row below
            // is in the ring; at the frame's last row all are); a round is due
            // when 32 are, or when the next row would overwrite the ring slot of
            // a row the oldest one needs.  Pending entries stay below KS_CAP.
            const int ready = (Ym == FH - 1) ? head : before;
            bool partial = false;
            if (ready - tail < 32 && ready > tail)
                partial = (S.cpos[tail & (KS_CAP - 1)] >> 5) - 1 <= Ym + 1 - KS_MR;
            if (ready - tail >= 32 || partial) {
                rd_ready = ready;
                rd_partial = partial;
                due = 1;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            Pd[h] = ks_fma(ks_f2(2.f, 2.f), dn[h], Dp[h]);
            Qs[h] = Sp[h];
            Dp[h] = dn[h];
            Sp[h] = sn[h];
        }
        return due;
    };
    int phase = 0;
    while (true) {
        int code = 0;
        switch (phase) {
#define EF_KS_STEP(K)                                                        \
    case K:                                                                  \
        if constexpr (K < U) {                                               \
            code = step(std::integral_constant<int, K>{});                   \
            if (code) {                                                      \
                phase = K;                                                   \
                goto stepped;                                                \
            }                                                                \
        }                                                                    \
        [[fallthrough]];
            EF_KS_STEP(0) EF_KS_STEP(1) EF_KS_STEP(2) EF_KS_STEP(3) EF_KS_STEP(4) EF_KS_STEP(5)
            EF_KS_STEP(6) EF_KS_STEP(7) EF_KS_STEP(8) EF_KS_STEP(9) EF_KS_STEP(10) EF_KS_STEP(11)
            EF_KS_STEP(12) EF_KS_STEP(13) EF_KS_STEP(14) EF_KS_STEP(15) EF_KS_STEP(16) EF_KS_STEP(17)
#undef EF_KS_STEP
            default: break;
        }
        phase = 0;  // the whole chain ran: the next block of U rows
        continue;
    stepped:
        if (code == 2) break;
        rounds(rd_ready, rd_partial);
        phase = phase + 1 == U ? 0 : phase + 1;
    }
    static_assert(KsCfg<R>::U <= 18, "step cases");
    if (be == me) {  // frame bottom: the row below the last magnitude row repeats its blurred row
        const float2 dn[2] = {Dp[0], Dp[1]}, sn[2] = {Sp[0], Sp[1]};
        emit(me, dn, sn);
    }
    // the strip's remaining candidates (their rows below are all in the ring)
    if (head > tail) ks_rounds<FUSED>(S, tail, head, true, X);
}

// One block = one warp = one task (block-uniform control flow: every branch
// around a shuffle or vote is visibly warp-uniform to the compiler).
template <int R, bool FUSED>
__global__ void __launch_bounds__(32, EF_K1S_MINW)
k1s_kernel(const uint8_t* __restrict__ src, FrameGeom g, FastParams P, uint8_t* __restrict__ labels,
           unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr, FgBits B, int seg, int nstrips,
           int nsegs) {
    __shared__ KsWarp S;
    pdl_wait();  // workspace counters and bit planes are reset by the previous kernel
    pdl_trigger();
    const int task = blockIdx.x;
    const int sy = task / nstrips, sx = task - sy * nstrips;
    const int xv0 = sx * KsCfg<R>::OW - KsCfg<R>::HXA;
    if (xv0 < 0 || xv0 + KS_COLS > g.W)
        k1s_task<R, FUSED, true>(src, g, P, labels, fix_list, hdr, B, seg, sx, sy, S);
    else
        k1s_task<R, FUSED, false>(src, g, P, labels, fix_list, hdr, B, seg, sx, sy, S);
}

// k1s runs where k1v3 would (W % 4 == 0, aligned buffers, radius 1..6) on a
// contiguous source (no peer halo rows); ef_set_k1_variant selects it
static std::atomic<int> g_k1_variant{getenv("EF_K1_VARIANT") ? atoi(getenv("EF_K1_VARIANT")) : 1};
static std::atomic<int> g_k1s_seg{getenv("EF_K1S_SEG") ? atoi(getenv("EF_K1S_SEG")) : 64};

void set_k1_variant(int v, int seg) {
    g_k1_variant.store(v);
    if (seg > 0) g_k1s_seg.store(seg);
}

bool k1s_selected(const FastParams& P, const FrameGeom& g) {
    return g_k1_variant.load() == 1 && !g.top && !g.bot && k1v2_supported(P, g) && P.r <= 4;
}

template <int R>
static cudaError_t launch_s(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                            uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                            cudaStream_t st) {
    const int seg = std::max(1, g_k1s_seg.load());
    const int nstrips = (g.W + KsCfg<R>::OW - 1) / KsCfg<R>::OW;
    const int nsegs = (g.rows + seg - 1) / seg;
    const long long tasks = (long long)nstrips * nsegs;
    if (batch > 65535 || tasks > 0x7fffffff) return cudaErrorInvalidValue;
    static std::atomic<uint64_t> configured{0};
    cudaError_t e = once_per_device(configured, [&] {
        cudaError_t r = cudaSuccess;
        for (auto k : {k1s_kernel<R, true>, k1s_kernel<R, false>})
            if (r == cudaSuccess)
                r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared);
        return r;
    });
    if (e != cudaSuccess) return e;
    auto kern = B.fg ? k1s_kernel<R, true> : k1s_kernel<R, false>;
    dim3 grid((unsigned)tasks, (unsigned)batch);
    return launch_pdl(kern, grid, dim3(32), 0, st, src, g, P, labels, fix_list, hdr, B, seg, nstrips,
                      nsegs);
}

cudaError_t launch_k1s(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                       uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                       cudaStream_t st) {
    switch (P.r) {
        case 1: return launch_s<1>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 2: return launch_s<2>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 3: return launch_s<3>(src, batch, g, P, labels, fix_list, hdr, B, st);
        case 4: return launch_s<4>(src, batch, g, P, labels, fix_list, hdr, B, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ef
