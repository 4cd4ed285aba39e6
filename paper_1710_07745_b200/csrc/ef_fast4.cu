// ef_fast4.cu -- K1 v4: single-pass streaming fused classify kernel.
//
// Same contract as ef_fast.cu / ef_fast2.cu (certified fp32 decisions; kFlag
// + fix list for the rest).  Structure, per warp, no block-level sharing:
//
//  * a strip of 128 computed columns (lane = 4 adjacent columns; OW output
//    columns, HXA halo columns each side) and two row blocks A = [Y0, Y0+HB)
//    and B = [Y0+HB, Y0+2HB) processed in lockstep: every fp32 value is an
//    (A, B) float2, so all stencil arithmetic is packed f32x2 (FFMA2/FADD2/FMUL2);
//  * one pass down the rows: 4-byte coalesced loads prefetched 2R rows ahead,
//    u8 -> fp32 by byte-permute + FADD2, vertical blur from a register ring of
//    the last 2R+1 input rows, horizontal blur with 64-bit neighbour shuffles,
//    Sobel with running sums (gx(j) = P + d(j+1), P' = d(j) + 2 d(j+1);
//    gy(j) = s(j+1) - s(j-1)) -- period-2 state, so the loop unrolls by
//    lcm(2R+1, 2) with no register moves;
//  * squared magnitudes go to an 8-row (A,B) ring in shared memory; 4-pixel
//    groups holding a possible edge (m^2 >= lo_lo^2) are queued per warp with
//    their gx/gy and classified 32 at a time (sector, NMS, thresholds,
//    certification); all other groups are written as the suppressed class.
//
// Border policy (np.pad edge per stage): input rows/columns clamp on load;
// blurred and squared-magnitude values at out-of-frame columns are replaced by
// the edge column (warp shuffle); magnitude rows -1 and FH alias rows 0 and
// FH-1 in the ring.
#include "ef_common.cuh"
#include "ef_internal.h"

namespace ef {

constexpr int V4_WARPS = 4;
constexpr int V4_THREADS = 32 * V4_WARPS;
constexpr int V4_COLS = 128;
constexpr int V4_MRING = 8;
constexpr int V4_QCAP = 96;

template <int R>
struct V4Cfg {
    static constexpr int HXA = R <= 2 ? 4 : 8;
    static constexpr int OW = V4_COLS - 2 * HXA;
    static constexpr int NR = 2 * R + 1;
    static constexpr int PER = (NR % 2) ? 2 * NR : NR;  // lcm(NR, 2)
    static constexpr int HB = 4 * PER - 4;             // rows per block: steps = HB + 4 = 4*PER
    static constexpr int STEPS = HB + 4;
};

struct V4Warp {
    float2 m[V4_MRING][V4_COLS];  // (A, B) squared magnitudes, ring of rows
    int qmeta[V4_QCAP];           // (local row << 8) | (strip << 5) | lane
    float4 qgx[V4_QCAP];
    float4 qgy[V4_QCAP];
};

struct V4Smem {
    V4Warp w[V4_WARPS];
};

__device__ __forceinline__ float2 f2v(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2v(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2v(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2v(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 sub2v(float2 a, float2 b) { return __fadd2_rn(a, f2v(-b.x, -b.y)); }

__device__ __forceinline__ double pack_d(float2 v) {
    return __hiloint2double(__float_as_int(v.y), __float_as_int(v.x));
}
__device__ __forceinline__ float2 unpack_d(double d) {
    return f2v(__int_as_float(__double2loint(d)), __int_as_float(__double2hiint(d)));
}

__device__ __noinline__ uint32_t v4_load_edge(const uint8_t* rowp, int c, int W) {
    uint32_t w = 0;
    for (int k = 0; k < 4; ++k) w |= (uint32_t)rowp[clampi(c + k, 0, W - 1)] << (8 * k);
    return w;
}

__device__ __forceinline__ uint32_t v4_load(const uint8_t* rowp, int c, int W, bool col_ok) {
    if (col_ok) return __ldg(reinterpret_cast<const unsigned int*>(rowp + c));
    return v4_load_edge(rowp, c, W);
}

// bytes k of (wa, wb) -> float2(A, B)
__device__ __forceinline__ float2 cvt2(uint32_t wa, uint32_t wb, unsigned sel) {
    return add2v(f2v(__int_as_float(__byte_perm(wa, 0x4B000000u, sel)),
                     __int_as_float(__byte_perm(wb, 0x4B000000u, sel))),
                 f2v(-8388608.0f, -8388608.0f));
}

__device__ __forceinline__ float sqrt_apx4(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Replace (A,B) values at out-of-frame columns by the edge column's values.
__device__ __forceinline__ void edge_fix2(float2 (&v)[4], int xv0, int lane, int W) {
    const int c = xv0 + 4 * lane;
    if (xv0 < 0) {
        const int L0 = (-xv0) >> 2, k0 = (-xv0) & 3;
        float2 e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) e[k] = unpack_d(__shfl_sync(0xffffffffu, pack_d(v[k]), L0));
        const float2 ev = k0 == 0 ? e[0] : (k0 == 1 ? e[1] : (k0 == 2 ? e[2] : e[3]));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (c + k < 0) v[k] = ev;
    }
    if (xv0 + V4_COLS > W) {
        const int last = W - 1 - xv0;
        const int L1 = last >> 2, k1 = last & 3;
        float2 e[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) e[k] = unpack_d(__shfl_sync(0xffffffffu, pack_d(v[k]), L1));
        const float2 ev = k1 == 0 ? e[0] : (k1 == 1 ? e[1] : (k1 == 2 ? e[2] : e[3]));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (c + k >= W) v[k] = ev;
    }
}

struct V4Cls {
    float lo_lo, lo_hi, hi_lo, hi_hi, e_nms, e_sec;
    int cls0;
    int W, FH, out0, Y0, HB, xv0;
    uint8_t* labels;
    unsigned long long out_base;
    unsigned long long* fix_list;
    WsHeader* hdr;
};

__device__ __forceinline__ int v4slot(int lr) { return (lr + 2 * V4_MRING) & (V4_MRING - 1); }

// Classify queued groups, 32 at a time, until the queue is empty.
__device__ __noinline__ void v4_flush(const V4Cls P, int qn, V4Warp& S, int lane) {
    const float t1 = 0.41421356237309503f;
    for (int base = 0; base < qn; base += 32) {
        const int e = base + lane;
        if (e < qn) {
            const int meta = S.qmeta[e];
            const int lr = meta >> 8, strip = (meta >> 5) & 1, cl = meta & 31;
            const float4 gx4 = S.qgx[e], gy4 = S.qgy[e];
            const float gxa[4] = {gx4.x, gx4.y, gx4.z, gx4.w};
            const float gya[4] = {gy4.x, gy4.y, gy4.z, gy4.w};
            const int Yc = P.Y0 + lr + strip * P.HB;
            const float2* mu = S.m[v4slot(lr - 1)];
            const float2* mc = S.m[v4slot(lr)];
            const float2* md = S.m[v4slot(lr + 1)];
            const unsigned long long rowbase = P.out_base + (unsigned long long)(Yc - P.out0) * P.W;
            const int cc0 = 4 * cl;
            uint32_t packed = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int cc = cc0 + k;
                auto pick = [&](const float2* row, int col) { return strip ? row[col].y : row[col].x; };
                const float c = sqrt_apx4(pick(mc, cc));
                int cls;
                if (c > P.hi_hi) cls = 2;
                else if (c >= P.hi_lo) cls = -1;
                else if (c > P.lo_hi) cls = 1;
                else if (c >= P.lo_lo) cls = -1;
                else cls = 0;
                bool flag = cls < 0;
                uint32_t lab = (uint32_t)P.cls0;
                if (!flag && cls != P.cls0) {
                    const float gx = gxa[k], gy = gya[k];
                    const float a = fabsf(gx), b = fabsf(gy);
                    const float uu = fmaf(t1, a, -b), vv = fmaf(t1, b, -a);
                    if (fabsf(uu) <= P.e_sec || fabsf(vv) <= P.e_sec) {
                        flag = true;
                    } else {
                        float n1, n2;
                        if (uu > 0.f) { n1 = pick(mc, cc - 1); n2 = pick(mc, cc + 1); }                       // 0
                        else if (vv > 0.f) { n1 = pick(mu, cc); n2 = pick(md, cc); }                          // 90
                        else if ((gx > 0.f) == (gy > 0.f)) { n1 = pick(mu, cc + 1); n2 = pick(md, cc - 1); }  // 45
                        else { n1 = pick(mu, cc - 1); n2 = pick(md, cc + 1); }                                // 135
                        const float d = c - sqrt_apx4(fmaxf(n1, n2));
                        if (d < -P.e_nms) lab = (uint32_t)P.cls0;
                        else if (d > P.e_nms) lab = (uint32_t)cls;
                        else flag = true;
                    }
                }
                if (flag) {
                    lab = kFlag;
                    const unsigned long long o = rowbase + (unsigned long long)(P.xv0 + cc);
                    const unsigned long long slot = atomicAdd(&P.hdr->fix_count, 1ull);
                    if (slot < P.hdr->fix_cap) P.fix_list[slot] = o;
                    else P.hdr->overflow = 1u;
                }
                packed |= lab << (8 * k);
            }
            *reinterpret_cast<uint32_t*>(P.labels + rowbase + P.xv0 + cc0) = packed;
        }
    }
}

template <int R, bool INTERIOR>
__device__ __forceinline__ void v4_warp(const uint8_t* __restrict__ img, const FrameGeom& g, const FastParams& P,
                                        int xv0, int Y0, V4Warp& S, int lane, const V4Cls& CP) {
    constexpr int NR = V4Cfg<R>::NR;
    constexpr int PER = V4Cfg<R>::PER;
    constexpr int HB = V4Cfg<R>::HB;
    constexpr int STEPS = V4Cfg<R>::STEPS;
    constexpr int HXA = V4Cfg<R>::HXA;
    constexpr int OW = V4Cfg<R>::OW;
    const int W = g.W, FH = g.full_H;
    const int c = xv0 + 4 * lane;
    const bool edge = !INTERIOR && (xv0 < 0 || xv0 + V4_COLS > W);
    const bool col_ok = INTERIOR || (c >= 0 && c + 3 < W);
    const bool out_lane = lane >= HXA / 4 && lane < (HXA + OW) / 4 && c < W;
    // rows: strip A input row for step s is Y0 - 2 + R + s; strip B adds HB
    const int rlo = max(0, g.g0), rhi = min(FH - 1, g.g0 + g.H - 1);
    const uint8_t* base = img - (ptrdiff_t)g.g0 * W + c;
    auto rowp = [&](int Y) { return base + (INTERIOR ? Y : min(max(Y, rlo), rhi)) * W; };
    const int oy0 = max(Y0, g.out0), oy1 = min(Y0 + 2 * HB, g.out0 + g.rows);

    float2 wf[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wf[k] = f2v(P.wf[k], P.wf[k]);
    const float cand_sq = P.lo_lo > 0.f ? P.lo_lo * P.lo_lo * (1.0f - 1.0f / 262144.0f) : -1.0f;
    const uint32_t fill = (uint32_t)P.cls0 * 0x01010101u;

    // input ring (A,B) per column; raw prefetch ring
    float2 p[NR][4];
    uint32_t rawA[NR], rawB[NR];
    const int iA0 = Y0 - 2 - R;  // input row index ii -> global row iA0 + ii (A), + HB (B)
#pragma unroll
    for (int ii = 0; ii < 2 * R; ++ii) {
        const uint32_t wa = v4_load(rowp(iA0 + ii) - c, c, W, col_ok);
        const uint32_t wb = v4_load(rowp(iA0 + HB + ii) - c, c, W, col_ok);
#pragma unroll
        for (int k = 0; k < 4; ++k) p[ii][k] = cvt2(wa, wb, 0x7540u | k);
    }
#pragma unroll
    for (int ii = 2 * R; ii < 4 * R; ++ii) {
        rawA[ii % NR] = v4_load(rowp(iA0 + ii) - c, c, W, col_ok);
        rawB[ii % NR] = v4_load(rowp(iA0 + HB + ii) - c, c, W, col_ok);
    }
    // Sobel running state, two alternating register sets
    float2 Pg[2][4], q[2][4], s1[2][4], s2[2][4];
    uint32_t* lab32 = reinterpret_cast<uint32_t*>(CP.labels + CP.out_base) + (c >> 2);
    const int Wq = W >> 2;
    int qn = 0, qstep = 0;

#pragma unroll 1
    for (int s0 = 0; s0 < STEPS; s0 += PER) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int s = s0 + u;
            const int ph = u & 1;  // Sobel state set used this step
            const int rs = u % NR;  // ring phase
            // newest input row ii = s + 2R; prefetch ii = s + 4R
            {
                const uint32_t wa = rawA[(rs + 2 * R) % NR], wb = rawB[(rs + 2 * R) % NR];
#pragma unroll
                for (int k = 0; k < 4; ++k) p[(rs + 2 * R) % NR][k] = cvt2(wa, wb, 0x7540u | k);
                rawA[(rs + 4 * R) % NR] = v4_load(rowp(iA0 + s + 4 * R) - c, c, W, col_ok);
                rawB[(rs + 4 * R) % NR] = v4_load(rowp(iA0 + HB + s + 4 * R) - c, c, W, col_ok);
            }
            // vertical pass: b row jb = Y0 - 2 + s (A), + HB (B)
            float2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2 acc = mul2v(wf[0], p[(rs + R) % NR][k]);
#pragma unroll
                for (int o = 1; o <= R; ++o)
                    acc = fma2v(wf[o], add2v(p[(rs + R - o) % NR][k], p[(rs + R + o) % NR][k]), acc);
                v[k] = acc;
            }
            // horizontal pass: e[j] = column c - 4 + j
            float2 e[12];
#pragma unroll
            for (int k = 0; k < 4; ++k) e[4 + k] = v[k];
#pragma unroll
            for (int k = 4 - R; k < 4; ++k) e[k] = unpack_d(__shfl_up_sync(0xffffffffu, pack_d(v[k]), 1));
#pragma unroll
            for (int k = 0; k < R; ++k) e[8 + k] = unpack_d(__shfl_down_sync(0xffffffffu, pack_d(v[k]), 1));
            float2 b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float2 acc = mul2v(wf[0], e[4 + k]);
#pragma unroll
                for (int o = 1; o <= R; ++o) acc = fma2v(wf[o], add2v(e[4 + k - o], e[4 + k + o]), acc);
                b[k] = acc;
            }
            if (edge) edge_fix2(b, xv0, lane, W);
            // Sobel pieces of row jb: d = b(x+1) - b(x-1), s = b(x-1) + 2b(x) + b(x+1)
            const float2 bl = unpack_d(__shfl_up_sync(0xffffffffu, pack_d(b[3]), 1));
            const float2 br = unpack_d(__shfl_down_sync(0xffffffffu, pack_d(b[0]), 1));
            const float2 two = f2v(2.f, 2.f);
            float2 d[4], sv[4];
            d[0] = sub2v(b[1], bl);
            d[1] = sub2v(b[2], b[0]);
            d[2] = sub2v(b[3], b[1]);
            d[3] = sub2v(br, b[2]);
            sv[0] = fma2v(two, b[0], add2v(bl, b[1]));
            sv[1] = fma2v(two, b[1], add2v(b[0], b[2]));
            sv[2] = fma2v(two, b[2], add2v(b[1], b[3]));
            sv[3] = fma2v(two, b[3], add2v(b[2], br));
            const int np = ph ^ 1;
            (void)rs;
            if (!INTERIOR) {
                // the reference pads the *blurred* image: b(-1) = b(0), b(FH) = b(FH-1).
                // In the running Sobel that means d/s(-1) := d/s(0) (fix the
                // carried state at jb == 0) and d/s(FH) := d/s(FH-1) (at jb == FH).
                const int jbA = Y0 - 2 + s, jbB = jbA + HB;
                const bool topA = jbA == 0, topB = jbB == 0, botA = jbA == FH, botB = jbB == FH;
                if (topA || topB || botA || botB) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (botA) { d[k].x = q[ph][k].x; sv[k].x = s1[ph][k].x; }
                        if (botB) { d[k].y = q[ph][k].y; sv[k].y = s1[ph][k].y; }
                        if (topA) { q[ph][k].x = d[k].x; s1[ph][k].x = sv[k].x; }
                        if (topB) { q[ph][k].y = d[k].y; s1[ph][k].y = sv[k].y; }
                    }
                }
            }
            // row jb-1: gx = P + d, gy = s(jb) - s(jb-2)   (valid from s >= 2)
            float2 m2[4], gxv[4], gyv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                gxv[k] = add2v(Pg[ph][k], d[k]);
                gyv[k] = sub2v(sv[k], s2[ph][k]);
                m2[k] = fma2v(gxv[k], gxv[k], mul2v(gyv[k], gyv[k]));
                Pg[np][k] = fma2v(two, d[k], q[ph][k]);  // for row jb: d(jb-1) + 2 d(jb)
                q[np][k] = d[k];
                s2[np][k] = s1[ph][k];
                s1[np][k] = sv[k];
            }
            if (edge) edge_fix2(m2, xv0, lane, W);
            // ring row of local row lr = jb - 1 - Y0 (A; B shares the slot)
            const int lr = s - 3;
            if (s >= 2) {
                float2* dst = &S.m[v4slot(lr)][4 * lane];
                const int YAm = Y0 + lr, YBm = YAm + HB;
                if (INTERIOR || (YAm >= 0 && YAm < FH && YBm >= 0 && YBm < FH)) {
                    *reinterpret_cast<float4*>(dst) = make_float4(m2[0].x, m2[0].y, m2[1].x, m2[1].y);
                    *reinterpret_cast<float4*>(dst + 2) = make_float4(m2[2].x, m2[2].y, m2[3].x, m2[3].y);
                } else {
                    // rows outside the frame are never stored: rows -1 / FH are
                    // the aliases written below (row FH's alias lands one step
                    // before row FH itself would be computed)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (YAm >= 0 && YAm < FH) dst[k].x = m2[k].x;
                        if (YBm >= 0 && YBm < FH) dst[k].y = m2[k].y;
                    }
                }
                if (!INTERIOR) {
                    // rows -1 / FH alias rows 0 / FH-1 (per strip)
                    const int YA = Y0 + lr, YB = YA + HB;
                    if (YA == 0 || YB == 0) {
                        float2* al = &S.m[v4slot(lr - 1)][4 * lane];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (YA == 0) al[k].x = m2[k].x;
                            if (YB == 0) al[k].y = m2[k].y;
                        }
                    }
                    if (YA == FH - 1 || YB == FH - 1) {
                        float2* al = &S.m[v4slot(lr + 1)][4 * lane];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (YA == FH - 1) al[k].x = m2[k].x;
                            if (YB == FH - 1) al[k].y = m2[k].y;
                        }
                    }
                }
            }
            // 1) queued entries (rows <= lr-1) are complete now that row lr is in
            //    the ring: classify them when 32 wait, when the oldest is 5 steps
            //    old (the 8-row ring reuses the slot of its row-1 at age 7), or at
            //    the end.  Flushing before enqueueing keeps qn <= 31 + 64 < QCAP.
            __syncwarp();
            if (qn >= 32 || (qn > 0 && s - qstep >= 5)) {
                v4_flush(CP, qn, S, lane);
                __syncwarp();
                qn = 0;
            }
            // 2) candidate detection for row lr (A: Y0+lr, B: +HB): groups
            //    certainly below `low` are written now, the rest are queued
            if (s >= 3) {
                const int YA = Y0 + lr, YB = YA + HB;
                const bool okA = out_lane && lr < HB && (INTERIOR || (YA >= oy0 && YA < oy1));
                const bool okB = out_lane && lr < HB && (INTERIOR || (YB >= oy0 && YB < oy1));
                const float mA = fmaxf(fmaxf(m2[0].x, m2[1].x), fmaxf(m2[2].x, m2[3].x));
                const float mB = fmaxf(fmaxf(m2[0].y, m2[1].y), fmaxf(m2[2].y, m2[3].y));
                const bool ca = okA && mA >= cand_sq;
                const bool cb = okB && mB >= cand_sq;
                if (okA && !ca) lab32[(long long)(YA - g.out0) * Wq] = fill;
                if (okB && !cb) lab32[(long long)(YB - g.out0) * Wq] = fill;
                const unsigned ba = __ballot_sync(0xffffffffu, ca);
                const unsigned bb = __ballot_sync(0xffffffffu, cb);
                const unsigned lt = (1u << lane) - 1u;
                if (ca) {
                    const int pos = qn + __popc(ba & lt);
                    S.qmeta[pos] = (lr << 8) | lane;
                    S.qgx[pos] = make_float4(gxv[0].x, gxv[1].x, gxv[2].x, gxv[3].x);
                    S.qgy[pos] = make_float4(gyv[0].x, gyv[1].x, gyv[2].x, gyv[3].x);
                }
                if (cb) {
                    const int pos = qn + __popc(ba) + __popc(bb & lt);
                    S.qmeta[pos] = (lr << 8) | (1 << 5) | lane;
                    S.qgx[pos] = make_float4(gxv[0].y, gxv[1].y, gxv[2].y, gxv[3].y);
                    S.qgy[pos] = make_float4(gyv[0].y, gyv[1].y, gyv[2].y, gyv[3].y);
                }
                const int added = __popc(ba) + __popc(bb);
                if (qn == 0 && added) qstep = s;
                qn += added;
            }
        }
    }
    // entries of the last output row need the final ring row, stored above
    __syncwarp();
    if (qn > 0) v4_flush(CP, qn, S, lane);
}

template <int R>
__global__ void __launch_bounds__(V4_THREADS, 3)
k1v4_kernel(const uint8_t* __restrict__ src, FrameGeom g, FastParams P, uint8_t* __restrict__ labels,
            unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr) {
    extern __shared__ __align__(16) unsigned char smraw4[];
    V4Smem& S = *reinterpret_cast<V4Smem*>(smraw4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int HB = V4Cfg<R>::HB;
    const int x0 = blockIdx.x * V4Cfg<R>::OW;
    const int xv0 = x0 - V4Cfg<R>::HXA;
    const int Y0 = g.out0 + (blockIdx.y * V4_WARPS + warp) * (2 * HB);
    const uint8_t* img = src + (size_t)blockIdx.z * g.H * g.W;
    V4Cls CP{P.lo_lo, P.lo_hi, P.hi_lo, P.hi_hi, P.e_nms, P.e_sec, P.cls0, g.W, g.full_H, g.out0, Y0, HB, xv0,
             labels, (unsigned long long)blockIdx.z * g.rows * g.W, fix_list, hdr};
    // decided for the whole CTA (block-uniform, so the compiler keeps the
    // warp shuffles convergent): every warp's rows, halo included, exist
    const int Yc0 = g.out0 + blockIdx.y * V4_WARPS * 2 * HB, Yc1 = Yc0 + V4_WARPS * 2 * HB;
    // (input rows are prefetched 2R rows past the last one used: Yc1 + 1 + 3R)
    const bool interior = xv0 >= 0 && xv0 + V4_COLS <= g.W && Yc0 - 2 - R >= max(g.g0, 0) &&
                          Yc1 + 2 + 3 * R <= min(g.full_H, g.g0 + g.H) && Yc1 <= g.out0 + g.rows;
    if (interior) v4_warp<R, true>(img, g, P, xv0, Y0, S.w[warp], lane, CP);
    else v4_warp<R, false>(img, g, P, xv0, Y0, S.w[warp], lane, CP);
}

bool k1v4_supported(const FastParams& P, const FrameGeom& g) { return P.r >= 1 && P.r <= 2 && (g.W % 4) == 0; }

template <int R>
static cudaError_t launch_v4r(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                              uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st) {
    const int smem = (int)sizeof(V4Smem);
    cudaError_t e = cudaFuncSetAttribute(k1v4_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    constexpr int rows_per_cta = V4_WARPS * 2 * V4Cfg<R>::HB;
    dim3 grid((g.W + V4Cfg<R>::OW - 1) / V4Cfg<R>::OW, (g.rows + rows_per_cta - 1) / rows_per_cta, (unsigned)batch);
    k1v4_kernel<R><<<grid, V4_THREADS, smem, st>>>(src, g, P, labels, fix_list, hdr);
    return cudaGetLastError();
}

cudaError_t launch_k1v4(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st) {
    switch (P.r) {
        case 1: return launch_v4r<1>(src, batch, g, P, labels, fix_list, hdr, st);
        case 2: return launch_v4r<2>(src, batch, g, P, labels, fix_list, hdr, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ef
