// ef_fast2.cu -- K1 v2: the fused classify kernel, warp-streaming layout.
//
// Same contract as ef_fast.cu (certified fp32 decisions, kFlag + fix list
// for the rest); different structure, built for instruction economy:
//
//  tile      128 computed columns (32 lanes x 4 adjacent columns per lane) x
//            64 output rows; OW = 128 - 2*HXA output columns (HXA column
//            halo on each side, 4 for radius <= 2, 8 for radius <= 4).
//  phase 1   each warp streams down a block of rows: one coalesced 4-byte
//            load per lane per input row (prefetched 2R rows ahead), u8 ->
//            fp32 by byte-permute + one FADD, vertical blur from a register
//            ring of the last 2R+1 rows, horizontal blur with the neighbour
//            lanes' columns from warp shuffles.  The blurred rows land in
//            shared memory (b tile: 68 x 128 fp32).
//  phase 2   each warp streams 16 output rows: Sobel from the b tile (period-3
//            register rings of the row differences/sums), magnitude, and a
//            per-warp 8-row ring of magnitudes in shared memory.  Pixels
//            certainly below `low` (most of them) are written as the
//            suppressed class right away; 4-pixel groups holding a possible
//            edge go to a per-warp queue and are classified 32 at a time
//            with every lane busy (sector, NMS, thresholds, certification).
//
// Border policy (np.pad edge at every stage): input rows/columns clamped on
// load; blurred and magnitude values at out-of-frame columns are replaced by
// the edge column's value (warp shuffle); magnitude rows -1 and H alias rows
// 0 and H-1 in the ring.
#include "ef_common.cuh"
#include "ef_internal.h"

namespace ef {

constexpr int V2_WARPS = 4;
constexpr int V2_THREADS = 32 * V2_WARPS;
constexpr int V2_COLS = 128;
constexpr int V2_TH = 64;
constexpr int V2_BROWS = V2_TH + 4;
constexpr int V2_ROWS_PER_WARP = V2_TH / V2_WARPS;
constexpr int MRING = 8;
constexpr int QCAP = 128;

struct V2Smem {
    float b[V2_BROWS][V2_COLS];
    float m[V2_WARPS][MRING][V2_COLS];
    int q[V2_WARPS][QCAP];
};

template <int R>
struct V2Cfg {
    static constexpr int HXA = R <= 2 ? 4 : 8;
    static constexpr int OW = V2_COLS - 2 * HXA;
    static constexpr int NR = 2 * R + 1;
};

__device__ __forceinline__ float u8f(uint32_t w, int k) {
    // byte k of w placed in the mantissa of 2^23: exact integer -> float
    return __int_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | (unsigned)k)) - 8388608.0f;
}

// Lanes whose 4 columns straddle the frame edge gather clamped bytes; kept
// out of line so the interior path is a single 4-byte load.
__device__ __noinline__ uint32_t load4_edge(const uint8_t* rowp, int c, int W) {
    uint32_t w = 0;
    for (int k = 0; k < 4; ++k) w |= (uint32_t)rowp[clampi(c + k, 0, W - 1)] << (8 * k);
    return w;
}

__device__ __forceinline__ uint32_t load4(const uint8_t* rowp, int c, int W, bool col_ok) {
    if (col_ok) return __ldg(reinterpret_cast<const unsigned int*>(rowp + c));
    return load4_edge(rowp, c, W);
}

__device__ __forceinline__ float sqrt_apx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Replace values at out-of-frame columns by the edge column's value.
__device__ __forceinline__ void edge_fix(float (&v)[4], int xv0, int lane, int W) {
    const int c = xv0 + 4 * lane;
    if (xv0 < 0) {
        const int L0 = (-xv0) >> 2, k0 = (-xv0) & 3;
        float e0 = __shfl_sync(0xffffffffu, v[0], L0), e1 = __shfl_sync(0xffffffffu, v[1], L0);
        float e2 = __shfl_sync(0xffffffffu, v[2], L0), e3 = __shfl_sync(0xffffffffu, v[3], L0);
        float e = k0 == 0 ? e0 : (k0 == 1 ? e1 : (k0 == 2 ? e2 : e3));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (c + k < 0) v[k] = e;
    }
    if (xv0 + V2_COLS > W) {
        const int last = W - 1 - xv0;
        const int L1 = last >> 2, k1 = last & 3;
        float e0 = __shfl_sync(0xffffffffu, v[0], L1), e1 = __shfl_sync(0xffffffffu, v[1], L1);
        float e2 = __shfl_sync(0xffffffffu, v[2], L1), e3 = __shfl_sync(0xffffffffu, v[3], L1);
        float e = k1 == 0 ? e0 : (k1 == 1 ? e1 : (k1 == 2 ? e2 : e3));
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (c + k >= W) v[k] = e;
    }
}

// ---------------------------------------------------------------- phase 1 --
template <int R>
__device__ __forceinline__ void v2_phase1(const uint8_t* __restrict__ img, const FrameGeom& g, int xv0, int y0,
                                          const FastParams& P, V2Smem& S, int warp, int lane) {
    constexpr int NR = V2Cfg<R>::NR;
    const int bg0 = max(y0 - 2, 0);
    const int bg1 = min(y0 + V2_TH + 2, g.full_H);
    const int nrows = bg1 - bg0;
    const int per = (nrows + V2_WARPS - 1) / V2_WARPS;
    const int ys = bg0 + warp * per;
    const int n = min(per, bg1 - ys);
    if (n <= 0) return;
    const int c = xv0 + 4 * lane;
    const int W = g.W;
    const bool edge = xv0 < 0 || xv0 + V2_COLS > W;
    const bool col_ok = c >= 0 && c + 3 < W;
    // rows clamp to the frame and to the rows present in the buffer
    const int rlo = max(0, g.g0), rhi = min(g.full_H - 1, g.g0 + g.H - 1);
    const uint8_t* base = img - (ptrdiff_t)g.g0 * W;
    auto rowp = [&](int Y) { return base + min(max(Y, rlo), rhi) * W; };
    float wf[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) wf[k] = P.wf[k];

    float p[NR][4];
    uint32_t raw[NR];
    // input row ii (0-based) is global row ys - R + ii
#pragma unroll
    for (int ii = 0; ii < 2 * R; ++ii) {
        uint32_t w = load4(rowp(ys - R + ii), c, W, col_ok);
#pragma unroll
        for (int k = 0; k < 4; ++k) p[ii][k] = u8f(w, k);
    }
#pragma unroll
    for (int ii = 2 * R; ii < 4 * R; ++ii) raw[ii % NR] = load4(rowp(ys - R + ii), c, W, col_ok);

    for (int u0 = 0; u0 < n; u0 += NR) {
#pragma unroll
        for (int s = 0; s < NR; ++s) {
            const int u = u0 + s;
            if (u >= n) break;
            {   // newest input row ii = u + 2R, prefetch ii = u + 4R
                const uint32_t w = raw[(s + 2 * R) % NR];
#pragma unroll
                for (int k = 0; k < 4; ++k) p[(s + 2 * R) % NR][k] = u8f(w, k);
                raw[(s + 4 * R) % NR] = load4(rowp(ys - R + u + 4 * R), c, W, col_ok);
            }
            float v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float acc = wf[0] * p[(s + R) % NR][k];
#pragma unroll
                for (int o = 1; o <= R; ++o)
                    acc = fmaf(wf[o], p[(s + R - o) % NR][k] + p[(s + R + o) % NR][k], acc);
                v[k] = acc;
            }
            // columns c-R .. c+3+R: e[j] is column c - R + j
            float e[4 + 2 * R];
#pragma unroll
            for (int k = 0; k < 4; ++k) e[R + k] = v[k];
#pragma unroll
            for (int o = 1; o <= R; ++o) {
                e[R - o] = __shfl_up_sync(0xffffffffu, v[4 - o], 1);
                e[R + 3 + o] = __shfl_down_sync(0xffffffffu, v[o - 1], 1);
            }
            float b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float acc = wf[0] * e[R + k];
#pragma unroll
                for (int o = 1; o <= R; ++o) acc = fmaf(wf[o], e[R + k - o] + e[R + k + o], acc);
                b[k] = acc;
            }
            if (edge) edge_fix(b, xv0, lane, W);
            const int lr = ys + u - (y0 - 2);
            *reinterpret_cast<float4*>(&S.b[lr][4 * lane]) = make_float4(b[0], b[1], b[2], b[3]);
        }
    }
}

// ---------------------------------------------------------------- phase 2 --
struct V2Out {
    uint8_t* labels;
    unsigned long long out_base;
    unsigned long long* fix_list;
    WsHeader* hdr;
};

__device__ __forceinline__ int mslot(int Y) { return (Y + MRING) & (MRING - 1); }

// Classify the 4 pixels of one queued group (certified; kFlag otherwise).
template <int R>
__device__ __forceinline__ void v2_classify_group(const FrameGeom& g, int xv0, int y0, int Yc, int cl,
                                                  const FastParams& P, V2Smem& S, int warp, const V2Out& O) {
    const int W = g.W, FH = g.full_H;
    const float t1 = 0.41421356237309503f;
    const float* mu = S.m[warp][mslot(Yc - 1)];
    const float* mc = S.m[warp][mslot(Yc)];
    const float* md = S.m[warp][mslot(Yc + 1)];
    const float* bu = S.b[clampi(Yc - 1, 0, FH - 1) - (y0 - 2)];
    const float* bm = S.b[Yc - (y0 - 2)];
    const float* bd = S.b[clampi(Yc + 1, 0, FH - 1) - (y0 - 2)];
    uint32_t packed = 0;
    const int cc0 = 4 * cl;
    const unsigned long long rowbase = O.out_base + (unsigned long long)(Yc - g.out0) * W;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int cc = cc0 + k;
        const float c = mc[cc];
        int cls;
        if (c > P.hi_hi) cls = 2;
        else if (c >= P.hi_lo) cls = -1;
        else if (c > P.lo_hi) cls = 1;
        else if (c >= P.lo_lo) cls = -1;
        else cls = 0;
        bool flag = cls < 0;
        uint32_t lab = (uint32_t)P.cls0;
        if (!flag && cls != P.cls0) {
            float dxu = bu[cc + 1] - bu[cc - 1];
            float dxm = bm[cc + 1] - bm[cc - 1];
            float dxd = bd[cc + 1] - bd[cc - 1];
            float su = fmaf(2.f, bu[cc], bu[cc - 1] + bu[cc + 1]);
            float sd = fmaf(2.f, bd[cc], bd[cc - 1] + bd[cc + 1]);
            float gx = fmaf(2.f, dxm, dxu + dxd);
            float gy = sd - su;
            float a = fabsf(gx), b = fabsf(gy);
            float uu = fmaf(t1, a, -b), vv = fmaf(t1, b, -a);
            if (fabsf(uu) <= P.e_sec || fabsf(vv) <= P.e_sec) {
                flag = true;
            } else {
                float n1, n2;
                if (uu > 0.f) { n1 = mc[cc - 1]; n2 = mc[cc + 1]; }                       // 0
                else if (vv > 0.f) { n1 = mu[cc]; n2 = md[cc]; }                          // 90
                else if ((gx > 0.f) == (gy > 0.f)) { n1 = mu[cc + 1]; n2 = md[cc - 1]; }  // 45
                else { n1 = mu[cc - 1]; n2 = md[cc + 1]; }                                // 135
                float d = c - fmaxf(n1, n2);
                if (d < -P.e_nms) lab = (uint32_t)P.cls0;
                else if (d > P.e_nms) lab = (uint32_t)cls;
                else flag = true;
            }
        }
        if (flag) {
            lab = kFlag;
            const unsigned long long o = rowbase + (unsigned long long)(xv0 + cc);
            unsigned long long slot = atomicAdd(&O.hdr->fix_count, 1ull);
            if (slot < O.hdr->fix_cap) O.fix_list[slot] = o;
            else O.hdr->overflow = 1u;
        }
        packed |= lab << (8 * k);
    }
    *reinterpret_cast<uint32_t*>(O.labels + rowbase + xv0 + cc0) = packed;
}

template <int R>
__device__ __forceinline__ void v2_flush(const FrameGeom& g, int xv0, int y0, int& qn, const FastParams& P,
                                         V2Smem& S, int warp, int lane, const V2Out& O) {
    // every queued group is classified; at most QCAP - 32 stay behind
    while (qn > 0) {
        const int take = min(qn, 32);
        if (lane < take) {
            const int e = S.q[warp][lane];
            v2_classify_group<R>(g, xv0, y0, y0 + (e >> 8), e & 255, P, S, warp, O);
        }
        const int rest = qn - take;
        int moved[QCAP / 32 - 1];
#pragma unroll
        for (int j = 0; j < QCAP / 32 - 1; ++j) moved[j] = (lane + 32 * j < rest) ? S.q[warp][32 + lane + 32 * j] : 0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < QCAP / 32 - 1; ++j)
            if (lane + 32 * j < rest) S.q[warp][lane + 32 * j] = moved[j];
        __syncwarp();
        qn = rest;
    }
}

template <int R>
__device__ __forceinline__ void v2_phase2(const FrameGeom& g, int xv0, int y0, const FastParams& P, V2Smem& S,
                                          int warp, int lane, const V2Out& O) {
    constexpr int HXA = V2Cfg<R>::HXA;
    constexpr int OW = V2Cfg<R>::OW;
    const int W = g.W, FH = g.full_H;
    const int oy0 = max(y0, g.out0), oy1 = min(y0 + V2_TH, g.out0 + g.rows);
    const int Ys = max(y0 + warp * V2_ROWS_PER_WARP, oy0);
    const int Ye = min(y0 + (warp + 1) * V2_ROWS_PER_WARP, oy1);
    if (Ys >= Ye) return;
    const bool edge = xv0 < 0 || xv0 + V2_COLS > W;
    const int c = xv0 + 4 * lane;
    // output lane: its 4 columns lie inside [x0, x0 + OW) and inside the frame
    const bool out_lane = lane >= HXA / 4 && lane < (HXA + OW) / 4 && c < W;
    const uint32_t fill = (uint32_t)P.cls0 * 0x01010101u;
    const float lo_lo = P.lo_lo;
    // label row pointer of the row being classified (advances one row per step)
    uint32_t* lab = reinterpret_cast<uint32_t*>(O.labels + O.out_base + (unsigned long long)(Ys - g.out0) * W + c);
    const int Wq = W >> 2;

    float d[3][4], s[3][4], mr[3][4];
    int qn = 0, qprev = 0;
    const int l = 4 * lane;
    // b rows jb = Ys-2 .. Ye+1 ; step index t = jb - (Ys-2)
    const int nsteps = Ye - Ys + 4;
    for (int t0 = 0; t0 < nsteps; t0 += 3) {
#pragma unroll
        for (int ph = 0; ph < 3; ++ph) {
            const int t = t0 + ph;
            if (t >= nsteps) break;
            const int jb = Ys - 2 + t;
            const float* brow = S.b[clampi(jb, 0, FH - 1) - (y0 - 2)];
            const float4 bb = *reinterpret_cast<const float4*>(brow + l);
            // neighbour lanes' edge columns (lane 0 / 31 get their own values:
            // only columns no output depends on are affected)
            const float bl = __shfl_up_sync(0xffffffffu, bb.w, 1);
            const float br = __shfl_down_sync(0xffffffffu, bb.x, 1);
            d[ph][0] = bb.y - bl;
            d[ph][1] = bb.z - bb.x;
            d[ph][2] = bb.w - bb.y;
            d[ph][3] = br - bb.z;
            s[ph][0] = fmaf(2.f, bb.x, bl + bb.y);
            s[ph][1] = fmaf(2.f, bb.y, bb.x + bb.z);
            s[ph][2] = fmaf(2.f, bb.z, bb.y + bb.w);
            s[ph][3] = fmaf(2.f, bb.w, bb.z + br);
            const int Ym = jb - 1;
            if (t >= 2) {
                // magnitude row Ym from rows jb-2 (ph+1 mod 3), jb-1 (ph+2 mod 3), jb (ph)
                const int pu = (ph + 1) % 3, pm = (ph + 2) % 3;
                float m4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float gx = fmaf(2.f, d[pm][k], d[pu][k] + d[ph][k]);
                    float gy = s[ph][k] - s[pu][k];
                    m4[k] = sqrt_apx(fmaf(gx, gx, gy * gy));
                }
                if (edge) edge_fix(m4, xv0, lane, W);
#pragma unroll
                for (int k = 0; k < 4; ++k) mr[ph][k] = m4[k];
                if (Ym >= 0 && Ym < FH) {
                    const float4 mv = make_float4(m4[0], m4[1], m4[2], m4[3]);
                    *reinterpret_cast<float4*>(&S.m[warp][mslot(Ym)][l]) = mv;
                    if (Ym == 0) *reinterpret_cast<float4*>(&S.m[warp][mslot(-1)][l]) = mv;
                    if (Ym == FH - 1) *reinterpret_cast<float4*>(&S.m[warp][mslot(FH)][l]) = mv;
                }
            }
            if (t >= 4) {
                // row Yc = jb - 2: its magnitudes were produced one step ago
                const int Yc = jb - 2;
                const int pp = (ph + 2) % 3;
                bool cand = false;
                if (out_lane) {
                    cand = fmaxf(fmaxf(mr[pp][0], mr[pp][1]), fmaxf(mr[pp][2], mr[pp][3])) >= lo_lo;
                    if (!cand) *lab = fill;
                }
                lab += Wq;
                const unsigned ballot = __ballot_sync(0xffffffffu, cand);
                if (cand) S.q[warp][qn + __popc(ballot & ((1u << lane) - 1u))] = ((Yc - y0) << 8) | lane;
                qn += __popc(ballot);
            }
        }
        // classify queued groups when 32 are waiting, when entries have already
        // waited one 3-step group (an entry for row Yc needs ring rows Yc-1..Yc+1;
        // the 8-row ring reuses the slot of Yc-1 at step jb = Yc+8, and two
        // groups after its enqueue step jb = Yc+2 is at most jb = Yc+7), or at the end
        if (qn >= 32 || qprev > 0 || t0 + 3 >= nsteps) {
            __syncwarp();
            v2_flush<R>(g, xv0, y0, qn, P, S, warp, lane, O);
        }
        qprev = qn;
    }
}

template <int R>
__global__ void __launch_bounds__(V2_THREADS)
k1v2_kernel(const uint8_t* __restrict__ src, FrameGeom g, FastParams P, uint8_t* __restrict__ labels,
            unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr) {
    extern __shared__ __align__(16) unsigned char smraw[];
    V2Smem& S = *reinterpret_cast<V2Smem*>(smraw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x0 = blockIdx.x * V2Cfg<R>::OW;
    const int xv0 = x0 - V2Cfg<R>::HXA;
    const int y0 = g.out0 + blockIdx.y * V2_TH;
    const uint8_t* img = src + (size_t)blockIdx.z * g.H * g.W;
    v2_phase1<R>(img, g, xv0, y0, P, S, warp, lane);
    __syncthreads();
    V2Out O{labels, (unsigned long long)blockIdx.z * g.rows * g.W, fix_list, hdr};
    v2_phase2<R>(g, xv0, y0, P, S, warp, lane, O);
}

bool k1v2_supported(const FastParams& P, const FrameGeom& g) { return P.r >= 1 && P.r <= 4 && (g.W % 4) == 0; }

template <int R>
static cudaError_t launch_r(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                            uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st) {
    const int smem = (int)sizeof(V2Smem);
    cudaError_t e = cudaFuncSetAttribute(k1v2_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.W + V2Cfg<R>::OW - 1) / V2Cfg<R>::OW, (g.rows + V2_TH - 1) / V2_TH, (unsigned)batch);
    k1v2_kernel<R><<<grid, V2_THREADS, smem, st>>>(src, g, P, labels, fix_list, hdr);
    return cudaGetLastError();
}

cudaError_t launch_k1v2(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st) {
    switch (P.r) {
        case 1: return launch_r<1>(src, batch, g, P, labels, fix_list, hdr, st);
        case 2: return launch_r<2>(src, batch, g, P, labels, fix_list, hdr, st);
        case 3: return launch_r<3>(src, batch, g, P, labels, fix_list, hdr, st);
        case 4: return launch_r<4>(src, batch, g, P, labels, fix_list, hdr, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace ef
