// ef_fast.cu -- K1: fused Gaussian + Sobel + magnitude + sector + NMS +
// double threshold on u8 frames, fp32 with certified decisions.
//
// Replaces gaussian_blur (filtering.py:66-91), sobel (gradient.py:73-90),
// non_max_suppress (nms.py:36-55) and double_threshold (hysteresis.py:54-60)
// for integer-valued inputs.  Every decision (threshold class, orientation
// sector, the two NMS comparisons) is taken in fp32 only when its margin
// exceeds the certified bound in FastParams (derived in ef_abi.cu, see
// DESIGN.md); otherwise the label byte is marked kFlag and the pixel index is
// appended to the fix list for the exact float64 recompute (ef_exact.cu).
//
// v1 layout: one CTA per 32x64 output tile, each stage staged through shared
// memory (input with halo -> horizontal pass -> vertical pass -> magnitude ->
// classify).  Interior tiles take the BORDER=false instantiation (no clamps).
#include "ef_common.cuh"
#include "ef_internal.h"

#include <cstdlib>

namespace ef {

constexpr int K1_TH = 32, K1_TW = 64, K1_THREADS = 256;

size_t k1_smem_bytes(int r) {
    int R = r + 2;
    size_t in = (size_t)(K1_TH + 2 * R) * (K1_TW + 2 * R);
    size_t h = (size_t)(K1_TH + 2 * R) * (K1_TW + 4);
    size_t b = (size_t)(K1_TH + 4) * (K1_TW + 4);
    size_t m = (size_t)(K1_TH + 2) * (K1_TW + 2);
    return (in + h + b + m) * sizeof(float);
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <bool BORDER>
__device__ __forceinline__ void k1_tile(const uint8_t* __restrict__ img, const FrameGeom& g, int x0,
                                        int y0, const FastParams& P, uint8_t* __restrict__ out,
                                        unsigned long long out_base, unsigned long long* __restrict__ fix_list,
                                        WsHeader* __restrict__ hdr, float* smf) {
    const int r = P.r, R = r + 2;
    const int W = g.W, FH = g.full_H;
    const int inW = K1_TW + 2 * R, inH = K1_TH + 2 * R;
    const int hW = K1_TW + 4, bW = K1_TW + 4, bH = K1_TH + 4, mW = K1_TW + 2, mH = K1_TH + 2;
    float* s_in = smf;
    float* s_h = s_in + inH * inW;
    float* s_b = s_h + inH * hW;
    float* s_m = s_b + bH * bW;
    const int tid = threadIdx.x;
    const int yend = g.out0 + g.rows;  // first global row not classified by this launch

    auto cy = [&](int Y) { return BORDER ? clampi(Y, 0, FH - 1) : Y; };
    auto cx = [&](int X) { return BORDER ? clampi(X, 0, W - 1) : X; };

    // 1. u8 tile + halo -> fp32 (replicate borders against the whole frame)
    for (int i = tid; i < inH * inW; i += K1_THREADS) {
        int ly = i / inW, lx = i - ly * inW;
        int Yl = y0 - R + ly;
        if (BORDER) Yl = clampi(cy(Yl), g.g0, g.g0 + g.H - 1);  // rows past the band halo feed no output
        s_in[i] = (float)img[(size_t)(Yl - g.g0) * W + cx(x0 - R + lx)];
    }
    __syncthreads();
    // 2. horizontal pass, folded symmetric taps (rows outside the frame hold
    //    the clamped row already)
    for (int i = tid; i < inH * hW; i += K1_THREADS) {
        int ly = i / hW, lx = i - ly * hW;
        if (BORDER) {
            int X = x0 - 2 + lx;
            if (X < 0 || X >= W) continue;
        }
        const float* c = s_in + ly * inW + lx + r;  // centre tap
        float acc = P.wf[0] * c[0];
        for (int k = 1; k <= r; ++k) acc = fmaf(P.wf[k], c[-k] + c[k], acc);
        s_h[i] = acc;
    }
    __syncthreads();
    // 3. vertical pass
    for (int i = tid; i < bH * bW; i += K1_THREADS) {
        int ly = i / bW, lx = i - ly * bW;
        if (BORDER) {
            int Y = y0 - 2 + ly, X = x0 - 2 + lx;
            if (Y < 0 || Y >= FH || X < 0 || X >= W) continue;
        }
        const float* c = s_h + (ly + r) * hW + lx;
        float acc = P.wf[0] * c[0];
        for (int k = 1; k <= r; ++k) acc = fmaf(P.wf[k], c[-k * hW] + c[k * hW], acc);
        s_b[i] = acc;
    }
    __syncthreads();
    auto Bf = [&](int Y, int X) -> float { return s_b[(cy(Y) - (y0 - 2)) * bW + (cx(X) - (x0 - 2))]; };
    auto sob = [&](int Y, int X, float& gx, float& gy) {
        float dxu = Bf(Y - 1, X + 1) - Bf(Y - 1, X - 1);
        float dxm = Bf(Y, X + 1) - Bf(Y, X - 1);
        float dxd = Bf(Y + 1, X + 1) - Bf(Y + 1, X - 1);
        float su = fmaf(2.f, Bf(Y - 1, X), Bf(Y - 1, X - 1) + Bf(Y - 1, X + 1));
        float sd = fmaf(2.f, Bf(Y + 1, X), Bf(Y + 1, X - 1) + Bf(Y + 1, X + 1));
        gx = fmaf(2.f, dxm, dxu + dxd);
        gy = sd - su;
    };
    // 4. magnitude on [y0-1, y0+TH+1) x [x0-1, x0+TW+1)
    for (int i = tid; i < mH * mW; i += K1_THREADS) {
        int ly = i / mW, lx = i - ly * mW;
        int Y = y0 - 1 + ly, X = x0 - 1 + lx;
        if (BORDER && (Y < 0 || Y >= FH || X < 0 || X >= W)) continue;
        float gx, gy;
        sob(Y, X, gx, gy);
        s_m[i] = sqrt_approx(fmaf(gx, gx, gy * gy));
    }
    __syncthreads();
    auto Mf = [&](int Y, int X) -> float { return s_m[(cy(Y) - (y0 - 1)) * mW + (cx(X) - (x0 - 1))]; };
    // 5. classify with certification
    const float t1 = 0.41421356237309503f;
    for (int i = tid; i < K1_TH * K1_TW; i += K1_THREADS) {
        int ly = i / K1_TW, lx = i - ly * K1_TW;
        int Y = y0 + ly, X = x0 + lx;
        if (BORDER && (Y >= yend || X >= W)) continue;
        float c = Mf(Y, X);
        // class of c: 0/1/2, or -1 when not certified
        int cls;
        if (c > P.hi_hi) cls = 2;
        else if (c >= P.hi_lo) cls = -1;
        else if (c > P.lo_hi) cls = 1;
        else if (c >= P.lo_lo) cls = -1;
        else cls = 0;
        bool flag = cls < 0;
        uint8_t lab = (uint8_t)P.cls0;
        if (!flag && cls != P.cls0) {
            float gx, gy;
            sob(Y, X, gx, gy);
            float a = fabsf(gx), b = fabsf(gy);
            float u = fmaf(t1, a, -b), v = fmaf(t1, b, -a);
            if (fabsf(u) <= P.e_sec || fabsf(v) <= P.e_sec) {
                flag = true;
            } else {
                int s = u > 0.f ? 0 : (v > 0.f ? 2 : ((gx > 0.f) == (gy > 0.f) ? 1 : 3));
                int dy1, dx1, dy2, dx2;
                nb_offsets(s, dy1, dx1, dy2, dx2);
                float d1 = c - Mf(Y + dy1, X + dx1), d2 = c - Mf(Y + dy2, X + dx2);
                if (d1 < -P.e_nms || d2 < -P.e_nms) lab = (uint8_t)P.cls0;    // suppressed
                else if (d1 > P.e_nms && d2 > P.e_nms) lab = (uint8_t)cls;  // kept
                else flag = true;
            }
        }
        unsigned long long o = out_base + (unsigned long long)(Y - g.out0) * W + X;
        if (flag) {
            out[o] = kFlag;
            unsigned long long slot = atomicAdd(&hdr->fix_count, 1ull);
            if (slot < hdr->fix_cap) fix_list[slot] = o;
            else hdr->overflow = 1u;
        } else {
            out[o] = lab;
        }
    }
}

__global__ void __launch_bounds__(K1_THREADS)
k1_classify_kernel(const uint8_t* __restrict__ src, FrameGeom g, FastParams P, uint8_t* __restrict__ labels,
                   unsigned long long* __restrict__ fix_list, WsHeader* __restrict__ hdr) {
    extern __shared__ float smf[];
    const int R = P.r + 2;
    const int x0 = blockIdx.x * K1_TW, y0 = g.out0 + blockIdx.y * K1_TH;
    const uint8_t* img = src + (size_t)blockIdx.z * g.H * g.W;
    const unsigned long long out_base = (unsigned long long)blockIdx.z * g.rows * g.W;
    bool border = x0 - R < 0 || y0 - R < 0 || x0 + K1_TW + R > g.W || y0 + K1_TH + R > g.full_H ||
                  y0 + K1_TH > g.out0 + g.rows;
    if (border) k1_tile<true>(img, g, x0, y0, P, labels, out_base, fix_list, hdr, smf);
    else k1_tile<false>(img, g, x0, y0, P, labels, out_base, fix_list, hdr, smf);
}

cudaError_t launch_k1(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                      uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, const FgBits& B,
                      cudaStream_t st) {
    if (k1v2_supported(P, g)) return launch_k1v2(src, batch, g, P, labels, fix_list, hdr, B, st);
    return launch_k1v1(src, batch, g, P, labels, fix_list, hdr, st);
}

// bit planes need the production classifier and a zero background class (it
// writes bits for classified candidates only; with low == 0 every pixel is
// foreground)
bool k1_emits_bits(const FastParams& P, const FrameGeom& g) { return k1v2_supported(P, g) && P.cls0 == 0; }

cudaError_t launch_k1v1(const uint8_t* src, int64_t batch, const FrameGeom& g, const FastParams& P,
                        uint8_t* labels, unsigned long long* fix_list, WsHeader* hdr, cudaStream_t st) {
    size_t smem = k1_smem_bytes(P.r);
    cudaError_t e = cudaFuncSetAttribute(k1_classify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.W + K1_TW - 1) / K1_TW, (g.rows + K1_TH - 1) / K1_TH, (unsigned)batch);
    k1_classify_kernel<<<grid, K1_THREADS, smem, st>>>(src, g, P, labels, fix_list, hdr);
    return cudaGetLastError();
}

}  // namespace ef
