#include <algorithm>
// ef_exact.cu -- exact float64 kernels in the reference's operation order.
//
//  ex_tile_kernel   full-frame exact pipeline on a tile (u8 or float64 input):
//                   labels and, optionally, every intermediate array
//                   (keep_intermediates) and the thinned-field maximum
//                   (auto_thresholds).  Replaces gaussian_blur
//                   (filtering.py:66-91), sobel (gradient.py:73-90),
//                   non_max_suppress (nms.py:36-55), double_threshold
//                   (hysteresis.py:54-60) for float64 inputs.
//  fix_kernel       recomputes, one warp per pixel, the label of every pixel
//                   the fp32 fast path could not certify.
//
// Borders: the reference pads every stage's output with np.pad(mode="edge")
// before the next stage reads it (filtering.py:51,82; gradient.py:77;
// nms.py:41).  Here every stage is computed only at in-image positions and
// every read of the previous stage clamps its coordinates into the image.
#include "ef_common.cuh"
#include "ef_internal.h"
#include "ef_launch.cuh"

namespace ef {

constexpr int EX_TH = 32, EX_TW = 32, EX_THREADS = 256;

size_t ex_smem_bytes(int r) {
    int R = r + 2;
    size_t in = (size_t)(EX_TH + 2 * R) * (EX_TW + 2 * R);
    size_t h = (size_t)(EX_TH + 2 * R) * (EX_TW + 4);
    size_t b = (size_t)(EX_TH + 4) * (EX_TW + 4);
    size_t m = (size_t)(EX_TH + 2) * (EX_TW + 2);
    return (in + h + b + m) * sizeof(double);
}

template <typename In>
__global__ void __launch_bounds__(EX_THREADS)
ex_tile_kernel(const In* __restrict__ src, int H, int W, ExactParams P, uint8_t* __restrict__ labels,
               double* blurred, double* gxo, double* gyo, double* mago, int64_t* orio, double* thino,
               unsigned long long* max_bits, WsHeader* hdr) {
    extern __shared__ double sm[];
    const int r = P.r, R = r + 2;
    const int x0 = blockIdx.x * EX_TW, y0 = blockIdx.y * EX_TH;
    const size_t fbase = (size_t)blockIdx.z * H * W;
    const In* img = src + fbase;
    const int inW = EX_TW + 2 * R, inH = EX_TH + 2 * R;
    const int hW = EX_TW + 4, bW = EX_TW + 4, bH = EX_TH + 4, mW = EX_TW + 2, mH = EX_TH + 2;
    double* s_in = sm;
    double* s_h = s_in + inH * inW;
    double* s_b = s_h + inH * hW;
    double* s_m = s_b + bH * bW;
    const int tid = threadIdx.x;

    // 1. input with replicate borders (image.py:53-57 sample_pixel_clamped)
    for (int i = tid; i < inH * inW; i += EX_THREADS) {
        int ly = i / inW, lx = i - ly * inW;
        int Y = clampi(y0 - R + ly, 0, H - 1), X = clampi(x0 - R + lx, 0, W - 1);
        s_in[i] = load_px(img + (size_t)Y * W + X);
    }
    __syncthreads();
    // 2. horizontal pass, filtering.py:52-54: out = w0*p[x-r]; out += w_i*p[x-r+i]
    for (int i = tid; i < inH * hW; i += EX_THREADS) {
        int ly = i / hW, lx = i - ly * hW;
        int X = x0 - 2 + lx;
        if (X < 0 || X >= W) continue;
        const double* row = s_in + ly * inW + lx;  // column of p[X - r]
        double acc = __dmul_rn(P.w[0], row[0]);
        for (int k = 1; k <= 2 * r; ++k) acc = __dadd_rn(acc, __dmul_rn(P.w[k], row[k]));
        s_h[i] = acc;
    }
    __syncthreads();
    // 3. vertical pass, filtering.py:60-62 (rows of h outside the image already
    //    hold the clamped row: the input rows were clamped)
    for (int i = tid; i < bH * bW; i += EX_THREADS) {
        int ly = i / bW, lx = i - ly * bW;
        int Y = y0 - 2 + ly, X = x0 - 2 + lx;
        if (Y < 0 || Y >= H || X < 0 || X >= W) continue;
        const double* col = s_h + ly * hW + lx;  // row Y - r sits at local row ly
        double acc = __dmul_rn(P.w[0], col[0]);
        for (int k = 1; k <= 2 * r; ++k) acc = __dadd_rn(acc, __dmul_rn(P.w[k], col[k * hW]));
        s_b[i] = acc;
        if (blurred && ly >= 2 && ly < 2 + EX_TH && lx >= 2 && lx < 2 + EX_TW)
            blurred[fbase + (size_t)Y * W + X] = acc;
    }
    __syncthreads();
    auto B = [&](int Y, int X) -> double {
        return s_b[(clampi(Y, 0, H - 1) - (y0 - 2)) * bW + (clampi(X, 0, W - 1) - (x0 - 2))];
    };
    // 4. magnitude on [y0-1, y0+TH+1) x [x0-1, x0+TW+1)
    for (int i = tid; i < mH * mW; i += EX_THREADS) {
        int ly = i / mW, lx = i - ly * mW;
        int Y = y0 - 1 + ly, X = x0 - 1 + lx;
        if (Y < 0 || Y >= H || X < 0 || X >= W) continue;
        double blk[3][3];
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) blk[dy][dx] = B(Y + dy - 1, X + dx - 1);
        double gx, gy;
        exact_sobel(blk, gx, gy);
        s_m[i] = exact_mag(gx, gy);
    }
    __syncthreads();
    auto M = [&](int Y, int X) -> double {
        return s_m[(clampi(Y, 0, H - 1) - (y0 - 1)) * mW + (clampi(X, 0, W - 1) - (x0 - 1))];
    };
    // 5. orientation, NMS (nms.py:44-52), threshold (hysteresis.py:57-59)
    double local_max = 0.0;
    for (int i = tid; i < EX_TH * EX_TW; i += EX_THREADS) {
        int ly = i / EX_TW, lx = i - ly * EX_TW;
        int Y = y0 + ly, X = x0 + lx;
        if (Y >= H || X >= W) continue;
        double blk[3][3];
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) blk[dy][dx] = B(Y + dy - 1, X + dx - 1);
        double gx, gy;
        exact_sobel(blk, gx, gy);
        int s = exact_sector(gx, gy, hdr ? (unsigned long long*)&hdr->stats.ambiguous : nullptr);
        int dy1, dx1, dy2, dx2;
        nb_offsets(s, dy1, dx1, dy2, dx2);
        double c = M(Y, X);
        double t = (c >= M(Y + dy1, X + dx1) && c >= M(Y + dy2, X + dx2)) ? c : 0.0;
        size_t o = fbase + (size_t)Y * W + X;
        if (labels) labels[o] = classify_exact(t, P.low, P.high);
        if (gxo) gxo[o] = gx;
        if (gyo) gyo[o] = gy;
        if (mago) mago[o] = c;
        if (orio) orio[o] = (int64_t)s * 45;
        if (thino) thino[o] = t;
        local_max = fmax(local_max, t);
    }
    if (max_bits) {
        // thinned values are >= 0, so their bit patterns order like integers
        unsigned long long bits = (unsigned long long)__double_as_longlong(local_max);
        for (int off = 16; off > 0; off >>= 1) {
            unsigned long long o = __shfl_down_sync(0xffffffffu, bits, off);
            bits = o > bits ? o : bits;
        }
        if ((tid & 31) == 0) atomicMax(max_bits, bits);
    }
}

// ---------------------------------------------------------------------------
// Fix-up: exact label of one pixel, one warp per pixel.
// b is needed on the 5x5 block around the pixel (clamped), h on the rows
// clamp(y-2-r) .. clamp(y+2+r) x the 5 clamped columns.
// ---------------------------------------------------------------------------
constexpr int FX_WARPS = 4;


// One fix-up by a group of G lanes (G = 16: two pixels per warp in flight);
// gl = lane within the group, gm = the group's lane mask.
template <bool PEER, int G>
__device__ void fix_pixel_group(const uint8_t* __restrict__ img, const FrameGeom& g, int y, int x,
                                const ExactParams& P, uint8_t* s_in, double* s_h, double* s_b, double* s_m,
                                uint8_t* out, unsigned long long* ambiguous, int gl, unsigned gm) {
    const int lane = gl;
    const int r = P.r, H = g.full_H, W = g.W;
    const int hy0 = clampi(y - 2 - r, 0, H - 1), hy1 = clampi(y + 2 + r, 0, H - 1);
    const int nhr = hy1 - hy0 + 1;
    // the input window, staged with every load of a batch issued before any is
    // stored (one L2 round trip per 8 bytes a lane needs, instead of one per
    // tap of a dependent multiply-add chain): rows [hy0, hy1], columns [c0, c1]
    // = every column clamp(clamp(x - 2 + i) - r + j) can name
    const int c0 = max(0, clampi(x - 2, 0, W - 1) - r), c1 = min(W - 1, clampi(x + 2, 0, W - 1) + r);
    const int ncols = c1 - c0 + 1, nwin = nhr * ncols;
    for (int base = 0; base < nwin; base += 8 * G) {
        uint8_t v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = base + q * G + lane;
            const int row = k / ncols;
            v[q] = k < nwin ? frame_row<PEER>(img, g, hy0 + row)[c0 + (k - row * ncols)] : 0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = base + q * G + lane;
            if (k < nwin) s_in[k] = v[q];
        }
    }
    __syncwarp(gm);
    // h(Y', clamp(x - 2 + i)) for Y' in [hy0, hy1], i in 0..4  (filtering.py:52-54)
    for (int k = lane; k < nhr * 5; k += G) {
        int row = k / 5, i = k - row * 5;
        int X = clampi(x - 2 + i, 0, W - 1);
        const uint8_t* p = s_in + row * ncols - c0;  // p[c] = input(hy0 + row, c) for c in [c0, c1]
        double acc = __dmul_rn(P.w[0], (double)p[clampi(X - r, 0, W - 1)]);
        for (int j = 1; j <= 2 * r; ++j)
            acc = __dadd_rn(acc, __dmul_rn(P.w[j], (double)p[clampi(X - r + j, 0, W - 1)]));
        s_h[k] = acc;
    }
    __syncwarp(gm);
    // b(y - 2 + j, x - 2 + i) for in-frame positions  (filtering.py:60-62)
    for (int q = lane; q < 25; q += G) {
        int j = q / 5, i = q - j * 5;
        int Y = y - 2 + j, X = x - 2 + i;
        if (Y >= 0 && Y < H && X >= 0 && X < W) {
            double acc = __dmul_rn(P.w[0], s_h[(clampi(Y - r, 0, H - 1) - hy0) * 5 + i]);
            for (int k = 1; k <= 2 * r; ++k)
                acc = __dadd_rn(acc, __dmul_rn(P.w[k], s_h[(clampi(Y - r + k, 0, H - 1) - hy0) * 5 + i]));
            s_b[j * 5 + i] = acc;
        }
    }
    __syncwarp(gm);
    auto Bv = [&](int Y, int X) {
        return s_b[(clampi(Y, 0, H - 1) - (y - 2)) * 5 + (clampi(X, 0, W - 1) - (x - 2))];
    };
    auto grad = [&](int Y, int X, double& gx, double& gy) {
        double blk[3][3];
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) blk[dy][dx] = Bv(Y + dy - 1, X + dx - 1);
        exact_sobel(blk, gx, gy);
    };
    // lanes 0..8: gradient magnitude at the 3x3 positions around the pixel
    // (clamped), in parallel -- the NMS needs the centre and two of them
    for (int q = lane; q < 9; q += G) {
        const int dy = q / 3 - 1, dx = q % 3 - 1;
        double gx, gy;
        grad(clampi(y + dy, 0, H - 1), clampi(x + dx, 0, W - 1), gx, gy);
        s_m[q] = exact_mag(gx, gy);
        if (q == 4) {
            s_m[9] = gx;
            s_m[10] = gy;
        }
    }
    __syncwarp(gm);
    if (lane == 0) {
        const double c = s_m[4];
        const int s = exact_sector(s_m[9], s_m[10], ambiguous);
        int dy1, dx1, dy2, dx2;
        nb_offsets(s, dy1, dx1, dy2, dx2);
        const double m1 = s_m[(dy1 + 1) * 3 + (dx1 + 1)], m2 = s_m[(dy2 + 1) * 3 + (dx2 + 1)];
        const double t = (c >= m1 && c >= m2) ? c : 0.0;
        *out = classify_exact(t, P.low, P.high);  // nms.py:51-52, hysteresis.py:57-59
    }
    __syncwarp(gm);
}

// output index -> (frame, global row, column)
__device__ __forceinline__ void out_coords(unsigned long long idx, const FrameGeom& g, unsigned long long& f,
                                           int& y, int& x) {
    unsigned long long per = (unsigned long long)g.rows * g.W;
    f = idx / per;
    unsigned long long rem = idx - f * per;
    int yo = (int)(rem / g.W);
    x = (int)(rem - (unsigned long long)yo * g.W);
    y = g.out0 + yo;
    EF_DCHECK(yo >= 0 && yo < g.rows && x >= 0 && x < g.W);
}

// the fused pipeline's foreground bit planes for a fixed pixel
__device__ __forceinline__ void fix_bits(const FgBits& B, const FrameGeom& g, unsigned long long f, int y, int x,
                                         uint8_t lab, uint8_t* lab_ptr, int gl) {
    if (!B.fg || gl != 0) return;
    lab_ptr[B.fin_off] = lab == 2 ? 1 : 0;  // final = strong (weak pixels are decided by the hysteresis)
    if (lab != 1 && lab != 2) return;
    const unsigned long long w = f * B.frame_words + (unsigned long long)(y - g.out0) * B.words + (unsigned)(x >> 6);
    atomicOr(&B.fg[w], 1ull << (x & 63));
    if (lab == 2) atomicOr(&B.st[w], 1ull << (x & 63));
}

// Fix-ups: every flagged pixel recomputed exactly by a group of 16 lanes (two
// pixels per warp in flight: the f64 chain per pixel is latency-bound).  The
// normal case walks K1's fix list; when the list overflowed, the same launch
// scans every label byte for flags instead (one kernel either way: a separate
// always-launched fallback kernel cost a ~3 us slot in the PDL chain).
// Dynamic shared memory: per group the input window, h, b and m, sized by r.
#ifndef EF_FX_G
#define EF_FX_G 16
#endif
constexpr int FX_G = EF_FX_G;  // lanes per fix-up
constexpr int FX_GROUPS = FX_WARPS * 32 / FX_G;

__host__ __device__ inline int fx_group_bytes(int r) {
    const int side = 2 * r + 5;
    return 8 * (side * 5 + 25 + 11) + ((side * side + 7) & ~7);
}

template <bool PEER>
__global__ void __launch_bounds__(FX_WARPS * 32)
fix_kernel(const uint8_t* __restrict__ src, int64_t batch, FrameGeom g, ExactParams P, uint8_t* labels,
           const unsigned long long* __restrict__ list, WsHeader* hdr, FgBits B) {
    extern __shared__ __align__(16) unsigned char fx_smem[];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int grp = threadIdx.x / FX_G, gl = lane & (FX_G - 1);
    const unsigned gm = (FX_G == 32 ? 0xffffffffu : ((1u << FX_G) - 1u)) << (lane & ~(FX_G - 1));
    const int side = 2 * P.r + 5;
    unsigned char* base = fx_smem + (size_t)grp * fx_group_bytes(P.r);
    double* s_h = reinterpret_cast<double*>(base);
    double* s_b = s_h + side * 5;
    double* s_m = s_b + 25;
    uint8_t* s_in = reinterpret_cast<uint8_t*>(s_m + 11);
    auto fix_one = [&](unsigned long long idx) {
        unsigned long long f;
        int y, x;
        out_coords(idx, g, f, y, x);
        fix_pixel_group<PEER, FX_G>(src + f * (unsigned long long)g.H * g.W, g, y, x, P, s_in, s_h, s_b, s_m,
                                    labels + idx, (unsigned long long*)&hdr->stats.ambiguous, gl, gm);
        fix_bits(B, g, f, y, x, labels[idx], labels + idx, gl);
    };
    if (!hdr->overflow) {
        const unsigned long long n = hdr->fix_count;  // <= fix_cap without overflow
        for (unsigned long long e = (unsigned long long)blockIdx.x * FX_GROUPS + grp; e < n;
             e += (unsigned long long)gridDim.x * FX_GROUPS)
            fix_one(list[e]);
    } else {
        // overflow: the list is incomplete; scan every label byte (a warp
        // ballots 32 bytes, its groups take the flagged ones in turn)
        const int warp = threadIdx.x >> 5, sub = lane / FX_G;
        const unsigned long long total = (unsigned long long)batch * g.rows * g.W;
        for (unsigned long long b0 = ((unsigned long long)blockIdx.x * FX_WARPS + warp) * 32; b0 < total;
             b0 += (unsigned long long)gridDim.x * FX_WARPS * 32) {
            const unsigned long long idx = b0 + lane;
            const bool flagged = idx < total && (labels[idx] & kFlag);
            unsigned mask = __ballot_sync(0xffffffffu, flagged);
            while (mask) {  // warp-uniform: one flagged byte per group per round
                int mine = -1;
#pragma unroll
                for (int k = 0; k < 32 / FX_G; ++k) {
                    const int l = mask ? __ffs(mask) - 1 : -1;
                    if (mask) mask &= mask - 1;
                    if (k == sub) mine = l;
                }
                if (mine >= 0) fix_one(b0 + mine);
                __syncwarp();
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long*)&hdr->stats.fixups, hdr->fix_count);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename In>
cudaError_t launch_exact(const In* src, int64_t batch, int H, int W, const ExactParams& P,
                         uint8_t* labels, double* blurred, double* gx, double* gy, double* mag,
                         int64_t* ori, double* thin, unsigned long long* max_bits, WsHeader* hdr,
                         cudaStream_t st) {
    size_t smem = ex_smem_bytes(P.r);
    auto kern = ex_tile_kernel<In>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((W + EX_TW - 1) / EX_TW, (H + EX_TH - 1) / EX_TH, (unsigned)batch);
    kern<<<grid, EX_THREADS, smem, st>>>(src, H, W, P, labels, blurred, gx, gy, mag, ori, thin,
                                         max_bits, hdr);
    return cudaGetLastError();
}

template cudaError_t launch_exact<uint8_t>(const uint8_t*, int64_t, int, int, const ExactParams&,
                                           uint8_t*, double*, double*, double*, double*, int64_t*,
                                           double*, unsigned long long*, WsHeader*, cudaStream_t);
template cudaError_t launch_exact<double>(const double*, int64_t, int, int, const ExactParams&,
                                          uint8_t*, double*, double*, double*, double*, int64_t*,
                                          double*, unsigned long long*, WsHeader*, cudaStream_t);

cudaError_t launch_fix(const uint8_t* src, int64_t batch, const FrameGeom& g, const ExactParams& P,
                       uint8_t* labels, const unsigned long long* list, WsHeader* hdr, const FgBits& B,
                       int sm_count, cudaStream_t st) {
    auto kern = (g.top || g.bot) ? fix_kernel<true> : fix_kernel<false>;
    const size_t smem = (size_t)FX_GROUPS * fx_group_bytes(P.r);
    // small launches get a small grid (the kernel grid-strides over the list, or
    // over every pixel when the list overflowed): 2368 mostly idle blocks cost
    // a 512x512 frame ~5 us
    const long long px = batch * (long long)g.rows * g.W;
    const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((long long)sm_count * 16, px / 4096));
    return launch_pdl(kern, dim3(blocks), dim3(FX_WARPS * 32), smem, st, src, batch, g, P, labels, list, hdr, B);
}

}  // namespace ef
