// ef_stages.cu -- stage-level kernels behind the reference's stage functions
// (exact float64, reference semantics).  These serve the drop-in stage API
// (non_max_suppress on an arbitrary GradientField, double_threshold on an
// arbitrary ThinnedField, quantize_orientation_array, the Laplacian operator);
// the fused path does not use them.
#include "ef_common.cuh"
#include "ef_internal.h"

namespace ef {

// nms.py:36-55 on given magnitude/orientation arrays (orientation in degrees).
__global__ void nms_kernel(const double* __restrict__ mag, const int64_t* __restrict__ ori, int H, int W,
                           double* __restrict__ thin, int* bad) {
    long long n = (long long)H * W;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int y = (int)(i / W), x = (int)(i - (long long)y * W);
        int64_t o = ori[i];
        int s = o == 0 ? 0 : (o == 45 ? 1 : (o == 90 ? 2 : (o == 135 ? 3 : -1)));
        double c = mag[i];
        if (s < 0) {  // the reference matches no direction: keep stays False
            thin[i] = 0.0;
            atomicExch(bad, 1);
            continue;
        }
        int dy1, dx1, dy2, dx2;
        nb_offsets(s, dy1, dx1, dy2, dx2);
        double n1 = mag[(long long)clampi(y + dy1, 0, H - 1) * W + clampi(x + dx1, 0, W - 1)];
        double n2 = mag[(long long)clampi(y + dy2, 0, H - 1) * W + clampi(x + dx2, 0, W - 1)];
        thin[i] = (c >= n1 && c >= n2) ? c : 0.0;
    }
}

// hysteresis.py:54-60
__global__ void threshold_kernel(const double* __restrict__ thin, long long n, double low, double high,
                                 uint8_t* __restrict__ labels) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        labels[i] = classify_exact(thin[i], low, high);
}

// gradient.py:37-44 on arbitrary float64 pairs
__global__ void quantize_kernel(const double* __restrict__ gx, const double* __restrict__ gy, long long n,
                                int64_t* __restrict__ ori) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        ori[i] = (int64_t)exact_sector(gx[i], gy[i], nullptr) * 45;
}

// gradient.py:93-107: 5-point Laplacian, replicate borders, taps in row-major
// order (0,1)+1 (1,0)+1 (1,1)-4 (1,2)+1 (2,1)+1 from +0.0.
__global__ void laplacian_kernel(const double* __restrict__ src, int H, int W, double* __restrict__ out) {
    long long n = (long long)H * W;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int y = (int)(i / W), x = (int)(i - (long long)y * W);
        auto P = [&](int yy, int xx) { return src[(long long)clampi(yy, 0, H - 1) * W + clampi(xx, 0, W - 1)]; };
        double a = 0.0;
        a = __dadd_rn(a, P(y - 1, x));
        a = __dadd_rn(a, P(y, x - 1));
        a = __dadd_rn(a, __dmul_rn(-4.0, P(y, x)));
        a = __dadd_rn(a, P(y, x + 1));
        a = __dadd_rn(a, P(y + 1, x));
        out[i] = a;
    }
}

static unsigned grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 65535 * 4 ? 65535 * 4 : b));
}

cudaError_t launch_nms(const double* mag, const int64_t* ori, int H, int W, double* thin, int* bad, cudaStream_t st) {
    nms_kernel<<<grid_for((long long)H * W), 256, 0, st>>>(mag, ori, H, W, thin, bad);
    return cudaGetLastError();
}
cudaError_t launch_threshold(const double* thin, long long n, double low, double high, uint8_t* labels,
                             cudaStream_t st) {
    threshold_kernel<<<grid_for(n), 256, 0, st>>>(thin, n, low, high, labels);
    return cudaGetLastError();
}
cudaError_t launch_quantize(const double* gx, const double* gy, long long n, int64_t* ori, cudaStream_t st) {
    quantize_kernel<<<grid_for(n), 256, 0, st>>>(gx, gy, n, ori);
    return cudaGetLastError();
}
cudaError_t launch_laplacian(const double* src, int H, int W, double* out, cudaStream_t st) {
    laplacian_kernel<<<grid_for((long long)H * W), 256, 0, st>>>(src, H, W, out);
    return cudaGetLastError();
}

}  // namespace ef
