// Narrow down: (A) mbarrier alone, (B) 1-D bulk copy, (C) 2-D tensor map, (D) 3-D tensor map
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

struct __align__(128) Sm { unsigned char in[48][128]; unsigned long long mbar; };
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ void wait_bar(unsigned bar) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar) : "memory");
}

template <int V>
__global__ void probe(const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
                      const unsigned char* src, unsigned char* out, int x, int y) {
    __shared__ Sm S;
    const unsigned bar = smem_u32(&S.mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (V == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
        } else if (V == 1) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(1024) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                             "r"(smem_u32(&S.in[0][0])), "l"(src), "r"(1024), "r"(bar) : "memory");
        } else if (V == 2) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(40 * 128) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                             "r"(smem_u32(&S.in[0][0])), "l"(&tm2), "r"(x), "r"(y), "r"(bar) : "memory");
        } else {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(40 * 128) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                             "r"(smem_u32(&S.in[0][0])), "l"(&tm3), "r"(x), "r"(y), "r"(0), "r"(bar) : "memory");
        }
    }
    wait_bar(bar);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = S.in[i / 128][i % 128];
}

int main() {
    const int W = 512, H = 512;
    std::vector<unsigned char> h(W * H);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 7 + (i / W) * 3);
    unsigned char *d, *o;
    cudaMalloc(&d, h.size());
    cudaMalloc(&o, 4096);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    CUtensorMap tm2, tm3;
    memset(&tm2, 0, sizeof tm2); memset(&tm3, 0, sizeof tm3);
    cuuint64_t d2[2] = {(cuuint64_t)W, (cuuint64_t)H}, s2[1] = {(cuuint64_t)W};
    cuuint32_t b2[2] = {128, 40}, e2[2] = {1, 1};
    printf("enc2 %d\n", (int)enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, (getenv("P") ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    cuuint64_t d3[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}, s3[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
    cuuint32_t b3[3] = {128, 40, 1}, e3[3] = {1, 1, 1};
    printf("enc3 %d\n", (int)enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, (getenv("P") ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    int v = atoi(getenv("V")); int X = atoi(getenv("X")), Y = atoi(getenv("Y"));
    if (v == 0) probe<0><<<1, 128>>>(tm2, tm3, d, o, X, Y);
    if (v == 1) probe<1><<<1, 128>>>(tm2, tm3, d, o, X, Y);
    if (v == 2) probe<2><<<1, 128>>>(tm2, tm3, d, o, X, Y);
    if (v == 3) probe<3><<<1, 128>>>(tm2, tm3, d, o, X, Y);
    printf("V=%d X=%d Y=%d P=%s: %s\n", v, X, Y, getenv("P")?"1":"0", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
