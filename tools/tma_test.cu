// Minimal TMA probe: 3-D u8 map, 128 x ROWS box into shared memory, copy back.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cstdlib>

constexpr int ROWS = 40;
struct __align__(128) Sm { unsigned char in[48][128]; unsigned long long mbar; };

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, unsigned char* out, int x, int y, int z) {
    __shared__ Sm S;
    const unsigned bar = smem_u32(&S.mbar);
    const void* desc = (VARIANT == 2) ? (const void*)gmap : (const void*)&tmap;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        if (VARIANT == 0 || VARIANT == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ROWS * 128) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
                "r"(smem_u32(&S.in[0][0])), "l"(desc), "r"(x), "r"(y), "r"(z), "r"(bar)
            : "memory");
    }
    unsigned done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar) : "memory");
    }
    for (int i = threadIdx.x; i < ROWS * 128; i += blockDim.x) out[i] = S.in[i / 128][i % 128];
}

int main() {
    const int W = 512, H = 512, B = 1;
    std::vector<unsigned char> h(W * H * B);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 7 + (i / W) * 3);
    unsigned char *d, *o;
    cudaMalloc(&d, h.size());
    cudaMalloc(&o, ROWS * 128);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    printf("encoder %p q=%d\n", fnp, (int)q);
    CUtensorMap tm;
    memset(&tm, 0, sizeof tm);
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)W, (cuuint64_t)W * H};
    cuuint32_t box[3] = {128, ROWS, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    CUtensorMap* gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &tm, sizeof tm, cudaMemcpyHostToDevice);
    int which = getenv("V") ? atoi(getenv("V")) : 0;
    for (int variant = which; variant <= which; ++variant) {
        cudaMemset(o, 0, ROWS * 128);
        if (variant == 0) probe<0><<<1, 128>>>(tm, gm, o, 100, 37, 0);
        else if (variant == 1) probe<1><<<1, 128>>>(tm, gm, o, 100, 37, 0);
        else probe<2><<<1, 128>>>(tm, gm, o, 100, 37, 0);
        cudaError_t e = cudaDeviceSynchronize();
        printf("variant %d: %s\n", variant, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<unsigned char> got(ROWS * 128);
        cudaMemcpy(got.data(), o, got.size(), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int rr = 0; rr < ROWS; ++rr)
            for (int c = 0; c < 128; ++c) bad += got[rr * 128 + c] != h[(37 + rr) * W + 100 + c];
        printf("variant %d mismatches %d\n", variant, bad);
    }
    return 0;
}
