// ef_launch.cuh -- programmatic dependent launch (PDL) for the kernel chain of
// one fused call.
//
// ef_canny_u8 is ~10 dependent kernels on one stream; a plain launch waits for
// the previous grid to drain before the next one is even scheduled (~2-3 us per
// boundary, measured as the duration of the empty fallback kernels).  Launched
// with programmatic stream serialisation, a kernel's CTAs may be scheduled
// while its predecessor finishes; every kernel of the chain therefore calls
// pdl_wait() before touching anything a predecessor wrote (griddepcontrol.wait
// returns once all prerequisite grids have completed and their memory is
// visible), and pdl_trigger() to let its successor launch early.  Kernels
// launched without the attribute are unaffected by either instruction.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>

namespace ef {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = getenv("EF_NO_PDL") == nullptr;  // A/B switch
    return on;
}

// Function attributes are per device; set them once per (call site, device)
// instead of on every launch (each cudaFuncSetAttribute is a driver call).
// `done` is a per-call-site bit set of devices already configured.
template <typename F>
cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& set) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = set();
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace ef
