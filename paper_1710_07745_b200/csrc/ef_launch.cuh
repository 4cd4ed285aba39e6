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

#include <cstdlib>
#include <utility>

namespace ef {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = getenv("EF_NO_PDL") == nullptr;  // A/B switch
    return on;
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
