// Programmatic dependent launch (PDL).  Every kernel of the denoising step is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so kernel i+1 is scheduled while kernel i
// drains (its CTAs fill the SMs kernel i no longer uses, run their prologue -- barrier init,
// TMEM allocation, tensor-map prefetch, the first weight tiles -- and then block in
// griddepcontrol.wait until kernel i has completed and its writes are visible).
//   pdl_wait()    before the first read of data produced by an earlier kernel on the stream
//                 (and before the first global write: kernel i may still read that buffer)
//   pdl_trigger() lets the dependent grid launch once every CTA of this grid has called it
// Both are no-ops for a launch without the attribute.  PP_PDL=0 (or pp_set_pdl(0), a
// measurement control: kernels then run strictly back to back, so per-kernel device times
// from CUPTI carry no early-start wait) disables the attribute for later launches / captures.
#pragma once
#include "util.hpp"

#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <utility>

namespace pp {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline std::atomic<int>& pdl_flag() {
    static std::atomic<int> on{[] {
        const char* v = std::getenv("PP_PDL");
        return (v && v[0] == '0') ? 0 : 1;
    }()};
    return on;
}
inline bool pdl_enabled() { return pdl_flag().load(std::memory_order_relaxed) != 0; }

// kernel<<<grid, block, smem, stream>>>(args...) with the PDL attribute (and an optional
// cluster dimension).
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = unsigned(cluster_x);
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace pp
