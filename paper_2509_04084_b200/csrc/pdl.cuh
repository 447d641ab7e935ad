// Programmatic dependent launch (sm_90+, used on sm_100a) for the short kernels of one iteration's
// chain (compress select/emit, merge).  A kernel launched with launch_pdl may be scheduled while its
// predecessor in the stream drains; every kernel of the chain calls pdl_wait() as its first
// statement, which blocks until the predecessor grid has completed and its writes are visible, so
// the overlap covers only launch and CTA scheduling, never data.  pdl_trigger() lets the successor
// be scheduled as soon as every CTA of this grid is resident.  Without a programmatic predecessor
// both are no-ops.  LOWDIFF_PDL=0 turns the launch attribute off (plain stream order).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace ld {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("LOWDIFF_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

// launch with the programmatic-serialization attribute when pdl, and the cooperative attribute
// (every CTA co-resident: grid barriers are safe) when coop
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_ex(bool pdl, bool coop, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl && pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (coop) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// kernel<<<grid, block, smem, s>>>(args...) with the programmatic-serialization attribute when pdl
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  return launch_pdl_ex(pdl, false, kernel, grid, block, smem, s, args...);
}

}  // namespace ld
