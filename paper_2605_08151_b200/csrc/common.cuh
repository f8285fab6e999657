// common.cuh — error plumbing shared by every translation unit of libspectre.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/spectre.h"

namespace spectre {

void set_last_error(const std::string& msg);

inline int cuda_fail(cudaError_t e, const char* what) {
  set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SPECTRE_ECUDA;
}

inline int arg_fail(const char* what) {
  set_last_error(std::string("invalid argument: ") + what);
  return SPECTRE_EINVAL;
}

}  // namespace spectre

#define SPECTRE_CUDA_TRY(expr)                                        \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) return ::spectre::cuda_fail(_e, #expr);    \
  } while (0)

#define SPECTRE_LAUNCH_CHECK(name)                                    \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::spectre::cuda_fail(_e, name);     \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

namespace spectre {

// Programmatic dependent launch: the kernel may start (prologue, weight
// prefetch) while its predecessor drains; it must call pdl_wait() before
// touching any buffer a previous kernel writes or reads.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();

// Every kernel uses the same (maximum) shared-memory carveout so consecutive
// kernels never force an L1/shared reconfiguration of the SMs.
cudaError_t ensure_carveout(const void* kern);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  if (cudaError_t e = ensure_carveout(reinterpret_cast<const void*>(kern))) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// PDL launch of a kernel in clusters of `cluster_x` CTAs (CTA pairs).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t s, int cluster_x, Args... args) {
  if (cudaError_t e = ensure_carveout(reinterpret_cast<const void*>(kern))) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace spectre

#define SPECTRE_LAUNCH_PDL(name, ...)                                  \
  do {                                                                 \
    cudaError_t _e = ::spectre::launch_pdl(__VA_ARGS__);               \
    if (_e != cudaSuccess) return ::spectre::cuda_fail(_e, name);      \
  } while (0)
