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
