// abi.cu — library-wide C ABI plumbing: version string and per-thread error text.
#include <cstdlib>
#include <mutex>
#include <unordered_set>
#include <string>

#include "common.cuh"

namespace spectre {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

// SPECTRE_PDL=0 disables programmatic dependent launch (A/B measurements).
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("SPECTRE_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

cudaError_t ensure_carveout(const void* kern) {
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  static const bool on = [] {
    const char* v = getenv("SPECTRE_CARVEOUT");
    return !(v && v[0] == '0');
  }();
  if (!on) return cudaSuccess;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(kern)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done.insert(kern);
  return e;
}

}  // namespace spectre

extern "C" const char* spectre_version(void) { return "spectre-b200 0.1.0 sm_100a"; }

extern "C" const char* spectre_last_error(void) { return spectre::g_last_error.c_str(); }
