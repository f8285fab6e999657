// abi.cu — library-wide C ABI plumbing: version string and per-thread error text.
#include <string>

#include "common.cuh"

namespace spectre {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace spectre

extern "C" const char* spectre_version(void) { return "spectre-b200 0.1.0 sm_100a"; }

extern "C" const char* spectre_last_error(void) { return spectre::g_last_error.c_str(); }
