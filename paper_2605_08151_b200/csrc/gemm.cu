// gemm.cu — host side of the tcgen05 GEMM: TMA descriptors, planning, launch.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm.h"
#include "gemm_tcgen05.cuh"

namespace spectre {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static int get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_last_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return SPECTRE_ECUDA;
  }
  return SPECTRE_OK;
}

// [outer][inner] bf16 row-major, box_inner-element inner boxes swizzled to
// their byte span (64 el -> 128B swizzle, 32 el -> 64B swizzle).
int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                   uint32_t box_outer, uint32_t box_inner) {
  if (int e = get_encoder()) return e;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (inner * 2) % 16)
    return arg_fail("tensor map: 16-byte alignment");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_inner == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SPECTRE_ECUDA;
  }
  return SPECTRE_OK;
}

template <int kEpi, int BK>
static int launch_one(const GemmPlan& p, cudaStream_t s) {
  auto kern = gemm_bf16_swapab<kEpi, BK>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kGemmSmemBytes));
    configured = true;
  }
  SPECTRE_LAUNCH_PDL("gemm_bf16_swapab", kern, dim3(p.grid), dim3(kGemmThreads), kGemmSmemBytes, s,
                     p.tmap_w, p.tmap_x, p.args);
  return SPECTRE_OK;
}

int gemm_default_bk() {
  static const int bk = [] {
    const char* v = getenv("SPECTRE_GEMM_BK");
    return (v && atoi(v) == 32) ? 32 : 64;
  }();
  return bk;
}

int gemm_plan(GemmPlan* p, const void* W, int N, int K, const void* X, int rows_cap, int epi,
              int splits, int max_stages, int bk, int tile_rows) {
  if (tile_rows != 128) tile_rows = 256;
  if (bk == 0) bk = gemm_default_bk();
  if (bk != 32 && bk != 64) return arg_fail("gemm_plan: bk must be 32 or 64");
  if (N < 1 || K < 64 || K % 64 || rows_cap < 64 || rows_cap % 64 || splits < 1)
    return arg_fail("gemm_plan: shape (K % 64, rows_cap multiple of 64)");
  if (epi == kSwiGLU && (N % 128 || splits != 1)) return arg_fail("gemm_plan: swiglu shape");
  if (epi == kArgmax && splits != 1) return arg_fail("gemm_plan: argmax needs splits == 1");
  *p = GemmPlan{};
  if (int e = make_tmap_bf16(&p->tmap_w, W, (uint64_t)K, (uint64_t)N, 128, bk)) return e;
  if (int e = make_tmap_bf16(&p->tmap_x, X, (uint64_t)K, (uint64_t)rows_cap, 64, bk)) return e;
  p->bk = bk;
  const int n_tiles = (N + tile_rows - 1) / tile_rows;
  p->epi = epi;
  p->args.tile_rows = tile_rows;
  p->grid = n_tiles * splits;
  p->args.N = N;
  p->args.K = K;
  p->args.rows_cap = rows_cap;
  p->args.splits = splits;
  p->args.max_stages = max_stages;
  p->n_tiles = n_tiles;
  p->n_amax_blocks = (N + 31) / 32;
  return SPECTRE_OK;
}

int gemm_run(const GemmPlan& p, cudaStream_t s) {
  if (p.bk == 64) {
    switch (p.epi) {
      case kPartial: return launch_one<kPartial, 64>(p, s);
      case kArgmax: return launch_one<kArgmax, 64>(p, s);
      default: return launch_one<kSwiGLU, 64>(p, s);
    }
  }
  switch (p.epi) {
    case kPartial: return launch_one<kPartial, 32>(p, s);
    case kArgmax: return launch_one<kArgmax, 32>(p, s);
    default: return launch_one<kSwiGLU, 32>(p, s);
  }
}

}  // namespace spectre

using namespace spectre;

extern "C" int spectre_gemm_bf16(const void* X, const void* W, const int32_t* t_dev,
                                 int32_t t_static, int32_t rows_cap, int32_t N, int32_t K,
                                 int32_t splits, int32_t epilogue, float* partial,
                                 float* amax_val, int32_t* amax_idx, void* act, int32_t ld_act,
                                 int32_t max_stages, void* stream) {
  GemmPlan p;
  // test knobs: max_stages < 0 forces 32-wide K blocks; >= 1000 selects 128-row tiles
  const int tile_rows = max_stages >= 1000 ? 128 : 256;
  if (max_stages >= 1000) max_stages -= 1000;
  const int bk = max_stages < 0 ? 32 : 64;
  if (int e = gemm_plan(&p, W, N, K, X, rows_cap, epilogue, splits,
                        max_stages < 0 ? -max_stages : max_stages, bk, tile_rows))
    return e;
  p.args.t_dev = t_dev;
  p.args.t_static = t_static;
  p.args.part = partial;
  p.args.amax_val = amax_val;
  p.args.amax_idx = amax_idx;
  p.args.act = reinterpret_cast<__nv_bfloat16*>(act);
  p.args.ld_act = ld_act;
  return gemm_run(p, as_stream(stream));
}
