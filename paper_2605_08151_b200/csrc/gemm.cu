// gemm.cu — host side of the tcgen05 GEMM: TMA descriptors, planning, launch.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>
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

static int num_sms_pub();

// 2-D fp32 / bf16 map for TMA stores: [outer][inner], box {box_inner, box_outer}, no swizzle.
static int make_tmap_store(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int esize,
                           uint64_t inner, uint64_t outer, uint32_t box_inner,
                           uint32_t box_outer) {
  if (int e = get_encoder()) return e;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled(store) failed: " + std::to_string((int)r));
    return SPECTRE_ECUDA;
  }
  return SPECTRE_OK;
}

int gemm_set_outputs(GemmPlan* p, float* part, float* amax_val, int* amax_idx, void* act,
                     int ld_act) {
  p->args.part = part;
  p->args.amax_val = amax_val;
  p->args.amax_idx = amax_idx;
  p->args.act = reinterpret_cast<__nv_bfloat16*>(act);
  p->args.ld_act = ld_act;
  if (p->epi == kPartial && part) {
    if ((p->args.N * 4) % 16) return arg_fail("gemm: partial rows must be 16-byte aligned");
    if (int e = make_tmap_store(&p->tmap_out, part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                (uint64_t)p->args.N,
                                (uint64_t)p->args.splits * p->args.rows_cap, 32, 16))
      return e;
  }
  if (p->epi == kSwiGLU && act) {
    if ((ld_act * 2) % 16) return arg_fail("gemm: act rows must be 16-byte aligned");
    if (int e = make_tmap_store(&p->tmap_out, act, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                (uint64_t)ld_act, (uint64_t)p->args.rows_cap, 16, 32))
      return e;
  }
  if (p->args.stream_k && p->args.sk_part) {
    if (int e = make_tmap_store(&p->tmap_sk, p->args.sk_part, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                256, (uint64_t)num_sms_pub() * 256, 128, 16))
      return e;
  }
  return SPECTRE_OK;
}

template <int kEpi, int BK, int kHalf, int kPair = 0>
static int launch_one(const GemmPlan& p, cudaStream_t s) {
  using Cfg = GemmCfg<kHalf>;
  auto kern = gemm_bf16_swapab<kEpi, BK, kHalf, kPair>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          Cfg::kSmem));
    configured = true;
  }
  if (kPair) {
    if (kHalf) return arg_fail("gemm: pair plans use the full config");
    if (getenv("SPECTRE_GEMM_PAIR_DBG")) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(p.grid);
      cfg.blockDim = dim3(Cfg::kThreads);
      cfg.dynamicSmemBytes = Cfg::kSmem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t q = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      printf("pair: max active clusters %d (%s), grid %d\n", n, cudaGetErrorString(q), p.grid);
    }
    cudaError_t e = launch_pdl_cluster(kern, dim3(p.grid), dim3(Cfg::kThreads), Cfg::kSmem, s, 2,
                                       p.tmap_w, p.tmap_x, p.tmap_out, p.tmap_sk, p.args);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_bf16_swapab (pair)");
    if (getenv("SPECTRE_GEMM_PAIR_DBG")) {
      e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_fail(e, "gemm_bf16_swapab (pair, sync)");
    }
    return SPECTRE_OK;
  }
  SPECTRE_LAUNCH_PDL("gemm_bf16_swapab", kern, dim3(p.grid), dim3(Cfg::kThreads),
                     Cfg::kSmem, s, p.tmap_w, p.tmap_x, p.tmap_out, p.tmap_sk, p.args);
  return SPECTRE_OK;
}

static int num_sms();

// CTA-pair launch for a wide single-job GEMM: every CTA owns exactly one
// 256-row tile (full K), the grid is an even number of CTAs in clusters of 2.
int gemm_set_pair(GemmPlan* p) {
  if (p->half || p->bk != 64 || p->epi != kSwiGLU || p->args.tile_rows != 256 || p->args.splits != 1 ||
      p->args.stream_k || p->n_tiles % 2 ||
      p->n_tiles > num_sms())
    return arg_fail("gemm_set_pair: one 256-row tile per CTA, BK 64, no split / stream-K");
  p->grid = p->n_tiles;
  p->args.pair = 1;
  return SPECTRE_OK;
}

// CTA-pair SwiGLU plan scheduled as (tile pair, 256-token chunk) units over
// every SM (an even grid): for large verify batches and for 256-row tile
// counts above one wave of CTAs.
int gemm_set_pair_units(GemmPlan* p) {
  if (p->half || p->bk != 64 || p->args.tile_rows != 256 || p->args.stream_k || p->n_tiles % 2 ||
      (p->epi == kArgmax && p->args.splits != 1))
    return arg_fail("gemm_set_pair_units: 256-row tiles, an even count, BK 64");
  p->grid = num_sms() & ~1;
  p->args.pair = 1;
  p->args.pair_units = 1;
  return SPECTRE_OK;
}

int gemm_default_bk() {
  static const int bk = [] {
    const char* v = getenv("SPECTRE_GEMM_BK");
    return (v && atoi(v) == 32) ? 32 : 64;
  }();
  return bk;
}

static int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

size_t gemm_sk_part_floats() { return (size_t)num_sms() * 256 * 256; }
static int num_sms_pub() { return num_sms(); }
int gemm_sk_grid() { return num_sms(); }

int gemm_plan(GemmPlan* p, const void* W, int N, int K, const void* X, int rows_cap, int epi,
              int splits, int max_stages, int bk, int tile_rows, float* sk_part, int* sk_flag) {
  if (tile_rows != 128) tile_rows = 256;
  if (bk == 0) bk = gemm_default_bk();
  if (bk != 32 && bk != 64) return arg_fail("gemm_plan: bk must be 32 or 64");
  if (N < 1 || K < 64 || K % 64 || rows_cap < 64 || rows_cap % 64 || splits < 1)
    return arg_fail("gemm_plan: shape (K % 64, rows_cap multiple of 64)");
  if (epi == kSwiGLU && (N % 2 || splits != 1)) return arg_fail("gemm_plan: swiglu shape");
  if (epi == kArgmax && splits != 1) return arg_fail("gemm_plan: argmax needs splits == 1");
  *p = GemmPlan{};
  if (int e = make_tmap_bf16(&p->tmap_w, W, (uint64_t)K, (uint64_t)N, 128, bk)) return e;
  if (int e = make_tmap_bf16(&p->tmap_x, X, (uint64_t)K, (uint64_t)rows_cap, 64, bk)) return e;
  p->bk = bk;
  const int n_tiles = (N + tile_rows - 1) / tile_rows;
  p->epi = epi;
  p->args.tile_rows = tile_rows;
  // persistent: at most one CTA per SM.  Full-K epilogues with a stream-K
  // workspace partition the iteration space over every SM (T <= 256).
  // stream-K only when every CTA owns >= a quarter of a tile's iterations
  // (a tile then spans <= 5 CTAs: the owner's fix-up stays short)
  const int k_iters = K / bk, total_iters = n_tiles * k_iters;
  p->args.stream_k = (epi != kPartial && sk_part && sk_flag && tile_rows == 256 &&
                      total_iters >= num_sms() * std::max(4, k_iters / 4)) ? 1 : 0;
  p->args.sk_part = sk_part;
  p->args.sk_flag = sk_flag;
  p->grid = p->args.stream_k ? num_sms() : std::min(n_tiles * splits, num_sms());
  p->args.N = N;
  p->args.K = K;
  p->args.rows_cap = rows_cap;
  p->args.splits = splits;
  p->args.max_stages = max_stages;
  p->n_tiles = n_tiles;
  p->n_amax_blocks = p->grid * 8;   // one (max, index) partial per CTA epilogue warp
  return SPECTRE_OK;
}

static int ksub_env() {
  static const int v = [] {
    const char* e = getenv("SPECTRE_GEMM_KSUB");   // k blocks per stage override (1 / 2)
    return e ? atoi(e) : 0;
  }();
  return v;
}

int gemm_run(const GemmPlan& p0, cudaStream_t s) {
  GemmPlan stripped;
  const GemmPlan* pp = &p0;
  static const int ksub_max_env = [] {
    const char* e = getenv("SPECTRE_GEMM_KSUBMAX");
    return e ? atoi(e) : 0;
  }();
  if ((ksub_env() && ksub_env() != p0.args.ksub) ||
      (ksub_max_env && ksub_max_env != p0.args.ksub_max)) {
    stripped = p0;
    if (ksub_env()) stripped.args.ksub = ksub_env();
    if (ksub_max_env) stripped.args.ksub_max = ksub_max_env;
    pp = &stripped;
  }
  const GemmPlan& p = *pp;
  if (p.args.pair) {
    if (p.bk != 64) return arg_fail("gemm: CTA pairs: BK 64");
    if (p.epi == kPartial) return launch_one<kPartial, 64, 0, 1>(p, s);
    if (p.epi == kArgmax) return launch_one<kArgmax, 64, 0, 1>(p, s);
    return launch_one<kSwiGLU, 64, 0, 1>(p, s);
  }
  if (p.half) {
    if (p.bk != 64 || p.epi == kArgmax) return arg_fail("gemm: half config needs BK 64, no argmax");
    if (p.epi == kPartial) return launch_one<kPartial, 64, 1>(p, s);
    return launch_one<kSwiGLU, 64, 1>(p, s);
  }
  if (p.bk == 64) {
    switch (p.epi) {
      case kPartial: return launch_one<kPartial, 64, 0>(p, s);
      case kArgmax: return launch_one<kArgmax, 64, 0>(p, s);
      default: return launch_one<kSwiGLU, 64, 0>(p, s);
    }
  }
  switch (p.epi) {
    case kPartial: return launch_one<kPartial, 32, 0>(p, s);
    case kArgmax: return launch_one<kArgmax, 32, 0>(p, s);
    default: return launch_one<kSwiGLU, 32, 0>(p, s);
  }
}

int gemm_set_pass_units(GemmPlan* p, int tokens) {
  if (p->half || p->args.tile_rows != 128 || p->epi != kPartial || p->args.stream_k ||
      tokens < 16 || tokens > 256 || tokens % 16)
    return arg_fail("gemm_set_pass_units: 128-row partial plans, 16..256 tokens per pass");
  p->args.pass_units = tokens;
  p->grid = num_sms();
  return SPECTRE_OK;
}

int gemm_set_half(GemmPlan* p) {
  if (p->args.tile_rows != 128 || p->epi == kArgmax || p->args.stream_k || p->bk != 64)
    return arg_fail("gemm_set_half: 128-row tiles, BK 64, partial / SwiGLU epilogue");
  p->half = 1;
  p->grid = std::min(p->n_tiles * p->args.splits, 2 * num_sms());
  return SPECTRE_OK;
}

}  // namespace spectre

using namespace spectre;

// stream-K workspace for the C-ABI entry point (tests, roofline bench)
static float* g_sk_part = nullptr;
static int* g_sk_flag = nullptr;
static int sk_workspace(float** part, int** flag) {
  if (!g_sk_part) {
    SPECTRE_CUDA_TRY(cudaMalloc(&g_sk_part, gemm_sk_part_floats() * sizeof(float)));
    SPECTRE_CUDA_TRY(cudaMalloc(&g_sk_flag, gemm_sk_grid() * sizeof(int)));
    SPECTRE_CUDA_TRY(cudaMemset(g_sk_flag, 0, gemm_sk_grid() * sizeof(int)));
  }
  *part = g_sk_part;
  *flag = g_sk_flag;
  return SPECTRE_OK;
}

// Partial (max, index) rows the argmax epilogue writes for an [N, K] weight.
extern "C" int32_t spectre_gemm_argmax_blocks(int32_t N, int32_t K) {
  (void)N;
  (void)K;
  return gemm_sk_grid() * 8;
}

extern "C" int spectre_gemm_bf16(const void* X, const void* W, const int32_t* t_dev,
                                 int32_t t_static, int32_t rows_cap, int32_t N, int32_t K,
                                 int32_t splits, int32_t epilogue, float* partial,
                                 float* amax_val, int32_t* amax_idx, void* act, int32_t ld_act,
                                 int32_t max_stages, void* stream) {
  GemmPlan p;
  // test knobs: max_stages < 0 forces 32-wide K blocks; >= 7000 (+1000: 128-row tiles)
  // token-pass units; >= 9000 CTA pairs over (tile pair, chunk) units; >= 4000 CTA pairs; >= 3000 the
  // half-SM config; >= 2000 disables stream-K; >= 1000 selects 128-row tiles
  bool sk = true;
  bool half = false;
  bool pair = false;
  bool punits = false, pair_units = false;
  if (max_stages >= 9000) {   // CTA pairs as (tile pair, 256-token chunk) units
    pair_units = true;
    max_stages -= 5000;
  }
  if (max_stages >= 7000) {   // 128-row partial plans as (tile, split, 256-token pass) units
    punits = true;
    max_stages -= 7000;
  }
  if (max_stages >= 4000) {   // CTA-pair launch (256-row tiles, no stream-K)
    pair = true;
    sk = false;
    max_stages -= 4000;
  }
  if (max_stages >= 3000) {
    half = true;
    sk = false;
    max_stages -= 3000;
  }
  if (max_stages >= 2000) {
    sk = false;
    max_stages -= 2000;
  }
  const int tile_rows = (half || max_stages >= 1000) ? 128 : 256;
  if (max_stages >= 1000) max_stages -= 1000;
  const int bk = max_stages < 0 ? 32 : 64;
  float* skp = nullptr;
  int* skf = nullptr;
  if (sk)
    if (int e = sk_workspace(&skp, &skf)) return e;
  if (int e = gemm_plan(&p, W, N, K, X, rows_cap, epilogue, splits,
                        max_stages < 0 ? -max_stages : max_stages, bk, tile_rows, skp, skf))
    return e;
  p.args.t_dev = t_dev;
  p.args.t_static = t_static;
  if (half)
    if (int e = gemm_set_half(&p)) return e;
  if (pair)
    if (int e = pair_units ? gemm_set_pair_units(&p) : gemm_set_pair(&p)) return e;
  if (punits)
    if (int e = gemm_set_pass_units(&p, 256)) return e;
  if (int e = gemm_set_outputs(&p, partial, amax_val, amax_idx, act, ld_act)) return e;
  if (const char* dg = getenv("SPECTRE_GEMM_DIAG")) p.args.diag = atoi(dg);
  static unsigned long long* stall = nullptr;
  if (getenv("SPECTRE_GEMM_STALL")) {   // producer / MMA wait and issue cycles per stage
    if (!stall) SPECTRE_CUDA_TRY(cudaMalloc(&stall, 2 * 148 * 4 * 8));
    SPECTRE_CUDA_TRY(cudaMemsetAsync(stall, 0, 2 * 148 * 4 * 8, as_stream(stream)));
    p.args.stall = stall;
    int r = gemm_run(p, as_stream(stream));
    std::vector<unsigned long long> h(2 * 148 * 4);
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(h.data(), stall, h.size() * 8, cudaMemcpyDeviceToHost,
                                     as_stream(stream)));
    SPECTRE_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    double e = 0, f = 0, is = 0, n = 0;
    for (int c = 0; c < p.grid; ++c) {
      e += h[c * 4];
      f += h[c * 4 + 1];
      is += h[c * 4 + 2];
      n += h[c * 4 + 3];
    }
    printf("stall grid %d stages/cta %.1f  per stage cycles: producer empty-wait %.0f  "
           "mma full-wait %.0f  mma issue %.0f\n",
           p.grid, n / p.grid, e / n, f / n, is / n);
    fflush(stdout);
    return r;
  }
  static unsigned long long* dbg = nullptr;
  if (getenv("SPECTRE_GEMM_DBG")) {
    if (!dbg) SPECTRE_CUDA_TRY(cudaMalloc(&dbg, 148 * 8 * 8));
    SPECTRE_CUDA_TRY(cudaMemsetAsync(dbg, 0, 148 * 8 * 8, as_stream(stream)));
    p.args.dbg = dbg;
    int r = gemm_run(p, as_stream(stream));
    std::vector<unsigned long long> h(148 * 8);
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, as_stream(stream)));
    SPECTRE_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < p.grid; ++c) if (h[c * 8] && h[c * 8] < t0) t0 = h[c * 8];
    for (int c = 0; c < p.grid; ++c) {
      printf("cta %3d start %7.2f", c, (h[c * 8] - t0) * 1e-3);
      for (int k = 1; k < 6; ++k) if (h[c * 8 + k]) printf("  j%d(r%llu) %7.2f", k - 1, h[c*8+k] >> 62, ((h[c * 8 + k] & ((1ull << 62) - 1)) - t0) * 1e-3);
      printf("  mma0done %7.2f  pollok %7.2f\n", (h[c * 8 + 7] - t0) * 1e-3, h[c*8+6] ? (h[c * 8 + 6] - t0) * 1e-3 : -1.0);
    }
    fflush(stdout);
    return r;
  }
  return gemm_run(p, as_stream(stream));
}
