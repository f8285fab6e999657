// gemm.h — internal C++ interface of the tcgen05 GEMM (used by engine.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm_tcgen05.cuh"

namespace spectre {

struct GemmPlan {
  CUtensorMap tmap_w;
  CUtensorMap tmap_x;
  CUtensorMap tmap_out;   // kPartial: part fp32 [splits*rows_cap][N]; kSwiGLU: act bf16
  CUtensorMap tmap_sk;    // stream-K partials fp32 [grid*256][256]
  GemmArgs args;
  int grid = 0;
  int epi = 0;
  int n_tiles = 0;        // weight tiles (args.tile_rows rows each)
  int n_amax_blocks = 0;  // argmax partial rows (grid * 8 epilogue warps)
  int bk = 32;            // K per pipeline stage (32: 64B swizzle, 64: 128B swizzle)
  int half = 0;           // half-SM launch config (two CTAs per SM, GemmCfg<1>)
};

int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                   uint32_t box_outer, uint32_t box_inner = 64);
// W: [N][K] bf16, X: [rows_cap][K] bf16.  Output pointers are filled by the caller.
// sk_part / sk_flag: stream-K workspace (gemm_sk_part_floats() floats, gemm_sk_grid()
// zeroed ints) for full-K epilogues; nullptr keeps one CTA per tile.
int gemm_plan(GemmPlan* p, const void* W, int N, int K, const void* X, int rows_cap, int epi,
              int splits, int max_stages = 0, int bk = 0, int tile_rows = 256,
              float* sk_part = nullptr, int* sk_flag = nullptr);
size_t gemm_sk_part_floats();
int gemm_sk_grid();
// Output buffers (call after gemm_plan): builds the TMA store maps.
int gemm_set_outputs(GemmPlan* p, float* part, float* amax_val, int* amax_idx, void* act,
                     int ld_act);
int gemm_run(const GemmPlan& p, cudaStream_t s);
// Switch a 128-row-tile partial / SwiGLU plan to the half-SM configuration.
int gemm_set_half(GemmPlan* p);
int gemm_set_pair(GemmPlan* p);   // CTA pairs (cta_group::2) for wide single-tile plans
int gemm_set_pair_units(GemmPlan* p);   // pairs over (tile pair, 256-token chunk) units
// Large-T partial plans (128-row tiles): (tile, split, `tokens`-token pass) units
// over every SM instead of split-K alone (fewer splits: less fp32 partial traffic)
int gemm_set_pass_units(GemmPlan* p, int tokens);

}  // namespace spectre
