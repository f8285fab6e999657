// model_kernels.cuh — forward-pass kernels other than the GEMM.
//
// Packed ragged batches: request b contributes n_new[b] consecutive token rows
// starting at q_off[b]; its new tokens sit at absolute positions
// pos0[b] .. pos0[b]+n_new[b]-1 and attend causally to its KV cache
// [0, pos0[b]+n_new[b]).  The same kernels serve the target's gamma-token
// verification pass, the draft's autoregressive steps (n_new = 1, or a short
// catch-up after a rollback) and prompt prefill chunks.
#pragma once

#include <cuda_bf16.h>
#include <cstdint>

namespace spectre {

struct AttnArgs {
  const __nv_bfloat16* q;    // [rows][n_q][hd]
  const int* q_off;          // [n_req]
  const int* n_new;          // [n_req]
  const int* pos0;           // [n_req]
  const int* slot;           // [n_req] KV slot
  int n_req, n_q, n_kv, ctx_cap;
  int layer_row0;            // first cache row of this layer in the K/V tensor maps
  int rb_max, split_max;     // 16-row m-tiles per request, key splits per request
  int chunk;                 // keys per split (multiple of 64)
  float scale_log2;          // hd^-0.5 * log2(e)
  float* part_o;             // [n_req][n_kv][rb_max][split_max][rows_blk][hd]
  float* part_ml;            // [n_req][n_kv][rb_max][split_max][rows_blk][2]
  int* done_cnt;             // [n_req][n_kv][rb_max] split arrivals (self-resetting)
  __nv_bfloat16* out;        // [rows][n_q][hd]
  int debug;                 // diagnostics: 1 skip math, 2 skip merge (timing only)
};


}  // namespace spectre
