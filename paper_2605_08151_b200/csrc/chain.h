// chain.h — host interface of the persistent draft-step chain kernel (chain.cu).
#pragma once

#include <cuda_runtime.h>

namespace spectre {

enum ChainPhase : int { kPhEmbed = 1, kPhGemmPartial = 2, kPhGemmSwiGLU = 3, kPhResid = 4,
                        kPhRope = 5 };

struct ChainArgs;

// The model buffers a chain reads and writes (ModelRT's workspace).
struct ChainModel {
  int rows_cap, d, n_q, n_kv, hd, ctx_cap;
  float eps;
  const int* t_dev;
  const int* tok;
  const void* embed;        // bf16 [V][d]
  float* h;                 // fp32 residual [rows_cap][d]
  void* x;                  // bf16 normalised activations [rows_cap][d]
  const int* tok_pos;
  const int* tok_slot;
  const float2* rope;       // [ctx_cap][hd/2] (cos, sin)
  void* q;                  // bf16 [rows_cap][n_q][hd]
  void* kc;                 // RoPE phase: this chain's layer bases of the KV cache
  void* vc;
  float* part;              // split-K partials shared by the chain's GEMMs
  unsigned* bar;            // zeroed phase counter
  int t_pre_wait;           // 1: row count written launches back (see chain.cu)
  unsigned long long* dbg;  // diagnostics (nullptr: off): per-phase globaltimer stamps
};
int chain_set_model(void* plan, const ChainModel& m);

void* chain_alloc();
void chain_free(void* plan);
ChainArgs* chain_args(void* plan);
// GEMM phase: W [N][K] bf16, X [rows_cap][K] bf16; kPhGemmPartial writes split-K
// partials to part [splits][rows_cap][N], kPhGemmSwiGLU writes act [rows_cap][N/2].
int chain_add_gemm(void* plan, const void* W, int N, int K, const void* X, int rows_cap, int epi,
                   float* part, void* act);
// Glue phase: kPhEmbed / kPhResid (RMSNorm weight norm_w) / kPhRope.
int chain_add_glue(void* plan, int kind, const float* norm_w);
int chain_splits(int N, int K);
// t_bound: the forward's token rows, an upper bound or the typical count (selects
// 64-, 128- or 256-token MMA passes; more rows than the pass run as several passes)
int chain_launch(const void* plan, cudaStream_t s, int t_bound);

}  // namespace spectre
