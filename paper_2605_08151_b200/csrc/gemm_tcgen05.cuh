// gemm_tcgen05.cuh — weight-streaming GEMM for the verify / draft forward passes.
//
//   Y[t, n] = sum_k X[t, k] * W[n, k]        X: [T, K] bf16, W: [N, K] bf16 (both K-major)
//
// Decode-shaped: N (weights) is large, T (tokens = B*gamma on the target,
// B on the draft) is small and data-dependent.  So the MMA is issued
// "swap-AB": UMMA_M = 128 weight rows, UMMA_N = T (runtime, multiple of 16,
// up to 2 x 256 columns of TMEM).  One CTA owns a 128-row weight tile and a
// K-range (split-K), warp-specialised:
//   warp 0      TMA producer: W tile (64 x 128) + ceil(T/64) X boxes per stage
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld -> registers -> fused epilogue
// Epilogues:
//   kPartial  fp32 split-K partials [split][t][n] (deterministic reduction
//             happens in the consumer kernel, so results are batch invariant)
//   kArgmax   per-tile (max, argmax) over the 128 rows for every token
//             (lm_head greedy epilogue; logits are never materialised)
//   kSwiGLU   weight rows interleaved [64 gate | 64 up] per tile:
//             a[t, f] = silu(gate) * up written as bf16 (gate/up fused)
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx.cuh"

namespace spectre {

enum GemmEpilogue : int { kPartial = 0, kArgmax = 1, kSwiGLU = 2 };

constexpr int kGemmThreads = 192;
constexpr int kGemmBlockN = 128;   // weight rows per tile (UMMA_M)
constexpr int kGemmBlockK = 64;    // K per stage (one 128-byte swizzle row)
constexpr int kGemmMaxStages = 8;

struct GemmArgs {
  int N, K;                 // weight rows, reduction length
  int rows_cap;             // X buffer rows (multiple of 64); tokens beyond 512 run
                            // as extra passes that re-stream the weight tile
  int smem_rows;            // X rows staged per stage = min(rows_cap, 512)
  const int* t_dev;         // runtime token count (nullptr: use t_static)
  int t_static;
  int splits;               // split-K factor
  int stages;
  // kPartial
  float* part;              // [splits][rows_cap][N]
  // kArgmax
  float* amax_val;          // [n_tiles][rows_cap]
  int* amax_idx;
  // kSwiGLU
  __nv_bfloat16* act;       // [rows_cap][ld_act]
  int ld_act;
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

template <int kEpi, uint32_t kTmemCols>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_swapab(const __grid_constant__ CUtensorMap tmap_w,
                 const __grid_constant__ CUtensorMap tmap_x, GemmArgs a) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int stages = a.stages;
  const int x_stage_bytes = a.smem_rows * 128;
  uint8_t* w_smem = smem;                                    // stages * 16 KB
  uint8_t* x_smem = smem + stages * 16384;                   // stages * rows_cap*128
  uint64_t* full = reinterpret_cast<uint64_t*>(x_smem + stages * x_stage_bytes);
  uint64_t* empty = full + kGemmMaxStages;
  uint64_t* tmem_full = empty + kGemmMaxStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  float* scratch = reinterpret_cast<float*>(smem + stages * (16384 + x_stage_bytes) + 1024);

  const int n_tiles = (a.N + kGemmBlockN - 1) / kGemmBlockN;
  const int tile = blockIdx.x % n_tiles;
  const int split = blockIdx.x / n_tiles;
  const int n0 = tile * kGemmBlockN;
  const int k_iters_total = a.K / kGemmBlockK;
  const int it_begin = (int)((long long)k_iters_total * split / a.splits);
  const int it_end = (int)((long long)k_iters_total * (split + 1) / a.splits);
  const int n_iters = it_end - it_begin;

  int T = a.t_dev ? *a.t_dev : a.t_static;
  T = T < 0 ? 0 : (T > a.rows_cap ? a.rows_cap : T);
  const int n_pass = (T + a.smem_rows - 1) / a.smem_rows;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (T == 0 || n_iters <= 0) {
    // nothing to compute (empty batch): partial epilogue must still zero its slice
    if (kEpi == kPartial && warp >= 2) {
      // no rows to write when T == 0; when n_iters == 0 (K < splits) write zeros
      const int row = ((warp & 3) << 5) + lane;
      const int n = n0 + row;
      if (n < a.N) {
        for (int t = 0; t < T; ++t)
          a.part[((size_t)split * a.rows_cap + t) * a.N + n] = 0.0f;
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();   // weights stream through once
      const uint64_t pol_x = policy_evict_last();    // activations are re-read by every tile
      int g = 0;  // global pipeline iteration
      for (int pass = 0; pass < n_pass; ++pass) {
        const int r0 = pass * a.smem_rows;
        const int rows = min(T - r0, a.smem_rows);
        const int x_boxes = (rows + 63) >> 6;
        const uint32_t tx = 16384u + (uint32_t)x_boxes * 8192u;
        for (int i = 0; i < n_iters; ++i, ++g) {
          const int s = g % stages;
          const uint32_t ph = (uint32_t)(g / stages) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], tx);
          const int kc = (it_begin + i) * kGemmBlockK;
          tma_load_2d(w_smem + s * 16384, &tmap_w, &full[s], kc, n0, pol_w);
          for (int b = 0; b < x_boxes; ++b)
            tma_load_2d(x_smem + s * x_stage_bytes + b * 8192, &tmap_x, &full[s], kc,
                        r0 + b * 64, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    int g = 0;
    for (int pass = 0; pass < n_pass; ++pass) {
      const int rows = min(T - pass * a.smem_rows, a.smem_rows);
      const int t_pad = (rows + 15) & ~15;
      const int n_chunk0 = t_pad < 256 ? t_pad : 256;
      const int n_chunk1 = t_pad - n_chunk0;
      const uint32_t id0 = idesc_bf16_f32(128, (uint32_t)n_chunk0);
      const uint32_t id1 = idesc_bf16_f32(128, (uint32_t)(n_chunk1 > 0 ? n_chunk1 : 16));
      if (pass > 0) {  // epilogue must have drained the accumulator
        mbar_wait(tmem_empty, (uint32_t)(pass - 1) & 1u);
        tc_fence_after();
      }
      for (int i = 0; i < n_iters; ++i, ++g) {
        const int s = g % stages;
        const uint32_t ph = (uint32_t)(g / stages) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t wa = smem_u32(w_smem + s * 16384);
          const uint32_t xa = smem_u32(x_smem + s * x_stage_bytes);
#pragma unroll
          for (int kk = 0; kk < kGemmBlockK / 16; ++kk) {
            const uint64_t ad = umma_desc_sw128(wa + kk * 32);
            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
            mma_bf16_ss(tmem_base, ad, umma_desc_sw128(xa + kk * 32), id0, acc);
            if (n_chunk1 > 0)
              mma_bf16_ss(tmem_base + 256, ad, umma_desc_sw128(xa + 256 * 128 + kk * 32), id1,
                          acc);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(tmem_full);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue warps 2..5 (TMEM lane quarter = warp % 4)
    const int q = warp & 3;
    const int row = (q << 5) + lane;
    const int n = n0 + row;
    const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
    for (int pass = 0; pass < n_pass; ++pass) {
    mbar_wait(tmem_full, (uint32_t)pass & 1u);
    tc_fence_after();
    const int r0 = pass * a.smem_rows;
    const int rows = min(T - r0, a.smem_rows);
    const int t_pad = (rows + 15) & ~15;
    for (int cc = 0; cc < t_pad; cc += 16) {
      float v[16];
      tmem_ld16(tq + (uint32_t)cc, v);
      const int c0 = r0 + cc;
      if (kEpi == kPartial) {
        if (n < a.N) {
          float* dst = a.part + ((size_t)split * a.rows_cap) * a.N + n;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < T) dst[(size_t)(c0 + j) * a.N] = v[j];
        }
      } else if (kEpi == kArgmax) {
        // (max, lowest index) over this warp's 32 rows, per token column
        float* sv = scratch;                                   // [4][16]
        int* si = reinterpret_cast<int*>(scratch + 64);        // [4][16]
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float best = (n < a.N) ? v[j] : -INFINITY;
          int bi = n;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
              best = ov;
              bi = oi;
            }
          }
          if (lane == 0) {
            sv[q * 16 + j] = best;
            si[q * 16 + j] = bi;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane < 16 && c0 + lane < T) {
          float best = sv[lane];
          int bi = si[lane];
          for (int w = 1; w < 4; ++w) {
            const float ov = sv[w * 16 + lane];
            const int oi = si[w * 16 + lane];
            if (ov > best || (ov == best && oi < bi)) {
              best = ov;
              bi = oi;
            }
          }
          a.amax_val[(size_t)tile * a.rows_cap + c0 + lane] = best;
          a.amax_idx[(size_t)tile * a.rows_cap + c0 + lane] = bi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      } else {  // kSwiGLU: rows [0,64) gate, [64,128) up of features f0 + row%64
        float* up = scratch;                                   // [64][17]
        if (row >= 64) {
#pragma unroll
          for (int j = 0; j < 16; ++j) up[(row - 64) * 17 + j] = v[j];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (row < 64) {
          const int f = tile * 64 + row;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (c0 + j < T) {
              const float g = v[j];
              a.act[(size_t)(c0 + j) * a.ld_act + f] =
                  __float2bfloat16_rn(silu_f(g) * up[row * 17 + j]);
            }
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    tc_fence_before();
    mbar_arrive(tmem_empty);   // accumulator drained for the next pass
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace spectre
