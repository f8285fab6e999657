// gemm_tcgen05.cuh — weight-streaming GEMM for the verify / draft forward passes.
//
//   Y[t, n] = sum_k X[t, k] * W[n, k]        X: [T, K] bf16, W: [N, K] bf16 (both K-major)
//
// Decode-shaped: N (weights) is large and streamed once from HBM; T (tokens:
// B*gamma on the target, ~B on the draft) is small and known only on the
// device.  The MMA is issued "swap-AB": UMMA_M = 128 weight rows, UMMA_N = T.
// One CTA owns a 256-row weight tile and a K range (split-K):
//   T <= 256 : one phase, two 128x(T) accumulators in TMEM (cols 0 / 256),
//              every X stage feeds both -> X is read from L2 once per 256 W rows
//   T  > 256 : per 128-row half, N = up to 512 tokens in two MMA chunks
// The pipeline depth is chosen at run time from T (small T -> up to 8
// stages in flight), so one launch configuration serves the gamma-token
// verify pass, 1-token draft steps and prefill chunks (CUDA-graph friendly).
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// tcgen05.mma issuer, warps 2..9 epilogue (tcgen05.ld -> fused epilogue).
// Epilogues:
//   kPartial  fp32 split-K partials [split][t][n]; the consumer reduces them
//             in a fixed order (deterministic, batch invariant)
//   kArgmax   (max, lowest index) per 32-row block and token: lm_head greedy
//             decoding without materialising logits
//   kSwiGLU   weight rows interleaved [64 gate | 64 up]: a = silu(g) * u (bf16)
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace spectre {

enum GemmEpilogue : int { kPartial = 0, kArgmax = 1, kSwiGLU = 2 };

constexpr int kGemmThreads = 320;      // 2 control warps + 8 epilogue warps
constexpr int kGemmTileN = 256;        // weight rows per CTA
// K per pipeline stage is a template parameter: 64 (128-byte swizzle rows) or
// 32 (64-byte rows: half-size stages -> twice as many in flight).
constexpr int kGemmMaxStages = 8;
constexpr int kGemmSmemBytes = 232448; // dynamic smem requested at launch
constexpr int kGemmScratch = 2 * 64 * 17 * 4 + 1024;
constexpr int kGemmPipeBytes = kGemmSmemBytes - 1024 - 1024 - kGemmScratch;

struct GemmArgs {
  int N, K;                 // weight rows, reduction length
  int rows_cap;             // X buffer rows (multiple of 64)
  const int* t_dev;         // runtime token count (nullptr: use t_static)
  int t_static;
  int splits;               // split-K factor
  int max_stages;           // cap on pipeline depth (tests / tuning)
  int tile_rows;            // weight rows per CTA: 256 (two accumulators) or 128
  float* part;              // kPartial: [splits][rows_cap][N]
  float* amax_val;          // kArgmax: [ceil(N/32)][rows_cap]
  int* amax_idx;
  __nv_bfloat16* act;       // kSwiGLU: [rows_cap][ld_act]
  int ld_act;
};

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

struct GemmPhase {
  int row_off;   // first weight row of this phase within the tile (0 or 128)
  int boxes;     // 128-row weight boxes per stage (2: T<=256, 1: T>256)
  int t0, nt;    // token rows of this phase
};

// Phases of one CTA's work: T <= 256 with a 256-row tile -> one phase, both
// 128-row boxes per stage; otherwise one phase per (128-row box, 512-token pass).
__device__ __forceinline__ int gemm_n_phases(int T, int tile_rows) {
  if (T <= 256 && tile_rows == 256) return 1;
  return (tile_rows / 128) * ((T + 511) / 512);
}
__device__ __forceinline__ GemmPhase gemm_phase(int T, int tile_rows, int p) {
  GemmPhase ph;
  if (T <= 256 && tile_rows == 256) {
    ph.row_off = 0;
    ph.boxes = 2;
    ph.t0 = 0;
    ph.nt = T;
  } else {
    const int per = (T + 511) / 512;
    ph.row_off = (p / per) * 128;
    ph.boxes = 1;
    ph.t0 = (p % per) * 512;
    ph.nt = min(512, T - ph.t0);
  }
  return ph;
}

template <int kEpi, int BK>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_swapab(const __grid_constant__ CUtensorMap tmap_w,
                 const __grid_constant__ CUtensorMap tmap_x, GemmArgs a) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  int T = a.t_dev ? *a.t_dev : a.t_static;
  T = T < 0 ? 0 : (T > a.rows_cap ? a.rows_cap : T);
  constexpr int kRow = BK * 2;              // bytes per K-row segment (swizzle span)
  constexpr int kWBox = 128 * kRow;         // one 128-row weight box
  constexpr int kXBox = 64 * kRow;          // one 64-row activation box
  // runtime stage layout: W bytes + X bytes per stage
  const bool wide = (T <= 256 && a.tile_rows == 256);
  const int w_bytes = wide ? 2 * kWBox : kWBox;
  const int x_rows = wide ? ((T + 63) & ~63) : min((T + 63) & ~63, 512);
  const int stage_bytes = w_bytes + x_rows * kRow;
  int stages = stage_bytes > 0 ? kGemmPipeBytes / stage_bytes : 1;
  stages = stages > kGemmMaxStages ? kGemmMaxStages : (stages < 1 ? 1 : stages);
  if (a.max_stages > 0 && stages > a.max_stages) stages = a.max_stages;

  uint8_t* pipe = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGemmPipeBytes);
  uint64_t* empty = full + kGemmMaxStages;
  uint64_t* tmem_full = empty + kGemmMaxStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  float* scratch = reinterpret_cast<float*>(smem + kGemmPipeBytes + 1024);

  const int n_tiles = (a.N + a.tile_rows - 1) / a.tile_rows;
  const int tile = blockIdx.x % n_tiles;
  const int split = blockIdx.x / n_tiles;
  const int n0 = tile * a.tile_rows;
  const int k_iters_total = a.K / BK;
  const int it_begin = (int)((long long)k_iters_total * split / a.splits);
  const int it_end = (int)((long long)k_iters_total * (split + 1) / a.splits);
  const int n_iters = it_end - it_begin;
  const int n_phases = gemm_n_phases(T, a.tile_rows);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < kGemmMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const bool producer = (warp == 0 && lane == 0);
  if (!producer) {  // everyone but the TMA lane waits for the previous kernel now
    pdl_wait();
    pdl_trigger();
  }
  if (T == 0 || n_iters <= 0) {
    if (producer) {
      pdl_wait();
      pdl_trigger();
    }
    if (kEpi == kPartial && warp >= 2) {  // K < splits: this split contributes zeros
      for (int r = threadIdx.x - 64; r < a.tile_rows; r += 256) {
        const int n = n0 + r;
        if (n < a.N)
          for (int t = 0; t < T; ++t) a.part[((size_t)split * a.rows_cap + t) * a.N + n] = 0.0f;
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();   // weights stream through once
      const uint64_t pol_x = policy_evict_last();    // activations are re-read by every tile
      // Weights never change: the first stages' weight tiles are requested
      // before waiting on the previous kernel (its tail overlaps our fill).
      const GemmPhase ph0 = gemm_phase(T, a.tile_rows, 0);
      const int pre = n_iters < stages ? n_iters : stages;
      {
        const int x_boxes = (ph0.nt + 63) >> 6;
        const uint32_t tx = (uint32_t)ph0.boxes * kWBox + (uint32_t)x_boxes * kXBox;
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], tx);
          const int kc = (it_begin + i) * BK;
          for (int b = 0; b < ph0.boxes; ++b)
            tma_load_2d(pipe + i * stage_bytes + b * kWBox, &tmap_w, &full[i], kc,
                        n0 + ph0.row_off + b * 128, pol_w);
        }
      }
      pdl_wait();
      pdl_trigger();
      int g = 0;
      for (int p = 0; p < n_phases; ++p) {
        const GemmPhase ph = gemm_phase(T, a.tile_rows, p);
        const int x_boxes = (ph.nt + 63) >> 6;
        const uint32_t tx = (uint32_t)ph.boxes * kWBox + (uint32_t)x_boxes * kXBox;
        for (int i = 0; i < n_iters; ++i, ++g) {
          const int s = g % stages;
          uint8_t* st = pipe + s * stage_bytes;
          const int kc = (it_begin + i) * BK;
          if (g >= pre) {
            const uint32_t par = (uint32_t)(g / stages) & 1u;
            mbar_wait(&empty[s], par ^ 1u);
            mbar_arrive_expect_tx(&full[s], tx);
            for (int b = 0; b < ph.boxes; ++b)
              tma_load_2d(st + b * kWBox, &tmap_w, &full[s], kc, n0 + ph.row_off + b * 128,
                          pol_w);
          }
          for (int b = 0; b < x_boxes; ++b)
            tma_load_2d(st + w_bytes + b * kXBox, &tmap_x, &full[s], kc, ph.t0 + b * 64, pol_x);
        }
      }
    } else {
      pdl_wait();
      pdl_trigger();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    int g = 0;
    for (int p = 0; p < n_phases; ++p) {
      const GemmPhase ph = gemm_phase(T, a.tile_rows, p);
      const int t_pad = (ph.nt + 15) & ~15;
      const int nc0 = t_pad < 256 ? t_pad : 256;
      const int nc1 = t_pad - nc0;
      const uint32_t id0 = idesc_bf16_f32(128, (uint32_t)nc0);
      const uint32_t id1 = idesc_bf16_f32(128, (uint32_t)(nc1 > 0 ? nc1 : 16));
      if (p > 0) {
        mbar_wait(tmem_empty, (uint32_t)(p - 1) & 1u);
        tc_fence_after();
      }
      for (int i = 0; i < n_iters; ++i, ++g) {
        const int s = g % stages;
        const uint32_t par = (uint32_t)(g / stages) & 1u;
        mbar_wait(&full[s], par);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(pipe + s * stage_bytes);
          const uint32_t xa = sa + (uint32_t)w_bytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
            const uint64_t bd = umma_desc_kmajor<kRow>(xa + kk * 32);
            if (ph.boxes == 2) {
              mma_bf16_ss(tmem_base, umma_desc_kmajor<kRow>(sa + kk * 32), bd, id0, acc);
              mma_bf16_ss(tmem_base + 256, umma_desc_kmajor<kRow>(sa + kWBox + kk * 32), bd, id0,
                          acc);
            } else {
              const uint64_t ad = umma_desc_kmajor<kRow>(sa + kk * 32);
              mma_bf16_ss(tmem_base, ad, bd, id0, acc);
              if (nc1 > 0)
                mma_bf16_ss(tmem_base + 256, ad, umma_desc_kmajor<kRow>(xa + 256 * kRow + kk * 32),
                            id1, acc);
            }
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(tmem_full);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue warps 2..9: lane quarter q = warp % 4, group = (warp-2)/4
    const int q = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int gtid = threadIdx.x - 64 - grp * 128;       // 0..127 within the group
    const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
    float* up = scratch + grp * (64 * 17);
    for (int p = 0; p < n_phases; ++p) {
      const GemmPhase ph = gemm_phase(T, a.tile_rows, p);
      mbar_wait(tmem_full, (uint32_t)p & 1u);
      tc_fence_after();
      const int t_pad = (ph.nt + 15) & ~15;
      // 2 boxes: group g reads accumulator g (all columns);
      // 1 box:   both groups read accumulator 0, alternating 16-column chunks
      const int box = ph.boxes == 2 ? grp : 0;
      const int col_base = ph.boxes == 2 ? 256 * grp : 0;
      const int chunk_step = ph.boxes == 2 ? 16 : 32;
      const int chunk0 = ph.boxes == 2 ? 0 : 16 * grp;
      const int row = ph.row_off + box * 128 + q * 32 + lane;  // row within the tile
      const int n = n0 + row;
      for (int cc = chunk0; cc < t_pad; cc += chunk_step) {
        float v[16];
        tmem_ld16(tq + (uint32_t)(col_base + cc), v);
        const int c0 = ph.t0 + cc;
        if (kEpi == kPartial) {
          if (n < a.N) {
            float* dst = a.part + ((size_t)split * a.rows_cap) * a.N + n;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (cc + j < ph.nt) dst[(size_t)(c0 + j) * a.N] = v[j];
          }
        } else if (kEpi == kArgmax) {
          const int blk = n >> 5;  // 32-row block of this warp
          const bool warp_live = (n - lane) < a.N;
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
            if (warp_live && lane == j && cc + j < ph.nt) {
              a.amax_val[(size_t)blk * a.rows_cap + c0 + j] = best;
              a.amax_idx[(size_t)blk * a.rows_cap + c0 + j] = bi;
            }
          }
        } else {  // kSwiGLU: lanes [0,64) gate, [64,128) up of the box's 64 features
          const int r = q * 32 + lane;
          if (r >= 64) {
#pragma unroll
            for (int j = 0; j < 16; ++j) up[(r - 64) * 17 + j] = v[j];
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
          if (r < 64) {
            const int f = (n0 + ph.row_off + box * 128) / 2 + r;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (cc + j < ph.nt)
                a.act[(size_t)(c0 + j) * a.ld_act + f] =
                    __float2bfloat16_rn(silu_f(v[j]) * up[r * 17 + j]);
          }
          asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        }
      }
      (void)gtid;
      tc_fence_before();
      mbar_arrive(tmem_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace spectre
