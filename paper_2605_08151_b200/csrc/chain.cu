// chain.cu — the draft model's decode step as few persistent launches.
//
// Everything between two attention launches of the draft runs as ONE kernel
// ("chain"): o-projection -> residual + RMSNorm -> gate/up + SwiGLU -> down ->
// residual + RMSNorm -> next layer's q/k/v -> RoPE + KV write (the first chain
// of a step starts with embedding + RMSNorm, the last one ends at the final
// norm).  Per layer that is 2 launches (chain + attention) instead of 8.
//
// Why: at the draft's decode shape (T = B = 64 tokens) every weight-streaming
// GEMM launch costs ~5 us of body (weights at ~5.3 TB/s, then the epilogue)
// plus ~5 us of launch / drain (scripts/time_draft_gemms.py: back-to-back
// split-K launches run at 10.7-13.5 us for 8-34 MB), and the glue kernels add
// their own turnovers.  Inside a chain the weight stream never stops: weights
// are static, so the TMA producer warp walks ALL of the chain's GEMM jobs
// ahead of the math, limited only by its shared-memory ring; only the
// activation loads wait for the phase barrier that publishes their producer's
// output.
//
// One CTA per SM (grid = SMs, all co-resident), 11 warps:
//   warp 0  weight producer (TMA, evict-first), runs across phase boundaries
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-9  epilogue (tcgen05.ld -> split-K partial / SwiGLU stores straight
//           from registers: each warp instruction writes whole 32-128 B runs) and
//           the glue phases (residual + RMSNorm, RoPE, embedding) in between
//   warp 10 activation producer (TMA), waits on the phase barriers
// Phase barrier: one monotonic arrival counter per chain launch (each CTA
// arrives once per phase after its results are globally visible; the last
// arrival of the last phase resets it for the next launch).
//
// Arithmetic: GEMMs are 128-row weight tiles, K split into fixed ranges that
// depend only on (N, K, splits) — never on T — and the reductions (split sum in
// split order, per-row RMS over a fixed tree) are per row, so every token's
// result is independent of the batch composition (batch invariance).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "chain.h"
#include "common.cuh"
#include "gemm.h"
#include "model_kernels.cuh"
#include "ptx.cuh"

namespace spectre {

#define CHAIN_TRY(x)             \
  do {                           \
    if (int _r = (x)) return _r; \
  } while (0)

constexpr int kChainThreads = 352;
constexpr int kChainEpiThreads = 256;          // warps 2..9
constexpr int kChainMaxPhases = 8;
// One ring of stages, each holding kKS consecutive 64-wide k blocks of a job's
// weights (128 rows: 16 KB per block) AND its activations (one pass of up to
// kPass tokens: kPass * 128 B per block): both producers fill their half of a
// stage (one full barrier, two arrivals + tx bytes) and ONE MMA commit
// releases it — the tcgen05 commit is the MMA issuer's expensive step at T = 64.
constexpr int kChainWBox = 128 * 128;           // one k block of weights
// kPass tokens per MMA pass: 64 (decode steps of <= 64 requests: two k blocks
// per stage, four stages: 128 KB of weights in flight, the activation half
// sized to the 64-token box), 128 (<= 128 tokens, e.g. the catch-up step
// after a fully accepted round: two k blocks per stage, three stages) or 256
// (larger batches, e.g. config 3's B = 256: one N = 256 MMA chain per job
// instead of two passes that stream every weight tile twice; one k block per
// stage, four stages).  They keep 128 / 96 / 64 KB of weights and 192 KB of
// ring in flight per SM.
template <int kPass, int kKS_ = (kPass <= 128 ? 2 : 1), int kStages_ = (kPass == 128 ? 3 : 4)>
struct ChainCfg {
  static constexpr int kKS = kKS_;
  static constexpr int kStages = kStages_;
  static constexpr int kXBlk = kPass * 128;     // one k block of activations
  static constexpr int kStageBytes = kKS * (kChainWBox + kXBlk);
  static constexpr int kSmem = 1024 + kStages * kStageBytes + 1024;
  static constexpr int kTmemCols = 2 * kPass;   // two accumulator buffers
  static_assert(kSmem <= 232448, "chain smem");
};

struct ChainGemm {
  int N, K, splits, tiles, kb;   // kb: K / 64
  int epi;                       // kPhGemmPartial / kPhGemmSwiGLU
  void* out;                     // partials [splits][rows_cap][N] f32 / act [rows_cap][N/2] bf16
};

struct ChainArgs {
  int n_phase;
  int n_gemm;
  int t_pre_wait;                // 1: the row count was written launches back (read it
                                 // before griddepcontrol.wait); 0: by the predecessor
  int kind[kChainMaxPhases];
  int gemm[kChainMaxPhases];     // GEMM phases: slot 0..3
  float* resid_part;             // per-resid-phase source: the shared split-K buffer
  int resid_splits[kChainMaxPhases];
  const float* norm_w[kChainMaxPhases];
  ChainGemm g[4];
  int rows_cap, d, n_q, n_kv, hd, ctx_cap;
  float eps;
  const int* t_dev;
  const int* tok;
  const __nv_bfloat16* embed;
  float* h;
  __nv_bfloat16* x;
  const int* tok_pos;
  const int* tok_slot;
  const float2* rope;
  __nv_bfloat16* q;
  __nv_bfloat16* kc;             // this chain's RoPE layer bases
  __nv_bfloat16* vc;
  int rope_splits;
  unsigned* bar;                 // phase arrival counter (self-resetting)
  unsigned long long* dbg;       // diagnostics: CTA 0's globaltimer stamps [64]: 0 start,
                                 // 1 + 2p / 2 + 2p phase p may start / done, 16 + 2p / 17 + 2p
                                 // first accumulator ready / outputs stored, 32 + p MMA
                                 // issuer's first full stage of phase p
};

struct ChainJob {
  int tile, k0, k1, split, t0, nt;
};

// Jobs of GEMM slot `g` owned by CTA c of G: units (pass, split, tile), tile fastest.
struct ChainSched {
  int units, c, G, T, pass_t;
  __device__ __forceinline__ void init(const ChainGemm& g, int T_, int c_, int G_, int pass_) {
    T = T_;
    c = c_;
    G = G_;
    pass_t = pass_;
    const int passes = (T + pass_t - 1) / pass_t;
    units = g.tiles * g.splits * passes;
  }
  __device__ __forceinline__ bool get(const ChainGemm& g, int i, ChainJob& j) const {
    const int u = c + i * G;
    if (u >= units) return false;
    const int per_pass = g.tiles * g.splits;
    const int pass = u / per_pass;
    const int r = u % per_pass;
    j.tile = r % g.tiles;
    j.split = r / g.tiles;
    j.k0 = (int)((long long)g.kb * j.split / g.splits);
    j.k1 = (int)((long long)g.kb * (j.split + 1) / g.splits);
    j.t0 = pass * pass_t;
    j.nt = min(pass_t, T - j.t0);
    return true;
  }
};

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void chain_wait_phase(const unsigned* bar, unsigned target) {
  while (ld_acquire_u32(bar) < target) {
  }
}

// fixed-tree sum over the 256 epilogue threads (named barrier 1)
__device__ __forceinline__ float chain_block_sum(float v, float* sh, int et) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((et & 31) == 0) sh[et >> 5] = v;
  asm volatile("bar.sync 1, %0;" ::"n"(kChainEpiThreads) : "memory");
  float r = 0.f;
#pragma unroll
  for (int w = 0; w < kChainEpiThreads / 32; ++w) r += sh[w];
  asm volatile("bar.sync 1, %0;" ::"n"(kChainEpiThreads) : "memory");
  return r;
}

constexpr int kChainSplitBatch = 8;   // split partials in flight per batch (register budget)

// x[t] = bf16(h[t] * rsqrt(mean(h[t]^2) + eps) * w), h[t] = embedding row or
// h[t] + sum of the split partials (in split order).  One row per CTA at a time,
// float4 per thread; every split partial of a float4 is loaded before the
// fixed-order sum, so the loads overlap instead of forming a latency chain.
// kJ float4 per thread (d <= 1024 kJ), kB split partials per batch: kJ * kB
// float4 loads in flight per thread
template <int kJ, int kB>
__device__ void chain_norm_rows_t(const ChainArgs& a, int T, int phase, int et, float* sh) {
  const int d = a.d, nv = d >> 2;
  const bool embed = a.kind[phase] == kPhEmbed;
  const float4* w4 = reinterpret_cast<const float4*>(a.norm_w[phase]);
  const int splits = a.resid_splits[phase];
  const size_t sstride = (size_t)a.rows_cap * nv;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    float4 v[kJ];
    float ss = 0.f;
    float4* h4 = reinterpret_cast<float4*>(a.h + (size_t)t * d);
    const float4* p4 = reinterpret_cast<const float4*>(a.resid_part) + (size_t)t * nv;
    if (embed) {
      const __nv_bfloat16* e = a.embed + (size_t)a.tok[t] * d;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int i = et + j * kChainEpiThreads;
        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < nv) {
          const uint2 raw = *reinterpret_cast<const uint2*>(e + 4 * i);
          const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
          const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
          v[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int i = et + j * kChainEpiThreads;
        v[j] = i < nv ? h4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // every (element, split) load of a batch in flight at once; per element
      // the sum stays h + p0 + p1 + ... (split order)
      for (int s0 = 0; s0 < splits; s0 += kB) {
        float4 ld[kJ][kB];
#pragma unroll
        for (int sp = 0; sp < kB; ++sp)
#pragma unroll
          for (int j = 0; j < kJ; ++j) {
            const int i = et + j * kChainEpiThreads;
            if (s0 + sp < splits && i < nv) ld[j][sp] = __ldcg(p4 + (s0 + sp) * sstride + i);
          }
#pragma unroll
        for (int sp = 0; sp < kB; ++sp)
#pragma unroll
          for (int j = 0; j < kJ; ++j)
            if (s0 + sp < splits) {
              v[j].x += ld[j][sp].x;
              v[j].y += ld[j][sp].y;
              v[j].z += ld[j][sp].z;
              v[j].w += ld[j][sp].w;
            }
      }
    }
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int i = et + j * kChainEpiThreads;
      if (i < nv) {
        h4[i] = v[j];
        ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
      }
    }
    ss = chain_block_sum(ss, sh, et);
    const float r = rsqrtf(ss / (float)d + a.eps);
    __nv_bfloat162* xo = reinterpret_cast<__nv_bfloat162*>(a.x + (size_t)t * d);
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int i = et + j * kChainEpiThreads;
      if (i < nv) {
        const float4 ww = w4[i];
        xo[2 * i] = __floats2bfloat162_rn(v[j].x * r * ww.x, v[j].y * r * ww.y);
        xo[2 * i + 1] = __floats2bfloat162_rn(v[j].z * r * ww.z, v[j].w * r * ww.w);
      }
    }
  }
}

__device__ void chain_norm_rows(const ChainArgs& a, int T, int phase, int et, float* sh) {
  const int nv = a.d >> 2;
  if (nv <= kChainEpiThreads) chain_norm_rows_t<1, 8>(a, T, phase, et, sh);
  else chain_norm_rows_t<2, 5>(a, T, phase, et, sh);   // d <= 2048 (chain_set_model)
}

// RoPE (rotate-half pairs (i, i + hd/2)) on the summed q/k/v partials; q to
// the q buffer, k / v into the KV cache at (slot, position).  Four consecutive
// pairs per item (float4 partial loads), all splits in flight.
__device__ void chain_rope(const ChainArgs& a, int T, int et) {
  const int half = a.hd / 2;
  const int heads = a.n_q + 2 * a.n_kv;
  const int N = heads * a.hd;
  const int n_quads = heads * half / 4;
  const size_t sstride = (size_t)a.rows_cap * N;
  const int splits = a.rope_splits;
  const int items = T * n_quads;
  for (int it = blockIdx.x * kChainEpiThreads + et; it < items;
       it += gridDim.x * kChainEpiThreads) {
    const int t = it / n_quads;
    const int c = (it % n_quads) * 4;            // first pair index
    const int head = c / half, i = c % half;
    const float* p0 = a.resid_part + (size_t)t * N + head * a.hd + i;
    float x0[4] = {0.f, 0.f, 0.f, 0.f}, x1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < splits; s0 += kChainSplitBatch / 2) {   // split order kept
      float4 la[kChainSplitBatch / 2], lb[kChainSplitBatch / 2];
#pragma unroll
      for (int sp = 0; sp < kChainSplitBatch / 2; ++sp)
        if (s0 + sp < splits) {
          la[sp] = __ldcg(reinterpret_cast<const float4*>(p0 + (s0 + sp) * sstride));
          lb[sp] = __ldcg(reinterpret_cast<const float4*>(p0 + (s0 + sp) * sstride + half));
        }
#pragma unroll
      for (int sp = 0; sp < kChainSplitBatch / 2; ++sp)
        if (s0 + sp < splits) {
          x0[0] += la[sp].x; x0[1] += la[sp].y; x0[2] += la[sp].z; x0[3] += la[sp].w;
          x1[0] += lb[sp].x; x1[1] += lb[sp].y; x1[2] += lb[sp].z; x1[3] += lb[sp].w;
        }
    }
    const int pos = a.tok_pos[t];
    __nv_bfloat16* dst;
    if (head < a.n_q) dst = a.q + ((size_t)t * a.n_q + head) * a.hd;
    else if (head < a.n_q + a.n_kv)
      dst = a.kc + (((size_t)a.tok_slot[t] * a.n_kv + (head - a.n_q)) * a.ctx_cap + pos) * a.hd;
    else
      dst = a.vc +
            (((size_t)a.tok_slot[t] * a.n_kv + (head - a.n_q - a.n_kv)) * a.ctx_cap + pos) * a.hd;
    float ra[4], rb[4];
    if (head < a.n_q + a.n_kv) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 cs = a.rope[(size_t)pos * half + i + k];
        ra[k] = x0[k] * cs.x - x1[k] * cs.y;
        rb[k] = x1[k] * cs.x + x0[k] * cs.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ra[k] = x0[k];
        rb[k] = x1[k];
      }
    }
    __nv_bfloat162 a01 = __floats2bfloat162_rn(ra[0], ra[1]), a23 = __floats2bfloat162_rn(ra[2], ra[3]);
    __nv_bfloat162 b01 = __floats2bfloat162_rn(rb[0], rb[1]), b23 = __floats2bfloat162_rn(rb[2], rb[3]);
    uint2 ua, ub;
    ua.x = *reinterpret_cast<uint32_t*>(&a01);
    ua.y = *reinterpret_cast<uint32_t*>(&a23);
    ub.x = *reinterpret_cast<uint32_t*>(&b01);
    ub.y = *reinterpret_cast<uint32_t*>(&b23);
    *reinterpret_cast<uint2*>(dst + i) = ua;
    *reinterpret_cast<uint2*>(dst + i + half) = ub;
  }
}

template <int kPass, int kKS, int kStages>
__global__ void __launch_bounds__(kChainThreads, 1)
k_chain(const __grid_constant__ CUtensorMap tw0, const __grid_constant__ CUtensorMap tw1,
        const __grid_constant__ CUtensorMap tw2, const __grid_constant__ CUtensorMap tw3,
        const __grid_constant__ CUtensorMap tx0, const __grid_constant__ CUtensorMap tx1,
        const __grid_constant__ CUtensorMap tx2, const __grid_constant__ CUtensorMap tx3,
        ChainArgs a) {
  using namespace ptx;
  using Cfg = ChainCfg<kPass, kKS, kStages>;
  constexpr int kChainKS = Cfg::kKS;
  constexpr int kChainStages = Cfg::kStages;
  constexpr int kChainXBlk = Cfg::kXBlk;
  constexpr int kChainStageBytes = Cfg::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* ring = smem;   // stage s: [KS weight blocks][KS activation blocks]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kChainStages * kChainStageBytes);
  uint64_t* empty = full + kChainStages;
  uint64_t* tmem_full = empty + kChainStages;       // [2]
  uint64_t* tmem_empty = tmem_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  float* sh = reinterpret_cast<float*>(tmem_slot + 4);   // 8 floats (block sums)

  const CUtensorMap* tw[4] = {&tw0, &tw1, &tw2, &tw3};
  const CUtensorMap* tx[4] = {&tx0, &tx1, &tx2, &tx3};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  auto row_count = [&]() {
    const int t = *a.t_dev;
    return t < 0 ? 0 : (t > a.rows_cap ? a.rows_cap : t);
  };
  // mid-step chains: the row count comes from the step's batch kernel, several
  // launches back (the preceding attention released this grid only after its
  // own wait); the first chain of a step follows the batch kernel directly
  int T = a.t_pre_wait ? row_count() : -1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kChainStages; ++s) {
      mbar_init(&full[s], 2);    // weight half + activation half
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], kChainEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- weight producer: every GEMM job of the chain, in order
    if (lane == 0) {
      for (int s = 0; s < a.n_gemm; ++s) prefetch_tmap(tw[s]);
      const uint64_t pol = policy_evict_first();
      int gw = 0;
      bool waited = false;
      if (T < 0) {
        pdl_wait();
        pdl_trigger();
        waited = true;
        T = row_count();
      }
      for (int p = 0; p < a.n_phase && T > 0; ++p) {
        if (a.kind[p] != kPhGemmPartial && a.kind[p] != kPhGemmSwiGLU) continue;
        const ChainGemm& g = a.g[a.gemm[p]];
        ChainSched sc;
        sc.init(g, T, c, G, kPass);
        ChainJob j;
        for (int i = 0; sc.get(g, i, j); ++i) {
          for (int kb = j.k0; kb < j.k1; kb += kChainKS, ++gw) {
            const int s = gw % kChainStages;
            const int nk = min(kChainKS, j.k1 - kb);
            if (gw >= kChainStages) {
              if (!waited) {   // the first ring's worth streams before the predecessor ends
                pdl_wait();
                pdl_trigger();
                waited = true;
              }
              mbar_wait(&empty[s], ((uint32_t)(gw / kChainStages) - 1u) & 1u);
            }
            mbar_arrive_expect_tx(&full[s], (uint32_t)nk * kChainWBox);
            for (int q = 0; q < nk; ++q)
              tma_load_2d(ring + s * kChainStageBytes + q * kChainWBox, tw[a.gemm[p]], &full[s],
                          (kb + q) * 64, j.tile * 128, pol);
          }
        }
      }
      if (!waited) {
        pdl_wait();
        pdl_trigger();
      }
    } else {
      pdl_wait();
      pdl_trigger();
    }
    __syncwarp();
  } else if (warp == 10) {
    // ---------------- activation producer: waits for each phase's inputs
    pdl_wait();
    pdl_trigger();
    if (T < 0) T = row_count();
    if (lane == 0 && T > 0) {
      for (int s = 0; s < a.n_gemm; ++s) prefetch_tmap(tx[s]);
      const uint64_t pol = policy_evict_last();
      int gx = 0;
      for (int p = 0; p < a.n_phase; ++p) {
        if (a.kind[p] != kPhGemmPartial && a.kind[p] != kPhGemmSwiGLU) continue;
        const ChainGemm& g = a.g[a.gemm[p]];
        ChainSched sc;
        sc.init(g, T, c, G, kPass);
        ChainJob j;
        // only CTAs with jobs wait: a CTA's own epilogue cannot finish a phase it
        // has jobs in before this wait passed, so no waiter can outlive the
        // counter reset at the end of the chain
        if (p > 0 && sc.get(g, 0, j)) {
          chain_wait_phase(a.bar, (unsigned)(G * p));
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int i = 0; sc.get(g, i, j); ++i) {
          const int boxes = (j.nt + 63) >> 6;
          for (int kb = j.k0; kb < j.k1; kb += kChainKS, ++gx) {
            const int s = gx % kChainStages;
            const int nk = min(kChainKS, j.k1 - kb);
            if (gx >= kChainStages)
              mbar_wait(&empty[s], ((uint32_t)(gx / kChainStages) - 1u) & 1u);
            mbar_arrive_expect_tx(&full[s], (uint32_t)(nk * boxes) * 8192u);
            uint8_t* xs = ring + s * kChainStageBytes + kChainKS * kChainWBox;
            for (int q = 0; q < nk; ++q)
              for (int b = 0; b < boxes; ++b)
                tma_load_2d(xs + q * kChainXBlk + b * 8192, tx[a.gemm[p]], &full[s],
                            (kb + q) * 64, j.t0 + b * 64, pol);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer
    pdl_wait();
    pdl_trigger();
    if (T < 0) T = row_count();
    int gw = 0, jn = 0;
    for (int p = 0; p < a.n_phase && T > 0; ++p) {
      if (a.kind[p] != kPhGemmPartial && a.kind[p] != kPhGemmSwiGLU) continue;
      const ChainGemm& g = a.g[a.gemm[p]];
      ChainSched sc;
      sc.init(g, T, c, G, kPass);
      ChainJob j;
      for (int i = 0; sc.get(g, i, j); ++i, ++jn) {
        const int buf = jn & 1;
        const uint32_t acc = tmem_base + (uint32_t)(buf * kPass);
        const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)((j.nt + 15) & ~15));
        if (jn >= 2) {
          mbar_wait(&tmem_empty[buf], ((uint32_t)(jn >> 1) - 1u) & 1u);
          tc_fence_after();
        }
        for (int kb = j.k0; kb < j.k1; kb += kChainKS, ++gw) {
          const int s = gw % kChainStages;
          const int nk = min(kChainKS, j.k1 - kb);
          mbar_wait(&full[s], (uint32_t)(gw / kChainStages) & 1u);
          tc_fence_after();
          if (a.dbg && c == 0 && lane == 0 && i == 0 && kb == j.k0) a.dbg[32 + p] = gtimer_ns();
          if (lane == 0) {
            for (int q = 0; q < nk; ++q) {
              const uint32_t wa = smem_u32(ring + s * kChainStageBytes + q * kChainWBox);
              const uint32_t xa =
                  smem_u32(ring + s * kChainStageBytes + kChainKS * kChainWBox + q * kChainXBlk);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ss(acc, umma_desc_kmajor<128>(wa + kk * 32),
                            umma_desc_kmajor<128>(xa + kk * 32), idesc,
                            (kb > j.k0 || q > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit(&tmem_full[buf]);
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue + glue warps 2..9
    pdl_wait();
    pdl_trigger();
    if (T < 0) T = row_count();
    const bool stamp = a.dbg && c == 0 && threadIdx.x == 64;
    if (stamp) a.dbg[0] = gtimer_ns();
    const int et = threadIdx.x - 64;           // 0..255
    const int q = warp & 3;                    // TMEM lane quarter
    const int grp = (warp - 2) >> 2;           // 0 / 1: alternating 32-token chunks
    int jn = 0;
    for (int p = 0; p < a.n_phase; ++p) {
      const int kind = a.kind[p];
      if (p > 0) {   // inputs of this phase: every CTA finished phase p - 1
        if (et == 0) chain_wait_phase(a.bar, (unsigned)(G * p));
        asm volatile("bar.sync 1, %0;" ::"n"(kChainEpiThreads) : "memory");
        if (stamp) a.dbg[1 + 2 * p] = gtimer_ns();       // phase p may start
      }
      if (T > 0 && (kind == kPhGemmPartial || kind == kPhGemmSwiGLU)) {
        const int gi = a.gemm[p];
        const ChainGemm& g = a.g[gi];
        ChainSched sc;
        sc.init(g, T, c, G, kPass);
        ChainJob j;
        for (int i = 0; sc.get(g, i, j); ++i, ++jn) {
          const int buf = jn & 1;
          mbar_wait(&tmem_full[buf], (uint32_t)(jn >> 1) & 1u);
          tc_fence_after();
          if (stamp && i == 0) a.dbg[16 + 2 * p] = gtimer_ns();
          const int t_pad = (j.nt + 15) & ~15;
          const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kPass);
          for (int cc = 32 * grp; cc < t_pad; cc += 64) {
            uint32_t r[32];
            tmem_ld32_issue(tq + (uint32_t)cc, r);
            tmem_ld_wait(r);
            float v[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) v[jj] = __uint_as_float(r[jj]);
            const int nvalid = min(32, j.nt - cc);
            if (kind == kPhGemmPartial) {
              // [split][t][n] partials straight from registers: for each token
              // the warp's 32 lanes write 128 consecutive bytes
              float* dst = static_cast<float*>(g.out) +
                           (size_t)(j.split * a.rows_cap + j.t0 + cc) * g.N + j.tile * 128 +
                           q * 32 + lane;
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (jj < nvalid) dst[(size_t)jj * g.N] = v[jj];
            } else {
              // SwiGLU straight from registers: even lanes tokens 0..15 of the
              // chunk, odd lanes 16..31; lane pairs share feature lane / 2
              const bool odd = lane & 1;
              const int n2 = g.N >> 1;
              __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g.out) +
                                   (size_t)(j.t0 + cc + (odd ? 16 : 0)) * n2 +
                                   ((j.tile * 128 + q * 32) >> 1) + (lane >> 1);
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) {
                const float send = odd ? v[jj] : v[jj + 16];
                const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                const float gt = odd ? recv : v[jj];
                const float up = odd ? v[jj + 16] : recv;
                float th;
                asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(0.5f * gt));
                if ((odd ? 16 : 0) + jj < nvalid)
                  dst[(size_t)jj * n2] = __float2bfloat16_rn(gt * fmaf(0.5f, th, 0.5f) * up);
              }
            }
          }
          tc_fence_before();
          mbar_arrive(&tmem_empty[buf]);
        }
        if (stamp) a.dbg[17 + 2 * p] = gtimer_ns();
      } else if (T > 0 && (kind == kPhResid || kind == kPhEmbed)) {
        chain_norm_rows(a, T, p, et, sh);
      } else if (T > 0 && kind == kPhRope) {
        chain_rope(a, T, et);
      }
      // arrive: the CTA barrier orders every epilogue thread's results before
      // thread 0's gpu-scope release (cumulative), which publishes them with
      // the arrival (one fence per CTA instead of one per thread)
      asm volatile("bar.sync 1, %0;" ::"n"(kChainEpiThreads) : "memory");
      if (stamp) a.dbg[2 + 2 * p] = gtimer_ns();         // this CTA finished phase p
      if (et == 0) {
        unsigned prev;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;"
                     : "=r"(prev) : "l"(a.bar) : "memory");
        // the last arrival of the last phase: every CTA is past every wait
        if (p == a.n_phase - 1 && prev == (unsigned)(G * a.n_phase) - 1u) atomicExch(a.bar, 0u);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

struct ChainPlan {
  GemmPlan gp[4];
  ChainArgs args;
  int n_gemm = 0;
};

static int chain_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// One split count per chain GEMM: about one job per SM at one pass, >= 3 k blocks per job.
int chain_splits(int N, int K) {
  const int tiles = (N + 127) / 128, kb = K / 64;
  int s = chain_sms() / tiles;
  if (s > 16) s = 16;
  if (s < 1) s = 1;
  while (s > 1 && kb / s < 3) --s;
  return s;
}

template <int kPass, int kKS = ChainCfg<kPass>::kKS, int kStages = ChainCfg<kPass>::kStages>
static int chain_launch_t(const ChainPlan& cp, cudaStream_t s) {
  using Cfg = ChainCfg<kPass, kKS, kStages>;
  static bool cfg = false;
  if (!cfg) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_chain<kPass, kKS, kStages>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
    cfg = true;
  }
  const GemmPlan* g = cp.gp;
  SPECTRE_LAUNCH_PDL("k_chain", (k_chain<kPass, kKS, kStages>), dim3(chain_sms()),
                     dim3(kChainThreads), Cfg::kSmem, s, g[0].tmap_w, g[1].tmap_w, g[2].tmap_w,
                     g[3].tmap_w, g[0].tmap_x, g[1].tmap_x, g[2].tmap_x, g[3].tmap_x, cp.args);
  return SPECTRE_OK;
}

int chain_launch(const void* plan_v, cudaStream_t s, int t_bound) {
  const ChainPlan& cp = *reinterpret_cast<const ChainPlan*>(plan_v);
  static const int pass256 = [] {   // SPECTRE_CHAIN_PASS=128: never the 256-token passes
    const char* v = getenv("SPECTRE_CHAIN_PASS");
    return v ? atoi(v) != 128 : 1;
  }();
  static const int pass64 = [] {   // SPECTRE_CHAIN_PASS64=0: never the 64-token passes
    const char* v = getenv("SPECTRE_CHAIN_PASS64");
    return v ? atoi(v) != 0 : 1;
  }();
  if (pass256 && t_bound > 128) return chain_launch_t<256>(cp, s);
  if (pass64 && t_bound <= 64) return chain_launch_t<64>(cp, s);
  return chain_launch_t<128>(cp, s);
}

void* chain_alloc() { return new ChainPlan(); }
void chain_free(void* p) { delete reinterpret_cast<ChainPlan*>(p); }
ChainArgs* chain_args(void* p) { return &reinterpret_cast<ChainPlan*>(p)->args; }

// Add a GEMM phase: W [N][K], X [rows_cap][K]; epi kPhGemmPartial (partials to
// part [splits][rows_cap][N]) or kPhGemmSwiGLU (act [rows_cap][N/2]).
int chain_add_gemm(void* plan_v, const void* W, int N, int K, const void* X, int rows_cap, int epi,
                   float* part, void* act) {
  ChainPlan& cp = *reinterpret_cast<ChainPlan*>(plan_v);
  ChainArgs& a = cp.args;
  if (cp.n_gemm >= 4 || a.n_phase >= kChainMaxPhases) return arg_fail("chain: too many phases");
  if (N % 128 || K % 64) return arg_fail("chain: N % 128, K % 64");
  const int gi = cp.n_gemm++;
  a.n_gemm = cp.n_gemm;
  const int splits = epi == kPhGemmSwiGLU ? 1 : chain_splits(N, K);
  GemmPlan& gp = cp.gp[gi];
  CHAIN_TRY(gemm_plan(&gp, W, N, K, X, rows_cap, epi == kPhGemmSwiGLU ? kSwiGLU : kPartial, splits, 0,
                64, 128));
  CHAIN_TRY(gemm_set_outputs(&gp, part, nullptr, nullptr, act, N / 2));
  ChainGemm& g = a.g[gi];
  g.N = N;
  g.K = K;
  g.out = epi == kPhGemmSwiGLU ? act : static_cast<void*>(part);
  g.splits = splits;
  g.tiles = N / 128;
  g.kb = K / 64;
  g.epi = epi;
  a.kind[a.n_phase] = epi;
  a.gemm[a.n_phase] = gi;
  ++a.n_phase;
  return SPECTRE_OK;
}

// Add a glue phase (kPhEmbed / kPhResid / kPhRope).  Resid / Rope read the
// split-K partials of the chain's LAST added GEMM.
int chain_add_glue(void* plan_v, int kind, const float* norm_w) {
  ChainPlan& cp = *reinterpret_cast<ChainPlan*>(plan_v);
  ChainArgs& a = cp.args;
  if (a.n_phase >= kChainMaxPhases) return arg_fail("chain: too many phases");
  if (kind == kPhResid || kind == kPhRope) {
    if (cp.n_gemm == 0 || a.g[cp.n_gemm - 1].epi != kPhGemmPartial)
      return arg_fail("chain: residual / RoPE phases follow a split-K GEMM");
    if (kind == kPhResid) a.resid_splits[a.n_phase] = a.g[cp.n_gemm - 1].splits;
    else a.rope_splits = a.g[cp.n_gemm - 1].splits;
  }
  a.kind[a.n_phase] = kind;
  a.gemm[a.n_phase] = -1;
  a.norm_w[a.n_phase] = norm_w;
  ++a.n_phase;
  return SPECTRE_OK;
}

int chain_set_model(void* plan_v, const ChainModel& m) {
  ChainArgs& a = reinterpret_cast<ChainPlan*>(plan_v)->args;
  if (m.d > 8 * kChainEpiThreads) return arg_fail("chain: d_model > 2048");
  a.rows_cap = m.rows_cap;
  a.d = m.d;
  a.n_q = m.n_q;
  a.n_kv = m.n_kv;
  a.hd = m.hd;
  a.ctx_cap = m.ctx_cap;
  a.eps = m.eps;
  a.t_dev = m.t_dev;
  a.tok = m.tok;
  a.embed = reinterpret_cast<const __nv_bfloat16*>(m.embed);
  a.h = m.h;
  a.x = reinterpret_cast<__nv_bfloat16*>(m.x);
  a.tok_pos = m.tok_pos;
  a.tok_slot = m.tok_slot;
  a.rope = m.rope;
  a.q = reinterpret_cast<__nv_bfloat16*>(m.q);
  a.kc = reinterpret_cast<__nv_bfloat16*>(m.kc);
  a.vc = reinterpret_cast<__nv_bfloat16*>(m.vc);
  a.resid_part = m.part;
  a.bar = m.bar;
  a.t_pre_wait = m.t_pre_wait;
  a.dbg = m.dbg;
  return SPECTRE_OK;
}

}  // namespace spectre
