// gemm_tcgen05.cuh — persistent weight-streaming GEMM for the verify / draft
// forward passes.
//
//   Y[t, n] = sum_k X[t, k] * W[n, k]        X: [T, K] bf16, W: [N, K] bf16 (both K-major)
//
// Decode-shaped: N (weights) is large and streamed once from HBM; T (tokens:
// B*gamma on the target, ~B on the draft) is small and known only on the
// device.  The MMA is issued "swap-AB": UMMA_M = 128 weight rows, UMMA_N = T.
// A tile is 256 weight rows (two TMEM accumulators share every activation
// stage, so X is read from L2 once per 256 W rows) or 128.
//
// Persistent: one CTA per SM walks a static schedule of accumulation jobs.
//   * stream-K (full-K epilogues, T <= 256): the n_tiles x K/BK iteration
//     space is cut into equal contiguous ranges, one per CTA, so every SM
//     streams the same number of weight bytes whatever N is (no wave
//     quantisation).  A tile cut by a range boundary is finished by its HEAD
//     owner (the CTA holding k = 0, which reaches it last in time): it adds
//     the fp32 partials of the tile's later segments (each the first
//     segment of the next CTAs) in k order, then runs the epilogue.  The cut
//     points depend only on (N, K, grid), never on T: results stay bit-
//     identical for any token count.
//   * split-K units (partial epilogue) / whole tiles (T > 256, prefill).
// TMEM accumulators are double-buffered whenever two fit (T <= 128 with
// 256-row tiles), so one job's epilogue overlaps the next job's MMAs, and the
// TMA ring runs across job boundaries.  The first stages' weight tiles are
// requested before griddepcontrol.wait (PDL): the weight stream starts while
// the previous kernel drains.
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + single-thread
// tcgen05.mma issuer, warps 2..9 epilogue (tcgen05.ld -> fused epilogue).
// Epilogues:
//   kPartial  fp32 split-K partials [split][t][n]; the consumer reduces them
//             in a fixed order (deterministic, batch invariant)
//   kArgmax   (max, lowest index) per (CTA, epilogue warp) and token over every
//             weight row the warp saw: lm_head greedy decoding without
//             materialising logits ([grid * 8][rows_cap] partials)
//   kSwiGLU   weight rows interleaved per pair [gate_i, up_i]: a = silu(g) * u
//             (bf16), combined with one shuffle (no shared-memory exchange)
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace spectre {

enum GemmEpilogue : int { kPartial = 0, kArgmax = 1, kSwiGLU = 2 };

constexpr int kGemmThreads = 320;      // full config: 2 control warps + 8 epilogue warps
constexpr int kGemmTileN = 256;        // weight rows per CTA tile
constexpr int kGemmMaxStages = 8;
constexpr int kGemmSmemBytes = 232448; // dynamic smem requested at launch
constexpr int kGemmScratch = 1024;
constexpr int kGemmStageOut = 2 * 16384;   // per epilogue group: [32 tokens][128 rows] fp32
constexpr int kGemmPipeBytes = kGemmSmemBytes - 1024 - 1024 - kGemmScratch - kGemmStageOut;

// Launch configurations.  Full: one CTA per SM (all 512 TMEM columns, ~227 KB
// shared memory).  Half (T <= 128 decode GEMMs): 128-row tiles, 4 epilogue
// warps, 256 TMEM columns, ~113 KB — two CTAs per SM, so the next kernel's
// CTAs become resident (and prefetch their weights under PDL) while this
// kernel's last CTAs drain.
template <int kHalf>
struct GemmCfg {
  static constexpr int kEpiWarps = kHalf ? 4 : 8;
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr int kTmemCols = kHalf ? 256 : 512;
  static constexpr int kSmem = kHalf ? 115712 : kGemmSmemBytes;
  static constexpr int kStageOut = (kEpiWarps / 4) * 16384;
  static constexpr int kPipe = kSmem - 1024 - 1024 - kGemmScratch - kStageOut;
  static constexpr int kPass = kHalf ? 256 : 512;   // tokens per one-box pass
  static constexpr int kMinBlocks = kHalf ? 2 : 1;
};

struct GemmArgs {
  int N, K;                 // weight rows, reduction length
  int rows_cap;             // X buffer rows (multiple of 64)
  const int* t_dev;         // runtime token count (nullptr: use t_static)
  int t_static;
  int splits;               // split-K factor (kPartial without stream-K)
  int max_stages;           // cap on pipeline depth (tests / tuning)
  int tile_rows;            // weight rows per tile: 256 (two accumulators) or 128
  int stream_k;             // full-K epilogues: equal iteration ranges per CTA
  float* part;              // kPartial: [splits][rows_cap][N] (written through tmap_out)
  float* amax_val;          // kArgmax: [grid * 8][rows_cap]
  int* amax_idx;
  __nv_bfloat16* act;       // kSwiGLU: [rows_cap][ld_act] (written through tmap_out)
  int ld_act;
  float* sk_part;           // stream-K: [grid][256 tokens][256 rows] fp32 segment partials
  int* sk_flag;             // stream-K: [grid] segment-ready flags (self-resetting)
  unsigned long long* dbg;  // diagnostics: per-CTA [8] globaltimer stamps (nullptr: off)
  int diag;                 // diagnostics (timing only): 1 skip MMAs, 2 skip epilogue math
  int ksub;                 // 1: one BK block per stage; 0: two when >= 2 such stages fit
  int ksub_max;             // most BK blocks per stage (0: 4)
  int pass_units;           // > 0: one-box plans schedule (tile, split, token pass of this
                            // many tokens) units over the CTAs (large T without split-K)
  int pair;                 // launched as CTA pairs (cluster 2): M=256 cta_group::2 MMAs
                            // whenever the tile is wide (T <= 256, 256-row tiles)
  int pair_units;           // pairs: (tile pair, 256-token chunk) units over every SM
                            // (chunk fastest) instead of one tile per CTA walking its chunks
  unsigned long long* stall;   // diagnostics: per CTA {producer empty-wait, MMA full-wait,
                               // MMA issue, stages} in cycles (null = off)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// one MUFU op: sigmoid(x) = 0.5 tanh(x/2) + 0.5 (tanh.approx: ~2^-11 relative,
// below the bf16 output's precision)
__device__ __forceinline__ float silu_tanh(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return x * fmaf(0.5f, t, 0.5f);
}

// One accumulation job of a CTA: a k-range of one tile and one token pass.
struct GemmJob {
  int tile, k0, k1;   // weight tile, k-iteration range [k0, k1)
  int row_off;        // first weight row of this pass within the tile (0 or 128)
  int boxes;          // 128-row weight boxes per stage (2: wide, 1 otherwise)
  int t0, nt;         // token rows of this pass
  int split;          // kPartial output slice
  int role;           // 0 plain, 1 stream-K head owner (has later segments), 2 contributor
};

// The static schedule, computed identically by the three warp roles.
struct GemmSched {
  int n_tiles, KI, G, c, T, tile_rows, splits, n_phases, pass, n_pu, n_ch;
  bool sk, wide;
  int it, hi, unit, phase;

  __device__ __forceinline__ static int iter_lo(int c, int G, int total) {
    return (int)((long long)total * c / G);
  }

  __device__ __forceinline__ bool has_iters(int cc) const {
    const int total = n_tiles * KI;
    return iter_lo(cc + 1, G, total) > iter_lo(cc, G, total);
  }

  // chunked: CTA-pair plans cover any T as wide jobs over 256-token chunks
  __device__ __forceinline__ void init(const GemmArgs& a, int T_, int BK, int pass_, bool chunked) {
    T = T_;
    pass = pass_;
    tile_rows = a.tile_rows;
    n_tiles = (a.N + tile_rows - 1) / tile_rows;
    KI = a.K / BK;
    G = gridDim.x;
    c = blockIdx.x;
    wide = chunked || (T <= 256 && tile_rows == 256);
    sk = a.stream_k && wide && !chunked;
    splits = sk ? 1 : a.splits;
    n_phases = wide ? (T + 255) / 256 : (tile_rows / 128) * ((T + pass - 1) / pass);
    // token-pass units: (tile, split, pass) spread over the CTAs, pass fastest
    // (CTAs sharing a weight tile run together: one HBM read, L2 for the rest)
    n_pu = (!wide && a.pass_units > 0 && tile_rows == 128) ? (T + a.pass_units - 1) / a.pass_units
                                                           : 0;
    if (n_pu > 0) {
      pass = a.pass_units;
      n_phases = 1;
    }
    // pair units: CTAs c, c + 1 (one cluster; G even) take units c + kG and
    // c + 1 + kG, i.e. the same chunk of tiles 2tp, 2tp + 1; neighbouring
    // pairs take the other chunks of the same tiles (one HBM read, L2 for the
    // rest).  n_tiles even, so both CTAs of a pair run out of units together.
    n_ch = (chunked && a.pair_units) ? (T + 255) / 256 : 0;
    const int total = n_tiles * KI;
    it = sk ? iter_lo(c, G, total) : 0;
    hi = sk ? iter_lo(c + 1, G, total) : 0;
    unit = c;
    phase = 0;
  }

  __device__ __forceinline__ bool next(GemmJob& j) {
    if (sk) {
      if (it >= hi) return false;
      j.tile = it / KI;
      j.k0 = it % KI;
      j.k1 = min(KI, j.k0 + (hi - it));
      it += j.k1 - j.k0;
      j.row_off = 0;
      j.boxes = 2;
      j.t0 = 0;
      j.nt = T;
      j.split = 0;
      j.role = j.k0 > 0 ? 2 : (j.k1 < KI ? 1 : 0);
      return true;
    }
    if (n_pu > 0) {
      if (unit >= n_tiles * splits * n_pu) return false;
      const int r = unit / n_pu;
      j.tile = r % n_tiles;
      j.split = r / n_tiles;
      j.k0 = (int)((long long)KI * j.split / splits);
      j.k1 = (int)((long long)KI * (j.split + 1) / splits);
      j.role = 0;
      j.row_off = 0;
      j.boxes = 1;
      j.t0 = (unit % n_pu) * pass;
      j.nt = min(pass, T - j.t0);
      unit += G;
      return true;
    }
    if (n_ch > 0) {   // (tile pair, split, chunk) units, chunk fastest
      if (unit >= n_tiles * splits * n_ch) return false;
      const int pr = unit >> 1;
      const int ch = pr % n_ch;
      const int r2 = pr / n_ch;
      j.tile = 2 * (r2 / splits) + (unit & 1);
      j.split = r2 % splits;
      j.k0 = (int)((long long)KI * j.split / splits);
      j.k1 = (int)((long long)KI * (j.split + 1) / splits);
      j.role = 0;
      j.row_off = 0;
      j.boxes = 2;
      j.t0 = ch * 256;
      j.nt = min(256, T - j.t0);
      unit += G;
      return true;
    }
    if (unit >= n_tiles * splits) return false;
    j.tile = unit % n_tiles;
    j.split = unit / n_tiles;
    j.k0 = (int)((long long)KI * j.split / splits);
    j.k1 = (int)((long long)KI * (j.split + 1) / splits);
    j.role = 0;
    if (wide) {   // 256-token chunks (one unless chunked)
      j.row_off = 0;
      j.boxes = 2;
      j.t0 = phase * 256;
      j.nt = min(256, T - j.t0);
    } else {
      const int per = (T + pass - 1) / pass;
      j.row_off = (phase / per) * 128;
      j.boxes = 1;
      j.t0 = (phase % per) * pass;
      j.nt = min(pass, T - j.t0);
    }
    if (++phase >= n_phases) {
      phase = 0;
      unit += G;
    }
    return true;
  }
};

// kPair: the CTA-pair instantiation (contains cta_group::2 instructions, so it
// must be launched in clusters of 2; it falls back to per-CTA MMAs when the
// tile is not wide).
template <int kEpi, int BK, int kHalf, int kPair = 0>
__global__ void __launch_bounds__(GemmCfg<kHalf>::kThreads, GemmCfg<kHalf>::kMinBlocks)
gemm_bf16_swapab(const __grid_constant__ CUtensorMap tmap_w,
                 const __grid_constant__ CUtensorMap tmap_x,
                 const __grid_constant__ CUtensorMap tmap_out,   // part fp32 / act bf16
                 const __grid_constant__ CUtensorMap tmap_sk,    // stream-K partials fp32
                 GemmArgs a) {
  using namespace ptx;
  using Cfg = GemmCfg<kHalf>;
  constexpr int kPipeB = Cfg::kPipe;
  constexpr int kStageOutB = Cfg::kStageOut;
  constexpr int kEpiThreads = 32 * Cfg::kEpiWarps;
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
  // CTA pair: each CTA holds its own 256 weight rows and HALF of the token
  // tile; one M=256 MMA per box spans both CTAs (the leader issues it).  Past
  // 256 tokens a pair walks the tokens in 256-token chunks (weights re-read
  // per chunk) so the MMAs stay M=256 x N=256 with both boxes sharing B.
  const bool pair = kPair && !kHalf && a.pair && a.tile_rows == 256;
  const int Tc = pair ? min(T, 256) : T;           // tokens per job
  const bool wide = (Tc <= 256 && a.tile_rows == 256);
  const int w_bytes = wide ? 2 * kWBox : kWBox;
  const uint32_t crank = kPair ? cluster_rank() : 0u;
  const bool leader = crank == 0;
  const int x_half = ((Tc + 15) & ~15) / 2;        // tokens held by each CTA of a pair
  const bool pu = !wide && a.pass_units > 0 && a.tile_rows == 128;   // token-pass units
  const int x_rows = pair ? ((x_half + 63) & ~63)
                          : (wide ? ((T + 63) & ~63)
                                  : min((T + 63) & ~63, pu ? a.pass_units : Cfg::kPass));
  // a stage holds `ksub` consecutive BK-wide k blocks (one expect-tx, one
  // MMA commit): fewer commit groups per byte when the MMAs are small (T=64)
  const int sub_bytes = w_bytes + x_rows * kRow;
  // two k blocks per stage whenever >= 2 such stages fit (measured: draft
  // SwiGLU 27.3 -> 22.5 us, draft lm_head 107 -> 98 us, target 128-row q/k/v/o
  // GEMMs -0.12 ms/round); a.ksub = 1 forces one block, >= 3 raises the minimum
  const int ksub_min_stages = a.ksub >= 2 ? a.ksub : 2;
  const int ksub_max = a.ksub_max > 0 ? a.ksub_max : 4;   // draft SwiGLU: 22.5 -> 21.1 us at 4
  int ksub = 1;
  if (a.ksub != 1)
    for (int c = ksub_max; c >= 2; --c)
      if (ksub_min_stages * c * sub_bytes <= kPipeB) {
        ksub = c;
        break;
      }
  const int stage_bytes = ksub * sub_bytes;
  int stages = stage_bytes > 0 ? kPipeB / stage_bytes : 1;
  stages = stages > kGemmMaxStages ? kGemmMaxStages : (stages < 1 ? 1 : stages);
  if (a.max_stages > 0 && stages > a.max_stages) stages = a.max_stages;
  // TMEM accumulator buffers: two whenever a job needs <= half the columns
  const int t_pad_all = ((pu ? min(Tc, a.pass_units) : Tc) + 15) & ~15;
  constexpr int kBufCols = Cfg::kTmemCols / 2;
  const int nbuf = ((wide && t_pad_all <= 128) || (!wide && t_pad_all <= kBufCols)) ? 2 : 1;
  const int half_stride = (wide && t_pad_all <= 128) ? 128 : 256;   // wide: 2nd accumulator

  uint8_t* pipe = smem;
  uint8_t* stage_out = smem + kPipeB;   // 1024-aligned: kPipe % 1024 == 0
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPipeB + kStageOutB);
  uint64_t* empty = full + kGemmMaxStages;
  uint64_t* tmem_full = empty + kGemmMaxStages;    // [2]
  uint64_t* tmem_empty = tmem_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_w);
    prefetch_tmap(&tmap_x);
    for (int s = 0; s < kGemmMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      // pair: both CTAs' epilogues arrive on the leader's barrier (the leader
      // issues every MMA into both TMEMs)
      mbar_init(&tmem_empty[b], (kPair && pair) ? 2 * kEpiThreads : kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (kPair && pair) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
    else tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();   // peer barriers initialised before any TMA signals them
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const bool producer = (warp == 0 && lane == 0);
  if (!producer) {  // everyone but the TMA lane waits for the previous kernel now
    pdl_wait();
    pdl_trigger();
  }
  GemmSched sched;
  sched.init(a, T, BK, Cfg::kPass, pair);
  if (a.dbg && threadIdx.x == 64) a.dbg[blockIdx.x * 8 + 0] = gtimer();
  const bool no_work = (T == 0);

  if (no_work) {
    if (producer) {
      pdl_wait();
      pdl_trigger();
    }
  } else if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();   // weights stream through once
      const uint64_t pol_x = policy_evict_last();    // activations are re-read by every tile
      GemmJob j;
      bool have = sched.next(j);
      // Weights never change: the first stages' weight tiles are requested
      // before waiting on the previous kernel (its tail overlaps our fill).
      int pre = 0;
      // pair: both CTAs' loads complete on the leader's barrier, which
      // expects both CTAs' bytes; the peer never arrives on it
      auto load_w = [&](void* dst, int s2, int c0, int c1) {
        if (kPair && pair) tma_load_2d_pair(dst, &tmap_w, mapa_shared(&full[s2], 0), c0, c1, pol_w);
        else tma_load_2d(dst, &tmap_w, &full[s2], c0, c1, pol_w);
      };
      auto load_x = [&](void* dst, int s2, int c0, int c1) {
        if (kPair && pair) tma_load_2d_pair(dst, &tmap_x, mapa_shared(&full[s2], 0), c0, c1, pol_x);
        else tma_load_2d(dst, &tmap_x, &full[s2], c0, c1, pol_x);
      };
      auto expect = [&](int s2, uint32_t bytes) {
        if (!pair) mbar_arrive_expect_tx(&full[s2], bytes);
        else if (leader) mbar_arrive_expect_tx(&full[s2], 2 * bytes);
      };
      // pair: this CTA's half of the job's (chunk's) tokens
      auto xh_of = [&](const GemmJob& jj) { return ((jj.nt + 15) & ~15) / 2; };
      auto x_boxes_of = [&](const GemmJob& jj) {
        return pair ? (xh_of(jj) + 63) >> 6 : (jj.nt + 63) >> 6;
      };
      if (have) {
        const int x_boxes = x_boxes_of(j);
        const uint32_t tx = (uint32_t)j.boxes * kWBox + (uint32_t)x_boxes * kXBox;
        pre = min((j.k1 - j.k0 + ksub - 1) / ksub, stages);
        for (int i = 0; i < pre; ++i) {
          const int kb = j.k0 + i * ksub, nk = min(ksub, j.k1 - kb);
          expect(i, tx * (uint32_t)nk);
          for (int q = 0; q < nk; ++q)
            for (int b = 0; b < j.boxes; ++b)
              load_w(pipe + i * stage_bytes + q * sub_bytes + b * kWBox, i, (kb + q) * BK,
                     j.tile * a.tile_rows + j.row_off + b * 128);
        }
      }
      pdl_wait();
      pdl_trigger();
      int g = 0;
      long long st_empty = 0;
      for (; have; have = sched.next(j)) {
        const int x_boxes = x_boxes_of(j);
        const uint32_t tx = (uint32_t)j.boxes * kWBox + (uint32_t)x_boxes * kXBox;
        const int n0 = j.tile * a.tile_rows + j.row_off;
        for (int k = j.k0; k < j.k1; k += ksub, ++g) {
          const int s = g % stages;
          const int nk = min(ksub, j.k1 - k);
          uint8_t* st = pipe + s * stage_bytes;
          if (g >= pre) {
            if (g >= stages) {
              const long long t_w = a.stall ? clock64() : 0;
              mbar_wait(&empty[s], ((uint32_t)(g / stages) & 1u) ^ 1u);
              if (a.stall) st_empty += clock64() - t_w;
            }
            expect(s, tx * (uint32_t)nk);
            for (int q = 0; q < nk; ++q)
              for (int b = 0; b < j.boxes; ++b)
                load_w(st + q * sub_bytes + b * kWBox, s, (k + q) * BK, n0 + b * 128);
          }
          const int x_t0 = pair ? (int)crank * xh_of(j) : 0;
          for (int q = 0; q < nk; ++q)
            for (int b = 0; b < x_boxes; ++b)
              load_x(st + q * sub_bytes + w_bytes + b * kXBox, s, (k + q) * BK,
                     j.t0 + x_t0 + b * 64);
        }
      }
      if (a.stall) a.stall[blockIdx.x * 4 + 0] = (unsigned long long)st_empty;
    } else {
      pdl_wait();
      pdl_trigger();
    }
    __syncwarp();   // reconverge the producer lane before the CTA-wide barrier
  } else if (warp == 1) {
    if (!pair || leader) {   // pair: the leader issues for both CTAs
    // ---------------- MMA issuer (one thread)
    int g = 0, jn = 0;
    long long st_full = 0, st_issue = 0;
    GemmJob j;
    while (sched.next(j)) {
      const int t_pad = (j.nt + 15) & ~15;
      const int nc0 = t_pad < 256 ? t_pad : 256;
      const int nc1 = t_pad - nc0;
      const uint32_t id0 = idesc_bf16_f32(pair ? 256 : 128, (uint32_t)nc0);
      const uint32_t id1 = idesc_bf16_f32(128, (uint32_t)(nc1 > 0 ? nc1 : 16));
      const int buf = jn % nbuf;
      const uint32_t acc = tmem_base + (uint32_t)(buf * kBufCols);
      if (jn >= nbuf) {
        mbar_wait(&tmem_empty[buf], (uint32_t)((jn / nbuf) - 1) & 1u);
        tc_fence_after();
      }
      for (int k = j.k0; k < j.k1; k += ksub, ++g) {
        const int s = g % stages;
        const int nk = min(ksub, j.k1 - k);
        const long long t_w = a.stall ? clock64() : 0;
        mbar_wait(&full[s], (uint32_t)(g / stages) & 1u);
        const long long t_i = a.stall ? clock64() : 0;
        st_full += t_i - t_w;
        tc_fence_after();
        if (lane == 0 && !(a.diag & 1)) {
          for (int q = 0; q < nk; ++q) {
          const uint32_t sa = smem_u32(pipe + s * stage_bytes + q * sub_bytes);
          const uint32_t xa = sa + (uint32_t)w_bytes;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t accf = (k > j.k0 || q > 0 || kk > 0) ? 1u : 0u;
            const uint64_t bd = umma_desc_kmajor<kRow>(xa + kk * 32);
            if (kPair && pair) {   // rows: this box in both CTAs; tokens: both CTAs' halves
              mma_bf16_ss_pair(acc, umma_desc_kmajor<kRow>(sa + kk * 32), bd, id0, accf);
              mma_bf16_ss_pair(acc + (uint32_t)half_stride,
                               umma_desc_kmajor<kRow>(sa + kWBox + kk * 32), bd, id0, accf);
            } else if (j.boxes == 2) {
              mma_bf16_ss(acc, umma_desc_kmajor<kRow>(sa + kk * 32), bd, id0, accf);
              mma_bf16_ss(acc + (uint32_t)half_stride,
                          umma_desc_kmajor<kRow>(sa + kWBox + kk * 32), bd, id0, accf);
            } else {
              const uint64_t ad = umma_desc_kmajor<kRow>(sa + kk * 32);
              mma_bf16_ss(acc, ad, bd, id0, accf);
              if (nc1 > 0)
                mma_bf16_ss(acc + 256, ad, umma_desc_kmajor<kRow>(xa + 256 * kRow + kk * 32),
                            id1, accf);
            }
          }
          }
          if (kPair && pair) mma_commit_pair(&empty[s]);
          else mma_commit(&empty[s]);
        } else if (lane == 0) {
          if (kPair && pair) mma_commit_pair(&empty[s]);
          else mma_commit(&empty[s]);
        }
        __syncwarp();
        if (a.stall) st_issue += clock64() - t_i;
      }
      if (lane == 0) {
        if (kPair && pair) mma_commit_pair(&tmem_full[buf]);
        else mma_commit(&tmem_full[buf]);
      }
      __syncwarp();
      ++jn;
    }
    if (a.stall && lane == 0) {
      a.stall[blockIdx.x * 4 + 1] = (unsigned long long)st_full;
      a.stall[blockIdx.x * 4 + 2] = (unsigned long long)st_issue;
      a.stall[blockIdx.x * 4 + 3] = (unsigned long long)g;
    }
    }
  } else {
    // ---------------- epilogue warps 2..9: lane quarter q = warp % 4, group = (warp-2)/4
    // Each thread owns one weight row (TMEM lane) and walks 32-column chunks
    // (tokens); one tcgen05.wait per chunk.
    const int q = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int etid = threadIdx.x - 64;                   // 0..255
    const int ewarp = etid >> 5;                         // 0..7
    // Outputs leave through TMA bulk-tensor stores staged in shared memory
    // (per group [32 tokens][128 rows]): plain per-thread stores are bounded
    // by outstanding-store slots (~20 GB/s per SM), bulk stores are not.
    const bool issuer = (warp == 2 + 4 * grp) && lane == 0;
    const int srow = q * 32 + lane;                      // row within the group's 128
    const int gbar = 1 + grp;
    int sbuf = 0;   // double-buffered staging: 2 x 8 KB per group
    int wbuf = 0;   // kPartial: per-warp double-buffered 2 KB boxes
    uint8_t* stg = stage_out + grp * 16384;
    auto stage_begin = [&]() {   // the store issued two steps ago has read its buffer
      stg = stage_out + grp * 16384 + sbuf * 8192;
      sbuf ^= 1;
      if (issuer) bulk_wait_read<1>();
      asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");
    };
    auto stage_end = [&]() {     // staged tile visible to the async proxy
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(gbar) : "memory");
    };
    int jn = 0;
    int amax_jobs = 0;   // jobs that wrote argmax slots (contributor segments do not)
    // pair units: a CTA's units cover scattered chunks, so its warps' slots
    // start at the identity and every unit merges (same lane writes and merges
    // a token: lane = token % 32)
    const bool amax_init = kEpi == kArgmax && sched.n_ch > 0 && !(a.diag & 2);
    if (amax_init)
      for (int t = lane; t < T; t += 32) {
        const size_t slot = ((size_t)blockIdx.x * 8 + ewarp) * a.rows_cap + t;
        a.amax_val[slot] = -INFINITY;
        a.amax_idx[slot] = 0x7fffffff;
      }
    GemmJob j;
    while (sched.next(j)) {
      const int buf = jn % nbuf;
      mbar_wait(&tmem_full[buf], (uint32_t)(jn / nbuf) & 1u);
      tc_fence_after();
      if (a.dbg && etid == 0 && jn == 0) a.dbg[blockIdx.x * 8 + 7] = gtimer();
      const int t_pad = (j.nt + 15) & ~15;
      // wide: group g reads accumulator g (all columns);
      // 1 box: both groups read accumulator 0, alternating 32-column chunks
      const int box = j.boxes == 2 ? grp : 0;
      const int col_base = buf * kBufCols + (j.boxes == 2 ? half_stride * grp : 0);
      constexpr int kGroups = Cfg::kEpiWarps / 4;
      const int chunk_step = j.boxes == 2 ? 32 : 32 * kGroups;
      const int chunk0 = j.boxes == 2 ? 0 : 32 * grp;
      const int trow = j.row_off + box * 128 + q * 32 + lane;   // row within the tile
      const int n = j.tile * a.tile_rows + trow;
      const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
      // stream-K head owner: the CTAs whose first segment continues this tile
      // (at most kSkMaxSeg - 1 of them: the plan only enables stream-K when
      // every CTA owns at least a quarter of a tile's iterations)
      constexpr int kSkMaxSeg = 8;
      int cl[kSkMaxSeg - 1];
      int ncl = 0;
      if (j.role == 1) {
        const int total = sched.n_tiles * sched.KI;
        const int tile_end = (j.tile + 1) * sched.KI;
        for (int cc = sched.c + 1;
             cc < sched.G && GemmSched::iter_lo(cc, sched.G, total) < tile_end; ++cc)
          if (sched.has_iters(cc) && ncl < kSkMaxSeg - 1) cl[ncl++] = cc;
        if (etid == 0) {   // one poller per owner (no polling storm on the flag lines)
          for (int i = 0; i < ncl; ++i)
            while (ld_acquire_gpu(a.sk_flag + cl[i]) == 0) {
            }
          __threadfence();
        }
        asm volatile("bar.sync 3, %0;" ::"r"(kEpiThreads) : "memory");
      }
      // TMEM loads are software-pipelined: chunk cc+step is in flight while
      // chunk cc is processed (columns past t_pad: unused)
      uint32_t rcur[32], rnext[32];
      if (chunk0 < t_pad && !(a.diag & 2)) {
        tmem_ld32_issue(tq + (uint32_t)(col_base + chunk0), rcur);
        tmem_ld_wait(rcur);
      }
      for (int cc = chunk0; cc < t_pad && !(a.diag & 2); cc += chunk_step) {
        const bool more = cc + chunk_step < t_pad;
        if (more) tmem_ld32_issue(tq + (uint32_t)(col_base + cc + chunk_step), rnext);
        float v[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) v[jj] = __uint_as_float(rcur[jj]);
        do {   // chunk body (a `continue` leaves the body, not the chunk loop)
        if (j.k1 <= j.k0) {   // empty k-range (K < splits): this split contributes zeros
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) v[jj] = 0.f;
        }
        const int c0 = j.t0 + cc;
        const int nvalid = min(32, j.nt - cc);           // live token columns of this chunk
        if (a.diag & 4) {   // diagnostics: TMEM loads only
          if (v[0] == 12345.f) a.part[0] = v[1];
          if (a.dbg && etid == 0 && cc == chunk0) a.dbg[blockIdx.x * 8 + 6] = gtimer();
          continue;
        }
        if (j.role == 2) {   // contributor: publish the raw segment sum ([col][256 rows])
#pragma unroll
          for (int h = 0; h < 2; ++h) {   // two 16-token halves
            stage_begin();
            float* st = reinterpret_cast<float*>(stg);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) st[jj * 128 + srow] = v[h * 16 + jj];
            stage_end();
            if (issuer) {
              tma_store_2d(&tmap_sk, stg, box * 128, sched.c * 256 + c0 + 16 * h);
              bulk_commit();
            }
          }
          continue;
        }
        if (j.role == 1) {   // owner: add later segments in k order
          for (int i = 0; i < ncl; ++i) {
            const float* src = a.sk_part + (size_t)cl[i] * (256 * 256) + trow + (size_t)c0 * 256;
            float add[32];
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) add[jj] = jj < nvalid ? __ldcg(src + jj * 256) : 0.f;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) v[jj] += add[jj];
          }
        }
        if (kEpi == kPartial) {
          if (a.diag & 8) {   // diagnostics: no staging / store
            if (v[0] == 12345.f) a.part[0] = v[1];
            continue;
          }
          // [split][t][n]: rows t >= T of the 16-token box land in unread
          // padding; columns past N are clipped by the tensor map.  Each warp
          // stages and stores its own 32 rows (box {32 rows, 16 tokens}), so
          // no cross-warp barrier per step.
#pragma unroll
          for (int h = 0; h < 2; ++h) {   // two 16-token halves
            if (h * 16 >= nvalid) break;
            float* wst = reinterpret_cast<float*>(stage_out + grp * 16384 + q * 4096 +
                                                  wbuf * 2048);
            wbuf ^= 1;
            if (lane == 0) bulk_wait_read<1>();   // the store two steps back has read it
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) wst[jj * 32 + lane] = v[h * 16 + jj];
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmap_out, wst, j.tile * a.tile_rows + j.row_off + box * 128 + q * 32,
                           j.split * a.rows_cap + c0 + 16 * h);
              bulk_commit();
            }
          }
        } else if (kEpi == kArgmax) {
          // (max, lowest index) over this warp's 32 rows for each of the 32
          // token columns: transpose-reduce butterfly (31 pair exchanges
          // instead of 32 x 5); afterwards lane l holds column l.
          float bv[32];
          int bi[32];
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            bv[jj] = (n < a.N) ? v[jj] : -INFINITY;
            bi[jj] = n;
          }
#pragma unroll
          for (int w = 16; w >= 1; w >>= 1) {
            const bool upper = (lane & w) != 0;
#pragma unroll
            for (int jj = 0; jj < w; ++jj) {
              // keep half [jj] (lower lanes) or [jj + w] (upper lanes); send the other
              const float send_v = upper ? bv[jj] : bv[jj + w];
              const int send_i = upper ? bi[jj] : bi[jj + w];
              const float keep_v = upper ? bv[jj + w] : bv[jj];
              const int keep_i = upper ? bi[jj + w] : bi[jj];
              const float ov = __shfl_xor_sync(0xffffffffu, send_v, w);
              const int oi = __shfl_xor_sync(0xffffffffu, send_i, w);
              const bool take = ov > keep_v || (ov == keep_v && oi < keep_i);
              bv[jj] = take ? ov : keep_v;
              bi[jj] = take ? oi : keep_i;
            }
          }
          // lane l now holds column c = bit-reverse-free index: lane bits select halves
          // high-to-low, so the surviving slot 0 of lane l is column l
          if (lane < nvalid) {
            const size_t slot = ((size_t)blockIdx.x * 8 + ewarp) * a.rows_cap + c0 + lane;
            float ov = bv[0];
            int oi = bi[0];
            // first coverage of a token by this warp: the CTA's first unit,
            // first row pass; later jobs merge with what the warp wrote
            if (amax_init || !(amax_jobs < sched.n_phases && j.row_off == 0)) {
              const float pv = a.amax_val[slot];
              const int pi = a.amax_idx[slot];
              if (pv > ov || (pv == ov && pi < oi)) {
                ov = pv;
                oi = pi;
              }
            }
            a.amax_val[slot] = ov;
            a.amax_idx[slot] = oi;
          }
        } else {
          // kSwiGLU: weight rows interleaved per row pair [gate_i, up_i]: lane
          // 2i holds gate_i, lane 2i+1 up_i.  Even lanes finish tokens 0..15 of
          // the chunk, odd lanes tokens 16..31.
          const bool odd = lane & 1;
          float out[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            // even lane needs up[jj] from its partner; odd lane needs gate[jj+16]
            const float send = odd ? v[jj] : v[jj + 16];
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const float g = odd ? recv : v[jj];
            const float u = odd ? v[jj + 16] : recv;
            out[jj] = silu_tanh(g) * u;
          }
          if (a.diag & 8) {   // diagnostics: no staging / store
            if (out[0] == 12345.f) a.part[0] = out[1];
            continue;
          }
          // each warp stages its own [32 tokens][16 features] bf16 box (its 32
          // rows = 16 row pairs) and stores it: no cross-warp barrier per chunk
          __nv_bfloat16* wst = reinterpret_cast<__nv_bfloat16*>(stage_out + grp * 16384 +
                                                                  q * 4096 + wbuf * 2048);
          wbuf ^= 1;
          if (lane == 0) bulk_wait_read<1>();   // the store two steps back has read it
          __syncwarp();
          const int fi = lane >> 1;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            wst[((odd ? 16 : 0) + jj) * 16 + fi] = __float2bfloat16_rn(out[jj]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmap_out, wst, (j.tile * a.tile_rows + j.row_off + box * 128 + q * 32) >> 1,
                         c0);
            bulk_commit();
          }
        }
              } while (0);
        if (more) {
          tmem_ld_wait(rnext);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) rcur[jj] = rnext[jj];
        }
      }
      if (a.dbg && etid == 0 && jn < 5) a.dbg[blockIdx.x * 8 + 1 + jn] = gtimer() | ((unsigned long long)j.role << 62);
      tc_fence_before();
      if (kPair && pair) {
        if (leader) mbar_arrive(&tmem_empty[buf]);
        else mbar_arrive_cluster(mapa_shared(&tmem_empty[buf], 0));
      } else {
        mbar_arrive(&tmem_empty[buf]);
      }
      if (j.role == 2) {
        // make the segment partial visible, then flag it (one thread, after all 256)
        if (issuer) {
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __threadfence();
        asm volatile("bar.sync 3, %0;" ::"r"(kEpiThreads) : "memory");
        if (etid == 0) atomicExch(a.sk_flag + sched.c, 1);
      } else if (j.role == 1) {
        asm volatile("bar.sync 3, %0;" ::"r"(kEpiThreads) : "memory");   // every owner thread read them
        if (etid == 0)
          for (int i = 0; i < ncl; ++i) a.sk_flag[cl[i]] = 0;   // self-reset
      }
      if (j.role != 2) ++amax_jobs;
      ++jn;
    }
    if (issuer || (kEpi != kArgmax && lane == 0)) {   // outputs complete (and visible to
      bulk_wait_all();                                // generic loads) before the grid does
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (kEpi == kArgmax && !(a.diag & 2) && !amax_init) {
      // every (CTA, warp) slot of every live token is defined: fill the tokens
      // this warp never covered (no job, or the other group's chunks of a
      // one-box pass) with the identity
      for (int t = lane; t < T; t += 32) {
        const bool covered = amax_jobs > 0 &&
                             (sched.wide || Cfg::kEpiWarps == 4 || (((t % 512) >> 5) & 1) == grp);
        if (!covered) {
          const size_t slot = ((size_t)blockIdx.x * 8 + ewarp) * a.rows_cap + t;
          a.amax_val[slot] = -INFINITY;
          a.amax_idx[slot] = 0x7fffffff;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();   // the leader's MMAs and both epilogues are done with both TMEMs
  if (warp == 1) {
    tc_fence_after();
    if (kPair && pair) tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
    else tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace spectre
