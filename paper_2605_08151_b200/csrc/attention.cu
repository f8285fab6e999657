// attention.cu — causal attention of a packed ragged batch of new tokens over
// each request's KV cache: the target's gamma-token verify pass, the draft's
// decode steps (one token, or a short catch-up after a rollback) and prefill
// chunks all use this kernel.
//
// HBM-bound (bytes = sum_req ctx * n_kv * hd * 2 * 2 per layer), so
// the design is about keeping the KV stream in flight:
//
//   * persistent CTAs, one per SM; work item = (key split, request, kv head,
//     block of query rows); items are split-major so the live ones form a
//     contiguous prefix and the static stride balances them;
//   * warp-specialised: one producer lane streams 64-key K/V stages with TMA
//     (2-D tensor map over the whole cache, 128-byte swizzle) into an
//     NS-deep mbarrier ring that runs ACROSS item boundaries; before
//     griddepcontrol.wait it already prefetches keys below pos0 (written by
//     earlier rounds), so the stream starts while the QKV kernel drains;
//   * 4 consumer warps per 16-row m-tile, warp w owning keys [16w, 16w+16) of
//     every stage: S = Q K^T and O += P V on mma.sync m16n8k16 from
//     ldmatrix'ed swizzled tiles, online softmax in the log2 domain;
//   * fixed-order merges: the 4 key-slice warps through shared memory, then
//     splits (the last split of an m-tile to arrive merges all of them in
//     split order).
//
// Every reduction boundary is an absolute key position (split = chunk keys,
// stage = 64, slice = 16), so a token's output is bit-identical whether it is
// computed in a verify pass, a prefill chunk or plain autoregressive decode.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "model_kernels.cuh"
#include "ptx.cuh"

namespace spectre {

template <int HD, int MT, int NG, int NS>
struct AttnCfg {
  static constexpr int kBoxes = HD / 64;                 // 128-byte swizzle boxes per key row
  static constexpr int kBoxBytes = 64 * 128;             // 64 keys x 64 elements
  static constexpr int kStageBytes = 2 * kBoxes * kBoxBytes;   // K + V of 64 keys
  static constexpr int kStages = NS;
  static constexpr int kCWarps = 4 * MT * NG;            // consumer warps
  static constexpr int kThreads = 32 * (kCWarps + 1);    // + producer warp
  static constexpr int kRows = 16 * MT;
  static constexpr int kLdO = HD + 4;
  static constexpr int kRing = kStages * kStageBytes;
  static constexpr int kQBytes = kRows * HD * 2;         // one Q slot (unpadded rows)
  static constexpr int kMergeBytes = MT * 4 * 16 * (kLdO + 2) * 4;
  static constexpr int kMetaBytes = 2 * 64;
  static constexpr int kBarBytes = (2 * kStages + 4) * 8 + 64 + 32 * 52 + 32 * 4;
  static constexpr int kSmem = 1024 + kRing + 2 * kQBytes + kMergeBytes + kMetaBytes + kBarBytes;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                          uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void bar_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Byte offset of (key row, element col) inside a stage's K (or V) half:
// boxes of 64 columns, 128-byte rows, 16-byte chunks XOR-swizzled by row & 7.
__device__ __forceinline__ uint32_t swz(int key, int col) {
  return (uint32_t)((col >> 6) * (64 * 128) + key * 128 + ((((col & 63) >> 3) ^ (key & 7)) << 4));
}

// Work item descriptor, resolved by the producer and handed to the consumers
// through shared memory (the consumers never chase global metadata).
struct AttnMeta {
  int valid, b, kvh, rblk, split, nn, p0, c0, c1, qoff, rows_total, n_split;
};

// Decode item `item` (split-major); returns false if it has no work.
__device__ __forceinline__ bool attn_item(const AttnArgs& a, int item, int n_rblk, int rows_blk,
                                          AttnMeta& it) {
  // (row block, split, request, kv head), row block slowest: the live items
  // of a typical launch (one row block, few splits) form a dense prefix
  const int n_pairs = a.n_req * a.n_kv;
  const int per_rblk = n_pairs * a.split_max;
  it.rblk = item / per_rblk;
  int r = item % per_rblk;
  it.split = r / n_pairs;
  r %= n_pairs;
  it.kvh = r % a.n_kv;
  it.b = r / a.n_kv;
  it.nn = a.n_new[it.b];
  if (it.nn <= 0) return false;
  it.rows_total = it.nn * (a.n_q / a.n_kv);
  if (it.rblk * rows_blk >= it.rows_total) return false;
  it.p0 = a.pos0[it.b];
  const int kv_len = it.p0 + it.nn;
  it.c0 = it.split * a.chunk;
  if (it.c0 >= kv_len) return false;
  it.c1 = min(it.c0 + a.chunk, kv_len);
  it.n_split = (kv_len + a.chunk - 1) / a.chunk;
  it.qoff = a.q_off[it.b];
  it.valid = 1;
  return true;
}

template <int HD, int MT, int NG, int NS>
__global__ void __launch_bounds__(AttnCfg<HD, MT, NG, NS>::kThreads, 1)
k_attn(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
       AttnArgs a) {
  using C = AttnCfg<HD, MT, NG, NS>;
  static_assert(C::kStages % NG == 0, "stage groups");
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* ring = smem;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem + C::kRing);   // [2][kRows][HD]
  float* sMerge = reinterpret_cast<float*>(smem + C::kRing + 2 * C::kQBytes);
  AttnMeta* meta = reinterpret_cast<AttnMeta*>(smem + C::kRing + 2 * C::kQBytes + C::kMergeBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(meta) + C::kMetaBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* ifull = empty + C::kStages;     // [2] item meta + Q landed
  uint64_t* iempty = ifull + 2;             // [2] item slot released by every consumer warp
  int* s_last = reinterpret_cast<int*>(iempty + 2);   // [MT]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int group = a.n_q / a.n_kv;
  const int n_rblk = a.rb_max / MT;
  const int n_items = a.n_req * a.n_kv * n_rblk * a.split_max;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::kCWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&ifull[s], 1);
      mbar_init(&iempty[s], C::kCWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == C::kCWarps) {
    // ------------------------------------------------------------ producer
    // The warp's 32 lanes resolve 32 candidate items at a time (independent
    // metadata loads in parallel) into a compact list; lane 0 then streams
    // the live ones.
    AttnMeta* list = reinterpret_cast<AttnMeta*>(s_last + 4);   // [32]
    int* row0s = reinterpret_cast<int*>(list + 32);               // [32]
    const uint64_t pol = policy_evict_first();   // every KV byte is read once per layer
    if (lane == 0) {
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
    }
    bool waited = false;
    int g = 0, ii = 0;
    auto stage = [&](int row0, int k0) {
      const int s = g % C::kStages;
      if (g >= C::kStages) mbar_wait(&empty[s], (uint32_t)((g / C::kStages) - 1) & 1u);
      uint8_t* st = ring + s * C::kStageBytes;
      mbar_arrive_expect_tx(&full[s], C::kStageBytes);
#pragma unroll
      for (int bx = 0; bx < C::kBoxes; ++bx) {
        tma_load_2d(st + bx * C::kBoxBytes, &tm_k, &full[s], bx * 64, row0 + k0, pol);
        tma_load_2d(st + (C::kBoxes + bx) * C::kBoxBytes, &tm_v, &full[s], bx * 64, row0 + k0,
                    pol);
      }
      ++g;
    };
    auto publish = [&](const AttnMeta& it) {   // meta + Q rows of this item -> slot ii & 1
      const int slot = ii & 1;
      if (ii >= 2) mbar_wait(&iempty[slot], (uint32_t)((ii >> 1) - 1) & 1u);
      meta[slot] = it;
      if (!it.valid) {
        mbar_arrive(&ifull[slot]);
        return;
      }
      const int R0 = it.rblk * C::kRows, R1 = min(it.rows_total, R0 + C::kRows);
      mbar_arrive_expect_tx(&ifull[slot], (uint32_t)(R1 - R0) * HD * 2);
      __nv_bfloat16* dst = sQ + (size_t)slot * C::kRows * HD;
      for (int R = R0; R < R1;) {
        const int j = R / group, hh = R % group;
        const int cnt = min(group - hh, R1 - R);
        bulk_load(dst + (size_t)(R - R0) * HD,
                  a.q + (((size_t)(it.qoff + j) * a.n_q) + it.kvh * group + hh) * HD,
                  (uint32_t)cnt * HD * 2, &ifull[slot]);
        R += cnt;
      }
      ++ii;
    };
    for (int base = blockIdx.x; base < n_items; base += 32 * gridDim.x) {
      AttnMeta it;
      const int item = base + lane * gridDim.x;
      const bool live = item < n_items && attn_item(a, item, n_rblk, C::kRows, it);
      const unsigned m = __ballot_sync(0xffffffffu, live);
      if (live) {
        const int k = __popc(m & ((1u << lane) - 1u));
        list[k] = it;
        row0s[k] = a.layer_row0 + (a.slot[it.b] * a.n_kv + it.kvh) * a.ctx_cap;
      }
      __syncwarp();
      if (lane == 0) {
        for (int k = 0; k < __popc(m); ++k) {
          const AttnMeta cur = list[k];
          const int row0 = row0s[k];
          int k0 = cur.c0;
          if (!waited) {
            // keys below pos0 were written by earlier rounds: stream them while
            // the QKV kernel (which writes Q and the new keys) is still running
            for (int n = 0; n < C::kStages && k0 + 64 <= cur.p0 && k0 < cur.c1; ++n, k0 += 64)
              stage(row0, k0);
            pdl_wait();
            pdl_trigger();
            waited = true;
          }
          publish(cur);
          for (; k0 < cur.c1; k0 += 64) stage(row0, k0);
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (!waited) {
        pdl_wait();
        pdl_trigger();
      }
      AttnMeta end{};
      end.valid = 0;
      publish(end);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  pdl_wait();
  pdl_trigger();
  // warp = (stage group ng, m-tile mt, key slice ks): group ng computes the
  // 64-key stages whose ABSOLUTE index k0/64 is ng mod NG (batch invariant)
  const int ng = warp / (4 * MT);
  const int mt = (warp >> 2) % MT;   // m-tile of this warp
  const int ks = warp & 3;           // 16-key slice of every 64-key stage
  const int g8 = lane >> 2, tq = lane & 3;
  constexpr int kMtThreads = 128 * NG;
  const int ltid = (ng * 4 + ks) * 32 + lane;   // 0..kMtThreads-1 within the m-tile
  float* mO = sMerge + mt * 4 * 16 * (C::kLdO + 2);     // [4 slices][16 rows][kLdO]
  float* mML = mO + 4 * 16 * C::kLdO;                   // [4][16][2]
  int g = 0;

  for (int ii = 0;; ++ii) {
    const int slot = ii & 1;
    mbar_wait(&ifull[slot], (uint32_t)(ii >> 1) & 1u);
    const AttnMeta it = meta[slot];
    if (!it.valid) break;
    const int row_lo = it.rblk * C::kRows + mt * 16;     // first query row of this m-tile
    const bool active = row_lo < it.rows_total;
    const int p_max = it.p0 + (min(it.rows_total, row_lo + 16) - 1) / group;
    uint32_t qf[HD / 16][4];
    float o[HD / 8][4];
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    int qpos[2];
    bool qvalid[2];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[n][e] = 0.f;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int R = row_lo + g8 + hr * 8;
      qvalid[hr] = R < it.rows_total;
      qpos[hr] = it.p0 + (qvalid[hr] ? R / group : 0);
    }
    if (active) {
      // rows past rows_total hold stale data: their scores are masked below
      const __nv_bfloat16* q = sQ + (size_t)slot * C::kRows * HD + (size_t)(mt * 16) * HD;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(smem_u32(q + (lane & 15) * HD + kk * 16 + (lane >> 4) * 8), qf[kk][0], qf[kk][1],
                qf[kk][2], qf[kk][3]);
    }

    for (int k0 = it.c0; k0 < it.c1; k0 += 64, ++g) {
      const int s = g % C::kStages;
      mbar_wait(&full[s], (uint32_t)(g / C::kStages) & 1u);
      const int kb = k0 + 16 * ks;                       // first key of this warp's slice
      if (active && kb <= p_max && (k0 >> 6) % NG == ng && !(a.debug & 1)) {
        const uint32_t sK = smem_u32(ring + s * C::kStageBytes);
        const uint32_t sV = sK + C::kBoxes * C::kBoxBytes;
        const int mi = lane >> 3;
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        float t0[4] = {0.f, 0.f, 0.f, 0.f}, t1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          uint32_t b0, b1, b2, b3;
          const int key = 16 * ks + (mi >> 1) * 8 + (lane & 7);
          ldsm_x4(sK + swz(key, kk * 16 + (mi & 1) * 8), b0, b1, b2, b3);
          if (kk & 1) {
            mma16816(t0, qf[kk], b0, b1);
            mma16816(t1, qf[kk], b2, b3);
          } else {
            mma16816(s0, qf[kk], b0, b1);
            mma16816(s1, qf[kk], b2, b3);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s0[e] += t0[e];
          s1[e] += t1[e];
        }
        // mask + online softmax; s0: keys kb+2tq+{0,1}, s1: kb+8+2tq+{0,1}
        float p[2][4];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          float v[4] = {s0[hr * 2], s0[hr * 2 + 1], s1[hr * 2], s1[hr * 2 + 1]};
          float mx = -INFINITY;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = kb + (e >> 1) * 8 + 2 * tq + (e & 1);
            v[e] *= a.scale_log2;
            if (!qvalid[hr] || key > qpos[hr]) v[e] = -INFINITY;
            mx = fmaxf(mx, v[e]);
          }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          const float m_new = fmaxf(mrow[hr], mx);
          const float corr = (m_new == -INFINITY) ? 1.f : exp2f(mrow[hr] - m_new);
          float rs = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            p[hr][e] = (v[e] == -INFINITY) ? 0.f : exp2f(v[e] - m_new);
            rs += p[hr][e];
          }
          rs += __shfl_xor_sync(0xffffffffu, rs, 1);
          rs += __shfl_xor_sync(0xffffffffu, rs, 2);
          lrow[hr] = lrow[hr] * corr + rs;
          mrow[hr] = m_new;
#pragma unroll
          for (int n = 0; n < HD / 8; ++n) {
            o[n][hr * 2] *= corr;
            o[n][hr * 2 + 1] *= corr;
          }
        }
        const uint32_t pa[4] = {pack_bf16(p[0][0], p[0][1]), pack_bf16(p[1][0], p[1][1]),
                                pack_bf16(p[0][2], p[0][3]), pack_bf16(p[1][2], p[1][3])};
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          const int key = 16 * ks + (mi & 1) * 8 + (lane & 7);
          ldsm_x4_t(sV + swz(key, dp * 16 + (mi >> 1) * 8), b0, b1, b2, b3);
          mma16816(o[2 * dp], pa, b0, b1);
          mma16816(o[2 * dp + 1], pa, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    if (active && !(a.debug & 2)) {   // uniform across the m-tile's warps
      if (NG == 2) {
        // ---- stage groups: group 1's state folds into group 0's (same lanes)
        if (ng == 1) {
#pragma unroll
          for (int hr = 0; hr < 2; ++hr) {
            const int r = g8 + hr * 8;
#pragma unroll
            for (int n = 0; n < HD / 8; ++n)
              *reinterpret_cast<float2*>(&mO[(ks * 16 + r) * C::kLdO + n * 8 + 2 * tq]) =
                  make_float2(o[n][hr * 2], o[n][hr * 2 + 1]);
            if (tq == 0) {
              mML[(ks * 16 + r) * 2] = mrow[hr];
              mML[(ks * 16 + r) * 2 + 1] = lrow[hr];
            }
          }
        }
        bar_named(2 + mt, kMtThreads);
        if (ng == 0) {
#pragma unroll
          for (int hr = 0; hr < 2; ++hr) {
            const int r = g8 + hr * 8;
            const float m1 = mML[(ks * 16 + r) * 2], l1 = mML[(ks * 16 + r) * 2 + 1];
            const float M = fmaxf(mrow[hr], m1);
            const float f0 = (mrow[hr] == -INFINITY) ? 0.f : exp2f(mrow[hr] - M);
            const float f1 = (m1 == -INFINITY) ? 0.f : exp2f(m1 - M);
#pragma unroll
            for (int n = 0; n < HD / 8; ++n) {
              const float2 v =
                  *reinterpret_cast<const float2*>(&mO[(ks * 16 + r) * C::kLdO + n * 8 + 2 * tq]);
              o[n][hr * 2] = o[n][hr * 2] * f0 + v.x * f1;
              o[n][hr * 2 + 1] = o[n][hr * 2 + 1] * f0 + v.y * f1;
            }
            lrow[hr] = lrow[hr] * f0 + l1 * f1;
            mrow[hr] = M;
          }
        }
        bar_named(2 + mt, kMtThreads);
      }
      // ---- merge the 4 key-slice warps of this m-tile (fixed order)
      if (ng == 0) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int r = g8 + hr * 8;
#pragma unroll
        for (int n = 0; n < HD / 8; ++n)
          *reinterpret_cast<float2*>(&mO[(ks * 16 + r) * C::kLdO + n * 8 + 2 * tq]) =
              make_float2(o[n][hr * 2], o[n][hr * 2 + 1]);
        if (tq == 0) {
          mML[(ks * 16 + r) * 2] = mrow[hr];
          mML[(ks * 16 + r) * 2 + 1] = lrow[hr];
        }
      }
      }
      bar_named(2 + mt, kMtThreads);
      const int mtg = it.rblk * MT + mt;                  // m-tile index within the request
      const size_t pbase = (((size_t)it.b * a.n_kv + it.kvh) * a.rb_max + mtg) * a.split_max;
      for (int c = ltid; c < 16 * HD / 4; c += kMtThreads) {
        const int r = (c * 4) / HD, dcol = (c * 4) % HD;
        const int R = row_lo + r;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, mML[(w * 16 + r) * 2]);
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        float Ls = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float mw = mML[(w * 16 + r) * 2];
          const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
          const float4 v = *reinterpret_cast<const float4*>(&mO[(w * 16 + r) * C::kLdO + dcol]);
          O.x += v.x * f;
          O.y += v.y * f;
          O.z += v.z * f;
          O.w += v.w * f;
          Ls += mML[(w * 16 + r) * 2 + 1] * f;
        }
        if (it.n_split == 1) {
          if (R < it.rows_total) {
            const float inv = 1.f / Ls;
            const int j = R / group, hh = R % group;
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
                a.out + (((size_t)(it.qoff + j)) * a.n_q + it.kvh * group + hh) * HD + dcol);
            dst[0] = __floats2bfloat162_rn(O.x * inv, O.y * inv);
            dst[1] = __floats2bfloat162_rn(O.z * inv, O.w * inv);
          }
        } else {
          const size_t pi = (pbase + it.split) * 16 + r;
          *reinterpret_cast<float4*>(&a.part_o[pi * HD + dcol]) = O;
          if (dcol == 0) {
            a.part_ml[pi * 2] = M;
            a.part_ml[pi * 2 + 1] = Ls;
          }
        }
      }
      if (it.n_split > 1) {
        // ---- last split of this m-tile to arrive merges all splits in split order
        __threadfence();
        bar_named(2 + mt, kMtThreads);
        if (ltid == 0) {
          int* cnt = a.done_cnt + ((size_t)it.b * a.n_kv + it.kvh) * a.rb_max + mtg;
          const int prev = atomicAdd(cnt, 1);
          s_last[mt] = (prev == it.n_split - 1);
          if (s_last[mt]) *cnt = 0;   // self-reset for the next launch
        }
        bar_named(2 + mt, kMtThreads);
        if (s_last[mt]) {
          __threadfence();
          for (int c = ltid; c < 16 * HD / 4; c += kMtThreads) {
            const int r = (c * 4) / HD, dcol = (c * 4) % HD;
            const int R = row_lo + r;
            if (R >= it.rows_total) continue;
            const int qp = it.p0 + R / group;
            const int ns = min(it.n_split, qp / a.chunk + 1);   // splits this row can see
            float M = -INFINITY;
            for (int sp = 0; sp < ns; ++sp)
              M = fmaxf(M, __ldcg(&a.part_ml[((pbase + sp) * 16 + r) * 2]));
            float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
            float Ls = 0.f;
            for (int sp = 0; sp < ns; ++sp) {
              const size_t pi = (pbase + sp) * 16 + r;
              const float ms = __ldcg(&a.part_ml[pi * 2]);
              const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
              const float4 v =
                  __ldcg(reinterpret_cast<const float4*>(&a.part_o[pi * HD + dcol]));
              O.x += v.x * f;
              O.y += v.y * f;
              O.z += v.z * f;
              O.w += v.w * f;
              Ls += __ldcg(&a.part_ml[pi * 2 + 1]) * f;
            }
            const float inv = 1.f / Ls;
            const int j = R / group, hh = R % group;
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
                a.out + (((size_t)(it.qoff + j)) * a.n_q + it.kvh * group + hh) * HD + dcol);
            dst[0] = __floats2bfloat162_rn(O.x * inv, O.y * inv);
            dst[1] = __floats2bfloat162_rn(O.z * inv, O.w * inv);
          }
        }
      }
      bar_named(2 + mt, kMtThreads);   // merge area free for the next item
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&iempty[slot]);
  }
}

// ------------------------------------------------------------------------
// Warp-per-item variant.  Every consumer warp owns whole work items (one
// 16-row m-tile of one request's kv head over one key split): it streams the
// item's K/V in 32-key stages through its own TMA ring (issued by its lane 0),
// keeps the online-softmax state of its 16 rows, and writes the output rows
// itself — no cross-warp merge, no named barriers.  Warp slots are laid out
// warp-major across CTAs (slot = warp * grid + cta), so all items of a
// typical launch (B * n_kv <= slots) are in flight at once and the SM-level
// balance problem of CTA-sized items disappears.  Same absolute reduction
// boundaries as the CTA kernel -> bit-identical tokens in verify / prefill /
// AR passes.
template <int HD, int NWARP, int NS>
struct AttnWCfg {
  static constexpr int kKeys = 32;                            // keys per stage
  static constexpr int kBoxes = HD / 64;
  static constexpr int kBoxBytes = kKeys * 128;               // 32 keys x 64 elements
  static constexpr int kStageBytes = 2 * kBoxes * kBoxBytes;  // K + V
  static constexpr int kWarpRing = NS * kStageBytes;
  static constexpr int kQBytes = 16 * HD * 2;
  static constexpr int kSmem = 1024 + NWARP * (kWarpRing + kQBytes) + NWARP * NS * 8 + 64;
};

__device__ __forceinline__ uint32_t swz32(int key, int col) {   // 32-row boxes
  return (uint32_t)((col >> 6) * (32 * 128) + key * 128 + ((((col & 63) >> 3) ^ (key & 7)) << 4));
}

template <int HD, int NWARP, int NS, int NP>
__global__ void __launch_bounds__(NWARP * 32, 1)
k_attn_w(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
         AttnArgs a) {
  // NP warps per item: warp `sub` of the group takes the stages whose
  // absolute index is sub mod NP (batch invariant), merged at the end.
  using C = AttnWCfg<HD, NWARP, NS>;
  static_assert(NWARP % NP == 0, "warp groups");
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * C::kWarpRing;
  __nv_bfloat16* sQ =
      reinterpret_cast<__nv_bfloat16*>(smem + NWARP * C::kWarpRing + warp * C::kQBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NWARP * (C::kWarpRing + C::kQBytes)) +
                   warp * NS;
  if (lane == 0) {
    for (int s2 = 0; s2 < NS; ++s2) mbar_init(&full[s2], 1);
    fence_barrier_init();
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  const int group = a.n_q / a.n_kv;
  const int n_rblk = a.rb_max;                 // 16-row m-tiles per request
  const int n_pairs = a.n_req * a.n_kv;
  const int n_items = n_pairs * a.split_max * n_rblk;
  const int slots = gridDim.x * (NWARP / NP);
  const int g8 = lane >> 2, tq = lane & 3;
  const int pw = warp / NP, sub = warp % NP;
  int g = 0;                                    // this warp's stage counter
  bool waited = false;

  for (int item = pw * gridDim.x + blockIdx.x; item < n_items; item += slots) {
    // (row block, split, request, kv head), row block slowest
    const int rblk = item / (n_pairs * a.split_max);
    int r = item % (n_pairs * a.split_max);
    const int split = r / n_pairs;
    r %= n_pairs;
    const int kvh = r % a.n_kv, b = r / a.n_kv;
    const int nn = a.n_new[b];
    if (nn <= 0) continue;
    const int rows_total = nn * group;
    const int row_lo = rblk * 16;
    if (row_lo >= rows_total) continue;
    const int p0 = a.pos0[b];
    const int kv_len = p0 + nn;
    const int c0 = split * a.chunk;
    if (c0 >= kv_len) continue;
    const int c1 = min(c0 + a.chunk, kv_len);
    const int p_max = p0 + (min(rows_total, row_lo + 16) - 1) / group;
    const int c_end = min(c1, p_max + 1);        // keys past every row's position are no-ops
    const int n_all = (c_end - c0 + C::kKeys - 1) / C::kKeys;   // stages of the item
    const int n_stages = (n_all - sub + NP - 1) / NP;             // this warp's share
    const int row0 = a.layer_row0 + (a.slot[b] * a.n_kv + kvh) * a.ctx_cap;
    const int g_item = g;
    auto issue = [&](int st) {   // local stage st (item stage st*NP+sub) -> slot (g_item+st)%NS
      const int gg = g_item + st;
      const int sl = gg % NS;
      uint8_t* dst = ring + sl * C::kStageBytes;
      const int k0 = c0 + (st * NP + sub) * C::kKeys;
      mbar_arrive_expect_tx(&full[sl], C::kStageBytes);
#pragma unroll
      for (int bx = 0; bx < C::kBoxes; ++bx) {
        tma_load_2d(dst + bx * C::kBoxBytes, &tm_k, &full[sl], bx * 64, row0 + k0, pol);
        tma_load_2d(dst + (C::kBoxes + bx) * C::kBoxBytes, &tm_v, &full[sl], bx * 64,
                    row0 + k0, pol);
      }
    };
    int pre = 0;
    if (!waited) {
      // keys below pos0 were written by earlier rounds: stream them before
      // the QKV epilogue kernel (which writes the new keys and Q) finishes
      while (pre < NS && pre < n_stages && c0 + (pre * NP + sub + 1) * C::kKeys <= p0) ++pre;
      if (lane == 0)
        for (int st = 0; st < pre; ++st) issue(st);
      pdl_wait();
      pdl_trigger();
      waited = true;
    }
    if (lane == 0)
      for (int st = pre; st < NS && st < n_stages; ++st) issue(st);
    // ---- Q rows of this m-tile -> smem -> fragments
    for (int c = lane; c < 16 * (HD / 8); c += 32) {
      const int rr = c / (HD / 8), ch = c % (HD / 8);
      const int R = row_lo + rr;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (R < rows_total) {
        const int j = R / group, hh = R % group;
        v = *reinterpret_cast<const uint4*>(
            a.q + (((size_t)(a.q_off[b] + j) * a.n_q) + kvh * group + hh) * HD + ch * 8);
      }
      *reinterpret_cast<uint4*>(sQ + rr * HD + ((ch ^ (rr & 7)) * 8)) = v;   // 16B-chunk swizzle
    }
    __syncwarp();
    uint32_t qf[HD / 16][4];
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      const int rr = lane & 15, ch = kk * 2 + (lane >> 4);
      ldsm_x4(smem_u32(sQ + rr * HD + ((ch ^ (rr & 7)) * 8)), qf[kk][0], qf[kk][1], qf[kk][2],
              qf[kk][3]);
    }
    float o[HD / 8][4];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[n][e] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    int qpos[2];
    bool qvalid[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int R = row_lo + g8 + hr * 8;
      qvalid[hr] = R < rows_total;
      qpos[hr] = p0 + (qvalid[hr] ? R / group : 0);
    }
    const int mi = lane >> 3;
    for (int st = 0; st < n_stages; ++st, ++g) {
      const int sl = g % NS;
      mbar_wait(&full[sl], (uint32_t)(g / NS) & 1u);
      const uint32_t sK = smem_u32(ring + sl * C::kStageBytes);
      const uint32_t sV = sK + C::kBoxes * C::kBoxBytes;
      const int kb = c0 + (st * NP + sub) * C::kKeys;
#pragma unroll
      for (int half16 = 0; half16 < 2; ++half16) {   // two 16-key steps per stage
        const int kofs = half16 * 16;
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        float t0[4] = {0.f, 0.f, 0.f, 0.f}, t1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          uint32_t b0, b1, b2, b3;
          const int key = kofs + (mi >> 1) * 8 + (lane & 7);
          ldsm_x4(sK + swz32(key, kk * 16 + (mi & 1) * 8), b0, b1, b2, b3);
          if (kk & 1) {
            mma16816(t0, qf[kk], b0, b1);
            mma16816(t1, qf[kk], b2, b3);
          } else {
            mma16816(s0, qf[kk], b0, b1);
            mma16816(s1, qf[kk], b2, b3);
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s0[e] += t0[e];
          s1[e] += t1[e];
        }
        const int kb16 = kb + kofs;
        float p[2][4];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          float v[4] = {s0[hr * 2], s0[hr * 2 + 1], s1[hr * 2], s1[hr * 2 + 1]};
          float mx = -INFINITY;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = kb16 + (e >> 1) * 8 + 2 * tq + (e & 1);
            v[e] *= a.scale_log2;
            if (!qvalid[hr] || key > qpos[hr]) v[e] = -INFINITY;
            mx = fmaxf(mx, v[e]);
          }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          const float m_new = fmaxf(mrow[hr], mx);
          const float corr = (m_new == -INFINITY) ? 1.f : exp2f(mrow[hr] - m_new);
          float rs = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            p[hr][e] = (v[e] == -INFINITY) ? 0.f : exp2f(v[e] - m_new);
            rs += p[hr][e];
          }
          rs += __shfl_xor_sync(0xffffffffu, rs, 1);
          rs += __shfl_xor_sync(0xffffffffu, rs, 2);
          lrow[hr] = lrow[hr] * corr + rs;
          mrow[hr] = m_new;
#pragma unroll
          for (int n = 0; n < HD / 8; ++n) {
            o[n][hr * 2] *= corr;
            o[n][hr * 2 + 1] *= corr;
          }
        }
        const uint32_t pa[4] = {pack_bf16(p[0][0], p[0][1]), pack_bf16(p[1][0], p[1][1]),
                                pack_bf16(p[0][2], p[0][3]), pack_bf16(p[1][2], p[1][3])};
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          uint32_t b0, b1, b2, b3;
          const int key = kofs + (mi & 1) * 8 + (lane & 7);
          ldsm_x4_t(sV + swz32(key, dp * 16 + (mi >> 1) * 8), b0, b1, b2, b3);
          mma16816(o[2 * dp], pa, b0, b1);
          mma16816(o[2 * dp + 1], pa, b2, b3);
        }
      }
      // every lane is done with this slot: refill it with stage st + NS
      __syncwarp();
      fence_proxy_async_smem();
      if (lane == 0 && st + NS < n_stages) issue(st + NS);
    }
    g = g_item + n_stages;
    if (NP == 2) {
      // fold warp 1's state into warp 0's (same lane layout) through warp 1's
      // now idle ring, fixed order (stages of parity 0, then parity 1)
      float* xch = reinterpret_cast<float*>(smem + (pw * NP + 1) * C::kWarpRing);
      if (sub == 1) {
#pragma unroll
        for (int n = 0; n < HD / 8; ++n)
#pragma unroll
          for (int e = 0; e < 4; ++e) xch[(n * 4 + e) * 32 + lane] = o[n][e];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          xch[(HD / 2 + hr * 2) * 32 + lane] = mrow[hr];
          xch[(HD / 2 + hr * 2 + 1) * 32 + lane] = lrow[hr];
        }
      }
      bar_named(1 + pw, 64);
      if (sub == 0) {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
          const float m1 = xch[(HD / 2 + hr * 2) * 32 + lane];
          const float l1 = xch[(HD / 2 + hr * 2 + 1) * 32 + lane];
          const float M = fmaxf(mrow[hr], m1);
          const float f0 = (mrow[hr] == -INFINITY) ? 0.f : exp2f(mrow[hr] - M);
          const float f1 = (m1 == -INFINITY) ? 0.f : exp2f(m1 - M);
#pragma unroll
          for (int n = 0; n < HD / 8; ++n) {
            o[n][hr * 2] = o[n][hr * 2] * f0 + xch[(n * 4 + hr * 2) * 32 + lane] * f1;
            o[n][hr * 2 + 1] = o[n][hr * 2 + 1] * f0 + xch[(n * 4 + hr * 2 + 1) * 32 + lane] * f1;
          }
          lrow[hr] = lrow[hr] * f0 + l1 * f1;
          mrow[hr] = M;
        }
      }
      bar_named(1 + pw, 64);   // warp 1's ring is free again
      fence_proxy_async_smem();
      if (sub == 1) continue;
    }
    // ---- output: this warp holds the whole split of its 16 rows
    const int n_split = (kv_len + a.chunk - 1) / a.chunk;
    const int qoff = a.q_off[b];
    if (n_split == 1) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int R = row_lo + g8 + hr * 8;
        if (R >= rows_total) continue;
        const float inv = 1.f / lrow[hr];
        const int j = R / group, hh = R % group;
        __nv_bfloat16* dst = a.out + (((size_t)(qoff + j)) * a.n_q + kvh * group + hh) * HD;
#pragma unroll
        for (int n = 0; n < HD / 8; ++n)
          *reinterpret_cast<__nv_bfloat162*>(dst + n * 8 + 2 * tq) =
              __floats2bfloat162_rn(o[n][hr * 2] * inv, o[n][hr * 2 + 1] * inv);
      }
      continue;
    }
    if (a.debug & 2) continue;   // diagnostics: no partial write / merge
    // multi-split (contexts past a.chunk): partial + last-arriver merge in split order
    const size_t pbase = (((size_t)b * a.n_kv + kvh) * a.rb_max + rblk) * a.split_max;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int rr = g8 + hr * 8;
      const size_t pi = (pbase + split) * 16 + rr;
#pragma unroll
      for (int n = 0; n < HD / 8; ++n)
        *reinterpret_cast<float2*>(&a.part_o[pi * HD + n * 8 + 2 * tq]) =
            make_float2(o[n][hr * 2], o[n][hr * 2 + 1]);
      if (tq == 0) {
        a.part_ml[pi * 2] = mrow[hr];
        a.part_ml[pi * 2 + 1] = lrow[hr];
      }
    }
    if (!(a.debug & 8)) __threadfence();   // debug 8: no fence (diagnostics only)
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      int* cnt = a.done_cnt + ((size_t)b * a.n_kv + kvh) * a.rb_max + rblk;
      const int prev = atomicAdd(cnt, 1);
      last = prev == n_split - 1;
      if (last) *cnt = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last || (a.debug & 4)) continue;   // debug 4: no merge (diagnostics only)
    __threadfence();
    // fixed trip count (16 * HD / 4 / 32): unrolled so every iteration's
    // partial loads are in flight together instead of one L2 round trip chain
    // per iteration (the merge was most of a split item's time)
#pragma unroll
    for (int c = lane; c < 16 * HD / 4; c += 32) {
      const int rr = (c * 4) / HD, dcol = (c * 4) % HD;
      const int R = row_lo + rr;
      if (R >= rows_total) continue;
      const int qp = p0 + R / group;
      const int ns = min(n_split, qp / a.chunk + 1);
      float M = -INFINITY;
      for (int sp = 0; sp < ns; ++sp)
        M = fmaxf(M, __ldcg(&a.part_ml[((pbase + sp) * 16 + rr) * 2]));
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
      float Ls = 0.f;
      for (int sp = 0; sp < ns; ++sp) {
        const size_t pi = (pbase + sp) * 16 + rr;
        const float ms = __ldcg(&a.part_ml[pi * 2]);
        const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
        const float4 v = __ldcg(reinterpret_cast<const float4*>(&a.part_o[pi * HD + dcol]));
        O.x += v.x * f;
        O.y += v.y * f;
        O.z += v.z * f;
        O.w += v.w * f;
        Ls += __ldcg(&a.part_ml[pi * 2 + 1]) * f;
      }
      const float inv = 1.f / Ls;
      const int j = R / group, hh = R % group;
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
          a.out + (((size_t)(qoff + j)) * a.n_q + kvh * group + hh) * HD + dcol);
      dst[0] = __floats2bfloat162_rn(O.x * inv, O.y * inv);
      dst[1] = __floats2bfloat162_rn(O.z * inv, O.w * inv);
    }
  }
  if (!waited) {
    pdl_wait();
    pdl_trigger();
  }
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

template <int HD, int MT, int NG, int NS>
static int launch_attn_t(const CUtensorMap& tk, const CUtensorMap& tv, AttnArgs a,
                         cudaStream_t s) {
  using C = AttnCfg<HD, MT, NG, NS>;
  static_assert(C::kSmem <= 232448, "attention smem");
  static bool cfg = false;
  if (!cfg) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_attn<HD, MT, NG, NS>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    cfg = true;
  }
  static const int per_sm = [] {
    int n = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_attn<HD, MT, NG, NS>, C::kThreads,
                                                  C::kSmem);
    return n < 1 ? 1 : n;
  }();
  a.rb_max = (a.rb_max + MT - 1) / MT * MT;   // whole row blocks of MT m-tiles
  const int items = a.n_req * a.n_kv * (a.rb_max / MT) * a.split_max;
  const int grid = cap_grid(std::min(items, per_sm * num_sms()));
  SPECTRE_LAUNCH_PDL("k_attn", k_attn<HD, MT, NG, NS>, dim3(grid), dim3(C::kThreads), C::kSmem,
                     s, tk, tv, a);
  return SPECTRE_OK;
}

static bool attn_two_per_sm() {
  static const bool v = [] {
    const char* e = getenv("SPECTRE_ATTN_2CTA");
    return e ? atoi(e) != 0 : false;
  }();
  return v;
}

static int attn_mtiles_cfg() {
  static const int v = [] {
    const char* e = getenv("SPECTRE_ATTN_MT");   // 0: one m-tile per item (default)
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int HD, int NWARP, int NS, int NP>
static int launch_attn_w_t(const CUtensorMap& tk, const CUtensorMap& tv, AttnArgs a,
                           int rows_per_req, cudaStream_t s) {
  using C = AttnWCfg<HD, NWARP, NS>;
  static_assert(C::kSmem <= 232448, "attention smem");
  static bool cfg = false;
  if (!cfg) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_attn_w<HD, NWARP, NS, NP>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    cfg = true;
  }
  a.rb_max = (rows_per_req + 15) / 16;
  SPECTRE_LAUNCH_PDL("k_attn_w", k_attn_w<HD, NWARP, NS, NP>, dim3(cap_grid(num_sms())),
                     dim3(NWARP * 32), C::kSmem, s, tk, tv, a);
  return SPECTRE_OK;
}

// Warp-per-item attention (32-key TMA boxes: tk32 / tv32).
int launch_attention_w(const CUtensorMap& tk32, const CUtensorMap& tv32, const AttnArgs& a,
                       int hd, int rows_per_req, cudaStream_t s) {
  if (a.chunk % 64 || a.chunk <= 0) return arg_fail("attention: chunk must be a multiple of 64");
  static const int v = [] {
    const char* e = getenv("SPECTRE_ATTN_WPAIR");   // warps per item (1 or 2)
    return e ? atoi(e) : 2;
  }();
  if (hd == 128) return launch_attn_w_t<128, 4, 3, 1>(tk32, tv32, a, rows_per_req, s);
  if (hd == 64) {
    if (v == 1) return launch_attn_w_t<64, 8, 3, 1>(tk32, tv32, a, rows_per_req, s);
    return launch_attn_w_t<64, 8, 3, 2>(tk32, tv32, a, rows_per_req, s);
  }
  return arg_fail("attention: head_dim must be 64 or 128");
}

// rows_per_req = the most query rows any request can have in this launch
// (new tokens x GQA group).  Default: one 16-row m-tile per item with two
// stage groups (requests with more rows get several row blocks);
// SPECTRE_ATTN_MT=1 covers all rows of a request in one item instead.
int launch_attention(const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& a, int hd,
                     int rows_per_req, cudaStream_t s) {
  const int mtiles = attn_mtiles_cfg() ? (rows_per_req + 15) / 16 : 1;
  if (a.chunk % 64 || a.chunk <= 0) return arg_fail("attention: chunk must be a multiple of 64");
  const bool two = attn_two_per_sm();
  if (hd == 128) {
    if (mtiles <= 1)
      return two ? launch_attn_t<128, 1, 2, 2>(tk, tv, a, s) : launch_attn_t<128, 1, 2, 4>(tk, tv, a, s);
    return launch_attn_t<128, 2, 1, 4>(tk, tv, a, s);
  }
  if (hd == 64) {
    if (mtiles <= 1)
      return two ? launch_attn_t<64, 1, 2, 4>(tk, tv, a, s) : launch_attn_t<64, 1, 2, 12>(tk, tv, a, s);
    if (mtiles <= 2) return launch_attn_t<64, 2, 1, 8>(tk, tv, a, s);
    return launch_attn_t<64, 3, 1, 8>(tk, tv, a, s);
  }
  return arg_fail("attention: head_dim must be 64 or 128");
}

}  // namespace spectre
