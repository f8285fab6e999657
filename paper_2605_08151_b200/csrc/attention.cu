// attention.cu — causal attention of a packed ragged batch of new tokens over
// each request's KV cache: the target's gamma-token verify pass, the draft's
// decode steps (one token, or a short catch-up after a rollback) and prefill
// chunks all use this kernel.
//
// HBM-bound (bytes = sum_req ctx * n_kv * hd * 2 * 2 per layer), so
// the design is about keeping every KV stream in flight at once:
//
//   * warp per work item (one 16-row m-tile of one request's kv head over one
//     key split); warp slots are laid out warp-major across the persistent
//     CTAs, so all B * n_kv items of a launch run concurrently and there is
//     no SM-level balance problem and no cross-warp merge;
//   * each warp streams its item's K/V in 32-key stages through its own
//     3-deep TMA ring (2-D tensor map over the whole cache, 128-byte
//     swizzle; keys below pos0 — written by earlier rounds — are requested
//     before griddepcontrol.wait);
//   * S = Q K^T and O += P V on mma.sync m16n8k16 from ldmatrix'ed swizzled
//     tiles (the per-kv-head row count, gamma x group = 16, is below a
//     tcgen05 tile), online softmax in the log2 domain;
//   * the draft (head_dim 64, one token per request) uses two warps per item
//     taking the stages of even / odd absolute index, folded through the
//     idle ring; contexts past the key split merge partials in split order.
//
// Every reduction boundary is an absolute key position (split, stage), so a
// token's output is bit-identical whether it is computed in a verify pass, a
// prefill chunk or plain autoregressive decode.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "model_kernels.cuh"
#include "ptx.cuh"

namespace spectre {

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
  static constexpr int kSmem = 1024 + NWARP * kWarpRing + NWARP * NS * 8 + 64;
};

__device__ __forceinline__ uint32_t swz32(int key, int col) {   // 32-row boxes
  return (uint32_t)((col >> 6) * (32 * 128) + key * 128 + ((((col & 63) >> 3) ^ (key & 7)) << 4));
}

// The work-item loop of one attention warp (also run by the draft chain's
// epilogue warps as its attention phase, chain.cu).  ring: this warp's NS-stage
// K/V ring (NS * kStageBytes, 1024-aligned), full: its NS initialised
// mbarriers; NP == 2: xch is the ring of the group's second warp (the state
// exchange buffer) and bar_id a named barrier for the pair.  warps_per_cta:
// attention warps per CTA (slot layout).  *waited: griddepcontrol.wait done;
// before it only keys of earlier rounds (below pos0) are streamed.
template <int HD, int NS, int NP>
__device__ void attn_warp_items(const CUtensorMap* tm_k, const CUtensorMap* tm_v,
                                const AttnArgs& a, int warp, int warps_per_cta, uint8_t* ring,
                                uint64_t* full, uint8_t* xch_ring, int bar_id, bool* waited_io) {
  using C = AttnWCfg<HD, 1, NS>;
  using namespace ptx;
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  const int group = a.n_q / a.n_kv;
  const int n_rblk = a.rb_max;                 // 16-row m-tiles per request
  const int n_pairs = a.n_req * a.n_kv;
  const int n_items = n_pairs * a.split_max * n_rblk;
  const int slots = gridDim.x * (warps_per_cta / NP);
  const int g8 = lane >> 2, tq = lane & 3;
  const int pw = warp / NP, sub = warp % NP;
  int g = 0;                                    // this warp's stage counter
  bool waited = *waited_io;

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
        tma_load_2d(dst + bx * C::kBoxBytes, tm_k, &full[sl], bx * 64, row0 + k0, pol);
        tma_load_2d(dst + (C::kBoxes + bx) * C::kBoxBytes, tm_v, &full[sl], bx * 64,
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
    // ---- Q fragments of this m-tile straight from global (m16n8k16 A layout:
    // regs 0 / 1 rows g8 / g8 + 8 at cols 2tq, regs 2 / 3 the same at cols 2tq + 8)
    uint32_t qf[HD / 16][4];
    {
      const __nv_bfloat16* qrow[2];
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int R = row_lo + g8 + hr * 8;
        qrow[hr] = nullptr;
        if (R < rows_total) {
          const int j = R / group, hh = R % group;
          qrow[hr] = a.q + (((size_t)(a.q_off[b] + j) * a.n_q) + kvh * group + hh) * HD;
        }
      }
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __nv_bfloat16* qr = qrow[e & 1];
          qf[kk][e] = qr ? *reinterpret_cast<const uint32_t*>(qr + kk * 16 + (e >> 1) * 8 + 2 * tq)
                         : 0u;
        }
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
      float* xch = reinterpret_cast<float*>(xch_ring);
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
      bar_named(bar_id, 64);
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
      bar_named(bar_id, 64);   // warp 1's ring is free again
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
  *waited_io = waited;
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
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NWARP * C::kWarpRing) + warp * NS;
  if (lane == 0) {
    for (int s2 = 0; s2 < NS; ++s2) mbar_init(&full[s2], 1);
    fence_barrier_init();
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  __syncwarp();
  bool waited = false;
  const int pw = warp / NP;
  attn_warp_items<HD, NS, NP>(&tm_k, &tm_v, a, warp, NWARP, smem + warp * C::kWarpRing, full,
                              smem + (pw * NP + NP - 1) * C::kWarpRing, 1 + pw, &waited);
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
  SPECTRE_LAUNCH_PDL("k_attn_w", k_attn_w<HD, NWARP, NS, NP>, dim3(num_sms()),
                     dim3(NWARP * 32), C::kSmem, s, tk, tv, a);
  return SPECTRE_OK;
}

// Warp-per-item attention (32-key TMA boxes: tk32 / tv32).
int launch_attention_w(const CUtensorMap& tk32, const CUtensorMap& tv32, const AttnArgs& a,
                       int hd, int rows_per_req, cudaStream_t s) {
  if (a.chunk % 64 || a.chunk <= 0) return arg_fail("attention: chunk must be a multiple of 64");
  // hd 128: 7 warps with 2-stage rings (one more warp per SM sub-partition
  // than 4 warps x 3 stages: the kernel is warp-latency bound, 1 warp per
  // SMSP issued every ~3.8 cycles; ncu r02f): config 3 (4,096 m-tile items)
  // 107.0 -> 90.3 us per launch, config 2 34.4 -> 33.4 us; 6 x 2: 103.3 / 33.6
  if (hd == 128) return launch_attn_w_t<128, 7, 2, 1>(tk32, tv32, a, rows_per_req, s);
  if (hd == 64) {
    // two warps per item (even / odd stages) while the (request, kv head,
    // key split) items of a decode step fit one wave of warp pairs (config 2:
    // 512), else one warp per item (config 3's B=256: 2,048 items; 40.5 ->
    // 35.1 us per launch).  Decided by the request count, not by this
    // forward's row bound (a catch-up step's extra m-tiles are mostly empty),
    // so one engine always uses one variant.
    const long long items = (long long)a.n_req * a.n_kv * a.split_max;
    // (one warp per item: 14 warps with 2-stage rings, 54.2 -> 48.6 us at
    // config 3; 12 x 2: 59.5 us)
    if (2 * items > 8ll * num_sms())
      return launch_attn_w_t<64, 14, 2, 1>(tk32, tv32, a, rows_per_req, s);
    return launch_attn_w_t<64, 8, 3, 2>(tk32, tv32, a, rows_per_req, s);
  }
  return arg_fail("attention: head_dim must be 64 or 128");
}

}  // namespace spectre
