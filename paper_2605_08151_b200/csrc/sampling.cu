// sampling.cu — temperature sampling and speculative rejection sampling
// (BASELINE config 3, T = 1).  The reference implements greedy verification
// only; this is the standard lossless speculative-sampling rule
// (SURVEY §8c): accept draft token x at position i with probability
// min(1, p_i(x) / q_i(x)); at the first rejection resample from
// norm(max(0, p_i - q_i)); if every candidate survives, the bonus token is
// drawn from p_{m}.  p = softmax(target logits / T), q = softmax(draft
// logits / T).
//
// Every draw is a Gumbel-max: argmax_k (log w_k + G_k) with G_k = -log(-log U_k)
// is an exact sample from w / sum(w), so a draw is ONE coalesced pass over the
// row (no CDF, no scan), fused with the online (max, sum exp) statistics the
// ratio tests need.  U_k is counter-based (SplitMix64 of a per-draw key and k),
// the key is (seed, purpose, request slot, output position): results are
// reproducible and independent of batch composition, and an AR draw and a
// speculative bonus draw at the same (request, position) use the same stream.
//
// Logits are materialised in fp32 by the lm_head GEMM (partial epilogue, one
// split) and read once per pass with float4 loads.  Every per-row reduction has
// a fixed order (per-thread strided order, then a fixed block tree).
#include <cuda_bf16.h>

#include "common.cuh"
#include "engine_state.cuh"
#include "protocol.cuh"

namespace spectre {

constexpr int kSampThreads = 512;
constexpr int kSampWarps = kSampThreads / 32;
enum : uint64_t { kStreamDraftSample = 4, kStreamAccept = 5, kStreamResample = 6,
                  kStreamRowSample = 7 };

__device__ __forceinline__ double u53s(uint64_t h) {
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

// G_k for element k of the draw keyed `key`: SplitMix64 state key + (k+1)*phi,
// 24-bit uniform in (0, 1), -log(-log U)
__device__ __forceinline__ float gumbel(uint64_t key, int k) {
  uint64_t z = key + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  const float u = ((float)(uint32_t)(z >> 40) + 0.5f) * (1.0f / 16777216.0f);
  return -__logf(-__logf(u));
}

// One pass's running state: online (max, sum exp) of x = logit / T and the
// Gumbel-max candidate (g, index).
struct RowAcc {
  float m, s, g;
  int gi;
  __device__ __forceinline__ void init() {
    m = -INFINITY;
    s = 0.f;
    g = -INFINITY;
    gi = 0x7fffffff;
  }
  __device__ __forceinline__ void add_stat(float x) {
    if (x > m) {
      s = s * __expf(m - x) + 1.f;
      m = x;
    } else {
      s += __expf(x - m);
    }
  }
  __device__ __forceinline__ void add_draw(float lw, int k) {   // log weight + Gumbel
    if (lw > g || (lw == g && k < gi)) {
      g = lw;
      gi = k;
    }
  }
  __device__ __forceinline__ void merge(const RowAcc& o) {
    if (o.m > m) {
      s = (m == -INFINITY ? 0.f : s * __expf(m - o.m)) + o.s;
      m = o.m;
    } else if (o.m != -INFINITY) {
      s += o.s * __expf(o.m - m);
    }
    add_draw(o.g, o.gi);
  }
};

// Fixed-tree block merge (xor butterfly in each warp, then warp 0 over the
// warps in index order); every thread gets the result.
__device__ RowAcc block_merge(RowAcc a, RowAcc* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    RowAcc b;
    b.m = __shfl_xor_sync(0xffffffffu, a.m, o);
    b.s = __shfl_xor_sync(0xffffffffu, a.s, o);
    b.g = __shfl_xor_sync(0xffffffffu, a.g, o);
    b.gi = __shfl_xor_sync(0xffffffffu, a.gi, o);
    // lanes l and l^o merge in the same order (lower lane first): identical results
    if (threadIdx.x & o) {
      RowAcc lo = b;
      lo.merge(a);
      a = lo;
    } else {
      a.merge(b);
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    RowAcc r = sh[0];
    for (int i = 1; i < kSampWarps; ++i) r.merge(sh[i]);
    sh[kSampWarps] = r;
  }
  __syncthreads();
  const RowAcc r = sh[kSampWarps];
  __syncthreads();
  return r;
}

// Statistics of x = l / T over a row and a Gumbel-max draw from softmax(x)
// (key 0: statistics only); kCopy also streams the row to `dst`.
template <bool kCopy, bool kDraw>
__device__ RowAcc row_pass(const float* __restrict__ l, int V, float inv_t, uint64_t key,
                           float* __restrict__ dst, RowAcc* sh) {
  RowAcc a;
  a.init();
  const int V4 = V >> 2;
  const float4* l4 = reinterpret_cast<const float4*>(l);
  // kB float4 loads of a thread in flight before any of them is consumed
  // (the per-element work would otherwise serialise one L2 / HBM round trip
  // per few loads); element order per thread is unchanged
  constexpr int kB = 8;
  int v = threadIdx.x;
  for (; v + (kB - 1) * kSampThreads < V4; v += kB * kSampThreads) {
    float4 q[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) q[u] = __ldg(l4 + v + u * kSampThreads);
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int vv = v + u * kSampThreads;
      if (kCopy) reinterpret_cast<float4*>(dst)[vv] = q[u];
      const float x[4] = {q[u].x * inv_t, q[u].y * inv_t, q[u].z * inv_t, q[u].w * inv_t};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a.add_stat(x[e]);
        if (kDraw) a.add_draw(x[e] + gumbel(key, 4 * vv + e), 4 * vv + e);
      }
    }
  }
  for (; v < V4; v += kSampThreads) {
    const float4 q = __ldg(l4 + v);
    if (kCopy) reinterpret_cast<float4*>(dst)[v] = q;
    const float x[4] = {q.x * inv_t, q.y * inv_t, q.z * inv_t, q.w * inv_t};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      a.add_stat(x[e]);
      if (kDraw) a.add_draw(x[e] + gumbel(key, 4 * v + e), 4 * v + e);
    }
  }
  for (int k = 4 * V4 + threadIdx.x; k < V; k += kSampThreads) {   // tail (V % 4)
    const float q = l[k];
    if (kCopy) dst[k] = q;
    a.add_stat(q * inv_t);
    if (kDraw) a.add_draw(q * inv_t + gumbel(key, k), k);
  }
  return block_merge(a, sh);
}

// ------------------------------------------------ per-row sample + stats
// Every live row of a forward: (m, s) of logits/T into stats[row]; the last
// row of each request also draws a token from p into out_tok[row] (admission,
// token 0 of the output, AR decoding, the bonus token of a verify pass — the
// other rows of a verify pass only need their statistics).  Key: (seed, 7,
// request slot, input position).
__device__ __forceinline__ uint64_t row_key(uint64_t seed, const BatchDev& bt, int row) {
  return mix64(seed, kStreamRowSample, (uint64_t)bt.slot[row], (uint64_t)bt.pos[row]);
}

__global__ void __launch_bounds__(kSampThreads) k_sample_rows(
    const float* __restrict__ logits, int V, BatchDev bt, float inv_t, uint64_t seed,
    float2* __restrict__ stats) {
  pdl_wait();
  pdl_trigger();
  __shared__ RowAcc sh[kSampWarps + 1];
  const int T = *bt.t_dev;
  for (int row = blockIdx.x; row < T; row += gridDim.x) {
    const int b = bt.slot[row];
    const float* l = logits + (size_t)row * V;
    if (row == bt.q_off[b] + bt.n_new[b] - 1) {
      const RowAcc r = row_pass<false, true>(l, V, inv_t, row_key(seed, bt, row), nullptr, sh);
      if (threadIdx.x == 0) {
        stats[row] = make_float2(r.m, r.s);
        bt.out_tok[row] = r.gi;
      }
    } else {
      const RowAcc r = row_pass<false, false>(l, V, inv_t, 0, nullptr, sh);
      if (threadIdx.x == 0) stats[row] = make_float2(r.m, r.s);
    }
  }
}

// ------------------------------------------------ draft sampling step
// The draft's token for request b at draft-history position hl = a q-draw
// from its last row; the logits row (streamed in the same pass) and its
// stats are kept in q-store slot hl % W (the accept step needs q at every
// candidate position).
__global__ void __launch_bounds__(kSampThreads) k_draft_sample(
    DecodeStateDev s, BatchDev bt, const float* __restrict__ logits, int V, float inv_t,
    float* __restrict__ qstore, float2* __restrict__ qstat, int W) {
  pdl_wait();
  pdl_trigger();
  __shared__ RowAcc sh[kSampWarps + 1];
  const int b = blockIdx.x;
  if (b >= s.n_req || bt.n_new[b] <= 0) return;
  if (!(s.gen_count[b] > 0 && s.gen_done[b] < s.gen_count[b])) return;
  const int row = bt.q_off[b] + bt.n_new[b] - 1;
  const int hl = s.hist_len[b];                       // output position being drafted
  const int slot = hl % W;
  const uint64_t key = mix64(s.seed, kStreamDraftSample, (uint64_t)b, (uint64_t)hl);
  const RowAcc r = row_pass<true, true>(logits + (size_t)row * V, V, inv_t, key,
                                        qstore + ((size_t)b * W + slot) * V, sh);
  if (threadIdx.x == 0) {
    qstat[b * W + slot] = make_float2(r.m, r.s);
    bt.out_tok[row] = r.gi;
  }
}

// ------------------------------------------------ speculative rejection sampling
// One CTA per verified request: accepted count a and the bonus/resample
// token, consumed by k_accept (which then runs the reference's commit /
// rollback / suffix-reuse rules unchanged).
__global__ void __launch_bounds__(kSampThreads) k_accept_sample(
    DecodeStateDev s, BatchDev bt, const float* __restrict__ logits, int V, float inv_t,
    const float2* __restrict__ tstat, const float* __restrict__ qstore,
    const float2* __restrict__ qstat, int W, int* __restrict__ out_a,
    int* __restrict__ out_bonus) {
  pdl_wait();
  pdl_trigger();
  __shared__ RowAcc sh[kSampWarps + 1];
  const int b = blockIdx.x;
  if (b >= s.n_req || s.vkind[b] == 0) return;
  const int m = s.vcand_n[b];
  const int row0 = bt.q_off[b];
  const int pos = s.pos[b];
  const uint64_t* cand = s.cand_tok + (size_t)b * (s.gamma + 1);
  int a = 0;
  for (; a < m; ++a) {   // uniform across the CTA
    const int x = (int)cand[a];
    const float2 ts = tstat[row0 + a];
    const float p = __expf(logits[(size_t)(row0 + a) * V + x] * inv_t - ts.x) / ts.y;
    const int slot = (pos + a) % W;
    const float2 qs = qstat[b * W + slot];
    const float q = __expf(qstore[((size_t)b * W + slot) * V + x] * inv_t - qs.x) / qs.y;
    const double u = u53s(mix64(s.seed, kStreamAccept, (uint64_t)b, (uint64_t)(pos + a)));
    if (!(u * (double)q < (double)p)) break;   // reject with probability 1 - p/q
  }
  const float* lp = logits + (size_t)(row0 + a) * V;
  const float2 ts = tstat[row0 + a];
  // Parallel rounds: the draft's fresh speculation starts AT the bonus position
  // (its head token is a proposal for the token this round emits).  It goes
  // through the same min(1, p/q) test instead of being matched against an
  // independently sampled bonus (probability sum_x p(x) q(x), ~0 at V = 128k);
  // accepted, it is the bonus and the rest of the segment stays cached;
  // rejected, the bonus is drawn from norm(max(0, p - q)) — whose weight at the
  // head token is 0, so k_accept's reuse rule (head == bonus) then discards the
  // segment.  The emitted token is distributed as p either way.
  bool head = false;
  if (a == m) {
    const bool fresh = s.r_serial[b] == s.q_serial[b] && s.r_round[b] == s.q_round[b];
    if (s.ctrl->mode == 'P' && fresh && s.gen_count[b] > 0 && s.gen_done[b] > 0 &&
        s.gen_start[b] == pos + a) {
      const int x = (int)s.hist[(size_t)b * s.hist_cap + s.gen_start[b]];
      const float p = __expf(lp[x] * inv_t - ts.x) / ts.y;
      const int slot = (pos + a) % W;
      const float2 qs = qstat[b * W + slot];
      const float q = __expf(qstore[((size_t)b * W + slot) * V + x] * inv_t - qs.x) / qs.y;
      const double u = u53s(mix64(s.seed, kStreamAccept, (uint64_t)b, (uint64_t)(pos + a)));
      if (u * (double)q < (double)p) {
        if (threadIdx.x == 0) {
          out_a[b] = a;
          out_bonus[b] = x;
        }
        return;
      }
      head = true;   // rejected: residual resample against the head's q
    }
  }
  // every candidate accepted: the bonus is row m's own draw from p (k_sample_rows)
  int y = a < m ? -1 : bt.out_tok[row0 + a];
  if (a < m || head) {
    // resample from norm(max(0, p - q)) at the rejected position: Gumbel-max
    // over log(p - q) where positive; an empty residual (p == q) keeps row a's
    // own draw from p (independent of the acceptance uniforms)
    const int slot = (pos + a) % W;
    const float* lq = qstore + ((size_t)b * W + slot) * V;
    const float2 qs = qstat[b * W + slot];
    const uint64_t key = mix64(s.seed, kStreamResample, (uint64_t)b, (uint64_t)(pos + a));
    const float4* p4 = reinterpret_cast<const float4*>(lp);
    const float4* q4 = reinterpret_cast<const float4*>(lq);
    const float inv_sp = 1.f / ts.y, inv_sq = 1.f / qs.y;
    RowAcc acc;
    acc.init();
    auto one = [&](float lpk, float lqk, int k) {
      const float w = __expf(lpk * inv_t - ts.x) * inv_sp - __expf(lqk * inv_t - qs.x) * inv_sq;
      if (w > 0.f) acc.add_draw(__logf(w) + gumbel(key, k), k);
    };
    const int V4 = V >> 2;
#pragma unroll 2
    for (int v = threadIdx.x; v < V4; v += kSampThreads) {
      const float4 pp = __ldg(p4 + v), qq = __ldg(q4 + v);
      one(pp.x, qq.x, 4 * v);
      one(pp.y, qq.y, 4 * v + 1);
      one(pp.z, qq.z, 4 * v + 2);
      one(pp.w, qq.w, 4 * v + 3);
    }
    for (int k = 4 * V4 + threadIdx.x; k < V; k += kSampThreads) one(lp[k], lq[k], k);
    const RowAcc r = block_merge(acc, sh);
    if (r.gi != 0x7fffffff) {
      y = r.gi;
    } else if (y < 0) {
      // empty residual (p == q) below the last row: row a's own draw from p,
      // the one k_sample_rows would have made (same key)
      y = row_pass<false, true>(lp, V, inv_t, row_key(s.seed, bt, row0 + a), nullptr, sh).gi;
    }
  }
  if (threadIdx.x == 0) {
    out_a[b] = a;
    out_bonus[b] = y;
  }
}

// ------------------------------------------------------------------ launchers
int launch_sample_rows(const float* logits, int V, const BatchDev& bt, int t_cap, float inv_t,
                       uint64_t seed, float2* stats, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_sample_rows", k_sample_rows, dim3((t_cap < 296 ? t_cap : 296)),
                     dim3(kSampThreads), 0, s, logits, V, bt, inv_t, seed, stats);
  return SPECTRE_OK;
}
int launch_draft_sample(const DecodeStateDev& st, const BatchDev& bt, const float* logits, int V,
                        float inv_t, float* qstore, float2* qstat, int W, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_draft_sample", k_draft_sample, dim3(st.n_req), dim3(kSampThreads), 0, s,
                     st, bt, logits, V, inv_t, qstore, qstat, W);
  return SPECTRE_OK;
}
int launch_accept_sample(const DecodeStateDev& st, const BatchDev& bt, const float* logits, int V,
                         float inv_t, const float2* tstat, const float* qstore,
                         const float2* qstat, int W, int* out_a, int* out_bonus,
                         cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_accept_sample", k_accept_sample, dim3(st.n_req), dim3(kSampThreads), 0, s,
                     st, bt, logits, V, inv_t, tstat, qstore, qstat, W, out_a, out_bonus);
  return SPECTRE_OK;
}

}  // namespace spectre
