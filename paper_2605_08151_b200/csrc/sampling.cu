// sampling.cu — temperature sampling and speculative rejection sampling
// (BASELINE config 3, T = 1).  The reference implements greedy verification
// only; this is the standard lossless speculative-sampling rule
// (SURVEY §8c): accept draft token x at position i with probability
// min(1, p_i(x) / q_i(x)); at the first rejection resample from
// norm(max(0, p_i - q_i)); if every candidate survives, the bonus token is
// drawn from p_{m}.  p = softmax(target logits / T), q = softmax(draft
// logits / T).  Every random draw is a counter-based uniform keyed by
// (seed, purpose, request, output position): results are reproducible and
// independent of batch composition.
//
// Logits are materialised in fp32 by the lm_head GEMM (partial epilogue, one
// split) — at most rows x V x 4 bytes (B=64, gamma=4: 164 MB), streamed once
// per reduction pass.  Every per-row reduction has a fixed order.
#include <cuda_bf16.h>

#include "common.cuh"
#include "engine_state.cuh"
#include "protocol.cuh"

namespace spectre {

constexpr int kSampThreads = 512;
enum : uint64_t { kStreamDraftSample = 4, kStreamAccept = 5, kStreamResample = 6,
                  kStreamRowSample = 7 };

__device__ __forceinline__ double u53s(uint64_t h) {
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

// Block reductions with a fixed tree (kSampThreads threads).
__device__ __forceinline__ float block_max(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < kSampThreads / 32 ? sh[l] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) sh[32] = v;
  }
  __syncthreads();
  v = sh[32];
  __syncthreads();
  return v;
}
__device__ __forceinline__ float block_sum(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < kSampThreads / 32 ? sh[l] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) sh[32] = v;
  }
  __syncthreads();
  v = sh[32];
  __syncthreads();
  return v;
}

// (max, sum exp) of logits/T over V: a thread owns a contiguous chunk.
struct RowStats {
  float m, s;
};
__device__ RowStats row_stats(const float* __restrict__ l, int V, float inv_t, float* sh) {
  const int per = (V + kSampThreads - 1) / kSampThreads;
  const int b0 = threadIdx.x * per, b1 = min(V, b0 + per);
  float m = -INFINITY;
  for (int y = b0; y < b1; ++y) m = fmaxf(m, l[y] * inv_t);
  m = block_max(m, sh);
  float s = 0.f;
  for (int y = b0; y < b1; ++y) s += __expf(l[y] * inv_t - m);
  s = block_sum(s, sh);
  return {m, s};
}

// Inverse-CDF draw over weights w(y) (>= 0) with total Z: the smallest y with
// cumsum(w)[y] > u*Z.  Chunked: per-thread sums -> block exclusive scan ->
// the owning thread scans its chunk.  `wfn(y)` returns the weight.
template <class W>
__device__ int sample_index(int V, double u, float Z, W wfn, float* sh, int* shi) {
  const int per = (V + kSampThreads - 1) / kSampThreads;
  const int b0 = threadIdx.x * per, b1 = min(V, b0 + per);
  float part = 0.f;
  for (int y = b0; y < b1; ++y) part += wfn(y);
  // inclusive scan of per-thread sums in thread order (fixed)
  sh[threadIdx.x] = part;
  __syncthreads();
  for (int d = 1; d < kSampThreads; d <<= 1) {
    const float x = threadIdx.x >= d ? sh[threadIdx.x - d] : 0.f;
    __syncthreads();
    sh[threadIdx.x] += x;
    __syncthreads();
  }
  const float total = sh[kSampThreads - 1];
  const float target = (float)(u * (double)total);
  const float incl = sh[threadIdx.x];
  const float excl = threadIdx.x > 0 ? sh[threadIdx.x - 1] : 0.f;   // exact chunk bounds
  if (threadIdx.x == 0) *shi = -1;
  __syncthreads();
  if (part > 0.f && target >= excl && target < incl) {
    float c = excl;
    int pick = b1 - 1;
    for (int y = b0; y < b1; ++y) {
      c += wfn(y);
      if (c > target) {
        pick = y;
        break;
      }
    }
    *shi = pick;   // exactly one thread's chunk contains the target
  }
  __syncthreads();
  int r = *shi;
  if (r < 0) {   // rounding at the very top of the CDF: last positive-weight token
    if (threadIdx.x == 0) {
      int last = V - 1;
      while (last > 0 && wfn(last) <= 0.f) --last;
      *shi = last;
    }
    __syncthreads();
    r = *shi;
  }
  __syncthreads();
  (void)Z;
  return r;
}

// ------------------------------------------------ per-row sample + stats
// Every live row of a forward: (m, s) of logits/T into stats[row], and a
// token sampled from p into out_tok[row] (used for admission, token 0 of the
// output, and AR decoding).  Uniform key: (seed, 7, request slot, position).
__global__ void __launch_bounds__(kSampThreads) k_sample_rows(
    const float* __restrict__ logits, int V, const int* __restrict__ t_dev,
    const int* __restrict__ tok_pos, const int* __restrict__ tok_slot, float inv_t,
    uint64_t seed, float2* __restrict__ stats, int* __restrict__ out_tok) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sh[kSampThreads + 64];
  __shared__ int shi;
  const int T = *t_dev;
  for (int row = blockIdx.x; row < T; row += gridDim.x) {
    const float* l = logits + (size_t)row * V;
    const RowStats st = row_stats(l, V, inv_t, sh);
    if (threadIdx.x == 0) stats[row] = make_float2(st.m, st.s);
    const double u = u53s(mix64(seed, kStreamRowSample, (uint64_t)tok_slot[row],
                                (uint64_t)tok_pos[row]));
    const int y = sample_index(V, u, st.s, [&](int k) { return __expf(l[k] * inv_t - st.m); },
                               sh, &shi);
    if (threadIdx.x == 0) out_tok[row] = y;
    __syncthreads();
  }
}

// ------------------------------------------------ draft sampling step
// The draft's token for request b at draft-history position hl = q-sample of
// its last row; the logits row and its stats are kept in q-store slot
// hl % W (the accept step needs q at every candidate position).
__global__ void __launch_bounds__(kSampThreads) k_draft_sample(
    DecodeStateDev s, BatchDev bt, const float* __restrict__ logits, int V, float inv_t,
    float* __restrict__ qstore, float2* __restrict__ qstat, int W) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sh[kSampThreads + 64];
  __shared__ int shi;
  const int b = blockIdx.x;
  if (b >= s.n_req || bt.n_new[b] <= 0) return;
  if (!(s.gen_count[b] > 0 && s.gen_done[b] < s.gen_count[b])) return;
  const int row = bt.q_off[b] + bt.n_new[b] - 1;
  const int hl = s.hist_len[b];                       // output position being drafted
  const float* l = logits + (size_t)row * V;
  const RowStats st = row_stats(l, V, inv_t, sh);
  const double u = u53s(mix64(s.seed, kStreamDraftSample, (uint64_t)b, (uint64_t)hl));
  const int y = sample_index(V, u, st.s, [&](int k) { return __expf(l[k] * inv_t - st.m); }, sh,
                             &shi);
  const int slot = hl % W;
  float* q = qstore + ((size_t)b * W + slot) * V;
  for (int k = threadIdx.x; k < V; k += kSampThreads) q[k] = l[k];
  if (threadIdx.x == 0) {
    qstat[b * W + slot] = make_float2(st.m, st.s);
    bt.out_tok[row] = y;
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
  __shared__ float sh[kSampThreads + 64];
  __shared__ int shi;
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
  const double u2 = u53s(mix64(s.seed, kStreamResample, (uint64_t)b, (uint64_t)(pos + a)));
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
  int y;
  if (a < m || head) {   // resample from norm(max(0, p - q)) at the rejected position
    const int slot = (pos + a) % W;
    const float* lq = qstore + ((size_t)b * W + slot) * V;
    const float2 qs = qstat[b * W + slot];
    auto wres = [&](int k) {
      const float p = __expf(lp[k] * inv_t - ts.x) / ts.y;
      const float q = __expf(lq[k] * inv_t - qs.x) / qs.y;
      return fmaxf(p - q, 0.f);
    };
    float z = 0.f;
    {
      const int per = (V + kSampThreads - 1) / kSampThreads;
      const int b0 = threadIdx.x * per, b1 = min(V, b0 + per);
      for (int k = b0; k < b1; ++k) z += wres(k);
      z = block_sum(z, sh);
    }
    if (z > 0.f) {
      y = sample_index(V, u2, z, wres, sh, &shi);
    } else {   // p == q: the residual is empty, draw from p
      y = sample_index(V, u2, ts.y, [&](int k) { return __expf(lp[k] * inv_t - ts.x); }, sh,
                       &shi);
    }
  } else {       // every candidate accepted: bonus from p_m
    y = sample_index(V, u2, ts.y, [&](int k) { return __expf(lp[k] * inv_t - ts.x); }, sh,
                     &shi);
  }
  if (threadIdx.x == 0) {
    out_a[b] = a;
    out_bonus[b] = y;
  }
}

// ------------------------------------------------------------------ launchers
int launch_sample_rows(const float* logits, int V, const int* t_dev, int t_cap,
                       const int* tok_pos, const int* tok_slot, float inv_t, uint64_t seed,
                       float2* stats, int* out_tok, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_sample_rows", k_sample_rows, dim3((t_cap < 296 ? t_cap : 296)),
                     dim3(kSampThreads), 0, s, logits, V, t_dev, tok_pos, tok_slot, inv_t, seed,
                     stats, out_tok);
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
