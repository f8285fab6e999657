// model_kernels.cu — RMSNorm / embedding, RoPE + KV-cache write, gamma-query
// attention over the KV cache, split combine, and the greedy argmax reduce.
//
// All reductions use a fixed order that depends only on absolute positions
// (never on how many tokens share the batch), so a token's logits are
// bit-identical in a verify pass and in plain autoregressive decoding.
#include <cuda_bf16.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "model_kernels.cuh"

namespace spectre {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t ptx_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed tree) for blockDim.x == 256
__device__ __forceinline__ float block_sum_256(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  float r = 0.f;
  if (threadIdx.x < 32) {
    r = threadIdx.x < 8 ? sh[threadIdx.x] : 0.f;
    r = warp_sum(r);
    if (threadIdx.x == 0) sh[8] = r;
  }
  __syncthreads();
  r = sh[8];
  __syncthreads();
  return r;
}

// --------------------------------------------------------- embed + RMSNorm
// h[t] = E[tok[t]] (fp32 residual), x[t] = bf16(h * rsqrt(mean(h^2)+eps) * w)
__global__ void __launch_bounds__(256) k_embed_rmsnorm(const int* __restrict__ tok,
                                                       const int* __restrict__ t_dev,
                                                       const __nv_bfloat16* __restrict__ E,
                                                       const float* __restrict__ w,
                                                       float* __restrict__ h,
                                                       __nv_bfloat16* __restrict__ x, int d,
                                                       float eps) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sh[16];
  const int T = *t_dev;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {   // grid-stride over the live rows
    const __nv_bfloat16* e = E + (size_t)tok[t] * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += 256) {
      const float v = __bfloat162float(e[i]);
      h[(size_t)t * d + i] = v;
      ss += v * v;
    }
    ss = block_sum_256(ss, sh);
    const float r = rsqrtf(ss / (float)d + eps);
    for (int i = threadIdx.x; i < d; i += 256)
      x[(size_t)t * d + i] = __float2bfloat16_rn(h[(size_t)t * d + i] * r * w[i]);
  }
}

// ---------------------------------------------- residual add (+split-K sum)
// h[t] += sum_s part[s][t]; x[t] = bf16(rmsnorm(h[t]) * w).  One CTA per token
// row, one float4 per thread; all split partials are loaded before the fixed-
// order sum so the loads overlap instead of forming a latency chain.
constexpr int kMaxSplits = 12;

// kS: most splits the kernel keeps in flight per chunk (register budget: with
// kS = 4 a 512-thread CTA fits twice per SM, so T=256 rows run in one wave)
// kFlat: every (chunk, split) load of a row in flight at once (splits <= kS)
template <int kVec, int kS = kMaxSplits, bool kFlat = false>
__global__ void __launch_bounds__(512) k_residual_rmsnorm_v(const float* __restrict__ part,
                                                             int splits, int rows_cap,
                                                             const int* __restrict__ t_dev,
                                                             const float* __restrict__ w,
                                                             float* __restrict__ h,
                                                             __nv_bfloat16* __restrict__ x,
                                                             int d, float eps) {
  __shared__ float sh[40];
  const int nv = d >> 2;
  const size_t sstride = (size_t)rows_cap * d / 4;
  const float4* w4 = reinterpret_cast<const float4*>(w);
  // Before griddepcontrol.wait: everything that does not come from the
  // preceding (split-K GEMM) launch.  The row count, the residual row and the
  // norm weight were written at least two launches back, and the preceding
  // launch itself waited for its predecessor before releasing this grid.
  const int T = *t_dev;
  float4 wv[kVec], hv[kVec];
  if ((int)blockIdx.x < T) {
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      if (i < nv) {
        wv[j] = __ldg(w4 + i);
        hv[j] = reinterpret_cast<const float4*>(h + (size_t)blockIdx.x * d)[i];
      }
    }
  }
  pdl_wait();
  pdl_trigger();
  for (int t = blockIdx.x; t < T; t += gridDim.x) {   // grid-stride over the live rows
  if (t != (int)blockIdx.x) {
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      if (i < nv) hv[j] = reinterpret_cast<const float4*>(h + (size_t)t * d)[i];
    }
  }
  const float4* p4 = reinterpret_cast<const float4*>(part + (size_t)t * d);
  float4 v[kVec];
  if constexpr (kFlat) {
    // every chunk's loads of kS splits in flight at once: one L2 round trip
    // per kS splits (per element still h + p0 + p1 + ..., split order)
#pragma unroll
    for (int j = 0; j < kVec; ++j) v[j] = hv[j];
    for (int s0 = 0; s0 < splits; s0 += kS) {
      float4 ld[kVec][kS];
#pragma unroll
      for (int j = 0; j < kVec; ++j)
#pragma unroll
        for (int sp = 0; sp < kS; ++sp) {
          const int i = threadIdx.x + j * blockDim.x;
          if (s0 + sp < splits && i < nv) ld[j][sp] = __ldg(p4 + (s0 + sp) * sstride + i);
        }
#pragma unroll
      for (int j = 0; j < kVec; ++j)
#pragma unroll
        for (int sp = 0; sp < kS; ++sp)
          if (s0 + sp < splits) {
            v[j].x += ld[j][sp].x; v[j].y += ld[j][sp].y;
            v[j].z += ld[j][sp].z; v[j].w += ld[j][sp].w;
          }
    }
  } else
#pragma unroll
  for (int j = 0; j < kVec; ++j) {   // one chunk's split loads in flight (register budget:
    const int i = threadIdx.x + j * blockDim.x;   // two 512-thread CTAs per SM)
    float4 acc = hv[j];
    // splits in batches of kS (in split order: h + p0 + p1 + ...)
    for (int s0 = 0; s0 < splits; s0 += kS) {
      float4 ld[kS];
#pragma unroll
      for (int sp = 0; sp < kS; ++sp)
        if (s0 + sp < splits && i < nv) ld[sp] = __ldg(p4 + (s0 + sp) * sstride + i);
#pragma unroll
      for (int sp = 0; sp < kS; ++sp)
        if (s0 + sp < splits) {
          acc.x += ld[sp].x; acc.y += ld[sp].y; acc.z += ld[sp].z; acc.w += ld[sp].w;
        }
    }
    v[j] = acc;
  }
  float ss = 0.f;
  float4* ho = reinterpret_cast<float4*>(h + (size_t)t * d);
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      ho[i] = v[j];
      ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
    }
  }
  // deterministic block reduction (fixed shuffle tree + fixed warp order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const int nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float r = threadIdx.x < nw ? sh[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (threadIdx.x == 0) sh[32] = r;
  }
  __syncthreads();
  const float r = rsqrtf(sh[32] / (float)d + eps);
  __nv_bfloat162* xo = reinterpret_cast<__nv_bfloat162*>(x + (size_t)t * d);
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      const float4 ww = wv[j];
      xo[2 * i] = __floats2bfloat162_rn(v[j].x * r * ww.x, v[j].y * r * ww.y);
      xo[2 * i + 1] = __floats2bfloat162_rn(v[j].z * r * ww.z, v[j].w * r * ww.w);
    }
  }
  __syncthreads();   // sh reused by the next row
  }
}

// ------------------------------------------- qkv epilogue: RoPE + KV write
// part: [splits][rows_cap][(n_q + 2 n_kv) * hd] fp32.  rope: [ctx_cap][hd/2] (cos, sin)
// Rotate-half convention: pairs (i, i + hd/2).  grid (token, pair block); one
// (i, i+hd/2) pair per thread, all split loads issued up front.
__global__ void __launch_bounds__(128) k_qkv_rope_kv(const float* __restrict__ part, int splits,
                                                     int rows_cap, const int* __restrict__ t_dev,
                                                     const int* __restrict__ tok_pos,
                                                     const int* __restrict__ tok_slot,
                                                     const float2* __restrict__ rope,
                                                     __nv_bfloat16* __restrict__ q,
                                                     __nv_bfloat16* __restrict__ kc,
                                                     __nv_bfloat16* __restrict__ vc, int n_q,
                                                     int n_kv, int hd, int ctx_cap) {
  pdl_wait();
  pdl_trigger();
  const int T = *t_dev;
  const int half = hd / 2;
  const int n_pairs = (n_q + 2 * n_kv) * half;
  const int per_tok = (n_pairs + 127) / 128;
  for (int wi = blockIdx.x; wi < T * per_tok; wi += gridDim.x) {   // (token, pair block)
  const int t = wi / per_tok;
  const int c = (wi % per_tok) * 128 + threadIdx.x;
  if (c >= n_pairs) continue;
  const int head = c / half, i = c % half;
  const int N = (n_q + 2 * n_kv) * hd;
  const float* p0 = part + (size_t)t * N + head * hd + i;
  const size_t sstride = (size_t)rows_cap * N;
  float la[kMaxSplits], lb[kMaxSplits];
#pragma unroll
  for (int sp = 0; sp < kMaxSplits; ++sp)
    if (sp < splits) {
      la[sp] = __ldg(p0 + sp * sstride);
      lb[sp] = __ldg(p0 + sp * sstride + half);
    }
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int sp = 0; sp < kMaxSplits; ++sp)
    if (sp < splits) {
      a += la[sp];
      b += lb[sp];
    }
  const int pos = tok_pos[t];
  if (head < n_q + n_kv) {
    const float2 cs = rope[(size_t)pos * half + i];
    const float ra = a * cs.x - b * cs.y;
    const float rb = b * cs.x + a * cs.y;
    if (head < n_q) {
      __nv_bfloat16* dst = q + ((size_t)t * n_q + head) * hd;
      dst[i] = __float2bfloat16_rn(ra);
      dst[i + half] = __float2bfloat16_rn(rb);
    } else {
      const size_t off = (((size_t)tok_slot[t] * n_kv + (head - n_q)) * ctx_cap + pos) * hd;
      kc[off + i] = __float2bfloat16_rn(ra);
      kc[off + i + half] = __float2bfloat16_rn(rb);
    }
  } else {
    const size_t off =
        (((size_t)tok_slot[t] * n_kv + (head - n_q - n_kv)) * ctx_cap + pos) * hd;
    vc[off + i] = __float2bfloat16_rn(a);
    vc[off + i + half] = __float2bfloat16_rn(b);
  }
  }
}

// Vectorised variant: four consecutive pairs per thread (float4 partial loads,
// 8-byte bf16 stores); per element the same split order and arithmetic.
__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* dst, float a0, float a1, float a2,
                                          float a3) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a0, a1), hi = __floats2bfloat162_rn(a2, a3);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = u;
}

// kB: split partials in flight per batch — 4 (80 registers) when the GEMM had
// <= 4 splits (target: 6.9 -> 4.8 us), all 12 otherwise (a 12-split draft
// q/k/v is latency-bound and would pay three round trips)
template <int kB>
__global__ void __launch_bounds__(128) k_qkv_rope_kv4(const float* __restrict__ part, int splits,
                                                      int rows_cap, const int* __restrict__ t_dev,
                                                      const int* __restrict__ tok_pos,
                                                      const int* __restrict__ tok_slot,
                                                      const float2* __restrict__ rope,
                                                      __nv_bfloat16* __restrict__ q,
                                                      __nv_bfloat16* __restrict__ kc,
                                                      __nv_bfloat16* __restrict__ vc, int n_q,
                                                      int n_kv, int hd, int ctx_cap) {
  // token count, positions, slots and the cos/sin table come from launches at
  // least two back (see k_residual_rmsnorm_v): fetch the first item's before
  // the wait, so only the split-K partial loads follow it
  const int T = *t_dev;
  const int half = hd / 2;
  const int n_quads = (n_q + 2 * n_kv) * half / 4;
  const int per_tok = (n_quads + 127) / 128;
  const int N = (n_q + 2 * n_kv) * hd;
  const size_t sstride = (size_t)rows_cap * N;
  int pos_pre = 0, slot_pre = 0;
  float4 c01_pre = make_float4(0.f, 0.f, 0.f, 0.f), c23_pre = c01_pre;
  if ((int)blockIdx.x < T * per_tok) {
    const int t = blockIdx.x / per_tok;
    const int c = ((blockIdx.x % per_tok) * 128 + threadIdx.x) * 4;
    pos_pre = tok_pos[t];
    slot_pre = tok_slot[t];
    if (c < n_quads * 4 && c / half < n_q + n_kv) {
      const float4* cs4 = reinterpret_cast<const float4*>(rope + (size_t)pos_pre * half + c % half);
      c01_pre = cs4[0];
      c23_pre = cs4[1];
    }
  }
  pdl_wait();
  pdl_trigger();
  for (int wi = blockIdx.x; wi < T * per_tok; wi += gridDim.x) {   // (token, quad block)
    const int t = wi / per_tok;
    const int c = ((wi % per_tok) * 128 + threadIdx.x) * 4;        // first pair index
    if (c >= n_quads * 4) continue;
    const bool first = wi == (int)blockIdx.x;
    const int head = c / half, i = c % half;
    const float* p0 = part + (size_t)t * N + head * hd + i;
    float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
    // splits in batches (same summation order), so more CTAs stay resident
    for (int s0 = 0; s0 < splits; s0 += kB) {
      float4 la[kB], lb[kB];
#pragma unroll
      for (int sp = 0; sp < kB; ++sp)
        if (s0 + sp < splits) {
          la[sp] = __ldg(reinterpret_cast<const float4*>(p0 + (s0 + sp) * sstride));
          lb[sp] = __ldg(reinterpret_cast<const float4*>(p0 + (s0 + sp) * sstride + half));
        }
#pragma unroll
      for (int sp = 0; sp < kB; ++sp)
        if (s0 + sp < splits) {
          a[0] += la[sp].x; a[1] += la[sp].y; a[2] += la[sp].z; a[3] += la[sp].w;
          b[0] += lb[sp].x; b[1] += lb[sp].y; b[2] += lb[sp].z; b[3] += lb[sp].w;
        }
    }
    const int pos = first ? pos_pre : tok_pos[t];
    const int slot = first ? slot_pre : tok_slot[t];
    if (head < n_q + n_kv) {
      float4 c01 = c01_pre, c23 = c23_pre;
      if (!first) {
        const float4* cs4 = reinterpret_cast<const float4*>(rope + (size_t)pos * half + i);
        c01 = cs4[0];
        c23 = cs4[1];
      }
      const float cx[4] = {c01.x, c01.z, c23.x, c23.z}, cy[4] = {c01.y, c01.w, c23.y, c23.w};
      float ra[4], rb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ra[k] = a[k] * cx[k] - b[k] * cy[k];
        rb[k] = b[k] * cx[k] + a[k] * cy[k];
      }
      __nv_bfloat16* dst;
      if (head < n_q) {
        dst = q + ((size_t)t * n_q + head) * hd;
      } else {
        dst = kc + (((size_t)slot * n_kv + (head - n_q)) * ctx_cap + pos) * hd;
      }
      st_bf16x4(dst + i, ra[0], ra[1], ra[2], ra[3]);
      st_bf16x4(dst + i + half, rb[0], rb[1], rb[2], rb[3]);
    } else {
      __nv_bfloat16* dst =
          vc + (((size_t)slot * n_kv + (head - n_q - n_kv)) * ctx_cap + pos) * hd;
      st_bf16x4(dst + i, a[0], a[1], a[2], a[3]);
      st_bf16x4(dst + i + half, b[0], b[1], b[2], b[3]);
    }
  }
}

// ------------------------------------------------------------ argmax reduce
// (max, lowest index) over the lm_head tiles for each token row.
__global__ void __launch_bounds__(256) k_argmax_reduce(const float* __restrict__ val,
                                                       const int* __restrict__ idx, int n_tiles,
                                                       int rows_cap,
                                                       const int* __restrict__ t_dev,
                                                       int* __restrict__ out_tok,
                                                       float* __restrict__ out_val) {
  pdl_wait();
  pdl_trigger();
  const int T = *t_dev;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {   // grid-stride over the live rows
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < n_tiles; i += 256) {
    const float v = val[(size_t)i * rows_cap + t];
    const int ix = idx[(size_t)i * rows_cap + t];
    if (v > best || (v == best && ix < bi)) {
      best = v;
      bi = ix;
    }
  }
  __shared__ float sv[8];
  __shared__ int si[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    out_tok[t] = bi;
    if (out_val) out_val[t] = best;
  }
  __syncthreads();   // sv / si reused by the next row
  }
}

// Row-group variant: lanes are 32 consecutive rows (coalesced 128 B loads of
// one slot), the 32 warps split the slots, then a fixed-order cross-warp
// reduction.  (max value, lowest index among equals) is order independent,
// so the result equals k_argmax_reduce's.
__global__ void __launch_bounds__(1024) k_argmax_reduce_rows(const float* __restrict__ val,
                                                            const int* __restrict__ idx,
                                                            int n_tiles, int rows_cap,
                                                            const int* __restrict__ t_dev,
                                                            int* __restrict__ out_tok,
                                                            float* __restrict__ out_val) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32][33];
  __shared__ int si[32][33];
  const int T = *t_dev;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t0 = blockIdx.x * 32; t0 < T; t0 += gridDim.x * 32) {
    const int t = t0 + lane;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    if (t < T) {
      int i = warp;
#pragma unroll 1
      for (; i + 224 < n_tiles; i += 256) {   // eight independent slots in flight
        float v[8];
        int ix[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = val[(size_t)(i + 32 * u) * rows_cap + t];
          ix[u] = idx[(size_t)(i + 32 * u) * rows_cap + t];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (v[u] > best || (v[u] == best && ix[u] < bi)) {
            best = v[u];
            bi = ix[u];
          }
      }
      for (; i < n_tiles; i += 32) {
        const float v = val[(size_t)i * rows_cap + t];
        const int ix = idx[(size_t)i * rows_cap + t];
        if (v > best || (v == best && ix < bi)) {
          best = v;
          bi = ix;
        }
      }
    }
    sv[warp][lane] = best;
    si[warp][lane] = bi;
    __syncthreads();
    if (warp == 0 && t < T) {
      for (int w = 1; w < 32; ++w)
        if (sv[w][lane] > best || (sv[w][lane] == best && si[w][lane] < bi)) {
          best = sv[w][lane];
          bi = si[w][lane];
        }
      out_tok[t] = bi;
      if (out_val) out_val[t] = best;
    }
    __syncthreads();   // sv / si reused by the next row group
  }
}

// RoPE table: rope[p][i] = (cos(p * theta^(-2i/hd)), sin(...)), double precision.
__global__ void k_rope_table(float2* rope, int ctx_cap, int hd, double theta) {
  const int half = hd / 2;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ctx_cap * half;
       c += gridDim.x * blockDim.x) {
    const int p = c / half, i = c % half;
    const double inv = pow(theta, -2.0 * i / (double)hd);
    double sn, cs;
    sincos((double)p * inv, &sn, &cs);
    rope[c] = make_float2((float)cs, (float)sn);
  }
}

// ------------------------------------------------------------------ launchers
// Row kernels are grid-stride loops over the device-side row count: a fixed
// grid of a few CTAs per SM instead of one CTA per row of capacity.
constexpr int kSms = 148;
static int rope_ctas_per_sm() {
  static const int v = [] {
    const char* e = getenv("SPECTRE_ROPE_CTAS");   // measured: 24 per SM (scalar), 8 (float4)
    return e ? atoi(e) : 0;
  }();
  return v;
}
static int resid_ctas_per_sm() {
  static const int v = [] {
    const char* e = getenv("SPECTRE_RESID_CTAS");
    return e ? atoi(e) : 2;
  }();
  return v;
}
int launch_embed_rmsnorm(const int* tok, const int* t_dev, int t_cap, const void* E,
                         const float* w, float* h, void* x, int d, float eps, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_embed_rmsnorm", k_embed_rmsnorm, dim3((std::min(t_cap, 2 * kSms))), dim3(256), 0, s, tok, t_dev,
                     reinterpret_cast<const __nv_bfloat16*>(E), w, h,
                     reinterpret_cast<__nv_bfloat16*>(x), d, eps);
  return SPECTRE_OK;
}

static bool resid_batched() {   // > 4 splits through the 4-at-a-time variant too
  static const bool v = [] {     // (measured: down-projection residual 7.0 -> ~5.6 us)
    const char* e = getenv("SPECTRE_RESID_BATCHED");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}


int launch_residual_rmsnorm(const float* part, int splits, int rows_cap, const int* t_dev,
                            int t_cap, const float* w, float* h, void* x, int d, float eps,
                            cudaStream_t s) {
  if (d % 4 || splits > kMaxSplits) return arg_fail("residual_rmsnorm: d % 4 / splits");
  const int nv = d / 4;
  const int threads = nv < 512 ? ((nv + 31) / 32) * 32 : 512;
  const int vec = (nv + threads - 1) / threads;
  auto* xb = reinterpret_cast<__nv_bfloat16*>(x);
  const dim3 grid((std::min(t_cap, resid_ctas_per_sm() * kSms)));
  if (vec <= 1)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<1>, grid, dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else if (vec <= 2 && (splits <= 4 || resid_batched()))
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<2, 4>, grid, dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else if (vec <= 2)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<2>, grid, dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  // d = 5120 (Qwen2.5-32B): every chunk's loads of 4 splits in flight at once
  // (T=896, 3 splits: 23.6 -> 17.9 us; the same at d = 4096 costs the second
  // CTA per SM and is slower, 4.67 -> 5.6 us)
  else if (vec <= 3)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", (k_residual_rmsnorm_v<3, 4, true>), grid, dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else if (vec <= 4)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<4>, grid, dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else
    return arg_fail("residual_rmsnorm: d > 8192");
  return SPECTRE_OK;
}

int launch_qkv_rope_kv(const float* part, int splits, int rows_cap, const int* t_dev, int t_cap,
                       const int* tok_pos, const int* tok_slot, const void* rope, void* q,
                       void* kc, void* vc, int n_q, int n_kv, int hd, int ctx_cap,
                       cudaStream_t s) {
  if (splits > kMaxSplits) return arg_fail("qkv_rope_kv: splits");
  const int pairs = (n_q + 2 * n_kv) * hd / 2;
  static const bool vec4 = [] {
    const char* e = getenv("SPECTRE_ROPE_VEC");   // 0: one pair per thread
    return e ? atoi(e) != 0 : true;
  }();
  if (vec4 && (hd / 2) % 4 == 0) {
    const int quads = pairs / 4;
    if (splits <= 4)
      SPECTRE_LAUNCH_PDL("k_qkv_rope_kv4", k_qkv_rope_kv4<4>,
                       dim3((std::min(t_cap * ((quads + 127) / 128),
                                              (rope_ctas_per_sm() ? rope_ctas_per_sm() : 8) * kSms))),
                       dim3(128), 0, s, part, splits, rows_cap, t_dev, tok_pos, tok_slot,
                       reinterpret_cast<const float2*>(rope), reinterpret_cast<__nv_bfloat16*>(q),
                       reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc),
                       n_q, n_kv, hd, ctx_cap);
    else
      SPECTRE_LAUNCH_PDL("k_qkv_rope_kv4", k_qkv_rope_kv4<kMaxSplits>,
                       dim3((std::min(t_cap * ((quads + 127) / 128),
                                              (rope_ctas_per_sm() ? rope_ctas_per_sm() : 8) * kSms))),
                       dim3(128), 0, s, part, splits, rows_cap, t_dev, tok_pos, tok_slot,
                       reinterpret_cast<const float2*>(rope), reinterpret_cast<__nv_bfloat16*>(q),
                       reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc),
                       n_q, n_kv, hd, ctx_cap);
    return SPECTRE_OK;
  }
  SPECTRE_LAUNCH_PDL("k_qkv_rope_kv", k_qkv_rope_kv,
                     dim3((std::min(t_cap * ((pairs + 127) / 128),
                                            (rope_ctas_per_sm() ? rope_ctas_per_sm() : 24) * kSms))),
                     dim3(128),
                     0, s, part, splits, rows_cap, t_dev, tok_pos, tok_slot,
                     reinterpret_cast<const float2*>(rope), reinterpret_cast<__nv_bfloat16*>(q),
                     reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc),
                     n_q, n_kv, hd, ctx_cap);
  return SPECTRE_OK;
}

int launch_argmax_reduce(const float* val, const int* idx, int n_tiles, int rows_cap,
                         const int* t_dev, int t_cap, int* out_tok, float* out_val,
                         cudaStream_t s) {
  static const bool rows = [] {
    const char* e = getenv("SPECTRE_ARGMAX_ROWS");   // 0: one CTA per row (strided slots)
    return e ? atoi(e) != 0 : true;
  }();
  if (rows) {
    SPECTRE_LAUNCH_PDL("k_argmax_reduce_rows", k_argmax_reduce_rows,
                       dim3((std::min((t_cap + 31) / 32, kSms))), dim3(1024), 0, s, val,
                       idx, n_tiles, rows_cap, t_dev, out_tok, out_val);
    return SPECTRE_OK;
  }
  SPECTRE_LAUNCH_PDL("k_argmax_reduce", k_argmax_reduce, dim3((std::min(t_cap, 2 * kSms))), dim3(256), 0, s, val, idx,
                     n_tiles, rows_cap, t_dev, out_tok, out_val);
  return SPECTRE_OK;
}

int launch_rope_table(void* rope, int ctx_cap, int hd, double theta, cudaStream_t s) {
  k_rope_table<<<256, 256, 0, s>>>(reinterpret_cast<float2*>(rope), ctx_cap, hd, theta);
  SPECTRE_LAUNCH_CHECK("k_rope_table");
  return SPECTRE_OK;
}

}  // namespace spectre
