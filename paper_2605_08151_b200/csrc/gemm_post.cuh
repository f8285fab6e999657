// gemm_post.cuh — split-K reduction phases fused into the producing GEMM.
//
// A split-K GEMM writes fp32 partials [split][t][n]; its consumer used to be
// a separate kernel (one kernel turnover per reduction).  Here the GEMM's own
// CTAs (all co-resident: one per SM) pass an in-kernel grid barrier after
// their epilogues and run the reduction:
//   kPostRope   sum partials -> RoPE -> q (bf16) + K/V cache write
//   kPostResid  h += sum partials; x = bf16(rmsnorm(h) * w)   (next block's input)
// The arithmetic is the standalone kernels' (model_kernels.cu): same split
// order (h + p0 + p1 + ...), fixed reduction trees; every row's result is
// independent of the token count (batch invariance).
#pragma once

#include <cuda_bf16.h>
#include <cstdint>

#include "common.cuh"

namespace spectre {

enum GemmPostKind : int { kPostNone = 0, kPostRope = 1, kPostResid = 2 };

struct GemmPost {
  int kind;
  int* gbar;               // [2] grid barrier {arrivals, generation} (self-resetting)
  // kPostRope
  const int* tok_pos;
  const int* tok_slot;
  const float2* rope;      // [ctx_cap][hd/2]
  __nv_bfloat16* q;        // [rows][n_q][hd]
  __nv_bfloat16* kc;       // layer base [slots][n_kv][ctx_cap][hd]
  __nv_bfloat16* vc;
  int n_q, n_kv, hd, ctx_cap;
  // kPostResid
  const float* w;          // [d] norm weight of the next block
  float* h;                // [rows][d] fp32 residual
  __nv_bfloat16* x;        // [rows][d] bf16 normalised input of the next GEMM
  float eps;
};

constexpr int kPostMaxSplits = 12;

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All CTAs of the grid: arrival counter + generation flip (one thread per
// CTA).  Waiters poll with plain acquire loads — read-modify-write polling
// serialises 148 CTAs on one L2 slice.
__device__ __forceinline__ void post_grid_sync(int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int gen = ld_acquire_gpu(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1) == (int)gridDim.x - 1) {
      atomicExch(bar, 0);
      __threadfence();
      atomicAdd(bar + 1, 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void post_rope(const GemmPost& p, const float* part, int splits,
                                          int rows_cap, int T) {
  const int half = p.hd / 2;
  const int n_pairs = (p.n_q + 2 * p.n_kv) * half;
  const int nt = blockDim.x;
  const int per_tok = (n_pairs + nt - 1) / nt;
  const int N = (p.n_q + 2 * p.n_kv) * p.hd;
  const size_t sstride = (size_t)rows_cap * N;
  for (int wi = blockIdx.x; wi < T * per_tok; wi += gridDim.x) {   // (token, pair block)
    const int t = wi / per_tok;
    const int c = (wi % per_tok) * nt + threadIdx.x;
    if (c >= n_pairs) continue;
    const int head = c / half, i = c % half;
    const float* p0 = part + (size_t)t * N + head * p.hd + i;
    float la[kPostMaxSplits], lb[kPostMaxSplits];
#pragma unroll
    for (int sp = 0; sp < kPostMaxSplits; ++sp)
      if (sp < splits) {
        la[sp] = __ldcg(p0 + sp * sstride);
        lb[sp] = __ldcg(p0 + sp * sstride + half);
      }
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int sp = 0; sp < kPostMaxSplits; ++sp)
      if (sp < splits) {
        a += la[sp];
        b += lb[sp];
      }
    const int pos = p.tok_pos[t];
    if (head < p.n_q + p.n_kv) {
      const float2 cs = p.rope[(size_t)pos * half + i];
      const float ra = a * cs.x - b * cs.y;
      const float rb = b * cs.x + a * cs.y;
      if (head < p.n_q) {
        __nv_bfloat16* dst = p.q + ((size_t)t * p.n_q + head) * p.hd;
        dst[i] = __float2bfloat16_rn(ra);
        dst[i + half] = __float2bfloat16_rn(rb);
      } else {
        const size_t off =
            (((size_t)p.tok_slot[t] * p.n_kv + (head - p.n_q)) * p.ctx_cap + pos) * p.hd;
        p.kc[off + i] = __float2bfloat16_rn(ra);
        p.kc[off + i + half] = __float2bfloat16_rn(rb);
      }
    } else {
      const size_t off =
          (((size_t)p.tok_slot[t] * p.n_kv + (head - p.n_q - p.n_kv)) * p.ctx_cap + pos) * p.hd;
      p.vc[off + i] = __float2bfloat16_rn(a);
      p.vc[off + i + half] = __float2bfloat16_rn(b);
    }
  }
}

template <int kVec>
__device__ __forceinline__ void post_resid_rows(const GemmPost& p, const float* part, int splits,
                                                int rows_cap, int T, int d, float* sh) {
  const int nv = d >> 2;
  const size_t sstride = (size_t)rows_cap * d / 4;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    float4 v[kVec];
    const float4* h4 = reinterpret_cast<const float4*>(p.h + (size_t)t * d);
    const float4* p4 = reinterpret_cast<const float4*>(part + (size_t)t * d);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      if (i < nv) {
        float4 acc = h4[i];
        float4 ld[kPostMaxSplits];
#pragma unroll
        for (int sp = 0; sp < kPostMaxSplits; ++sp)
          if (sp < splits) ld[sp] = __ldcg(p4 + sp * sstride + i);
#pragma unroll
        for (int sp = 0; sp < kPostMaxSplits; ++sp)
          if (sp < splits) {
            acc.x += ld[sp].x;
            acc.y += ld[sp].y;
            acc.z += ld[sp].z;
            acc.w += ld[sp].w;
          }
        v[j] = acc;
      }
    }
    float ss = 0.f;
    float4* ho = reinterpret_cast<float4*>(p.h + (size_t)t * d);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      if (i < nv) {
        ho[i] = v[j];
        ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
      }
    }
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
    const float r = rsqrtf(sh[32] / (float)d + p.eps);
    const float4* w4 = reinterpret_cast<const float4*>(p.w);
    __nv_bfloat162* xo = reinterpret_cast<__nv_bfloat162*>(p.x + (size_t)t * d);
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      if (i < nv) {
        const float4 ww = w4[i];
        xo[2 * i] = __floats2bfloat162_rn(v[j].x * r * ww.x, v[j].y * r * ww.y);
        xo[2 * i + 1] = __floats2bfloat162_rn(v[j].z * r * ww.z, v[j].w * r * ww.w);
      }
    }
    __syncthreads();   // sh reused by the next row
  }
}

__device__ __forceinline__ void post_resid(const GemmPost& p, const float* part, int splits,
                                           int rows_cap, int T, int d, float* sh) {
  const int kvec = (d / 4 + blockDim.x - 1) / blockDim.x;
  if (kvec <= 1) post_resid_rows<1>(p, part, splits, rows_cap, T, d, sh);
  else if (kvec <= 2) post_resid_rows<2>(p, part, splits, rows_cap, T, d, sh);
  else if (kvec <= 3) post_resid_rows<3>(p, part, splits, rows_cap, T, d, sh);
  else post_resid_rows<4>(p, part, splits, rows_cap, T, d, sh);
}

}  // namespace spectre
