// model_kernels.cu — RMSNorm / embedding, RoPE + KV-cache write, gamma-query
// attention over the KV cache, split combine, and the greedy argmax reduce.
//
// All reductions use a fixed order that depends only on absolute positions
// (never on how many tokens share the batch), so a token's logits are
// bit-identical in a verify pass and in plain autoregressive decoding.
#include <cuda_bf16.h>

#include <cfloat>

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
  __shared__ float sh[16];
  const int t = blockIdx.x;
  if (t >= *t_dev) return;
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

// ---------------------------------------------- residual add (+split-K sum)
// h[t] += sum_s part[s][t]; x[t] = bf16(rmsnorm(h[t]) * w).  One CTA per token
// row, one float4 per thread; all split partials are loaded before the fixed-
// order sum so the loads overlap instead of forming a latency chain.
constexpr int kMaxSplits = 12;

template <int kVec>
__global__ void __launch_bounds__(512) k_residual_rmsnorm_v(const float* __restrict__ part,
                                                             int splits, int rows_cap,
                                                             const int* __restrict__ t_dev,
                                                             const float* __restrict__ w,
                                                             float* __restrict__ h,
                                                             __nv_bfloat16* __restrict__ x,
                                                             int d, float eps) {
  __shared__ float sh[40];
  const int t = blockIdx.x;
  if (t >= *t_dev) return;
  const int nv = d >> 2;
  float4 v[kVec];
  const float4* h4 = reinterpret_cast<const float4*>(h + (size_t)t * d);
  const size_t sstride = (size_t)rows_cap * d / 4;
  const float4* p4 = reinterpret_cast<const float4*>(part + (size_t)t * d);
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      float4 acc = h4[i];
      float4 ld[kMaxSplits];
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp)
        if (sp < splits) ld[sp] = __ldg(p4 + sp * sstride + i);
#pragma unroll
      for (int sp = 0; sp < kMaxSplits; ++sp)
        if (sp < splits) {
          acc.x += ld[sp].x; acc.y += ld[sp].y; acc.z += ld[sp].z; acc.w += ld[sp].w;
        }
      v[j] = acc;
    }
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
  const float4* w4 = reinterpret_cast<const float4*>(w);
  __nv_bfloat162* xo = reinterpret_cast<__nv_bfloat162*>(x + (size_t)t * d);
#pragma unroll
  for (int j = 0; j < kVec; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < nv) {
      const float4 ww = w4[i];
      xo[2 * i] = __floats2bfloat162_rn(v[j].x * r * ww.x, v[j].y * r * ww.y);
      xo[2 * i + 1] = __floats2bfloat162_rn(v[j].z * r * ww.z, v[j].w * r * ww.w);
    }
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
  const int t = blockIdx.x;
  if (t >= *t_dev) return;
  const int half = hd / 2;
  const int c = blockIdx.y * 128 + threadIdx.x;
  const int n_pairs = (n_q + 2 * n_kv) * half;
  if (c >= n_pairs) return;
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

// ------------------------------------------------------------- attention
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
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// grid (split_max, rb_max, n_req * n_kv), 128 threads.  Each CTA: one request,
// one kv head, a block of 16*MT query rows (token-major x group heads) and up
// to 512 keys; warp w owns keys [c0 + 128 w, +128) in 4 x 32-key steps with
// an online softmax, then the 4 warps merge in fixed order.
template <int HD, int MT>
__global__ void __launch_bounds__(kAttnThreads) k_attention(AttnArgs a) {
  constexpr int ROWS = 16 * MT;
  constexpr int LD = HD + 8;  // padded smem row (elements)
  extern __shared__ __align__(16) uint8_t smem_attn[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sKV = sQ + ROWS * LD;  // per warp: K[32][LD], V[32][LD]

  const int split = blockIdx.x, rb = blockIdx.y;
  const int b = blockIdx.z / a.n_kv, kvh = blockIdx.z % a.n_kv;
  const int group = a.n_q / a.n_kv;
  const int nn = a.n_new[b];
  const int rows_total = nn * group;
  if (rb * ROWS >= rows_total) return;
  const int p0 = a.pos0[b];
  const int kv_len = p0 + nn;
  const int c0 = split * kAttnChunk;
  if (c0 >= kv_len) return;
  const int last_row = min(rows_total, (rb + 1) * ROWS) - 1;
  const int p_max = p0 + last_row / group;  // largest query position in this block
  const int qoff = a.q_off[b];
  const size_t kv_base = ((size_t)a.slot[b] * a.n_kv + kvh) * a.ctx_cap;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // ---- Q tile
  for (int c = tid; c < ROWS * (HD / 8); c += kAttnThreads) {
    const int r = c / (HD / 8), ch = c % (HD / 8);
    const int R = rb * ROWS + r;
    const bool valid = R < rows_total;
    const int j = valid ? R / group : 0, hh = valid ? R % group : 0;
    const __nv_bfloat16* src = a.q + (((size_t)(qoff + j) * a.n_q) + kvh * group + hh) * HD + ch * 8;
    cp_async16(ptx_smem(sQ + r * LD + ch * 8), src, valid);
  }
  cp_async_wait_all();
  __syncthreads();

  __nv_bfloat16* sK = sKV + warp * 2 * 32 * LD;
  __nv_bfloat16* sV = sK + 32 * LD;
  float o[MT][HD / 8][4];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[m][n][e] = 0.f;
  float mrow[MT][2], lrow[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    mrow[m][0] = mrow[m][1] = -INFINITY;
    lrow[m][0] = lrow[m][1] = 0.f;
  }
  const int g = lane >> 2, tq = lane & 3;
  // query position of the two rows this thread owns in each m-tile
  int qpos[MT][2];
  bool qvalid[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int R = rb * ROWS + m * 16 + g + hr * 8;
      qvalid[m][hr] = R < rows_total;
      qpos[m][hr] = p0 + (qvalid[m][hr] ? R / group : 0);
    }

  for (int it = 0; it < 4; ++it) {
    const int kb = c0 + warp * 128 + it * kAttnSub;
    if (kb > p_max || kb >= c0 + kAttnChunk) break;
    // ---- load 32 keys of K and V (zero-fill beyond kv_len)
    for (int c = lane; c < 32 * (HD / 8); c += 32) {
      const int r = c / (HD / 8), ch = c % (HD / 8);
      const bool valid = kb + r < kv_len;
      const size_t off = (kv_base + (valid ? kb + r : 0)) * HD + ch * 8;
      cp_async16(ptx_smem(sK + r * LD + ch * 8), a.k + off, valid);
      cp_async16(ptx_smem(sV + r * LD + ch * 8), a.v + off, valid);
    }
    cp_async_wait_all();
    __syncwarp();
    // ---- S = Q K^T  (MT x 4 n-tiles of 8 keys)
    float s[MT][4][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[m][n][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t af[MT][4];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r = m * 16 + (lane & 15);
        const int cc = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(ptx_smem(sQ + r * LD + cc), af[m][0], af[m][1], af[m][2], af[m][3]);
      }
#pragma unroll
      for (int np = 0; np < 2; ++np) {  // n-tile pairs (16 keys)
        const int mi = lane >> 3;
        const int r = np * 16 + (mi >> 1) * 8 + (lane & 7);
        const int cc = kk * 16 + (mi & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ptx_smem(sK + r * LD + cc), b0, b1, b2, b3);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          mma16816(s[m][2 * np], af[m][0], af[m][1], af[m][2], af[m][3], b0, b1);
          mma16816(s[m][2 * np + 1], af[m][0], af[m][1], af[m][2], af[m][3], b2, b3);
        }
      }
    }
    // ---- mask + online softmax (log2 domain)
#pragma unroll
    for (int m = 0; m < MT; ++m) {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        float mx = -INFINITY;
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = kb + n * 8 + 2 * tq + e;
            float v = s[m][n][hr * 2 + e] * a.scale_log2;
            if (!qvalid[m][hr] || key > qpos[m][hr]) v = -INFINITY;
            s[m][n][hr * 2 + e] = v;
            mx = fmaxf(mx, v);
          }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(mrow[m][hr], mx);
        const float corr = (m_new == -INFINITY) ? 1.f : exp2f(mrow[m][hr] - m_new);
        float rs = 0.f;
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float v = s[m][n][hr * 2 + e];
            const float p = (v == -INFINITY) ? 0.f : exp2f(v - m_new);
            s[m][n][hr * 2 + e] = p;
            rs += p;
          }
        rs += __shfl_xor_sync(0xffffffffu, rs, 1);
        rs += __shfl_xor_sync(0xffffffffu, rs, 2);
        lrow[m][hr] = lrow[m][hr] * corr + rs;
        mrow[m][hr] = m_new;
#pragma unroll
        for (int n = 0; n < HD / 8; ++n) {
          o[m][n][hr * 2] *= corr;
          o[m][n][hr * 2 + 1] *= corr;
        }
      }
    }
    // ---- O += P V   (2 k-steps of 16 keys)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t pa[MT][4];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        pa[m][0] = pack_bf16(s[m][2 * ks][0], s[m][2 * ks][1]);
        pa[m][1] = pack_bf16(s[m][2 * ks][2], s[m][2 * ks][3]);
        pa[m][2] = pack_bf16(s[m][2 * ks + 1][0], s[m][2 * ks + 1][1]);
        pa[m][3] = pack_bf16(s[m][2 * ks + 1][2], s[m][2 * ks + 1][3]);
      }
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {  // dim-tile pairs
        const int mi = lane >> 3;
        const int r = ks * 16 + (mi & 1) * 8 + (lane & 7);
        const int cc = dp * 16 + (mi >> 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(ptx_smem(sV + r * LD + cc), b0, b1, b2, b3);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          mma16816(o[m][2 * dp], pa[m][0], pa[m][1], pa[m][2], pa[m][3], b0, b1);
          mma16816(o[m][2 * dp + 1], pa[m][0], pa[m][1], pa[m][2], pa[m][3], b2, b3);
        }
      }
    }
    __syncwarp();
  }

  // ---- merge the 4 warps in fixed order (smem reuse of the K/V area)
  __syncthreads();
  float* sO = reinterpret_cast<float*>(sKV);            // [4][ROWS][HD]
  float* sML = sO + 4 * ROWS * HD;                      // [4][ROWS][2]
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int r = m * 16 + g + hr * 8;
#pragma unroll
      for (int n = 0; n < HD / 8; ++n) {
        sO[(warp * ROWS + r) * HD + n * 8 + 2 * tq] = o[m][n][hr * 2];
        sO[(warp * ROWS + r) * HD + n * 8 + 2 * tq + 1] = o[m][n][hr * 2 + 1];
      }
      if (tq == 0) {
        sML[(warp * ROWS + r) * 2] = mrow[m][hr];
        sML[(warp * ROWS + r) * 2 + 1] = lrow[m][hr];
      }
    }
  __syncthreads();
  const size_t pidx =
      (((size_t)b * a.n_kv + kvh) * a.rb_max + rb) * a.split_max + split;
  for (int c = tid; c < ROWS * HD; c += kAttnThreads) {
    const int r = c / HD, dcol = c % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sML[(w * ROWS + r) * 2]);
    float O = 0.f, Lsum = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = sML[(w * ROWS + r) * 2];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      O += sO[(w * ROWS + r) * HD + dcol] * f;
      Lsum += sML[(w * ROWS + r) * 2 + 1] * f;
    }
    a.part_o[(pidx * ROWS + r) * HD + dcol] = O;
    if (dcol == 0) {
      a.part_ml[(pidx * ROWS + r) * 2] = M;
      a.part_ml[(pidx * ROWS + r) * 2 + 1] = Lsum;
    }
  }
}

// grid (rb_max, n_req * n_kv), 128 threads: merge splits -> out (bf16)
template <int HD, int MT>
__global__ void __launch_bounds__(128) k_attn_combine(AttnArgs a) {
  constexpr int ROWS = 16 * MT;
  const int rb = blockIdx.x;
  const int b = blockIdx.y / a.n_kv, kvh = blockIdx.y % a.n_kv;
  const int group = a.n_q / a.n_kv;
  const int nn = a.n_new[b];
  const int rows_total = nn * group;
  if (rb * ROWS >= rows_total) return;
  const int kv_len = a.pos0[b] + nn;
  const int n_split = (kv_len + kAttnChunk - 1) / kAttnChunk;
  const int qoff = a.q_off[b];
  for (int c = threadIdx.x; c < ROWS * HD; c += 128) {
    const int r = c / HD, dcol = c % HD;
    const int R = rb * ROWS + r;
    if (R >= rows_total) continue;
    // only splits that start at or before this row's query position hold keys
    const int qp = a.pos0[b] + R / group;
    const int ns = min(n_split, qp / kAttnChunk + 1);
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) {
      const size_t pidx = (((size_t)b * a.n_kv + kvh) * a.rb_max + rb) * a.split_max + s;
      M = fmaxf(M, a.part_ml[(pidx * ROWS + r) * 2]);
    }
    float O = 0.f, Lsum = 0.f;
    for (int s = 0; s < ns; ++s) {
      const size_t pidx = (((size_t)b * a.n_kv + kvh) * a.rb_max + rb) * a.split_max + s;
      const float ms = a.part_ml[(pidx * ROWS + r) * 2];
      const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
      O += a.part_o[(pidx * ROWS + r) * HD + dcol] * f;
      Lsum += a.part_ml[(pidx * ROWS + r) * 2 + 1] * f;
    }
    const int j = R / group, hh = R % group;
    a.out[(((size_t)(qoff + j)) * a.n_q + kvh * group + hh) * HD + dcol] =
        __float2bfloat16_rn(O / Lsum);
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
  const int t = blockIdx.x;
  if (t >= *t_dev) return;
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
static int attn_smem(int hd, int mt) {
  const int rows = 16 * mt, ld = hd + 8;
  const int load = (rows * ld + 4 * 2 * 32 * ld) * 2;
  const int merge = rows * ld * 2 + (4 * rows * hd + 4 * rows * 2) * 4;
  return load > merge ? load : merge;
}

template <int HD, int MT>
static int launch_attn_t(const AttnArgs& a, cudaStream_t s) {
  static bool cfg = false;
  const int smem = attn_smem(HD, MT);
  if (!cfg) {
    SPECTRE_CUDA_TRY(
        cudaFuncSetAttribute(k_attention<HD, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cfg = true;
  }
  dim3 grid(a.split_max, a.rb_max, a.n_req * a.n_kv);
  k_attention<HD, MT><<<grid, kAttnThreads, smem, s>>>(a);
  SPECTRE_LAUNCH_CHECK("k_attention");
  k_attn_combine<HD, MT><<<dim3(a.rb_max, a.n_req * a.n_kv), 128, 0, s>>>(a);
  SPECTRE_LAUNCH_CHECK("k_attn_combine");
  return SPECTRE_OK;
}

int launch_attention(const AttnArgs& a, int hd, int mt, cudaStream_t s) {
  if (hd == 128 && mt == 1) return launch_attn_t<128, 1>(a, s);
  if (hd == 128 && mt == 2) return launch_attn_t<128, 2>(a, s);
  if (hd == 64 && mt == 1) return launch_attn_t<64, 1>(a, s);
  if (hd == 64 && mt == 2) return launch_attn_t<64, 2>(a, s);
  return arg_fail("attention: head_dim must be 64 or 128, mt 1 or 2");
}

int launch_embed_rmsnorm(const int* tok, const int* t_dev, int t_cap, const void* E,
                         const float* w, float* h, void* x, int d, float eps, cudaStream_t s) {
  k_embed_rmsnorm<<<t_cap, 256, 0, s>>>(tok, t_dev, reinterpret_cast<const __nv_bfloat16*>(E),
                                        w, h, reinterpret_cast<__nv_bfloat16*>(x), d, eps);
  SPECTRE_LAUNCH_CHECK("k_embed_rmsnorm");
  return SPECTRE_OK;
}

int launch_residual_rmsnorm(const float* part, int splits, int rows_cap, const int* t_dev,
                            int t_cap, const float* w, float* h, void* x, int d, float eps,
                            cudaStream_t s) {
  if (d % 4 || splits > kMaxSplits) return arg_fail("residual_rmsnorm: d % 4 / splits");
  const int nv = d / 4;
  const int threads = nv < 512 ? ((nv + 31) / 32) * 32 : 512;
  const int vec = (nv + threads - 1) / threads;
  auto* xb = reinterpret_cast<__nv_bfloat16*>(x);
  if (vec <= 1)
    k_residual_rmsnorm_v<1><<<t_cap, threads, 0, s>>>(part, splits, rows_cap, t_dev, w, h, xb, d,
                                                      eps);
  else if (vec <= 2)
    k_residual_rmsnorm_v<2><<<t_cap, threads, 0, s>>>(part, splits, rows_cap, t_dev, w, h, xb, d,
                                                      eps);
  else if (vec <= 4)
    k_residual_rmsnorm_v<4><<<t_cap, threads, 0, s>>>(part, splits, rows_cap, t_dev, w, h, xb, d,
                                                      eps);
  else
    return arg_fail("residual_rmsnorm: d > 8192");
  SPECTRE_LAUNCH_CHECK("k_residual_rmsnorm");
  return SPECTRE_OK;
}

int launch_qkv_rope_kv(const float* part, int splits, int rows_cap, const int* t_dev, int t_cap,
                       const int* tok_pos, const int* tok_slot, const void* rope, void* q,
                       void* kc, void* vc, int n_q, int n_kv, int hd, int ctx_cap,
                       cudaStream_t s) {
  if (splits > kMaxSplits) return arg_fail("qkv_rope_kv: splits");
  const int pairs = (n_q + 2 * n_kv) * hd / 2;
  k_qkv_rope_kv<<<dim3(t_cap, (pairs + 127) / 128), 128, 0, s>>>(
      part, splits, rows_cap, t_dev, tok_pos, tok_slot, reinterpret_cast<const float2*>(rope),
      reinterpret_cast<__nv_bfloat16*>(q), reinterpret_cast<__nv_bfloat16*>(kc),
      reinterpret_cast<__nv_bfloat16*>(vc), n_q, n_kv, hd, ctx_cap);
  SPECTRE_LAUNCH_CHECK("k_qkv_rope_kv");
  return SPECTRE_OK;
}

int launch_argmax_reduce(const float* val, const int* idx, int n_tiles, int rows_cap,
                         const int* t_dev, int t_cap, int* out_tok, float* out_val,
                         cudaStream_t s) {
  k_argmax_reduce<<<t_cap, 256, 0, s>>>(val, idx, n_tiles, rows_cap, t_dev, out_tok, out_val);
  SPECTRE_LAUNCH_CHECK("k_argmax_reduce");
  return SPECTRE_OK;
}

int launch_rope_table(void* rope, int ctx_cap, int hd, double theta, cudaStream_t s) {
  k_rope_table<<<256, 256, 0, s>>>(reinterpret_cast<float2*>(rope), ctx_cap, hd, theta);
  SPECTRE_LAUNCH_CHECK("k_rope_table");
  return SPECTRE_OK;
}

}  // namespace spectre
