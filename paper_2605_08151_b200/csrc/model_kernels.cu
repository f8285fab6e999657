// model_kernels.cu — RMSNorm / embedding, RoPE + KV-cache write, gamma-query
// attention over the KV cache, split combine, and the greedy argmax reduce.
//
// All reductions use a fixed order that depends only on absolute positions
// (never on how many tokens share the batch), so a token's logits are
// bit-identical in a verify pass and in plain autoregressive decoding.
#include <cuda_bf16.h>

#include <algorithm>
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Persistent attention.  A grid of one or more CTAs per SM walks the work
// items (request, kv head, block of 16 query rows, split of `chunk` keys).
// Rows are token-major x GQA heads (4 tokens x 4 heads = one 16-row MMA tile
// for a gamma=4 verify).  Inside an item, warp w of NW owns keys
// [c0 + w*chunk/NW, +chunk/NW) and streams them in 16-key steps through two
// cp.async buffers (step i+1 loading while step i runs S = Q K^T, the online
// softmax and O += P V on mma.sync m16n8k16).  The NW warps merge in a fixed
// order, write the split's partial, and the last split of a row block to
// finish merges all splits in split order into the bf16 output.  Chunk / warp
// / step boundaries are absolute key positions: a token's result does not
// depend on the rest of the batch.
template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32) k_attention(AttnArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int ROWS = 16;
  constexpr int STEP = 16;
  constexpr int LD = HD + 8;           // padded smem row: conflict-free ldmatrix
  constexpr int TILE = STEP * LD;      // one K or V step tile (elements)
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) uint8_t smem_attn[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sKV = sQ + ROWS * LD;  // per warp: 2 buffers x (K, V)
  __shared__ int s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int group = a.n_q / a.n_kv;
  const int g = lane >> 2, tq = lane & 3;
  __nv_bfloat16* wbuf = sKV + warp * 4 * TILE;
  const int n_items = a.n_req * a.n_kv * a.rb_max * a.split_max;
  const int per_warp = a.chunk / NW;

  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int split = item % a.split_max;
    const int rb = (item / a.split_max) % a.rb_max;
    const int bk = item / (a.split_max * a.rb_max);
    const int b = bk / a.n_kv, kvh = bk % a.n_kv;
    const int nn = a.n_new[b];
    const int rows_total = nn * group;
    if (rb * ROWS >= rows_total) continue;
    const int p0 = a.pos0[b];
    const int c0 = split * a.chunk;
    const int last_row = min(rows_total, (rb + 1) * ROWS) - 1;
    const int p_max = p0 + last_row / group;   // largest query position of the block
    if (c0 > p_max) continue;                  // chunk entirely in the causal future
    const int kv_len = p0 + nn;
    const int qoff = a.q_off[b];
    const size_t kv_base = ((size_t)a.slot[b] * a.n_kv + kvh) * a.ctx_cap;

    for (int c = tid; c < ROWS * (HD / 8); c += NT) {
      const int r = c / (HD / 8), ch = c % (HD / 8);
      const int R = rb * ROWS + r;
      const bool valid = R < rows_total;
      const int j = valid ? R / group : 0, hh = valid ? R % group : 0;
      const __nv_bfloat16* src =
          a.q + (((size_t)(qoff + j) * a.n_q) + kvh * group + hh) * HD + ch * 8;
      cp_async16(ptx_smem(sQ + r * LD + ch * 8), src, valid);
    }
    cp_async_commit();

    const int w0 = c0 + warp * per_warp;
    const int w_end = min(w0 + per_warp, p_max + 1);
    const int steps = w_end > w0 ? (w_end - w0 + STEP - 1) / STEP : 0;
    auto issue = [&](int st) {
      const int kb = w0 + st * STEP;
      __nv_bfloat16* sK = wbuf + (st & 1) * 2 * TILE;
      __nv_bfloat16* sV = sK + TILE;
#pragma unroll
      for (int c = lane; c < STEP * (HD / 8); c += 32) {
        const int r = c / (HD / 8), ch = c % (HD / 8);
        const bool valid = kb + r < kv_len;
        const size_t off = (kv_base + (valid ? kb + r : 0)) * HD + ch * 8;
        cp_async16(ptx_smem(sK + r * LD + ch * 8), a.k + off, valid);
        cp_async16(ptx_smem(sV + r * LD + ch * 8), a.v + off, valid);
      }
      cp_async_commit();
    };
    if (steps > 0) issue(0);
    if (steps > 1) issue(1);
    if (steps > 1) cp_async_wait<2>();
    else if (steps > 0) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();   // Q tile visible to every warp

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
      const int R = rb * ROWS + g + hr * 8;
      qvalid[hr] = R < rows_total;
      qpos[hr] = p0 + (qvalid[hr] ? R / group : 0);
    }

    // Q fragments stay in registers for the whole item
    uint32_t qf[HD / 16][4];
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
      ldsm_x4(ptx_smem(sQ + (lane & 15) * LD + kk * 16 + (lane >> 4) * 8), qf[kk][0], qf[kk][1],
              qf[kk][2], qf[kk][3]);

    for (int st = 0; st < steps; ++st) {
      if (st + 1 < steps) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncwarp();
      const int kb = w0 + st * STEP;
      const __nv_bfloat16* sK = wbuf + (st & 1) * 2 * TILE;
      const __nv_bfloat16* sV = sK + TILE;
      // two independent accumulation chains per n-tile (even / odd k-steps)
      float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
      float t0[4] = {0.f, 0.f, 0.f, 0.f}, t1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        uint32_t b0, b1, b2, b3;
        const int mi = lane >> 3;
        ldsm_x4(ptx_smem(sK + ((mi >> 1) * 8 + (lane & 7)) * LD + kk * 16 + (mi & 1) * 8), b0, b1,
                b2, b3);
        if (kk & 1) {
          mma16816(t0, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
          mma16816(t1, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
        } else {
          mma16816(s0, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
          mma16816(s1, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s0[e] += t0[e];
        s1[e] += t1[e];
      }
      // mask + online softmax (log2 domain); s0: keys kb+2tq+{0,1}, s1: kb+8+2tq+{0,1}
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
      // P (A fragment of the 16-key k-step) x V
      const uint32_t pa0 = pack_bf16(p[0][0], p[0][1]);
      const uint32_t pa1 = pack_bf16(p[1][0], p[1][1]);
      const uint32_t pa2 = pack_bf16(p[0][2], p[0][3]);
      const uint32_t pa3 = pack_bf16(p[1][2], p[1][3]);
#pragma unroll
      for (int dp = 0; dp < HD / 16; ++dp) {
        const int mi = lane >> 3;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(ptx_smem(sV + ((mi & 1) * 8 + (lane & 7)) * LD + dp * 16 + (mi >> 1) * 8), b0,
                  b1, b2, b3);
        mma16816(o[2 * dp], pa0, pa1, pa2, pa3, b0, b1);
        mma16816(o[2 * dp + 1], pa0, pa1, pa2, pa3, b2, b3);
      }
      __syncwarp();
      if (st + 2 < steps) issue(st + 2);
    }

    // ---- merge the NW warps in fixed order (reuses the K/V area)
    __syncthreads();
    float* sO = reinterpret_cast<float*>(sKV);   // [NW][ROWS][HD]
    float* sML = sO + NW * ROWS * HD;            // [NW][ROWS][2]
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int r = g + hr * 8;
#pragma unroll
      for (int n = 0; n < HD / 8; ++n)
        *reinterpret_cast<float2*>(&sO[(warp * ROWS + r) * HD + n * 8 + 2 * tq]) =
            make_float2(o[n][hr * 2], o[n][hr * 2 + 1]);
      if (tq == 0) {
        sML[(warp * ROWS + r) * 2] = mrow[hr];
        sML[(warp * ROWS + r) * 2 + 1] = lrow[hr];
      }
    }
    __syncthreads();
    const size_t pidx = (((size_t)b * a.n_kv + kvh) * a.rb_max + rb) * a.split_max + split;
    for (int c = tid; c < ROWS * HD / 4; c += NT) {
      const int r = (c * 4) / HD, dcol = (c * 4) % HD;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, sML[(w * ROWS + r) * 2]);
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
      float Lsum = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float mw = sML[(w * ROWS + r) * 2];
        const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
        const float4 v = *reinterpret_cast<const float4*>(&sO[(w * ROWS + r) * HD + dcol]);
        O.x += v.x * f;
        O.y += v.y * f;
        O.z += v.z * f;
        O.w += v.w * f;
        Lsum += sML[(w * ROWS + r) * 2 + 1] * f;
      }
      *reinterpret_cast<float4*>(&a.part_o[(pidx * ROWS + r) * HD + dcol]) = O;
      if (dcol == 0) {
        a.part_ml[(pidx * ROWS + r) * 2] = M;
        a.part_ml[(pidx * ROWS + r) * 2 + 1] = Lsum;
      }
    }
    // ---- last split of this row block merges all splits in split order
    __threadfence();
    __syncthreads();
    const int n_split = (p_max + 1 + a.chunk - 1) / a.chunk;   // splits with c0 <= p_max
    if (tid == 0) {
      int* cnt = a.done_cnt + ((size_t)b * a.n_kv + kvh) * a.rb_max + rb;
      const int prev = atomicAdd(cnt, 1);
      s_last = (prev == n_split - 1);
      if (s_last) *cnt = 0;  // self-reset for the next launch
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const size_t base = (((size_t)b * a.n_kv + kvh) * a.rb_max + rb) * a.split_max;
      for (int c = tid; c < ROWS * HD / 4; c += NT) {
        const int r = (c * 4) / HD, dcol = (c * 4) % HD;
        const int R = rb * ROWS + r;
        if (R >= rows_total) continue;
        const int qp = p0 + R / group;
        const int ns = min(n_split, qp / a.chunk + 1);
        float M = -INFINITY;
        for (int sp = 0; sp < ns; ++sp)
          M = fmaxf(M, __ldcg(&a.part_ml[((base + sp) * ROWS + r) * 2]));
        float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
        float Lsum = 0.f;
        for (int sp = 0; sp < ns; ++sp) {
          const float ms = __ldcg(&a.part_ml[((base + sp) * ROWS + r) * 2]);
          const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          const float4 v = __ldcg(reinterpret_cast<const float4*>(
              &a.part_o[((base + sp) * ROWS + r) * HD + dcol]));
          O.x += v.x * f;
          O.y += v.y * f;
          O.z += v.z * f;
          O.w += v.w * f;
          Lsum += __ldcg(&a.part_ml[((base + sp) * ROWS + r) * 2 + 1]) * f;
        }
        const float inv = 1.f / Lsum;
        const int j = R / group, hh = R % group;
        __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
            a.out + (((size_t)(qoff + j)) * a.n_q + kvh * group + hh) * HD + dcol);
        dst[0] = __floats2bfloat162_rn(O.x * inv, O.y * inv);
        dst[1] = __floats2bfloat162_rn(O.z * inv, O.w * inv);
      }
    }
    __syncthreads();  // smem reused by the next item
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
template <int HD, int NW>
static int attn_smem() {
  constexpr int ld = HD + 8;
  constexpr int load = (16 * ld + NW * 4 * 16 * ld) * 2;
  constexpr int merge = 16 * ld * 2 + (NW * 16 * HD + NW * 16 * 2) * 4;
  return load > merge ? load : merge;
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

template <int HD, int NW>
static int launch_attn_t(const AttnArgs& a, cudaStream_t s) {
  static bool cfg = false;
  const int smem = attn_smem<HD, NW>();
  if (!cfg) {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_attention<HD, NW>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cfg = true;
  }
  int per_sm = 1;
  SPECTRE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_attention<HD, NW>,
                                                                 NW * 32, smem));
  per_sm = std::max(1, per_sm);
  const int items = a.n_req * a.n_kv * a.rb_max * a.split_max;
  const int grid = std::min(items, per_sm * num_sms());
  SPECTRE_LAUNCH_PDL("k_attention", k_attention<HD, NW>, dim3(grid), dim3(NW * 32), smem, s, a);
  return SPECTRE_OK;
}

int launch_attention(const AttnArgs& a, int hd, int mt, cudaStream_t s) {
  (void)mt;  // rows are processed in 16-row blocks (rb_max of them)
  if (hd == 128) return launch_attn_t<128, 8>(a, s);
  if (hd == 64) return launch_attn_t<64, 8>(a, s);
  return arg_fail("attention: head_dim must be 64 or 128");
}

int launch_embed_rmsnorm(const int* tok, const int* t_dev, int t_cap, const void* E,
                         const float* w, float* h, void* x, int d, float eps, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_embed_rmsnorm", k_embed_rmsnorm, dim3(t_cap), dim3(256), 0, s, tok, t_dev,
                     reinterpret_cast<const __nv_bfloat16*>(E), w, h,
                     reinterpret_cast<__nv_bfloat16*>(x), d, eps);
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
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<1>, dim3(t_cap), dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else if (vec <= 2)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<2>, dim3(t_cap), dim3(threads),
                       0, s, part, splits, rows_cap, t_dev, w, h, xb, d, eps);
  else if (vec <= 4)
    SPECTRE_LAUNCH_PDL("k_residual_rmsnorm", k_residual_rmsnorm_v<4>, dim3(t_cap), dim3(threads),
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
  SPECTRE_LAUNCH_PDL("k_qkv_rope_kv", k_qkv_rope_kv, dim3(t_cap, (pairs + 127) / 128), dim3(128),
                     0, s, part, splits, rows_cap, t_dev, tok_pos, tok_slot,
                     reinterpret_cast<const float2*>(rope), reinterpret_cast<__nv_bfloat16*>(q),
                     reinterpret_cast<__nv_bfloat16*>(kc), reinterpret_cast<__nv_bfloat16*>(vc),
                     n_q, n_kv, hd, ctx_cap);
  return SPECTRE_OK;
}

int launch_argmax_reduce(const float* val, const int* idx, int n_tiles, int rows_cap,
                         const int* t_dev, int t_cap, int* out_tok, float* out_val,
                         cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_argmax_reduce", k_argmax_reduce, dim3(t_cap), dim3(256), 0, s, val, idx,
                     n_tiles, rows_cap, t_dev, out_tok, out_val);
  return SPECTRE_OK;
}

int launch_rope_table(void* rope, int ctx_cap, int hd, double theta, cudaStream_t s) {
  k_rope_table<<<256, 256, 0, s>>>(reinterpret_cast<float2*>(rope), ctx_cap, hd, theta);
  SPECTRE_LAUNCH_CHECK("k_rope_table");
  return SPECTRE_OK;
}

}  // namespace spectre
