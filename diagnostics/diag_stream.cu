// diag_stream.cu — diagnostics: per-SM streaming rate of the data-movement
// engines the hot kernels use (timing only; not on the decode path).
//   mode 0: 2-D TMA boxes {64 el, 128 rows} of a [rows][K] bf16 matrix (GEMM weights)
//   mode 1: 1-D cp.async.bulk of `stage_bytes` contiguous bytes
//   mode 2: 2-D TMA boxes {64 el, 256 rows}
// One CTA per SM, one producer lane keeping `stages` stages in flight, one
// consumer warp releasing them.  Each CTA streams its own contiguous share.
#include <cuda.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "gemm.h"
#include "ptx.cuh"

namespace spectre {

__global__ void __launch_bounds__(64, 1)
k_diag_stream(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tx,
              const uint8_t* src, size_t bytes_per_cta, int mode, int stages, int stage_bytes,
              int K, int rows_per_cta, int x_boxes, int stagger) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);   // X boxes at +4096
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int n = (int)(bytes_per_cta / stage_bytes);
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int kb = K / 64;                        // 64-element k blocks per row
      const int box_rows = mode == 2 ? 256 : 128;
      for (int g = 0; g < n; ++g) {
        const int s = g % stages;
        if (g >= stages) mbar_wait(&empty[s], (uint32_t)((g / stages) - 1) & 1u);
        uint8_t* st = smem + s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes + x_boxes * 8192);
        if (x_boxes) {   // shared activation boxes (same for every CTA) at this k block
          const int kx = stagger ? (g + blockIdx.x * 7) % kb : g % kb;
          for (int b = 0; b < x_boxes; ++b)
            tma_load_2d(smem + stages * stage_bytes + 4096 + (s * x_boxes + b) * 8192, &tx,
                        &full[s], kx * 64, b * 64, policy_evict_last());
        }
        if (mode == 1) {
          bulk_load(st, src + (size_t)blockIdx.x * bytes_per_cta + (size_t)g * stage_bytes,
                    stage_bytes, &full[s]);
        } else {
          // stage = stage_bytes / (box_rows*128) boxes walking k then rows (GEMM order)
          // GEMM order: a stage = the same 64-element k block of `boxes` row boxes
          const int boxes = stage_bytes / (box_rows * 128);
          const int kblk = g % kb, rg = g / kb;
          for (int b = 0; b < boxes; ++b)
            tma_load_2d(st + b * box_rows * 128, &tm, &full[s], kblk * 64,
                        blockIdx.x * rows_per_cta + (rg * boxes + b) * box_rows, pol);
        }
      }
    }
  } else {
    for (int g = 0; g < n; ++g) {
      const int s = g % stages;
      mbar_wait(&full[s], (uint32_t)(g / stages) & 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

}  // namespace spectre

using namespace spectre;

// Streams `bytes_per_cta` per CTA over `grid` CTAs; returns elapsed ms via events.
extern "C" int spectre_diag_stream(const void* buf, int64_t bytes_per_cta, int32_t grid,
                                   int32_t mode, int32_t stages, int32_t stage_bytes, int32_t K,
                                   int32_t x_boxes, int32_t stagger, const void* xbuf,
                                   float* ms_out, void* stream) {
  cudaStream_t s = as_stream(stream);
  CUtensorMap tm{};
  const int box_rows = mode == 2 ? 256 : 128;
  const int rows_per_cta = (int)(bytes_per_cta / (K * 2));
  if (mode != 1) {
    if (int e = make_tmap_bf16(&tm, buf, (uint64_t)K, (uint64_t)rows_per_cta * grid, box_rows, 64))
      return e;
  }
  if (mode != 1 && stage_bytes % (box_rows * 128)) return arg_fail("diag: stage < box");
  CUtensorMap tx{};
  if (x_boxes) {
    if (int e = make_tmap_bf16(&tx, xbuf, (uint64_t)K, (uint64_t)64 * x_boxes, 64, 64)) return e;
  }
  const int smem = stages * stage_bytes + 4096 + stages * x_boxes * 8192 + 1024;
  if (smem > 232448) return arg_fail("diag: smem");
  SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_diag_stream, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  k_diag_stream<<<grid, 64, smem, s>>>(tm, tx, reinterpret_cast<const uint8_t*>(buf),
                                       (size_t)bytes_per_cta, mode, stages, stage_bytes, K,
                                       rows_per_cta, x_boxes, stagger);
  cudaEventRecord(e1, s);
  SPECTRE_CUDA_TRY(cudaEventSynchronize(e1));
  SPECTRE_LAUNCH_CHECK("k_diag_stream");
  cudaEventElapsedTime(ms_out, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return SPECTRE_OK;
}

// TMEM load latency/throughput: 8 warps x `iters` x tcgen05.ld.32x32b.x32 (+ wait each).
namespace spectre {
__global__ void __launch_bounds__(320, 1) k_diag_tmem(int iters, int shape, unsigned long long* out) {
  using namespace ptx;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot;
  unsigned long long t0 = clock64();
  float acc = 0.f;
  if (warp >= 2) {
    const uint32_t tq = base + ((uint32_t)((warp & 3) * 32) << 16);
    for (int i = 0; i < iters; ++i) {
      float v[32];
      tmem_ld32(tq + (uint32_t)((i * 32) & 511), v);
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k];
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && warp >= 2) out[blockIdx.x * 8 + warp - 2] = t1 - t0;
  if (acc == 1234.5f) out[0] = 0;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(base);
  }
}
}  // namespace spectre

extern "C" int spectre_diag_tmem(int32_t iters, unsigned long long* out_dev, void* stream) {
  k_diag_tmem<<<1, 320, 0, as_stream(stream)>>>(iters, 0, out_dev);
  SPECTRE_LAUNCH_CHECK("k_diag_tmem");
  return SPECTRE_OK;
}

// MMA round trip: one thread issues `nmma` tcgen05.mma (M=128, N=n, K=16
// each, operands in shared memory), commits to an mbarrier and waits for it;
// `out` gets the average cycles per iteration (per CTA).  pipelined=1 keeps
// `depth` commits in flight (like the GEMM ring) and reports cycles per
// iteration of the steady state.
namespace spectre {
__global__ void __launch_bounds__(128, 1)
k_diag_mma(int iters, int nmma, int n, int depth, unsigned long long* out) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t acc = slot;
  if (warp == 1 && lane == 0) {
    const uint32_t sa = smem_u32(smem);
    const uint32_t sb = sa + 128 * 128;
    const uint32_t id = idesc_bf16_f32(128, (uint32_t)n);
    unsigned long long t0 = 0;
    // depth >= 1: commit per iteration, wait `depth` commits back;
    // 0: commit per iteration, no waits; -1: one commit at the end
    const int D = depth > 0 ? depth : 1;
    unsigned long long t_issue = 0;
    for (int it = 0; it < iters + 8; ++it) {
      if (it == 8) t0 = clock64();
      const int s = it % D;
      if (depth > 0 && it >= depth) mbar_wait(&bars[s], (uint32_t)((it / depth) - 1) & 1u);
      for (int k = 0; k < nmma; ++k)
        mma_bf16_ss(acc, umma_desc_kmajor<128>(sa + (k & 3) * 32),
                    umma_desc_kmajor<128>(sb + (k & 3) * 32), id, it > 0 || k > 0);
      if (depth >= 0) mma_commit(depth > 0 ? &bars[s] : &bars[15]);
    }
    t_issue = clock64();
    if (depth > 0) {
      for (int it = iters + 8 - depth; it < iters + 8; ++it) {
        const int s = it % depth;
        mbar_wait(&bars[s], (uint32_t)(it / depth) & 1u);
      }
    } else {
      mma_commit(&bars[14]);
      mbar_wait(&bars[14], 0u);
    }
    const unsigned long long t1 = clock64();
    if (gridDim.x == 1) out[1] = (t_issue - t0) / (unsigned long long)iters;
    out[blockIdx.x] = (t1 - t0) / (unsigned long long)iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(acc);
  }
}
}  // namespace spectre

namespace spectre {
template <int NM>
__global__ void __launch_bounds__(128, 1) k_diag_mma_u(int iters, int n, unsigned long long* out) {
  using namespace ptx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t acc = slot;
  if (warp == 1 && lane == 0) {
    const uint32_t sa = smem_u32(smem);
    const uint32_t sb = sa + 128 * 128;
    const uint32_t id = idesc_bf16_f32(128, (uint32_t)n);
    uint64_t ad[NM], bd[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      ad[k] = umma_desc_kmajor<128>(sa + (k & 3) * 32 + (k >> 2) * 16384);
      bd[k] = umma_desc_kmajor<128>(sb + (k & 3) * 32);
    }
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int s = it & 7;
      if (it >= 8) mbar_wait(&bars[s], (uint32_t)((it >> 3) - 1) & 1u);
#pragma unroll
      for (int k = 0; k < NM; ++k) {
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(acc),
                     "l"(ad[k]), "l"(bd[k]), "r"(id)
                     : "memory");
      }
      mma_commit(&bars[s]);
    }
    for (int it = iters - 8; it < iters; ++it) mbar_wait(&bars[it & 7], (uint32_t)(it >> 3) & 1u);
    out[0] = (clock64() - t0) / (unsigned long long)iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(acc);
  }
}
}  // namespace spectre

extern "C" int spectre_diag_mma_unrolled(int32_t nm, int32_t n, uint64_t* cycles_out) {
  unsigned long long* d = nullptr;
  SPECTRE_CUDA_TRY(cudaMalloc(&d, 8));
  const int smem = 2 * 16384 + 256 * 128 + 1024;
  auto run = [&](auto kern) -> int {
    SPECTRE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<1, 128, smem>>>(2000, n, d);
    SPECTRE_CUDA_TRY(cudaDeviceSynchronize());
    return 0;
  };
  int r = nm == 1 ? run(k_diag_mma_u<1>) : nm == 4 ? run(k_diag_mma_u<4>)
        : nm == 8 ? run(k_diag_mma_u<8>) : run(k_diag_mma_u<16>);
  if (r) return r;
  cudaMemcpy(cycles_out, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return SPECTRE_OK;
}

extern "C" int spectre_diag_mma(int32_t grid, int32_t iters, int32_t nmma, int32_t n,
                                int32_t depth, uint64_t* cycles_out, void* stream) {
  if (depth < -1 || depth > 14 || n < 16 || n > 256 || n % 16) return arg_fail("diag_mma");
  cudaStream_t s = as_stream(stream);
  unsigned long long* d = nullptr;
  SPECTRE_CUDA_TRY(cudaMalloc(&d, (grid + 1) * 8));
  const int smem = 128 * 128 + 256 * 128 + 1024;
  SPECTRE_CUDA_TRY(cudaFuncSetAttribute(k_diag_mma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        smem));
  k_diag_mma<<<grid, 128, smem, s>>>(iters, nmma, n, depth, d);
  SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
  SPECTRE_LAUNCH_CHECK("k_diag_mma");
  std::vector<unsigned long long> h(grid + 1);
  cudaMemcpy(h.data(), d, (grid + 1) * 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (grid == 1) {   // [0] total per iteration, [1] issue-only per iteration
    cycles_out[0] = h[0];
    cycles_out[1] = h[1];
    return SPECTRE_OK;
  }
  unsigned long long sum = 0;
  for (int i = 0; i < grid; ++i) sum += h[i];
  *cycles_out = sum / grid;
  return SPECTRE_OK;
}
