// mt19937.cu — the draft proposer's uniform stream.
//
// The reference draws one rng.random() per proposed token from
// random.Random(f"{seed}:draft") (sim.py:250, oracle.py:83-85): CPython's
// MT19937 seeded by init_by_array and read through genrand_res53.  The
// seeding (a few hundred sequential integer ops) is done on the host; the
// stream itself is generated on the device: one CTA of 624 threads performs
// the twist in four dependency-ordered phases and tempers in parallel.
#include <cstring>
#include <string>

#include "common.cuh"

namespace spectre {

constexpr int kN = 624, kM = 397;
constexpr uint32_t kMatrixA = 0x9908b0dfu, kUpper = 0x80000000u, kLower = 0x7fffffffu;

static void init_genrand(uint32_t* mt, uint32_t s) {
  mt[0] = s;
  for (int i = 1; i < kN; ++i) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
}

__device__ __forceinline__ uint32_t temper(uint32_t y) {
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

__device__ __forceinline__ uint32_t twist_one(uint32_t cur, uint32_t next, uint32_t far) {
  const uint32_t y = (cur & kUpper) | (next & kLower);
  return far ^ (y >> 1) ^ ((y & 1u) ? kMatrixA : 0u);
}

// In-place twist of s[624] by 624 threads.  new[i] depends on old[i], old[i+1]
// and old/new[i+397 mod 624]; the four phases respect those dependencies.
__device__ void twist(uint32_t* s) {
  const int i = threadIdx.x;
  uint32_t v = 0;
  // phase 1: i in [0, 227): all inputs old
  if (i < kN - kM) v = twist_one(s[i], s[i + 1], s[i + kM]);
  __syncthreads();
  if (i < kN - kM) s[i] = v;
  __syncthreads();
  // phase 2: i in [227, 454): far input new[i-227] (phase 1), next old
  if (i >= kN - kM && i < 2 * (kN - kM)) v = twist_one(s[i], s[i + 1], s[i + kM - kN]);
  __syncthreads();
  if (i >= kN - kM && i < 2 * (kN - kM)) s[i] = v;
  __syncthreads();
  // phase 3: i in [454, 623): far input new[i-227] in [227,396) (phase 2)
  if (i >= 2 * (kN - kM) && i < kN - 1) v = twist_one(s[i], s[i + 1], s[i + kM - kN]);
  __syncthreads();
  if (i >= 2 * (kN - kM) && i < kN - 1) s[i] = v;
  __syncthreads();
  // phase 4: i = 623: next = new[0], far = new[396]
  if (i == kN - 1) s[i] = twist_one(s[kN - 1], s[0], s[kM - 1]);
  __syncthreads();
}

// state[0..624) words + state[624] = index.  Emits 2n 32-bit words into out
// (viewed as uint32), then converts each pair in place to genrand_res53.
__global__ void __launch_bounds__(kN, 1) k_mt_uniforms(uint32_t* state, double* out, int64_t n) {
  __shared__ uint32_t s[kN];
  __shared__ int s_idx;
  const int i = threadIdx.x;
  s[i] = state[i];
  if (i == 0) s_idx = (int)state[kN];
  __syncthreads();
  uint32_t* w = reinterpret_cast<uint32_t*>(out);
  const int64_t words = 2 * n;
  int64_t produced = 0;
  int idx = s_idx;
  while (produced < words) {
    if (idx >= kN) {
      twist(s);
      idx = 0;
    }
    const int64_t avail = kN - idx;
    const int64_t take = (words - produced) < avail ? (words - produced) : avail;
    if (i < take) w[produced + i] = temper(s[idx + i]);
    produced += take;
    idx += (int)take;
    __syncthreads();
  }
  state[i] = s[i];
  if (i == 0) state[kN] = (uint32_t)idx;
  __syncthreads();
  __threadfence_block();
  for (int64_t k = i; k < n; k += kN) {
    const uint32_t a = w[2 * k] >> 5, b = w[2 * k + 1] >> 6;
    out[k] = ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
  }
}

}  // namespace spectre

using namespace spectre;

// CPython _randommodule.c init_by_array semantics.
extern "C" int spectre_mt19937_init_by_array(const uint32_t* key, int32_t key_len,
                                             uint32_t* state_out) {
  if (!key || key_len < 1 || !state_out) return arg_fail("spectre_mt19937_init_by_array");
  uint32_t mt[kN];
  init_genrand(mt, 19650218u);
  int i = 1, j = 0;
  int k = (kN > key_len ? kN : key_len);
  for (; k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    i++;
    j++;
    if (i >= kN) {
      mt[0] = mt[kN - 1];
      i = 1;
    }
    if (j >= key_len) j = 0;
  }
  for (k = kN - 1; k; k--) {
    mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    i++;
    if (i >= kN) {
      mt[0] = mt[kN - 1];
      i = 1;
    }
  }
  mt[0] = 0x80000000u;
  std::memcpy(state_out, mt, sizeof(mt));
  state_out[kN] = kN;
  return SPECTRE_OK;
}

extern "C" int spectre_mt19937_uniforms(uint32_t* state_dev, double* out, int64_t n,
                                        void* stream) {
  if (!state_dev || n < 0 || (n > 0 && !out)) return arg_fail("spectre_mt19937_uniforms");
  if (n == 0) return SPECTRE_OK;
  k_mt_uniforms<<<1, kN, 0, as_stream(stream)>>>(state_dev, out, n);
  SPECTRE_LAUNCH_CHECK("k_mt_uniforms");
  return SPECTRE_OK;
}
