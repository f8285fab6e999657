// protocol.cuh — device restatement of SPECTRE's per-request round operations.
//
// Shared by the oracle-mode decode loop (oracle_mode.cu) and the model-mode
// accept/assemble kernels.  Each function names the reference routine it
// implements (paths relative to /root/reference/pkg/src/specsim/).
// All floating-point controller arithmetic uses explicit _rn intrinsics so no
// FMA contraction can change a bit relative to the reference's IEEE doubles.
#pragma once

#include <cstdint>

namespace spectre {

constexpr uint64_t kPad = ~0ull;                 // core.py:16-18
constexpr uint64_t kDisagree = 0x5BD1E995ull;    // oracle.py:15
constexpr double kExitParallelMargin = 1.10;     // sim.py:199
// `round` controller re-probe (model mode only; not in the reference): the
// ordinary-round r-hat drift that triggers re-measuring r and T_par / T_ord,
// and the fewest rounds between two probes
constexpr double kReprobeDelta = 0.15;
constexpr int kReprobeMinRounds = 16;

enum CandKind : int32_t { kCached = 1, kRepaired = 2, kPadded = 3, kFallback = 4 };

// oracle.py:22-36 — the target's greedy stream in oracle mode.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t stream,
                                                   uint64_t req, uint64_t pos) {
  uint64_t x = seed * 0x9E3779B97F4A7C15ull + stream * 0xD6E8FEB86659FD93ull +
               req * 0xC2B2AE3D27D4EB4Full + pos * 0x165667B19E3779F9ull +
               0x2545F4914F6CDD1Dull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// oracle.py:53-57 / :62-64 — PAD is remapped to 0.
__host__ __device__ __forceinline__ uint64_t stream_token(uint64_t seed, uint64_t stream,
                                                          uint64_t req, uint64_t pos) {
  uint64_t t = mix64(seed, stream, req, pos);
  return t == kPad ? 0ull : t;
}

__device__ __forceinline__ uint64_t ref_token(uint64_t seed, uint64_t req, uint64_t pos) {
  return stream_token(seed, 0, req, pos);
}

// analytics.py:57-70 — r* = (g-1) L T_D / ((T_T + (g-1) T_D)(L - 1)).
__device__ __forceinline__ double critical_fallback_ratio(double L, int gamma,
                                                          double t_target, double t_draft) {
  const double g1 = (double)(gamma - 1);
  const double num = __dmul_rn(__dmul_rn(g1, L), t_draft);
  const double den = __dmul_rn(__dadd_rn(t_target, __dmul_rn(g1, t_draft)), __dsub_rn(L, 1.0));
  return __ddiv_rn(num, den);
}

// d*x + (1-d)*y in the reference's operation order (sim.py:677-678,
// target_engine.py:402).
__device__ __forceinline__ double ema_step(double d, double x, double y) {
  return __dadd_rn(__dmul_rn(d, x), __dmul_rn(__dsub_rn(1.0, d), y));
}

// sim.py:447-467 (hybrid branch) + analytics.py:73-75.  mode: 0 none, 'O', 'P'.
// Returns the mode for this round; r_star_out receives the threshold used.
__device__ __forceinline__ int choose_mode_hybrid(int prev_mode, bool has_ema, double r_hat_ema,
                                                  bool has_L, double L, int gamma,
                                                  double t_target, double t_draft,
                                                  double* r_star_out) {
  const double r_hat = has_ema ? r_hat_ema : 0.0;
  double r_star;
  if (!has_L || L <= 1.0 + 1e-9) {
    r_star = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  } else {
    r_star = critical_fallback_ratio(L, gamma, t_target, t_draft);
  }
  *r_star_out = r_star;
  if (prev_mode == 'P') {
    return (r_hat > __dmul_rn(r_star, kExitParallelMargin)) ? 'O' : 'P';
  }
  return (r_hat <= r_star) ? 'P' : 'O';
}

// ---------------------------------------------------------------------------
// Draft-side session ops over a token history held in global memory.
// ---------------------------------------------------------------------------

// draft_engine.py:246-280 + apply_recovery :82-99.  `tok(k)` yields the k-th
// token of the synced delta (committed[start + k]).  Returns the new length
// and the first invalidated position (for KV rollback in model mode) via
// *invalid_from (== new length when nothing was invalidated).
template <typename TokFn, typename RefFn>
__device__ __forceinline__ int32_t session_on_sync(uint64_t* h, int32_t hl, int32_t start,
                                                   int32_t ntok, TokFn tok, RefFn ref,
                                                   int32_t* invalid_from) {
  *invalid_from = 0x7fffffff;
  if (start > hl) {
    // gap: rebuild the verified prefix (draft_engine.py:255-266)
    for (int32_t q = 0; q < start; ++q) h[q] = ref(q);
    for (int32_t k = 0; k < ntok; ++k) h[start + k] = tok(k);
    *invalid_from = 0;
    return start + ntok;
  }
  const int32_t overlap = min(ntok, hl - start);
  int32_t diverged = overlap;
  for (int32_t k = 0; k < overlap; ++k) {
    if (tok(k) != h[start + k]) { diverged = k; break; }
  }
  if (diverged < overlap || start + ntok > hl) {
    const int32_t delta = start + diverged;
    const int32_t vlen = start + ntok;
    const int32_t ov = min(vlen, hl);
    if (delta < ov) {
      for (int32_t q = delta; q < vlen; ++q) h[q] = tok(q - start);
      *invalid_from = delta;
      return vlen;
    } else if (vlen > hl) {
      for (int32_t q = hl; q < vlen; ++q) h[q] = tok(q - start);
      return vlen;
    }
  }
  return hl;
}

// draft_engine.py:412-431.
template <typename RefFn>
__device__ __forceinline__ int32_t session_rebase(uint64_t* h, int32_t hl, int32_t anchor,
                                                  RefFn ref, int32_t* invalid_from) {
  *invalid_from = 0x7fffffff;
  if (anchor < hl) {
    *invalid_from = anchor;
    return anchor;
  }
  for (int32_t q = hl; q < anchor; ++q) h[q] = ref(q);
  return anchor > hl ? anchor : hl;
}

// ---------------------------------------------------------------------------
// Target-side ops.
// ---------------------------------------------------------------------------

// Longest exact-match prefix (oracle.py:99-104); PAD never matches because
// the reference stream never emits it.  `ref(q)` = target greedy token at q.
template <typename RefFn>
__device__ __forceinline__ int32_t verify_prefix(const uint64_t* cand, int32_t len, int32_t start,
                                                 RefFn ref) {
  int32_t accepted = 0;
  for (int32_t k = 0; k < len; ++k) {
    if (cand[k] != ref(start + accepted)) break;
    ++accepted;
  }
  return accepted;
}

// target_engine.py:252-279 — returns the new cached length (0 = rollback) and
// fills cached[] / *cached_start.
__device__ __forceinline__ int32_t reuse_or_discard(const uint64_t* prep, int32_t plen,
                                                    int32_t pstart, const uint64_t* committed,
                                                    int32_t pos, bool done, uint64_t* cached,
                                                    int32_t* cached_start) {
  if (plen <= 0 || done) return 0;
  if (pstart > pos) return 0;
  const int32_t overlap_end = min(pstart + plen, pos);
  for (int32_t p = pstart; p < overlap_end; ++p) {
    if (prep[p - pstart] != committed[p]) return 0;
  }
  const int32_t off = pos - pstart;
  const int32_t n = plen - off;
  if (n <= 0) return 0;
  for (int32_t k = 0; k < n; ++k) cached[k] = prep[off + k];
  *cached_start = pos;
  return n;
}

}  // namespace spectre
