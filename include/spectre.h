/*
 * spectre.h — C ABI of the B200-native SPECTRE decode loop (libspectre.so).
 *
 * Plain pointers and sizes only; every device pointer is a CUDA device
 * address, every `stream` is a cudaStream_t passed as void*.  All entry
 * points return 0 on success and a negative SPECTRE_E* code on failure;
 * protocol violations detected on the device are reported through the
 * scalar output word (see SpectreOracleOutputs.scalars) and surfaced by the
 * host layer as ProtocolViolation (target_engine.py:19-20).
 *
 * The reference (`specsim`, pure Python) exposes its decode loop through
 * duck-typed Python APIs rather than an FFI; each entry point below names the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/specsim/).  INTEGRATION.md shows the ctypes stub a
 * maintainer would add on the reference side.
 */
#ifndef SPECTRE_H_
#define SPECTRE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPECTRE_OK 0
#define SPECTRE_EINVAL (-1)
#define SPECTRE_ECUDA (-2)
#define SPECTRE_ENOMEM (-3)
#define SPECTRE_EUNSUPPORTED (-4)

/* PAD token of the oracle mode: the maximum 64-bit value (core.py:16-18). */
#define SPECTRE_PAD UINT64_MAX

/* Variants (sim.py:55-67). */
#define SPECTRE_VARIANT_AR 0
#define SPECTRE_VARIANT_ORDINARY 1
#define SPECTRE_VARIANT_PARALLEL 2
#define SPECTRE_VARIANT_HYBRID 3

/* ---------------------------------------------------------------- version */
/* Library build identifier ("spectre-b200 <semver> sm_100a"). */
const char* spectre_version(void);
/* Last CUDA / argument error message of the calling thread. */
const char* spectre_last_error(void);

/* ------------------------------------------- synthetic model pair (K8) ----
 * Replaces TokenStreamOracle.reference_token / prompt_token
 * (oracle.py:53-67): out[i] = stream value of (seed, stream_id, req[i], pos[i])
 * with PAD remapped to 0.  stream_id 0 = output stream, 1 = prompt stream.
 */
int spectre_oracle_stream(uint64_t seed, int32_t stream_id, const int64_t* req,
                          const int64_t* pos, uint64_t* out, int64_t n,
                          void* stream);

/* Replaces TokenStreamOracle.draft_propose (oracle.py:69-88) for a batch of
 * segments: segment s proposes count[s] tokens of request req[s] from
 * start[s]; token j keeps the reference value iff uniforms[off[s]+j] < alpha,
 * else ref ^ 0x5BD1E995.  out is [n_seg, max_count] row-major. */
int spectre_oracle_propose(uint64_t seed, double alpha, const int64_t* req,
                           const int64_t* start, const int32_t* count,
                           const int64_t* off, const double* uniforms,
                           uint64_t* out, int32_t max_count, int64_t n_seg,
                           void* stream);

/* Replaces TokenStreamOracle.verify (oracle.py:90-113) for a batch of
 * candidates ([n_cand, width] row-major, PAD-padded, len[c] real slots):
 * accepted[c], bonus[c]; new_position = start + accepted + 1. */
int spectre_oracle_verify(uint64_t seed, const int64_t* req, const int64_t* start,
                          const uint64_t* cand, const int32_t* len, int32_t width,
                          int32_t* accepted, uint64_t* bonus, int64_t n_cand,
                          void* stream);

/* ------------------------------------------------ draft RNG (MT19937) ----
 * The reference draws the proposer's uniforms from
 * random.Random(f"{seed}:draft") (sim.py:250).  Host side: init_by_array
 * over the caller-supplied key words (Python's str-seed expansion,
 * int.from_bytes(s + sha512(s)), little-endian 32-bit words); writes the
 * 624-word state + index (=624) to state_out[625].  Device side: fills
 * out[0..n) with genrand_res53 uniforms continuing from the state in
 * state_dev[625] (updated in place). */
int spectre_mt19937_init_by_array(const uint32_t* key, int32_t key_len,
                                  uint32_t* state_out);
int spectre_mt19937_uniforms(uint32_t* state_dev, double* out, int64_t n,
                             void* stream);

/* ---------------------------------------- the decode loop, oracle mode ----
 * Replaces specsim.run(config, variant) (sim.py:989-1005) in the fault-free
 * regime: the whole round loop — controller (sim.py:431-467), candidate
 * assembly (target_engine.py:132-221), draft sync/rebase/propose
 * (draft_engine.py:72-120, 246-300, 412-431), verify, commit, suffix reuse,
 * rollback set and r-hat (target_engine.py:227-308) and the simulated clock —
 * runs on the device in one persistent kernel with no host round trip. */
typedef struct SpectreOracleConfig {
  uint64_t seed;
  int32_t n_requests;
  int32_t max_concurrency;
  int32_t gamma;
  int32_t output_len;
  int32_t variant;          /* SPECTRE_VARIANT_* */
  int32_t fairness_period;
  int32_t has_fixed_l;      /* fixed_threshold_l given */
  int32_t max_rounds;       /* capacity of the per-round trace buffers */
  double alpha;
  double t_target;
  double t_draft;
  double delay;             /* constant transport delay (core.py:98) */
  double t_target_slope;
  double ema_decay;
  double fixed_threshold_l;
} SpectreOracleConfig;

typedef struct SpectreOracleOutputs {
  /* per request */
  uint64_t* committed;      /* [n_requests * output_len] */
  int32_t* committed_pos;   /* [n_requests] */
  double* admitted_at;      /* [n_requests] */
  double* finished_at;      /* [n_requests] */
  /* per round, [max_rounds] each */
  int32_t* round_mode;      /* 'O', 'P', 'F' */
  int32_t* round_participants;
  int32_t* round_delta;     /* committed tokens this round */
  int32_t* round_n_roll;    /* |R_n| (target_engine.py:285-302) */
  int32_t* round_content_sum;
  int32_t* round_content_n;
  int32_t* round_queries;   /* draft queries sent this round */
  int32_t* round_draft_tokens;
  int32_t* round_n_padded;  /* PADDED candidates (the paper's fallback r) */
  double* round_started;
  double* round_dispatch;
  double* round_commit;
  double* round_draft_start; /* NaN when no draft round ran */
  double* round_draft_done;
  double* round_r_hat_ema;
  double* round_accepted_len_ema;
  double* round_r_star;
  /* scalars: [0] rounds, [1] rng draws, [2] error code, [3] error request,
   * [4] requests finished */
  int64_t* scalars;
} SpectreOracleOutputs;

/* Device workspace the loop needs (bytes, 256-aligned). */
size_t spectre_oracle_workspace_bytes(const SpectreOracleConfig* cfg);

int spectre_oracle_run(const SpectreOracleConfig* cfg, const double* arrivals,
                       const double* uniforms, int64_t n_uniforms,
                       void* workspace, const SpectreOracleOutputs* out,
                       void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRE_H_ */
