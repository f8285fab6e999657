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
  /* draft latency model (draft_engine.py:158-164, 205-216): a round's step
   * latency is t_draft + t_draft_slope * max(0, queries - t_draft_free_batch),
   * with t_draft already scaled by the prompt-compression factor and alpha
   * already the compression-adjusted alpha; t_draft_init is the target's
   * T_D^mix before the first reply (sim.py:283-288) */
  double t_draft_slope;
  double t_draft_init;
  int32_t t_draft_free_batch;
  /* reply deadline (core.py:123, 2 * t_target by default): a conservative
   * parallel round (gamma * T_D^mix > t_target, sim.py:143-146) commits when
   * its replies land, which must be before this deadline (sim.py:599-606) */
  double reply_timeout;
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


/* ------------------------------------------------ tcgen05 GEMM (K1/K3) ----
 * Y[t, n] = sum_k X[t, k] W[n, k]; X [rows_cap, K] bf16, W [N, K] bf16.
 * The token count is t_dev[0] when t_dev != NULL (graph-capturable), else
 * t_static.  epilogue 0: fp32 split-K partials [splits][rows_cap][N];
 * 1: (max, argmax) partials [spectre_gemm_argmax_blocks(N, K)][rows_cap]
 * (lm_head greedy; reduce over the first dimension, lowest index on ties);
 * 2: SwiGLU over row-pair-interleaved gate/up weights [g0, u0, g1, u1, ...]
 * -> act [rows_cap][ld_act] bf16.  Exposed for unit tests and the roofline bench; the engine calls the
 * same kernels internally. */
int32_t spectre_gemm_argmax_blocks(int32_t N, int32_t K);
int spectre_gemm_bf16(const void* X, const void* W, const int32_t* t_dev, int32_t t_static,
                      int32_t rows_cap, int32_t N, int32_t K, int32_t splits,
                      int32_t epilogue, float* partial, float* amax_val, int32_t* amax_idx,
                      void* act, int32_t ld_act, int32_t max_stages, void* stream);

/* ------------------------------------------------ model mode (C2..C5) -----
 * Replaces the reference's model pair (TokenStreamOracle, oracle.py:47-113)
 * with a Llama-shaped bf16 target and draft on the device, and
 * specsim.run's round loop (sim.py:514-760) with the device-resident round:
 * controller -> [ordinary: draft repair] -> assemble -> verify forward ->
 * [parallel: draft speculation overlapped on a second stream] -> accept.
 * Weights and KV caches are caller-owned device buffers; the engine owns
 * only the workspace carved from `workspace`. */
typedef struct SpectreModelDims {
  int32_t d_model;
  int32_t n_layers;
  int32_t n_q_heads;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t ffn;
  int32_t vocab;
  float rms_eps;
  double rope_theta;
} SpectreModelDims;

typedef struct SpectreModelWeights {
  const void* embed;        /* [vocab][d] bf16 */
  const float* attn_norm;   /* [L][d] */
  const void* wqkv;         /* [L][(nq + 2 nkv) hd][d] bf16 */
  const void* wo;           /* [L][d][nq hd] bf16 */
  const float* mlp_norm;    /* [L][d] */
  const void* wgu;          /* [L][2 ffn][d] bf16, row-pair gate/up interleave */
  const void* wd;           /* [L][d][ffn] bf16 */
  const float* final_norm;  /* [d] */
  const void* lm_head;      /* [vocab][d] bf16 */
  void* k_cache;            /* [L][n_req][nkv][ctx_cap][hd] bf16 */
  void* v_cache;
} SpectreModelWeights;

#define SPECTRE_CTRL_REFERENCE 0  /* r* from config t_target / t_draft (sim.py:431-445) */
#define SPECTRE_CTRL_MEASURED 1   /* r* from device-timed T_T and T_D (paper Eq.) */
#define SPECTRE_CTRL_ROUND 2      /* r* from measured parallel / ordinary round times */

typedef struct SpectreDecodeConfig {
  uint64_t seed;
  int32_t n_req;
  int32_t gamma;
  int32_t output_len;
  int32_t prompt_len;
  int32_t variant;          /* SPECTRE_VARIANT_* */
  int32_t controller;       /* SPECTRE_CTRL_* */
  int32_t r_kind;           /* 0: r-hat = |R|/B (reference); 1: PADDED fraction */
  int32_t max_rounds;       /* trace capacity */
  int32_t ctx_cap;          /* KV capacity per request (absolute positions) */
  int32_t has_fixed_l;
  double alpha;             /* draft keep probability (controlled noise) */
  double t_target;          /* CTRL_REFERENCE latencies (s) */
  double t_draft;
  double ema_decay;
  double fixed_threshold_l;
  double temperature;       /* 0: greedy verification; > 0: speculative rejection
                               sampling at this temperature (config 3) */
  int32_t role;             /* SPECTRE_ROLE_*: both models, or one side of a
                               disaggregated pair (config 5) */
  int32_t breaker_threshold;  /* circuit breaker (target_engine.py:337-380): this
                                 many consecutive speculative rounds with a
                                 missing draft reply disable speculation ... */
  int32_t breaker_cooldown;   /* ... for this many rounds.  <= 0: defaults 3 / 5
                                 (core.py:93-94) */
  int32_t draft_prompt_keep;  /* draft prompt compression (draft_engine.py:123-131,
                                 StreamingLLM head/tail retention): the draft model
                                 sees only the first and the last `keep` prompt
                                 tokens, re-indexed to positions 0 .. 2 keep - 1;
                                 0 (or 2 keep >= prompt_len): the whole prompt */
  /* background (regular) tenants of the draft model and the speculative-priority
   * fairness scheduler (draft_engine.py:134-155, 302-394; core.py:79-85):
   * background_requests greedy draft-model requests of background_output_len
   * tokens share every draft round with the speculative queries; a round
   * serves at most draft_capacity items, speculative first; after
   * fairness_period consecutive speculative rounds with regular work waiting,
   * one round serves regular items only.  0 requests: no background load. */
  int32_t background_requests;
  int32_t background_output_len;
  int32_t fairness_period;
  int32_t draft_capacity;
  /* reply deadline in rounds (core.py:123, reply_timeout = 2 t_target): a
   * missing draft reply is declared a timeout (breaker strike, sim.py:653-665)
   * at the commit reply_timeout_rounds - 1 rounds after it was due.  <= 0: 2 */
  int32_t reply_timeout_rounds;
  /* non-stationary acceptance (config 4 drift workload): from draft output
   * position alpha_switch_pos on, the draft keep probability is alpha_late
   * instead of alpha.  alpha_switch_pos <= 0: alpha throughout */
  int32_t alpha_switch_pos;
  double alpha_late;
} SpectreDecodeConfig;

#define SPECTRE_ROLE_BOTH 0
#define SPECTRE_ROLE_TARGET 1   /* verify side: controller, assembly, verify, accept */
#define SPECTRE_ROLE_DRAFT 2    /* draft server: sync / rollback, speculation */

size_t spectre_engine_workspace_bytes(const SpectreModelDims* target,
                                      const SpectreModelDims* draft,
                                      const SpectreDecodeConfig* cfg);
/* Returns an opaque handle (NULL on error, see spectre_last_error). */
void* spectre_engine_create(const SpectreModelDims* target, const SpectreModelWeights* tw,
                            const SpectreModelDims* draft, const SpectreModelWeights* dw,
                            const SpectreDecodeConfig* cfg, void* workspace,
                            size_t workspace_bytes);
int spectre_engine_destroy(void* engine);

/* Disaggregated rounds (config 5: draft on its own GPU, target replicas on
 * others; the reference's draft server / target endpoints, draft_engine.py /
 * target_engine.py, joined by sim.py's channels).  The host drives one
 * round as BEGIN (target: controller, returns the mode) -> exchange
 * target->draft -> DRAFT (draft server) ∥ VERIFY (target) -> exchange
 * draft->target -> ACCEPT (target).  Returns the mode for BEGIN. */
#define SPECTRE_STEP_BEGIN 0
#define SPECTRE_STEP_DRAFT 1
#define SPECTRE_STEP_VERIFY 2
#define SPECTRE_STEP_ACCEPT 3
int spectre_engine_step(void* engine, int32_t step, int32_t mode, void* stream);
/* Copy the per-request state one side needs from the other for requests
 * [src_req0, src_req0+n) of `src` into [dst_req0, ...) of `dst` (peer copies
 * when the engines live on different GPUs).  direction 0: target -> draft
 * (per-request mode and query tags, committed tokens, positions, cache
 * flags); 1: draft -> target (draft history window, generation counters,
 * reply tags, draft timing).  Every query carries a (round, serial) tag and
 * the draft stamps its reply with it; the target uses a reply only when the
 * tags match its outstanding query (target_engine.py:314-331), so a lost or
 * superseded reply (an exchange that never ran) degrades that request to a
 * FALLBACK / PADDED candidate and counts towards the circuit breaker.
 * DRAFT with mode 'M' serves shards that chose different modes in one
 * draft phase (per-request mode from the last direction-0 exchange). */
int spectre_engine_exchange(void* src, void* dst, int32_t direction, int32_t src_req0,
                            int32_t dst_req0, int32_t n, void* stream);
/* Enable direct peer access between two GPUs (both directions; idempotent). */
int spectre_enable_peer_access(int32_t dev_a, int32_t dev_b);
/* One process per GPU: export a device pointer (an engine workspace) as a
 * CUDA IPC handle + offset into its allocation; a peer process opens it
 * (peer access enabled lazily) and attaches a layout-only engine view built
 * from the owner's dims and config.  spectre_engine_exchange between a local
 * engine and an attached view writes directly into the peer's state.  An
 * attached view supports only exchange and destroy. */
#define SPECTRE_IPC_HANDLE_BYTES 64
int spectre_ipc_export(const void* dev_ptr, uint8_t* handle_out, uint64_t* offset_out);
int spectre_ipc_open(const uint8_t* handle, uint64_t offset, void** base_out,
                     void** dev_ptr_out);
int spectre_ipc_close(void* base);
void* spectre_engine_attach(const SpectreModelDims* target, const SpectreModelDims* draft,
                            const SpectreDecodeConfig* cfg, void* workspace,
                            size_t workspace_bytes);
/* Prefill both models with prompts [n_req][prompt_len] (device int32) and
 * commit output token 0 (target greedy) — admission (target_engine.py:105-126). */
int spectre_engine_prefill(void* engine, const int32_t* prompts, void* stream);
/* Run decode rounds on `stream` (draft work forks to an internal stream).
 * Captures the round into a CUDA graph on first use (conditional nodes pick
 * ordinary / parallel work on the device; use_graph=0 launches eagerly with
 * one mode read-back per round).  Stops after max_rounds or when every
 * request is done; *rounds_run receives the count (host-synchronising). */
int spectre_engine_run(void* engine, int32_t max_rounds, int32_t use_graph,
                       int32_t* rounds_run, void* stream);
/* 1: the device-resident WHILE/IF round graph is in use; 2: graph capture
 * failed and rounds run eagerly (reason in spectre_last_error); 0: not built. */
int spectre_engine_graph_status(void* engine);
/* Copy device state out: committed tokens [n_req][output_len] int64,
 * committed_pos [n_req] int32, per-round trace (see SpectreRoundTrace). */
typedef struct SpectreRoundTrace {
  int32_t* mode;            /* 'O' 'P' 'F' */
  int32_t* participants;
  int32_t* delta;
  int32_t* n_roll;
  int32_t* content_sum;
  int32_t* content_n;
  int32_t* n_padded;
  int64_t* t_round_ns;      /* device %globaltimer spans */
  int64_t* t_verify_ns;
  int64_t* t_draft_ns;
  double* r_hat_ema;
  double* accepted_len_ema;
  double* r_star;
  int32_t* n_stale;         /* queried requests whose reply was missing or
                               superseded at commit (target_engine.py:314-331) */
  int32_t* n_regular;       /* background items scheduled with this round's speculation */
  int32_t* n_forced;        /* background items of a forced regular round (0: none) */
  int32_t* fair_counter;    /* FairnessCounter.consecutive_speculative after the round */
  int32_t* timeout;         /* round flagged a timeout round (RoundTrace.timeout) */
} SpectreRoundTrace;
int spectre_engine_read(void* engine, int64_t* committed, int32_t* committed_pos,
                        const SpectreRoundTrace* trace, int32_t* n_rounds, void* stream);
/* Asynchronous device-to-device copy of the committed tokens (int64,
 * [n_req][output_len]) on `stream` — the per-step output of the decode. */
int spectre_engine_read_committed(void* engine, int64_t* committed, void* stream);
/* Background tenants: generated tokens [background_requests][background_output_len]
 * int32 and per-request counts (device pointers), totals[2] = {tokens generated,
 * requests completed} (host).  Synchronous. */
int spectre_engine_read_background(void* engine, int32_t* tokens, int32_t* emitted,
                                   int32_t* totals, void* stream);
/* Measurement: launch the draft's mid-layer chain kernels back to back `reps`
 * times on `stream` (current draft batch); returns the launches issued and the
 * weight bytes of one pass in *weight_bytes. */
int spectre_engine_launch_chains(void* engine, int32_t reps, int64_t* weight_bytes,
                                 void* stream);
/* One forward pass over a packed ragged batch (tests / roofline):
 * which 0 = target, 1 = draft.  tok/pos/slot [T]; per request q_off, n_new,
 * pos0 [n_req] (n_new 0 = not participating).  out_tok [T] greedy argmax;
 * out_x (optional) [T][d] bf16 final-normed hidden state. */
int spectre_engine_forward(void* engine, int32_t which, const int32_t* tok,
                           const int32_t* pos, const int32_t* slot, int32_t T,
                           const int32_t* q_off, const int32_t* n_new, const int32_t* pos0,
                           int32_t* out_tok, void* out_x, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SPECTRE_H_ */
