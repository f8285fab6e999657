// engine_state.cuh — device-resident state of the model-mode decode loop.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace spectre {

// Packed ragged batch fed to one forward pass (see model_kernels.cuh).
struct BatchDev {
  int* tok;      // [rows_cap]
  int* pos;      // [rows_cap] absolute positions
  int* slot;     // [rows_cap] KV slot (request index)
  int* t_dev;    // [1] token rows this pass
  int* q_off;    // [n_req]
  int* n_new;    // [n_req]
  int* pos0;     // [n_req]
  int* rslot;    // [n_req] (identity)
  int* out_tok;  // [rows_cap] greedy argmax per row
};

// Controller + clock, one instance.
struct CtrlDev {
  int mode;          // this round: 'O', 'P', 'F'; 0 = finished
  int prev_mode;     // hybrid memory (sim.py:281, 466)
  int has_ema;
  int has_L;
  double ema;        // r-hat EMA (sim.py:673-678)
  double L;          // accepted-length EMA (target_engine.py:386-407)
  int round;         // rounds completed
  int round_limit;   // stop after this many rounds (set per run call)
  int round_base;    // rounds completed when the current run call started
  int n_active;
  int error;         // protocol violation code (0 = none)
  int error_req;
  long long t_round_begin, t_verify_begin, t_verify_end, t_draft_begin, t_draft_end;
  int draft_steps;   // steps in the draft phase of this round
  int has_tT, has_tD, has_tpar, has_tord;
  double tT, tD, tpar, tord;   // measured EMAs (seconds)
  double r_star;
  // `round` controller: the paper's r measured directly — PADDED fraction of
  // steady parallel rounds (a parallel round after a parallel round)
  int has_rpar, last_mode;
  double rpar;
  int has_rho;       // T_par / T_ord measured at the same context (steady P round vs
  double rho;        // the ordinary EMA at that time): round times grow with context
  // re-probe: r-hat over ordinary rounds only, its value when r / rho were last
  // measured, and the parallel rounds still owed by a running probe
  int has_ema_ord, has_probe_ref, probe_left, probe_round;
  int p_streak;      // consecutive parallel rounds up to the last accepted one
  double ema_ord, probe_ref;
  // circuit breaker (target_engine.py:337-380); round ids are 1-based as in sim.py:519
  int streak, disabled_until, activations;
  int n_stale;       // this round: queried requests without a matching reply
  // background (regular) draft tenants and the speculative-priority fairness
  // scheduler (draft_engine.py:134-155, 302-394): FairnessCounter, totals, and
  // this round's schedule (regular items in the forced round / the round that
  // served the speculative queries)
  int fair_counter, bg_tokens, bg_completed, ph_forced, ph_regular;
  int pending_timeout;   // last speculative round's unanswered queries (timeout_lag)
};

struct RoundTraceDev {
  int* mode;
  int* participants;
  int* delta;
  int* n_roll;
  int* content_sum;
  int* content_n;
  int* n_padded;
  long long* t_round_ns;
  long long* t_verify_ns;
  long long* t_draft_ns;
  double* r_hat_ema;
  double* accepted_len_ema;
  double* r_star;
  int* n_stale;
  int* n_regular;     // regular items scheduled with this round's speculation
  int* n_forced;      // regular items of a forced regular round (0: none)
  int* fair_counter;  // FairnessCounter.consecutive_speculative after the round
  int* timeout;       // the round was flagged a timeout round (breaker input)
};

struct DecodeStateDev {
  int n_req, gamma, out_len, prompt_len, vocab, variant, controller, r_kind, max_rounds;
  int dprompt_len;   // prompt tokens the draft model sees (compression, draft_engine.py:123-131)
  int has_fixed_l;
  int hist_cap;      // draft history capacity (output positions)
  uint64_t seed;
  double alpha, t_target, t_draft, ema_decay, fixed_l;
  int alpha_switch;  // draft output position where alpha_late takes over (INT_MAX: never)
  double alpha_late;
  // per request (SoA)
  int* pos;          // committed_pos
  int* done;
  int* synced;
  int* cached_len;
  int* cached_start;
  int* in_rollback;
  int* hist_len;
  int* kvd;          // draft KV valid length (output positions)
  int* gen_count;    // draft tokens to generate this phase (0: not queried)
  int* gen_done;
  int* gen_start;
  int* vkind;        // verify candidate kind this round
  int* vcand_n;      // non-seed candidate tokens
  int* delta;
  int* rolled;
  uint64_t* committed;   // [n_req][out_len]
  uint64_t* hist;        // [n_req][hist_cap]
  uint64_t* cached_tok;  // [n_req][gamma + 1]
  uint64_t* cand_tok;    // [n_req][gamma + 1]
  CtrlDev* ctrl;
  RoundTraceDev trace;
  cudaGraphConditionalHandle h_ord, h_par, h_ar, h_loop;
  int use_handles;
  int sampling;          // 1: accept from samp_a / samp_bonus (rejection sampling)
  int* samp_a;           // [n_req] accepted candidates
  int* samp_bonus;       // [n_req] bonus / resampled token
  int breaker_threshold, breaker_cooldown;
  int timeout_lag;       // rounds between a missing reply and its timeout (reply_timeout / T_T - 1)
  // query / reply versioning (target_engine.py:314-331, sim.py:816-844)
  int* req_mode;         // [n_req] this round's mode per request (draft side: 'M' phases)
  int* q_round;          // [n_req] outstanding query tag (target side)
  int* q_serial;
  int* r_round;          // [n_req] tag of the reply held in hist / gen_* (draft stamps)
  int* r_serial;
  // background tenants: draft-model requests decoding autoregressively in the
  // draft's KV slots n_req .. n_req + n_bg - 1 (batch entries b = n_req + j)
  int n_bg, bg_out_len, fair_period, draft_cap;
  int* bg_remaining;     // [n_bg] tokens still to generate
  int* bg_ctx;           // [n_bg] positions with KV = the next input's position
  int* bg_last;          // [n_bg] next input token
  int* bg_emitted;       // [n_bg] tokens generated so far
  int* bg_round_left;    // [n_bg] tokens still to emit in the current draft round
  int* bg_out;           // [n_bg][bg_out_len] generated tokens
};

// launchers (model_protocol.cu)
int launch_compress_prompts(const int* prompts, int P, int keep, int n_req, int* out,
                            cudaStream_t s);
int launch_prefill_batch(const int* prompts, int prompt_len, int n_req, int c0, int cs,
                         const BatchDev& bt, cudaStream_t s);
int launch_admit(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s);
int launch_round_begin(const DecodeStateDev& st, cudaStream_t s);
int launch_set_round_limit(const DecodeStateDev& st, int extra, cudaStream_t s);
int launch_draft_prep(const DecodeStateDev& st, const BatchDev& bt, int which, cudaStream_t s);
int launch_bg_prompts(uint64_t seed, int n_req, int n_bg, int P, int vocab, int* out,
                      cudaStream_t s);
int launch_bg_init(const DecodeStateDev& st, const int* dprompts, int P, cudaStream_t s);
int launch_bg_forced_prep(const DecodeStateDev& st, const BatchDev& bt, int which,
                          cudaStream_t s);
int launch_bg_forced_append(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s);
int launch_draft_append(const DecodeStateDev& st, const BatchDev& bt, int which, int last,
                        cudaStream_t s);
int launch_verify_prep(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s);
int launch_accept(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s);
// sampling.cu
int launch_sample_rows(const float* logits, int V, const BatchDev& bt, int t_cap, float inv_t,
                       uint64_t seed, float2* stats, cudaStream_t s);
int launch_draft_sample(const DecodeStateDev& st, const BatchDev& bt, const float* logits, int V,
                        float inv_t, float* qstore, float2* qstat, int W, cudaStream_t s);
int launch_accept_sample(const DecodeStateDev& st, const BatchDev& bt, const float* logits, int V,
                         float inv_t, const float2* tstat, const float* qstore,
                         const float2* qstat, int W, int* out_a, int* out_bonus,
                         cudaStream_t s);

}  // namespace spectre
