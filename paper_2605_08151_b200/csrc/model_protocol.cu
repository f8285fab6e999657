// model_protocol.cu — the model-mode round: controller, draft sync / rebase /
// catch-up, candidate assembly, fused accept (greedy verify + bonus + commit +
// suffix reuse + rollback statistics + EMA updates), all on the device.
//
// The per-request rules are the reference's (protocol.cuh cites them); only
// the "model pair" differs: the target's greedy token at output position q is
// the argmax row of the verify forward instead of the hash stream, and draft
// tokens come from the draft forward (+ controlled noise) instead of the
// alpha-proposer.  Compiled with -fmad=false (controller doubles).
#include "common.cuh"
#include "engine_state.cuh"
#include "protocol.cuh"

namespace spectre {

constexpr int kProtoThreads = 1024;

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// block-wide exclusive scan of v (requests strided by blockDim); returns total.
__device__ int block_exclusive_scan(int v, int* out, int idx, int n, int* sh) {
  // single pass when n <= blockDim
  const int tid = threadIdx.x;
  sh[tid] = (idx < n) ? v : 0;
  __syncthreads();
  for (int d = 1; d < blockDim.x; d <<= 1) {
    const int x = tid >= d ? sh[tid - d] : 0;
    __syncthreads();
    sh[tid] += x;
    __syncthreads();
  }
  if (idx < n) *out = sh[tid] - v;
  const int total = sh[blockDim.x - 1];
  __syncthreads();
  return total;
}

__device__ __forceinline__ double u53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

// draft "controlled noise": keep the draft's greedy token with probability
// alpha, else replace it with a different token (deterministic per position).
// From output position alpha_switch on the keep probability is alpha_late
// (non-stationary acceptance: the drift workload of config 4).
__device__ __forceinline__ int noisy_draft_token(const DecodeStateDev& s, int req, int pos,
                                                 int tok) {
  const double alpha = pos >= s.alpha_switch ? s.alpha_late : s.alpha;
  if (alpha >= 1.0) return tok;
  const uint64_t h = mix64(s.seed, 2, (uint64_t)req, (uint64_t)pos);
  if (u53(h) < alpha) return tok;
  const uint64_t r = mix64(s.seed, 3, (uint64_t)req, (uint64_t)pos);
  return (int)(((uint64_t)tok + 1 + r % (uint64_t)(s.vocab - 1)) % (uint64_t)s.vocab);
}

// ------------------------------------------------------------ prefill helpers
__global__ void k_prefill_batch(const int* prompts, int prompt_len, int n_req, int c0, int cs,
                                BatchDev bt) {
  pdl_wait();
  pdl_trigger();
  const int b = threadIdx.x + blockIdx.x * blockDim.x;
  const int n = min(cs, prompt_len - c0);
  if (b == 0) *bt.t_dev = n * n_req;
  if (b >= n_req) return;
  bt.q_off[b] = b * n;
  bt.n_new[b] = n;
  bt.pos0[b] = c0;
  bt.rslot[b] = b;
  for (int j = 0; j < n; ++j) {
    bt.tok[b * n + j] = prompts[(size_t)b * prompt_len + c0 + j];
    bt.pos[b * n + j] = c0 + j;
    bt.slot[b * n + j] = b;
  }
}

// After the target's last prompt chunk: admission commits output token 0
// (target_engine.py:105-126) and resets every round-protocol field.
__global__ void k_admit(DecodeStateDev s, BatchDev bt) {
  pdl_wait();
  pdl_trigger();
  const int b = threadIdx.x + blockIdx.x * blockDim.x;
  if (b == 0) {
    CtrlDev& c = *s.ctrl;
    c.mode = 0;
    c.prev_mode = 0;
    c.has_ema = c.has_L = 0;
    c.ema = c.L = 0.0;
    c.round = 0;
    c.round_limit = 0x7fffffff;
    c.n_active = s.n_req;
    c.error = 0;
    c.error_req = -1;
    c.has_tT = c.has_tD = c.has_tpar = c.has_tord = 0;
    c.tT = c.tD = c.tpar = c.tord = 0.0;
    c.has_rpar = 0;
    c.rpar = 0.0;
    c.has_rho = 0;
    c.rho = 0.0;
    c.has_ema_ord = c.has_probe_ref = c.probe_left = c.p_streak = 0;
    c.probe_round = 0;
    c.ema_ord = c.probe_ref = 0.0;
    c.last_mode = 0;
    c.r_star = 0.0;
    c.streak = c.disabled_until = c.activations = 0;
    c.n_stale = 0;
    c.fair_counter = c.bg_tokens = c.bg_completed = c.ph_forced = c.ph_regular = 0;
    c.pending_timeout = 0;
  }
  if (b >= s.n_req) return;
  s.req_mode[b] = 0;
  s.q_round[b] = s.r_round[b] = -1;
  s.q_serial[b] = 0;
  s.r_serial[b] = -1;
  const int row = bt.q_off[b] + bt.n_new[b] - 1;
  s.committed[(size_t)b * s.out_len] = (uint64_t)bt.out_tok[row];
  s.pos[b] = 1;
  s.done[b] = s.out_len <= 1;
  s.synced[b] = 0;
  s.cached_len[b] = 0;
  s.in_rollback[b] = 1;
  s.hist_len[b] = 0;
  s.kvd[b] = 0;
  s.gen_count[b] = 0;
  s.vkind[b] = 0;
}

// ------------------------------------------------------------ round begin
// Controller (sim.py:447-467) + conditional-node selection.
__device__ int round_choose_mode(DecodeStateDev& s, CtrlDev& c);

// Thread 0 picks the mode; every thread then stamps its requests' queries
// with a (round, serial) tag (sim.py:492-512: ordinary queries requests
// without a cache at round_tag = round, parallel queries all at round + 1).
__global__ void __launch_bounds__(kProtoThreads) k_round_begin(DecodeStateDev s) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_mode;
  CtrlDev& c = *s.ctrl;
  if (threadIdx.x == 0) s_mode = round_choose_mode(s, c);
  __syncthreads();
  const int mode = s_mode;
  const int round_id = c.round + 1;
  for (int b = threadIdx.x; b < s.n_req; b += blockDim.x) {
    s.req_mode[b] = mode;
    if (!s.done[b] && (mode == 'P' || (mode == 'O' && s.cached_len[b] == 0))) {
      s.q_serial[b] += 1;
      s.q_round[b] = mode == 'P' ? round_id + 1 : round_id;
    }
  }
}

__device__ int round_choose_mode(DecodeStateDev& s, CtrlDev& c) {
  c.t_round_begin = globaltimer();
  c.t_draft_begin = c.t_draft_end = 0;
  c.draft_steps = 0;
  c.n_stale = 0;
  c.ph_forced = c.ph_regular = 0;
  int mode = 0;
  if (c.n_active > 0 && c.error == 0 && c.round < s.max_rounds && c.round < c.round_limit) {
    if (s.variant == SPECTRE_VARIANT_AR) mode = 'F';
    // breaker window: speculation off, controller untouched (sim.py:520-533)
    else if (c.round + 1 < c.disabled_until) mode = 'F';
    else if (s.variant == SPECTRE_VARIANT_ORDINARY) mode = 'O';
    else if (s.variant == SPECTRE_VARIANT_PARALLEL) mode = 'P';
    else {
      const bool hasL = s.has_fixed_l ? true : (c.has_L != 0);
      const double L = s.has_fixed_l ? s.fixed_l : c.L;
      double r_star;
      if (s.controller == SPECTRE_CTRL_REFERENCE || !(c.has_tT && c.has_tD)) {
        if (s.controller == SPECTRE_CTRL_ROUND) {
          // explore: measure one round of each mode before trusting the model
          if (!c.has_tord) { mode = 'O'; }
          else if (!c.has_tpar) { mode = 'P'; }
        }
        if (mode == 0)
          mode = choose_mode_hybrid(c.prev_mode, c.has_ema != 0, c.ema, hasL, L, s.gamma,
                                    s.t_target, s.t_draft, &r_star);
        else
          r_star = 0.0;
      } else if (s.controller == SPECTRE_CTRL_MEASURED) {
        mode = choose_mode_hybrid(c.prev_mode, c.has_ema != 0, c.ema, hasL, L, s.gamma, c.tT,
                                  c.tD, &r_star);
      } else {  // SPECTRE_CTRL_ROUND: r* = L (1 - T_par / T_ord) / (L - 1)
        if (!c.has_tord) {
          mode = 'O';
          r_star = 0.0;
        } else if (!c.has_tpar) {
          mode = 'P';
          r_star = 0.0;
        } else if (c.probe_left > 0) {
          // re-probe in progress: one more parallel round (the steady one)
          mode = 'P';
          --c.probe_left;
          r_star = c.r_star;
        } else {
          // r: the PADDED fraction parallel rounds actually produced (the
          // paper's r) once measured; before that the reference's r-hat.  At
          // T=1 r-hat from ordinary rounds (~0.75) under-predicts it (~1.0)
          const double r_hat = c.has_rpar ? c.rpar : (c.has_ema ? c.ema : 0.0);
          if (!hasL || L <= 1.0 + 1e-9) {
            r_star = __longlong_as_double(0x7ff0000000000000ll);
          } else {
            // T_par / T_ord from rounds at the same context; a T_par measured
            // early against a T_ord that keeps growing would inflate r*
            const double ratio = c.has_rho ? c.rho : __ddiv_rn(c.tpar, c.tord);
            r_star = __ddiv_rn(__dmul_rn(L, __dsub_rn(1.0, ratio)), __dsub_rn(L, 1.0));
          }
          if (c.prev_mode == 'P')
            mode = (r_hat > __dmul_rn(r_star, kExitParallelMargin)) ? 'O' : 'P';
          else
            mode = (r_hat <= r_star) ? 'P' : 'O';
          // r and T_par / T_ord are only measured in parallel rounds: while
          // ordinary rounds run they go stale.  When the ordinary-round r-hat
          // has moved by more than kReprobeDelta since they were measured,
          // spend two parallel rounds (switch-over + steady) re-measuring them
          if (mode == 'O' && c.has_ema_ord && c.has_probe_ref &&
              c.round - c.probe_round >= kReprobeMinRounds &&
              fabs(__dsub_rn(c.ema_ord, c.probe_ref)) > kReprobeDelta) {
            mode = 'P';
            c.probe_left = 1;
            c.probe_round = c.round;
          }
        }
      }
      c.r_star = r_star;
      c.prev_mode = mode;
    }
  }
  c.mode = mode;
  if (s.use_handles) {
    cudaGraphSetConditional(s.h_ord, mode == 'O' ? 1u : 0u);
    cudaGraphSetConditional(s.h_par, mode == 'P' ? 1u : 0u);
    cudaGraphSetConditional(s.h_ar, mode == 'F' ? 1u : 0u);
  }
  return mode;
}

// ------------------------------------------------------------ background tenants
// Regular (non-speculative) draft-model requests sharing the draft server
// (draft_engine.py:302-394): background request j decodes greedily in the
// draft's KV slot n_req + j, batch entry b = n_req + j.  Each draft round
// schedules speculative items first and fills the remaining capacity with
// ready regular items in FIFO order; once `fair_period` consecutive rounds
// served speculation while regular work waited, one round serves only regular
// items (schedule_round, draft_engine.py:134-155).  A scheduled regular item
// emits min(remaining, steps) tokens, one per draft step (:389-394).

// Synthetic background prompts: TokenStreamOracle prompt stream of request ids
// 1,000,000 + j (sim.py _BG_BASE) mod V, written after the n_req speculative rows.
__global__ void k_bg_prompts(uint64_t seed, int n_req, int n_bg, int P, int vocab, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_bg * P; i += gridDim.x * blockDim.x) {
    const int j = i / P, k = i % P;
    out[(size_t)(n_req + j) * P + k] =
        (int)(stream_token(seed, 1, 1000000ull + (uint64_t)j, (uint64_t)k) % (uint64_t)vocab);
  }
}

// After the draft's prefill: every background request re-feeds its last prompt
// token (its KV is recomputed bit-identically) and owes bg_out_len tokens.
__global__ void k_bg_init(DecodeStateDev s, const int* dprompts, int P) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s.n_bg) return;
  s.bg_remaining[j] = s.bg_out_len;
  s.bg_ctx[j] = P - 1;
  s.bg_last[j] = dprompts[(size_t)(s.n_req + j) * P + P - 1];
  s.bg_emitted[j] = 0;
  s.bg_round_left[j] = 0;
}

// The draft's greedy token for background request j (row `row` of the pass).
__device__ __forceinline__ void bg_consume(DecodeStateDev& s, const BatchDev& bt, int j, int row) {
  const int tok = bt.out_tok[row];
  if (s.bg_emitted[j] < s.bg_out_len) s.bg_out[(size_t)j * s.bg_out_len + s.bg_emitted[j]] = tok;
  s.bg_emitted[j] += 1;
  s.bg_last[j] = tok;
  s.bg_ctx[j] += 1;
  s.bg_remaining[j] -= 1;
  s.bg_round_left[j] -= 1;
  atomicAdd(&s.ctrl->bg_tokens, 1);
  if (s.bg_remaining[j] == 0) atomicAdd(&s.ctrl->bg_completed, 1);
}

// FIFO rank of background entry b among the ready ones (block-wide; every
// thread of the block must call it).  *total = ready count.
__device__ int bg_ready_rank(const DecodeStateDev& s, int b, bool ready, int* total, int* sh) {
  int rank = 0;
  *total = block_exclusive_scan(ready ? 1 : 0, &rank, b - s.n_req, s.n_bg, sh);
  return rank;
}

// Phase start: a forced regular round (one step, regular items only) when the
// counter is due and regular work waits; otherwise an empty pass.
__global__ void __launch_bounds__(kProtoThreads) k_bg_forced_prep(DecodeStateDev s, BatchDev bt,
                                                                  int which_mode) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sh[kProtoThreads];
  __shared__ int s_forced;
  CtrlDev& c = *s.ctrl;
  const int b = threadIdx.x;
  const int nb = s.n_req + s.n_bg;
  const bool selected = which_mode == 'M' || c.mode == which_mode;
  if (threadIdx.x == 0 && selected) c.t_draft_begin = globaltimer();
  const int j = b - s.n_req;
  const bool ready = selected && j >= 0 && j < s.n_bg && s.bg_remaining[j] > 0;
  int total = 0;
  const int rank = bg_ready_rank(s, b, ready, &total, sh);
  if (threadIdx.x == 0) {
    s_forced = (selected && total > 0 && c.fair_counter >= s.fair_period) ? 1 : 0;
    c.ph_forced = s_forced ? min(total, s.draft_cap) : 0;
    if (s_forced) c.fair_counter = 0;
  }
  __syncthreads();
  const bool sched = s_forced && ready && rank < s.draft_cap;
  if (j >= 0 && j < s.n_bg) s.bg_round_left[j] = sched ? 1 : 0;
  int off = 0;
  const int rows = block_exclusive_scan(sched ? 1 : 0, &off, b, nb, sh);
  if (b < nb) {
    bt.q_off[b] = off;
    bt.n_new[b] = sched ? 1 : 0;
    bt.rslot[b] = b;
    if (sched) {
      bt.pos0[b] = s.bg_ctx[j];
      bt.tok[off] = s.bg_last[j];
      bt.pos[off] = s.bg_ctx[j];
      bt.slot[off] = b;
    }
  }
  if (threadIdx.x == 0) *bt.t_dev = rows;
}

__global__ void __launch_bounds__(kProtoThreads) k_bg_forced_append(DecodeStateDev s,
                                                                    BatchDev bt) {
  pdl_wait();
  pdl_trigger();
  const int j = threadIdx.x;
  if (j < s.n_bg && s.bg_round_left[j] > 0 && bt.n_new[s.n_req + j] > 0)
    bg_consume(s, bt, j, bt.q_off[s.n_req + j]);
}

// ------------------------------------------------------------ draft phase
// which_mode: 'O' (repair gamma-1 tokens anchored at committed_pos) or 'P'
// (speculate gamma tokens from the history tail).  Sync + rebase + catch-up
// batch for the draft's first step (draft_engine.py:246-280, 412-431).
__global__ void __launch_bounds__(kProtoThreads) k_draft_prep(DecodeStateDev s, BatchDev bt,
                                                              int which_mode) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sh[kProtoThreads];
  CtrlDev& c = *s.ctrl;
  const int mode = c.mode;
  const bool mixed = which_mode == 'M';   // per-request modes (disaggregated shards)
  if (!mixed && mode != which_mode) {  // phase not selected this round: empty batch
    if (threadIdx.x == 0) *bt.t_dev = 0;
    if (threadIdx.x < s.n_req + s.n_bg) bt.n_new[threadIdx.x] = 0;
    return;
  }
  // with background tenants the phase started at the forced-round slot
  if (threadIdx.x == 0 && s.n_bg == 0) c.t_draft_begin = globaltimer();
  const int b = threadIdx.x;
  int n_new = 0, kvd = 0, hl = 0;
  if (b < s.n_req) {
    bt.rslot[b] = b;
    s.gen_count[b] = 0;
    const bool active = !s.done[b];
    const int rm = mixed ? s.req_mode[b] : which_mode;
    const bool queried = active && (rm == 'P' || (rm == 'O' && s.cached_len[b] == 0));
    if (queried) {
      s.r_round[b] = s.q_round[b];     // the reply answers this query
      s.r_serial[b] = s.q_serial[b];
      uint64_t* h = s.hist + (size_t)b * s.hist_cap;
      const uint64_t* com = s.committed + (size_t)b * s.out_len;
      const int pos = s.pos[b];
      const int start = s.synced[b];
      int inv;
      auto ref = [&](int32_t q) { return com[q]; };  // verified prefix (q < pos)
      hl = session_on_sync(h, s.hist_len[b], start, pos - start,
                           [&](int32_t k) { return com[start + k]; }, ref, &inv);
      kvd = min(s.kvd[b], inv);
      s.synced[b] = pos;
      const int count = rm == 'O' ? s.gamma - 1 : s.gamma;
      if (rm == 'O' || hl + count > s.hist_cap) {
        // repair anchor (sim.py:550-555) / speculation-window cap
        hl = session_rebase(h, hl, pos, ref, &inv);
        kvd = min(kvd, inv);
      }
      kvd = min(kvd, hl - 1);
      n_new = hl - kvd;
      s.hist_len[b] = hl;
      s.kvd[b] = kvd;
      s.gen_count[b] = count;
      s.gen_done[b] = 0;
      s.gen_start[b] = hl;
    }
  }
  if (s.n_bg > 0) {
    // the round serving this phase's queries: speculative items first, the
    // remaining capacity to ready regular items (FIFO); steps = the queries'
    // count, 1 without speculation (draft_engine.py:134-155, 334-344)
    const int n_spec = __syncthreads_count(b < s.n_req && s.gen_count[b] > 0);
    const int j = b - s.n_req;
    const bool ready = j >= 0 && j < s.n_bg && s.bg_remaining[j] > 0;
    int n_ready = 0;
    const int rank = bg_ready_rank(s, b, ready, &n_ready, sh);
    const int reg_cap = max(0, s.draft_cap - n_spec);
    const bool sched = ready && rank < reg_cap;
    const int steps_ref = n_spec > 0 ? (which_mode == 'O' ? s.gamma - 1 : s.gamma) : 1;
    if (j >= 0 && j < s.n_bg) s.bg_round_left[j] = sched ? min(s.bg_remaining[j], steps_ref) : 0;
    if (sched) n_new = 1;
    if (threadIdx.x == 0) {
      c.ph_regular = min(n_ready, reg_cap);
      c.fair_counter = n_spec > 0 ? min(c.fair_counter + 1, s.fair_period) : 0;
    }
  }
  int off = 0;
  const int total = block_exclusive_scan(n_new, &off, b, s.n_req + s.n_bg, sh);
  if (b >= s.n_req && b < s.n_req + s.n_bg) {   // background rows
    const int j = b - s.n_req;
    bt.q_off[b] = off;
    bt.n_new[b] = n_new;
    bt.rslot[b] = b;
    if (n_new) {
      bt.pos0[b] = s.bg_ctx[j];
      bt.tok[off] = s.bg_last[j];
      bt.pos[off] = s.bg_ctx[j];
      bt.slot[off] = b;
    }
  }
  if (b < s.n_req) {
    bt.q_off[b] = off;
    bt.n_new[b] = n_new;
    bt.pos0[b] = s.dprompt_len + kvd;
    const uint64_t* h = s.hist + (size_t)b * s.hist_cap;
    for (int j = 0; j < n_new; ++j) {
      bt.tok[off + j] = (int)h[kvd + j];
      bt.pos[off + j] = s.dprompt_len + kvd + j;
      bt.slot[off + j] = b;
    }
  }
  if (threadIdx.x == 0) {
    *bt.t_dev = total;
    c.draft_steps = which_mode == 'O' ? s.gamma - 1 : s.gamma;
  }
}

// After each draft forward: append the (noised) greedy token, next 1-token batch.
__global__ void __launch_bounds__(kProtoThreads) k_draft_append(DecodeStateDev s, BatchDev bt,
                                                                int which_mode, int last_step) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sh[kProtoThreads];
  CtrlDev& c = *s.ctrl;
  if (which_mode != 'M' && c.mode != which_mode) {
    if (threadIdx.x == 0) *bt.t_dev = 0;
    if (threadIdx.x < s.n_req + s.n_bg) bt.n_new[threadIdx.x] = 0;
    return;
  }
  const int b = threadIdx.x;
  int n_new = 0;
  const int jb = b - s.n_req;   // background entry
  if (jb >= 0 && jb < s.n_bg && bt.n_new[b] > 0 && s.bg_round_left[jb] > 0) {
    bg_consume(s, bt, jb, bt.q_off[b]);
    if (s.bg_round_left[jb] > 0) n_new = 1;
  }
  if (b < s.n_req && s.gen_count[b] > 0 && s.gen_done[b] < s.gen_count[b]) {
    const int row = bt.q_off[b] + bt.n_new[b] - 1;
    uint64_t* h = s.hist + (size_t)b * s.hist_cap;
    const int hl = s.hist_len[b];
    const int tok = noisy_draft_token(s, b, hl, bt.out_tok[row]);
    h[hl] = (uint64_t)tok;
    s.kvd[b] = hl;            // every fed token now has KV; the new one does not
    s.hist_len[b] = hl + 1;
    s.gen_done[b] += 1;
    if (s.gen_done[b] < s.gen_count[b]) n_new = 1;
  }
  int off = 0;
  const int total = block_exclusive_scan(n_new, &off, b, s.n_req + s.n_bg, sh);
  if (jb >= 0 && jb < s.n_bg) {
    bt.q_off[b] = off;
    bt.n_new[b] = n_new;
    if (n_new) {
      bt.pos0[b] = s.bg_ctx[jb];
      bt.tok[off] = s.bg_last[jb];
      bt.pos[off] = s.bg_ctx[jb];
      bt.slot[off] = b;
    }
  }
  if (b < s.n_req) {
    bt.q_off[b] = off;
    bt.n_new[b] = n_new;
    const int hl = s.hist_len[b];
    bt.pos0[b] = s.dprompt_len + hl - 1;
    if (n_new) {
      bt.tok[off] = (int)s.hist[(size_t)b * s.hist_cap + hl - 1];
      bt.pos[off] = s.dprompt_len + hl - 1;
      bt.slot[off] = b;
    }
  }
  if (threadIdx.x == 0) {
    *bt.t_dev = total;
    if (last_step) c.t_draft_end = globaltimer();
  }
}

// ------------------------------------------------------------ target phase
// Candidate assembly (target_engine.py:132-221) -> verify batch rows
// [pending bonus @ pos-1, candidate tokens @ pos ...].
__global__ void __launch_bounds__(kProtoThreads) k_verify_prep(DecodeStateDev s, BatchDev bt) {
  pdl_wait();
  pdl_trigger();
  __shared__ int sh[kProtoThreads];
  CtrlDev& c = *s.ctrl;
  const int mode = c.mode;
  if (threadIdx.x == 0) c.t_verify_begin = globaltimer();
  const int b = threadIdx.x;
  int n_new = 0;
  int kind = 0, m = 0;
  if (b < s.n_req && mode != 0 && !s.done[b]) {
    const int pos = s.pos[b];
    uint64_t* cand = s.cand_tok + (size_t)b * (s.gamma + 1);
    if (mode == 'F') {
      kind = kFallback;
    } else if (s.cached_len[b] > 0 && !s.in_rollback[b]) {
      if (s.cached_start[b] != pos) {
        s.ctrl->error = 7;
        s.ctrl->error_req = b;
      }
      kind = kCached;
      m = s.cached_len[b];
      const uint64_t* ct = s.cached_tok + (size_t)b * (s.gamma + 1);
      for (int j = 0; j < m; ++j) cand[j] = ct[j];
    } else if (mode == 'O' &&
               (s.r_serial[b] != s.q_serial[b] || s.r_round[b] != s.q_round[b])) {
      // repair reply missing or superseded: FALLBACK (sim.py:568-577)
      kind = kFallback;
      atomicAdd(&s.ctrl->n_stale, 1);
    } else if (mode == 'O') {
      kind = kRepaired;
      m = s.gamma - 1;
      if (s.gen_start[b] != pos || s.gen_done[b] != m) {
        s.ctrl->error = 7;
        s.ctrl->error_req = b;
      }
      const uint64_t* h = s.hist + (size_t)b * s.hist_cap;
      for (int j = 0; j < m; ++j) cand[j] = h[pos + j];
    } else {
      kind = kPadded;
    }
    n_new = 1 + m;
  }
  if (b < s.n_req) {
    s.vkind[b] = kind;
    s.vcand_n[b] = m;
  }
  int off = 0;
  const int total = block_exclusive_scan(n_new, &off, b, s.n_req, sh);
  if (b < s.n_req) {
    const int pos = s.pos[b];
    bt.q_off[b] = off;
    bt.n_new[b] = n_new;
    bt.pos0[b] = s.prompt_len + pos - 1;
    bt.rslot[b] = b;
    if (n_new) {
      const uint64_t* com = s.committed + (size_t)b * s.out_len;
      const uint64_t* cand = s.cand_tok + (size_t)b * (s.gamma + 1);
      bt.tok[off] = (int)com[pos - 1];
      bt.pos[off] = s.prompt_len + pos - 1;
      bt.slot[off] = b;
      for (int j = 0; j < m; ++j) {
        bt.tok[off + 1 + j] = (int)cand[j];
        bt.pos[off + 1 + j] = s.prompt_len + pos + j;
        bt.slot[off + 1 + j] = b;
      }
    }
  }
  if (threadIdx.x == 0) *bt.t_dev = total;
}

// Fused accept: greedy exact-prefix verification (oracle.py:90-113 with the
// target argmax as the reference stream), bonus emission, commit
// (target_engine.py:227-249), rollback set (:285-302), suffix reuse
// (:252-279), r-hat / L EMAs (sim.py:673-678, target_engine.py:396-402),
// trace row, and the decode-loop condition.  KV rollback is implicit: the
// target's valid KV length is prompt_len + committed_pos - 1 and the draft's
// is tracked in kvd, so rejected rows are simply overwritten next time.
__global__ void __launch_bounds__(kProtoThreads) k_accept(DecodeStateDev s, BatchDev bt) {
  pdl_wait();
  pdl_trigger();
  __shared__ long long s_tv;
  __shared__ int s_trip;
  CtrlDev& c = *s.ctrl;
  const int mode = c.mode;
  if (threadIdx.x == 0) {
    s_tv = globaltimer();
    s_trip = 0;
  }
  __syncthreads();
  if (mode == 0) {
    if (threadIdx.x == 0 && s.use_handles) cudaGraphSetConditional(s.h_loop, 0u);
    return;
  }
  const int b = threadIdx.x;
  const int G = s.gamma + 1;
  if (b < s.n_req && s.vkind[b] != 0) {
    const int kind = s.vkind[b];
    const int m = s.vcand_n[b];
    const int row0 = bt.q_off[b];
    const uint64_t* cand = s.cand_tok + (size_t)b * G;
    uint64_t* com = s.committed + (size_t)b * s.out_len;
    int pos = s.pos[b];
    int a = 0;
    uint64_t bonus;
    if (s.sampling) {   // rejection sampling outcome (sampling.cu:k_accept_sample)
      a = s.samp_a[b];
      bonus = (uint64_t)s.samp_bonus[b];
    } else {            // greedy exact-prefix verification (oracle.py:99-107)
      while (a < m && cand[a] == (uint64_t)bt.out_tok[row0 + a]) ++a;
      bonus = (uint64_t)bt.out_tok[row0 + a];
    }
    const int accepted_count = a + (kind == kCached ? 0 : 1);
    const int real = kind == kRepaired ? s.gamma : (kind == kCached ? m : 1);
    // this round's prepared segment (parallel mode): the draft's speculation,
    // used only if its reply answers this round's query (target_engine.py:314-331)
    const bool fresh = s.r_serial[b] == s.q_serial[b] && s.r_round[b] == s.q_round[b];
    if (mode == 'P' && !fresh) atomicAdd(&s.ctrl->n_stale, 1);
    const bool prep = (mode == 'P') && fresh && s.gen_count[b] > 0;
    const uint64_t* h = s.hist + (size_t)b * s.hist_cap;
    const int pstart = s.gen_start[b];
    const int plen = prep ? s.gen_done[b] : 0;
    int rolled = accepted_count < real;
    if (!rolled && plen > 0 && h[pstart] != bonus) rolled = 1;
    const int end = min(pos + a + 1, s.out_len);
    for (int q = pos; q < end; ++q) com[q] = (q - pos < a) ? cand[q - pos] : bonus;
    const int delta = end - pos;
    pos = end;
    const int done = pos >= s.out_len;
    s.pos[b] = pos;
    s.done[b] = done;
    int cst = 0;
    const int cl = reuse_or_discard(h + pstart, plen, pstart, com, pos, done,
                                    s.cached_tok + (size_t)b * G, &cst);
    s.cached_len[b] = cl;
    s.cached_start[b] = cst;
    s.in_rollback[b] = cl == 0;
    s.delta[b] = delta;
    s.rolled[b] = rolled;
  }
  // per-request outcomes staged in shared memory by every thread, so the
  // in-order (bit-exact) estimator loop below reads smem, not global memory
  __shared__ int s_kind[kProtoThreads], s_delta[kProtoThreads];
  __shared__ unsigned char s_roll[kProtoThreads], s_done[kProtoThreads];
  __syncthreads();
  if (threadIdx.x < s.n_req) {
    const int r = threadIdx.x;
    s_kind[r] = s.vkind[r];
    s_delta[r] = s.delta[r];
    s_roll[r] = (unsigned char)s.rolled[r];
    s_done[r] = (unsigned char)s.done[r];
    s.vkind[r] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t_now = globaltimer();
    int P = 0, dsum = 0, nroll = 0, csum = 0, cn = 0, npad = 0;
    for (int r = 0; r < s.n_req; ++r) {
      const int k = s_kind[r];
      if (k == 0) continue;
      ++P;
      dsum += s_delta[r];
      nroll += s_roll[r];
      if (k == kPadded) ++npad;
      if (k == kCached || k == kRepaired) {
        csum += s_delta[r];
        ++cn;
        const double dv = (double)s_delta[r];
        if (!c.has_L) {
          c.L = dv;
          c.has_L = 1;
        } else {
          c.L = ema_step(s.ema_decay, c.L, dv);
        }
      }
      if (s_done[r]) --c.n_active;
    }
    const int num = s.r_kind == 1 ? npad : nroll;
    const double r_hat = __ddiv_rn((double)num, (double)(P > 0 ? P : 1));
    if (mode != 'F') {
      if (!c.has_ema) {
        c.ema = r_hat;
        c.has_ema = 1;
      } else {
        c.ema = ema_step(s.ema_decay, c.ema, r_hat);
      }
    }
    const double tv = (double)(s_tv - c.t_verify_begin) * 1e-9;
    const double tr = (double)(t_now - c.t_round_begin) * 1e-9;
    const double d = s.ema_decay;
    if (!c.has_tT) { c.tT = tv; c.has_tT = 1; } else { c.tT = ema_step(d, c.tT, tv); }
    if (c.t_draft_end > 0 && c.draft_steps > 0) {
      const double td = (double)(c.t_draft_end - c.t_draft_begin) * 1e-9 / c.draft_steps;
      if (!c.has_tD) { c.tD = td; c.has_tD = 1; } else { c.tD = ema_step(d, c.tD, td); }
    }
    // per-committed-token cost of each mode, normalised to the round shape.
    // The first parallel round after another mode is the switch-over (no
    // prepared segments: all PADDED, sim.py:455-458) — neither its time nor
    // its PADDED fraction is the steady parallel round's
    if (mode == 'P' && c.last_mode == 'P') {
      // the first steady round of a parallel streak replaces what earlier
      // streaks measured (stale: other context, other r); later rounds blend
      const bool fresh = c.p_streak == 1;
      if (!c.has_tpar || fresh) { c.tpar = tr; c.has_tpar = 1; } else { c.tpar = ema_step(d, c.tpar, tr); }
      const double rp = __ddiv_rn((double)npad, (double)(P > 0 ? P : 1));
      if (!c.has_rpar || fresh) { c.rpar = rp; c.has_rpar = 1; } else { c.rpar = ema_step(d, c.rpar, rp); }
      if (c.has_tord) {
        const double rv = __ddiv_rn(tr, c.tord);
        if (!c.has_rho || fresh) { c.rho = rv; c.has_rho = 1; } else { c.rho = ema_step(d, c.rho, rv); }
      }
      // r / rho are fresh: remember the ordinary-round r-hat they belong to
      c.probe_ref = c.has_ema_ord ? c.ema_ord : r_hat;
      c.has_probe_ref = 1;
      c.probe_round = c.round;
    } else if (mode == 'O') {
      // no T_ord sample from the run's first round: at low L the round
      // controller's r* = L (1 - T_par / T_ord) / (L - 1) turns a single
      // noisy sample into a wrong mode for the whole run (config 4, gamma 4,
      // alpha 0.1: hybrid 0.95 of ordinary), so it explores a second
      // ordinary round and takes T_ord there, next to its parallel probe
      if (c.round > 0) {
        if (!c.has_tord) { c.tord = tr; c.has_tord = 1; } else { c.tord = ema_step(d, c.tord, tr); }
      }
      if (!c.has_ema_ord) { c.ema_ord = r_hat; c.has_ema_ord = 1; }
      else { c.ema_ord = ema_step(d, c.ema_ord, r_hat); }
    }
    c.p_streak = mode == 'P' ? c.p_streak + 1 : 0;
    c.last_mode = mode;
    const int ri = c.round;
    // circuit breaker after a speculative round (sim.py:703-718,
    // target_engine.py:356-380).  A reply absent at commit never arrives (the
    // exchange is synchronous); the target declares its query timed out once it
    // is reply_timeout old (sim.py:653-665): with reply_timeout = 2 T_T that is
    // at the NEXT round's commit (timeout_lag = 1), as in the reference
    int timed_out = 0;
    if (mode != 'F') {
      timed_out = s.timeout_lag > 0 ? (c.pending_timeout > 0) : (c.n_stale > 0);
      c.pending_timeout = c.n_stale;
      const int round_id = ri + 1;
      const int streak = timed_out ? c.streak + 1 : 0;
      if (streak >= s.breaker_threshold) {
        c.streak = 0;
        c.disabled_until = round_id + s.breaker_cooldown + 1;
        c.activations += 1;
        c.pending_timeout = 0;   // every outstanding query is abandoned (sim.py:711-718)
        s_trip = 1;
      } else {
        c.streak = streak;
      }
    }
    if (mode == 'F') c.pending_timeout = 0;   // no queries in flight
    if (ri < s.max_rounds) {
      s.trace.timeout[ri] = timed_out;
      s.trace.n_stale[ri] = c.n_stale;
      s.trace.mode[ri] = mode;
      s.trace.participants[ri] = P;
      s.trace.delta[ri] = dsum;
      s.trace.n_roll[ri] = nroll;
      s.trace.content_sum[ri] = csum;
      s.trace.content_n[ri] = cn;
      s.trace.n_padded[ri] = npad;
      s.trace.t_round_ns[ri] = t_now - c.t_round_begin;
      s.trace.t_verify_ns[ri] = s_tv - c.t_verify_begin;
      s.trace.t_draft_ns[ri] = c.t_draft_end > 0 ? c.t_draft_end - c.t_draft_begin : 0;
      s.trace.r_hat_ema[ri] = c.ema;
      s.trace.accepted_len_ema[ri] = c.has_L ? c.L : 0.0;
      s.trace.r_star[ri] = c.r_star;
      s.trace.n_regular[ri] = c.ph_regular;
      s.trace.n_forced[ri] = c.ph_forced;
      s.trace.fair_counter[ri] = c.fair_counter;
    }
    c.round = ri + 1;
    if (s.use_handles)
      cudaGraphSetConditional(s.h_loop, (c.n_active > 0 && c.error == 0 &&
                                         c.round < s.max_rounds && c.round < c.round_limit)
                                            ? 1u
                                            : 0u);
  }
  __syncthreads();
  if (s_trip) {   // the window invalidates all in-flight speculation (sim.py:711-718)
    for (int r = threadIdx.x; r < s.n_req; r += blockDim.x) {
      s.cached_len[r] = 0;
      s.in_rollback[r] = 1;
      s.q_serial[r] += 1;   // outstanding queries cleared: no late reply can match
    }
  }
}

// host-free round budget: stop after `extra` more rounds
__global__ void k_set_round_limit(DecodeStateDev s, int extra) {
  pdl_wait();
  pdl_trigger();
  CtrlDev& c = *s.ctrl;
  const long long lim = (long long)c.round + extra;
  c.round_limit = lim > 0x7fffffff ? 0x7fffffff : (int)lim;
  c.round_base = c.round;
}

// ------------------------------------------------------------------ launchers
int launch_bg_prompts(uint64_t seed, int n_req, int n_bg, int P, int vocab, int* out,
                      cudaStream_t s) {
  if (n_bg <= 0) return SPECTRE_OK;
  k_bg_prompts<<<(n_bg * P + 255) / 256, 256, 0, s>>>(seed, n_req, n_bg, P, vocab, out);
  SPECTRE_LAUNCH_CHECK("k_bg_prompts");
  return SPECTRE_OK;
}
int launch_bg_init(const DecodeStateDev& st, const int* dprompts, int P, cudaStream_t s) {
  if (st.n_bg <= 0) return SPECTRE_OK;
  SPECTRE_LAUNCH_PDL("k_bg_init", k_bg_init, dim3((st.n_bg + 255) / 256), dim3(256), 0, s, st,
                     dprompts, P);
  return SPECTRE_OK;
}
int launch_bg_forced_prep(const DecodeStateDev& st, const BatchDev& bt, int which,
                          cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_bg_forced_prep", k_bg_forced_prep, dim3(1), dim3(kProtoThreads), 0, s,
                     st, bt, which);
  return SPECTRE_OK;
}
int launch_bg_forced_append(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_bg_forced_append", k_bg_forced_append, dim3(1), dim3(kProtoThreads), 0,
                     s, st, bt);
  return SPECTRE_OK;
}
int launch_set_round_limit(const DecodeStateDev& st, int extra, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_set_round_limit", k_set_round_limit, dim3(1), dim3(1), 0, s, st, extra);
  return SPECTRE_OK;
}
// Draft prompt compression (draft_engine.py:123-131): keep the first and the
// last `keep` tokens of every prompt, contiguous (StreamingLLM-style re-indexing).
__global__ void k_compress_prompts(const int* __restrict__ prompts, int P, int keep, int n_req,
                                   int* __restrict__ out) {
  const int Pd = 2 * keep;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_req * Pd; i += gridDim.x * blockDim.x) {
    const int b = i / Pd, j = i % Pd;
    out[i] = prompts[(size_t)b * P + (j < keep ? j : P - Pd + j)];
  }
}

int launch_compress_prompts(const int* prompts, int P, int keep, int n_req, int* out,
                            cudaStream_t s) {
  k_compress_prompts<<<(n_req * 2 * keep + 255) / 256, 256, 0, s>>>(prompts, P, keep, n_req, out);
  SPECTRE_LAUNCH_CHECK("k_compress_prompts");
  return SPECTRE_OK;
}

int launch_prefill_batch(const int* prompts, int prompt_len, int n_req, int c0, int cs,
                         const BatchDev& bt, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_prefill_batch", k_prefill_batch, dim3((n_req + 255) / 256), dim3(256), 0, s,
                     prompts, prompt_len, n_req, c0, cs, bt);
  return SPECTRE_OK;
}
int launch_admit(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_admit", k_admit, dim3((st.n_req + 255) / 256), dim3(256), 0, s, st, bt);
  return SPECTRE_OK;
}
int launch_round_begin(const DecodeStateDev& st, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_round_begin", k_round_begin, dim3(1), dim3(256), 0, s, st);
  return SPECTRE_OK;
}
int launch_draft_prep(const DecodeStateDev& st, const BatchDev& bt, int which, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_draft_prep", k_draft_prep, dim3(1), dim3(kProtoThreads), 0, s, st, bt, which);
  return SPECTRE_OK;
}
int launch_draft_append(const DecodeStateDev& st, const BatchDev& bt, int which, int last,
                        cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_draft_append", k_draft_append, dim3(1), dim3(kProtoThreads), 0, s, st, bt,
                     which, last);
  return SPECTRE_OK;
}
int launch_verify_prep(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_verify_prep", k_verify_prep, dim3(1), dim3(kProtoThreads), 0, s, st, bt);
  return SPECTRE_OK;
}
int launch_accept(const DecodeStateDev& st, const BatchDev& bt, cudaStream_t s) {
  SPECTRE_LAUNCH_PDL("k_accept", k_accept, dim3(1), dim3(kProtoThreads), 0, s, st, bt);
  return SPECTRE_OK;
}

}  // namespace spectre
