// oracle_mode.cu — the decode loop on the synthetic model pair, fully on device.
//
// K8 (stream / propose / verify batch kernels) and the persistent round-loop
// kernel that restates specsim.run in the fault-free regime
// (sim.py:338-760, target_engine.py:105-308, draft_engine.py:72-120,246-431).
// Compiled with -fmad=false; the controller and the simulated clock also use
// explicit _rn intrinsics, so every double matches the reference bit for bit.
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "protocol.cuh"

namespace spectre {

// ---------------------------------------------------------------- K8 batch ops

__global__ void k_oracle_stream(uint64_t seed, uint64_t stream_id, const int64_t* __restrict__ req,
                                const int64_t* __restrict__ pos, uint64_t* __restrict__ out,
                                int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = stream_token(seed, stream_id, (uint64_t)req[i], (uint64_t)pos[i]);
  }
}

__global__ void k_oracle_propose(uint64_t seed, double alpha, const int64_t* __restrict__ req,
                                 const int64_t* __restrict__ start,
                                 const int32_t* __restrict__ count,
                                 const int64_t* __restrict__ off,
                                 const double* __restrict__ uniforms, uint64_t* __restrict__ out,
                                 int32_t max_count, int64_t n_seg) {
  const int64_t total = n_seg * max_count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / max_count;
    const int32_t j = (int32_t)(i % max_count);
    if (j >= count[s]) {
      out[i] = kPad;
      continue;
    }
    const uint64_t ref = ref_token(seed, (uint64_t)req[s], (uint64_t)(start[s] + j));
    out[i] = uniforms[off[s] + j] < alpha ? ref : (ref ^ kDisagree);
  }
}

__global__ void k_oracle_verify(uint64_t seed, const int64_t* __restrict__ req,
                                const int64_t* __restrict__ start,
                                const uint64_t* __restrict__ cand, const int32_t* __restrict__ len,
                                int32_t width, int32_t* __restrict__ accepted,
                                uint64_t* __restrict__ bonus, int64_t n) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (uint64_t)req[c];
    const int32_t st = (int32_t)start[c];
    auto ref = [&](int32_t q) { return ref_token(seed, r, (uint64_t)q); };
    const int32_t a = verify_prefix(cand + c * width, len[c], st, ref);
    accepted[c] = a;
    bonus[c] = ref(st + a);
  }
}

// ------------------------------------------------------- the decode-loop kernel

struct OracleWS {
  int32_t* pos;
  int32_t* rnd;
  int32_t* synced;
  int32_t* done;
  int32_t* in_rollback;
  int32_t* cached_len;
  int32_t* cached_start;
  int32_t* hist_len;
  int32_t* prep_len;
  int32_t* prep_start;
  int32_t* rng_off;
  int32_t* kind;
  int32_t* delta;
  int32_t* rolled;
  uint64_t* cached_tok;  // [n][G]
  uint64_t* prep_tok;    // [n][G]
  uint64_t* cand_tok;    // [n][G]
  uint64_t* hist;        // [n][HC]
  int64_t hist_cap;
  int32_t G;
};

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t ws_layout(const SpectreOracleConfig& c, char* base, OracleWS* ws) {
  const size_t n = (size_t)c.n_requests;
  const int32_t G = c.gamma + 1;
  const int64_t HC = (int64_t)c.output_len * (c.gamma + 1) + 2 * c.gamma + 8;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += align256(bytes);
    return p;
  };
  int32_t** i32s[] = {&ws->pos,        &ws->rnd,        &ws->synced,   &ws->done,
                      &ws->in_rollback, &ws->cached_len, &ws->cached_start,
                      &ws->hist_len,   &ws->prep_len,   &ws->prep_start, &ws->rng_off,
                      &ws->kind,       &ws->delta,      &ws->rolled};
  for (auto p : i32s) *p = reinterpret_cast<int32_t*>(take(n * sizeof(int32_t)));
  ws->cached_tok = reinterpret_cast<uint64_t*>(take(n * G * sizeof(uint64_t)));
  ws->prep_tok = reinterpret_cast<uint64_t*>(take(n * G * sizeof(uint64_t)));
  ws->cand_tok = reinterpret_cast<uint64_t*>(take(n * G * sizeof(uint64_t)));
  ws->hist = reinterpret_cast<uint64_t*>(take(n * (size_t)HC * sizeof(uint64_t)));
  ws->hist_cap = HC;
  ws->G = G;
  return off;
}

enum OracleError : int64_t {
  kErrNone = 0,
  kErrCommitGap = 1,
  kErrRegression = 2,
  kErrHistoryOverflow = 3,
  kErrUniformsExhausted = 4,
  kErrLateReply = 5,       // parallel reply would miss the commit (or, conservative,
                           // the reply deadline): outside domain
  kErrTraceOverflow = 6,
  kErrMisanchored = 7,
};

constexpr int kLoopThreads = 512;

__device__ __forceinline__ void block_fail(int64_t* scalars, int64_t code, int64_t req) {
  if (atomicCAS(reinterpret_cast<unsigned long long*>(&scalars[2]), 0ull,
                (unsigned long long)code) == 0ull) {
    scalars[3] = req;
  }
}

__global__ void __launch_bounds__(kLoopThreads, 1)
k_oracle_decode_loop(SpectreOracleConfig cfg, const double* __restrict__ arrivals,
                     const double* __restrict__ uniforms, int64_t n_uniforms, OracleWS ws,
                     SpectreOracleOutputs out) {
  const int tid = threadIdx.x;
  const int n = cfg.n_requests;
  const int g = cfg.gamma;
  const int G = ws.G;
  const int OL = cfg.output_len;
  const uint64_t seed = cfg.seed;
  const bool spec = cfg.variant != SPECTRE_VARIANT_AR;

  __shared__ double s_now, s_ema, s_L, s_rstar;
  __shared__ double s_tdm;   // target's last reply T_D^mix (sim.py:283-288, 833-834)
  __shared__ int s_has_ema, s_has_L, s_prev_mode, s_mode, s_round, s_admitted, s_limit,
      s_active, s_lo, s_stop, s_finished;
  __shared__ long long s_cursor;
  __shared__ int s_scan[kLoopThreads];
  __shared__ int s_carry;

  if (tid == 0) {
    s_now = arrivals[0];
    s_limit = 0;
    s_admitted = 0;
    s_active = 0;
    s_lo = 0;
    s_round = 0;
    s_has_ema = 0;
    s_has_L = 0;
    s_ema = 0.0;
    s_tdm = cfg.t_draft_init;
    s_L = 0.0;
    s_prev_mode = 0;
    s_cursor = 0;
    s_stop = 0;
    s_finished = 0;
    out.scalars[2] = 0;
    out.scalars[3] = -1;
  }
  __syncthreads();

  while (true) {
    // ---- admission (sim.py:405-427) and idle wait for the next ARRIVAL
    if (tid == 0) {
      while (true) {
        while (s_admitted < n && s_admitted <= s_limit && s_active < cfg.max_concurrency) {
          const int r = s_admitted++;
          const uint64_t first = ref_token(seed, r, 0);
          out.committed[(int64_t)r * OL] = first;
          ws.pos[r] = 1;
          ws.rnd[r] = 0;
          ws.synced[r] = 0;
          ws.in_rollback[r] = 1;
          ws.cached_len[r] = 0;
          ws.hist_len[r] = 0;
          ws.prep_len[r] = 0;
          out.admitted_at[r] = s_now;
          if (1 >= OL) {
            ws.done[r] = 1;
            out.finished_at[r] = s_now;
            out.committed_pos[r] = 1;
            ++s_finished;
          } else {
            ws.done[r] = 0;
            ++s_active;
          }
        }
        if (s_active > 0) break;
        if (s_admitted >= n) {
          s_stop = 1;
          break;
        }
        s_now = arrivals[s_admitted];
        s_limit = s_admitted;
      }
      while (s_lo < s_admitted && ws.done[s_lo]) ++s_lo;
      if (!s_stop) {
        if (s_round >= cfg.max_rounds) {
          block_fail(out.scalars, kErrTraceOverflow, -1);
          s_stop = 1;
        }
      }
      if (!s_stop) {
        // ---- controller (sim.py:447-467)
        int mode = 'F';
        double r_star = __longlong_as_double(0x7ff8000000000000ll);
        if (spec) {
          if (cfg.variant == SPECTRE_VARIANT_ORDINARY) {
            mode = 'O';
          } else if (cfg.variant == SPECTRE_VARIANT_PARALLEL) {
            mode = 'P';
          } else {
            const bool hasL = cfg.has_fixed_l ? true : (s_has_L != 0);
            const double L = cfg.has_fixed_l ? cfg.fixed_threshold_l : s_L;
            // T_D fed to the controller = the last reply's t_d_mix
            mode = choose_mode_hybrid(s_prev_mode, s_has_ema != 0, s_ema, hasL, L, g,
                                      cfg.t_target, s_tdm, &r_star);
            s_prev_mode = mode;
          }
        }
        s_mode = mode;
        s_rstar = r_star;
        s_round += 1;
        s_carry = 0;
      }
    }
    __syncthreads();
    if (s_stop) break;

    const int mode = s_mode;
    const int lo = s_lo, hi = s_admitted;
    const int ridx = s_round - 1;
    const long long cursor = s_cursor;

    // ---- draws per queried request, exclusive scan in active order
    // (RNG consumption order: draft_engine.py:314-321, 362-376)
    for (int base = lo; base < hi; base += kLoopThreads) {
      const int i = base + tid;
      int cnt = 0;
      if (i < hi && !ws.done[i] && spec) {
        if (mode == 'O') cnt = ws.cached_len[i] == 0 ? g - 1 : 0;
        else if (mode == 'P') cnt = g;
      }
      s_scan[tid] = cnt;
      __syncthreads();
      for (int d = 1; d < kLoopThreads; d <<= 1) {
        int v = tid >= d ? s_scan[tid - d] : 0;
        __syncthreads();
        s_scan[tid] += v;
        __syncthreads();
      }
      if (i < hi) ws.rng_off[i] = s_carry + s_scan[tid] - cnt;
      __syncthreads();
      if (tid == kLoopThreads - 1) s_carry += s_scan[tid];
      __syncthreads();
    }
    const int total_draws = s_carry;
    if (tid == 0 && cursor + total_draws > n_uniforms) {
      block_fail(out.scalars, kErrUniformsExhausted, -1);
    }
    __syncthreads();
    if (out.scalars[2] != 0) break;

    // ---- per-request round body: sync/rebase/propose, assemble, verify,
    // commit, rollback flag, suffix reuse.
    for (int i = lo + tid; i < hi; i += kLoopThreads) {
      if (ws.done[i]) continue;
      const uint64_t r = (uint64_t)i;
      uint64_t* committed = out.committed + (int64_t)i * OL;
      uint64_t* h = ws.hist + (int64_t)i * ws.hist_cap;
      uint64_t* prep = ws.prep_tok + (int64_t)i * G;
      uint64_t* cached = ws.cached_tok + (int64_t)i * G;
      uint64_t* cand = ws.cand_tok + (int64_t)i * G;
      auto ref = [&](int32_t q) { return ref_token(seed, r, (uint64_t)q); };
      int32_t pos = ws.pos[i];
      int32_t prep_len = 0, prep_start = 0;
      const bool queried = spec && ((mode == 'P') || (mode == 'O' && ws.cached_len[i] == 0));
      // parallel: assemble from the state BEFORE the query (sim.py:594-598)
      int32_t kind, cstart, clen;
      if (mode == 'F') {
        kind = kFallback;
        cand[0] = committed[pos - 1];
        cstart = pos - 1;
        clen = 1;
      } else if (ws.cached_len[i] > 0 && !ws.in_rollback[i]) {
        if (ws.cached_start[i] != pos) block_fail(out.scalars, kErrMisanchored, i);
        kind = kCached;
        const int32_t cl = ws.cached_len[i];
        for (int k = 0; k < g; ++k) cand[k] = k < cl ? cached[k] : kPad;
        cstart = pos;
        clen = g;
      } else {
        kind = (mode == 'P') ? kPadded : kRepaired;
        cand[0] = committed[pos - 1];
        cstart = pos - 1;
        clen = g;
        for (int k = 1; k < g; ++k) cand[k] = kPad;  // PADDED; REPAIRED overwrites
      }
      if (queried) {
        // _sync_payload + DraftServer.on_sync (sim.py:473-477, draft_engine.py:246-280)
        const int32_t start = ws.synced[i];
        int32_t inv;
        int32_t hl = session_on_sync(
            h, ws.hist_len[i], start, pos - start,
            [&](int32_t k) { return committed[start + k]; }, ref, &inv);
        ws.synced[i] = pos;
        const int32_t count = (mode == 'O') ? g - 1 : g;
        if (mode == 'O') hl = session_rebase(h, hl, pos, ref, &inv);  // anchor = committed_pos
        if (hl + count > ws.hist_cap) {
          block_fail(out.scalars, kErrHistoryOverflow, i);
        } else {
          // generate_speculative -> draft_propose (oracle.py:69-88)
          const double* u = uniforms + cursor + ws.rng_off[i];
          for (int j = 0; j < count; ++j) {
            const uint64_t rt = ref(hl + j);
            const uint64_t t = (u[j] < cfg.alpha) ? rt : (rt ^ kDisagree);
            h[hl + j] = t;
            if (mode == 'O') cand[1 + j] = t;
            else prep[j] = t;
          }
          if (mode == 'O') {
            if (hl != pos) block_fail(out.scalars, kErrMisanchored, i);
          } else {
            prep_len = count;
            prep_start = hl;
          }
          hl += count;
        }
        ws.hist_len[i] = hl;
      }
      // ---- verify (oracle.py:90-113)
      const int32_t acc = verify_prefix(cand, clen, cstart, ref);
      const uint64_t bonus = ref(cstart + acc);
      const int32_t new_pos = cstart + acc + 1;
      int32_t real = 0;
      for (int k = 0; k < clen; ++k) real += cand[k] != kPad;
      // ---- rollback set membership (target_engine.py:285-302)
      int rolled = acc < real;
      if (!rolled && prep_len > 0 && prep[0] != bonus) rolled = 1;
      // ---- commit_round (target_engine.py:227-249)
      if (cstart > pos) block_fail(out.scalars, kErrCommitGap, i);
      if (new_pos <= pos) block_fail(out.scalars, kErrRegression, i);
      const int32_t end = min(new_pos, OL);
      for (int32_t q = pos; q < end; ++q) committed[q] = ref(q);
      const int32_t delta = max(end - pos, 0);
      pos += delta;
      const int32_t done = pos >= OL;
      ws.pos[i] = pos;
      ws.rnd[i] += 1;
      ws.done[i] = done;
      // ---- reuse_or_discard_suffix (target_engine.py:252-279)
      int32_t cst = 0;
      const int32_t cl =
          reuse_or_discard(prep, prep_len, prep_start, committed, pos, done, cached, &cst);
      ws.cached_len[i] = cl;
      ws.cached_start[i] = cst;
      ws.in_rollback[i] = cl == 0;
      ws.kind[i] = kind;
      ws.delta[i] = delta;
      ws.rolled[i] = rolled;
      if (done) out.committed_pos[i] = pos;
    }
    __syncthreads();

    // ---- round accounting, EMA updates, clock (sim.py:667-760) — serial in
    // active order because the L estimator is an order-dependent EMA.
    if (tid == 0) {
      int participants = 0, delta_sum = 0, n_roll = 0, csum = 0, cn = 0, queries = 0,
          n_padded = 0;
      for (int i = lo; i < hi; ++i) {
        if (ws.kind[i] == 0) continue;  // not active this round
        ++participants;
        delta_sum += ws.delta[i];
        n_roll += ws.rolled[i];
        const int k = ws.kind[i];
        if (k == kCached || k == kRepaired) {
          csum += ws.delta[i];
          ++cn;
          const double dv = (double)ws.delta[i];
          if (!s_has_L) {
            s_L = dv;
            s_has_L = 1;
          } else {
            s_L = ema_step(cfg.ema_decay, s_L, dv);
          }
        }
        if (k == kPadded) ++n_padded;
        if (spec && (mode == 'P' || (mode == 'O' && k == kRepaired))) ++queries;
      }
      const double r_hat = __ddiv_rn((double)n_roll, (double)participants);
      if (spec) {
        if (!s_has_ema) {
          s_ema = r_hat;
          s_has_ema = 1;
        } else {
          s_ema = ema_step(cfg.ema_decay, s_ema, r_hat);
        }
      }
      // simulated clock (sim.py:542-622; draft_engine.py:323-353)
      const double now = s_now;
      const double nan = __longlong_as_double(0x7ff8000000000000ll);
      double dispatch = now, dstart = nan, ddone = nan;
      int steps = 0;
      // draft step latency of this round: all-speculative base (compression
      // factor applied on the host) + contention slope beyond the free batch
      // (draft_engine.py:158-164, 335-344)
      const int over = queries > cfg.t_draft_free_batch ? queries - cfg.t_draft_free_batch : 0;
      const double tdm = __dadd_rn(cfg.t_draft, __dmul_rn(cfg.t_draft_slope, (double)over));
      // conservative_mode_check on the last reply's T_D^mix (sim.py:143-146, 599-602)
      const bool conservative = mode == 'P' && __dmul_rn((double)g, s_tdm) > cfg.t_target;
      if (mode == 'O' && queries > 0) {
        steps = g - 1;
        dstart = __dadd_rn(now, cfg.delay);
        ddone = __dadd_rn(dstart, __dmul_rn((double)steps, tdm));
        dispatch = __dadd_rn(ddone, cfg.delay);
        s_tdm = tdm;
      } else if (mode == 'P') {
        steps = g;
        dstart = __dadd_rn(now, cfg.delay);
        ddone = __dadd_rn(dstart, __dmul_rn((double)steps, tdm));
        s_tdm = tdm;
      }
      const double t_t =
          __dadd_rn(cfg.t_target, __dmul_rn(cfg.t_target_slope, (double)(participants - 1)));
      double commit = __dadd_rn(dispatch, t_t);
      if (mode == 'P') {
        const double reply = __dadd_rn(ddone, cfg.delay);
        if (conservative) {
          // _try_commit waits for every queried reply (sim.py:624-640, 841-844);
          // they must land before the wait deadline (no timeout in the domain)
          if (!(__dsub_rn(reply, dispatch) < __dsub_rn(cfg.reply_timeout, 1e-12)))
            block_fail(out.scalars, kErrLateReply, -1);
          if (reply > commit) commit = reply;
        } else if (!(reply < commit)) {
          block_fail(out.scalars, kErrLateReply, -1);
        }
      }
      out.round_mode[ridx] = mode;
      out.round_participants[ridx] = participants;
      out.round_delta[ridx] = delta_sum;
      out.round_n_roll[ridx] = n_roll;
      out.round_content_sum[ridx] = csum;
      out.round_content_n[ridx] = cn;
      out.round_queries[ridx] = queries;
      out.round_draft_tokens[ridx] = queries * steps;
      out.round_n_padded[ridx] = n_padded;
      out.round_started[ridx] = now;
      out.round_dispatch[ridx] = dispatch;
      out.round_commit[ridx] = commit;
      out.round_draft_start[ridx] = dstart;
      out.round_draft_done[ridx] = ddone;
      out.round_r_hat_ema[ridx] = s_has_ema ? s_ema : nan;
      out.round_accepted_len_ema[ridx] = s_has_L ? s_L : nan;
      out.round_r_star[ridx] = s_rstar;
      // finish requests, reset per-round marks
      for (int i = lo; i < hi; ++i) {
        if (ws.kind[i] == 0) continue;
        if (ws.done[i]) {
          out.finished_at[i] = commit;
          --s_active;
          ++s_finished;
        }
        ws.kind[i] = 0;
      }
      s_cursor = cursor + total_draws;
      s_now = commit;
      // arrivals that have fired by `commit` (ARRIVAL seq < VERIFY_DONE seq)
      int lim = s_limit;
      while (lim + 1 < n && arrivals[lim + 1] <= commit) ++lim;
      s_limit = lim;
      if (s_finished >= n) s_stop = 1;
    }
    __syncthreads();
    if (s_stop || out.scalars[2] != 0) break;
  }
  if (tid == 0) {
    out.scalars[0] = s_round;
    out.scalars[1] = s_cursor;
    out.scalars[4] = s_finished;
  }
}

// kind[] must start zeroed: initialise in a tiny kernel.
__global__ void k_zero_i32(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

static int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

}  // namespace spectre

using namespace spectre;

extern "C" int spectre_oracle_stream(uint64_t seed, int32_t stream_id, const int64_t* req,
                                     const int64_t* pos, uint64_t* out, int64_t n,
                                     void* stream) {
  if (n < 0 || (n > 0 && (!req || !pos || !out))) return arg_fail("spectre_oracle_stream");
  if (stream_id != 0 && stream_id != 1) return arg_fail("stream_id must be 0 or 1");
  if (n == 0) return SPECTRE_OK;
  k_oracle_stream<<<grid_for(n), 256, 0, as_stream(stream)>>>(seed, (uint64_t)stream_id, req, pos,
                                                               out, n);
  SPECTRE_LAUNCH_CHECK("k_oracle_stream");
  return SPECTRE_OK;
}

extern "C" int spectre_oracle_propose(uint64_t seed, double alpha, const int64_t* req,
                                      const int64_t* start, const int32_t* count,
                                      const int64_t* off, const double* uniforms, uint64_t* out,
                                      int32_t max_count, int64_t n_seg, void* stream) {
  if (n_seg < 0 || max_count < 0) return arg_fail("spectre_oracle_propose");
  if (n_seg == 0 || max_count == 0) return SPECTRE_OK;
  k_oracle_propose<<<grid_for(n_seg * max_count), 256, 0, as_stream(stream)>>>(
      seed, alpha, req, start, count, off, uniforms, out, max_count, n_seg);
  SPECTRE_LAUNCH_CHECK("k_oracle_propose");
  return SPECTRE_OK;
}

extern "C" int spectre_oracle_verify(uint64_t seed, const int64_t* req, const int64_t* start,
                                     const uint64_t* cand, const int32_t* len, int32_t width,
                                     int32_t* accepted, uint64_t* bonus, int64_t n_cand,
                                     void* stream) {
  if (n_cand < 0 || width < 1) return arg_fail("spectre_oracle_verify");
  if (n_cand == 0) return SPECTRE_OK;
  k_oracle_verify<<<grid_for(n_cand), 256, 0, as_stream(stream)>>>(seed, req, start, cand, len,
                                                                   width, accepted, bonus, n_cand);
  SPECTRE_LAUNCH_CHECK("k_oracle_verify");
  return SPECTRE_OK;
}

extern "C" size_t spectre_oracle_workspace_bytes(const SpectreOracleConfig* cfg) {
  if (!cfg || cfg->n_requests < 1 || cfg->gamma < 1 || cfg->output_len < 1) return 0;
  OracleWS ws;
  return ws_layout(*cfg, nullptr, &ws);
}

extern "C" int spectre_oracle_run(const SpectreOracleConfig* cfg, const double* arrivals,
                                  const double* uniforms, int64_t n_uniforms, void* workspace,
                                  const SpectreOracleOutputs* out, void* stream) {
  if (!cfg || !arrivals || !workspace || !out) return arg_fail("spectre_oracle_run: null");
  if (cfg->n_requests < 1 || cfg->gamma < 1 || cfg->output_len < 1 || cfg->max_concurrency < 1 ||
      cfg->max_rounds < 1 || cfg->variant < 0 || cfg->variant > 3)
    return arg_fail("spectre_oracle_run: config");
  if (cfg->variant != SPECTRE_VARIANT_AR && (cfg->gamma < 2 || !uniforms))
    return arg_fail("spectre_oracle_run: speculative variants need gamma >= 2 and uniforms");
  OracleWS ws;
  const size_t bytes = ws_layout(*cfg, reinterpret_cast<char*>(workspace), &ws);
  (void)bytes;
  cudaStream_t s = as_stream(stream);
  k_zero_i32<<<grid_for(cfg->n_requests), 256, 0, s>>>(ws.kind, cfg->n_requests);
  SPECTRE_LAUNCH_CHECK("k_zero_i32");
  k_oracle_decode_loop<<<1, kLoopThreads, 0, s>>>(*cfg, arrivals, uniforms, n_uniforms, ws, *out);
  SPECTRE_LAUNCH_CHECK("k_oracle_decode_loop");
  return SPECTRE_OK;
}
