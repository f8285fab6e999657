// engine.cu — model-mode runtime: forward-pass sequencing for the target and
// the draft, prefill/admission, and the decode round as a CUDA graph whose
// ordinary / parallel branches are conditional nodes selected on the device
// (no host round trip per round), looped by a device-side WHILE node.
//
// Round DAG (one WHILE iteration):
//   round_begin (controller) ─┬─► IF(ordinary){ draft repair (γ-1 steps) ─► verify }
//                             ├─► IF(parallel){ fork: draft speculation (γ steps) ∥ verify; join }
//                             └─► IF(ar){ verify }
//                                        ─► accept (rejection-sampling pre-pass when T > 0)
// In parallel rounds the draft and the target are forked onto two streams and
// joined before the accept.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "chain.h"
#include "common.cuh"
#include "engine_state.cuh"
#include "gemm.h"
#include "model_kernels.cuh"

namespace spectre {

int launch_attention_w(const CUtensorMap& tk32, const CUtensorMap& tv32, const AttnArgs& a,
                       int hd, int rows_per_req, cudaStream_t s);
int launch_embed_rmsnorm(const int* tok, const int* t_dev, int t_cap, const void* E,
                         const float* w, float* h, void* x, int d, float eps, cudaStream_t s);
int launch_residual_rmsnorm(const float* part, int splits, int rows_cap, const int* t_dev,
                            int t_cap, const float* w, float* h, void* x, int d, float eps,
                            cudaStream_t s);
int launch_qkv_rope_kv(const float* part, int splits, int rows_cap, const int* t_dev, int t_cap,
                       const int* tok_pos, const int* tok_slot, const void* rope, void* q,
                       void* kc, void* vc, int n_q, int n_kv, int hd, int ctx_cap,
                       cudaStream_t s);
int launch_argmax_reduce(const float* val, const int* idx, int n_tiles, int rows_cap,
                         const int* t_dev, int t_cap, int* out_tok, float* out_val,
                         cudaStream_t s);
int launch_rope_table(void* rope, int ctx_cap, int hd, double theta, cudaStream_t s);

#define TRY(x)                 \
  do {                         \
    int _r = (x);              \
    if (_r) return _r;         \
  } while (0)

struct Bump {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (n * sizeof(T) + 255) & ~size_t(255);
    return p;
  }
};

static inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

static int tile_rows_default(int fallback) {
  const char* v = getenv("SPECTRE_TILE_ROWS");
  if (!v) return fallback;
  return atoi(v) == 128 ? 128 : 256;
}

// Keys per attention item.  Key splits only pay when (request, kv head)
// items are too few to fill the SMs: with n_req * n_kv >= SMs one item per
// (request, head) already keeps every SM busy, and a split adds a partial
// round trip + merge (measured at ctx 1093, C2: target 110 vs ~61 us).
static int attn_chunk_default(int n_items, int ctx_cap) {
  if (const char* v = getenv("SPECTRE_ATTN_CHUNK")) {
    const int c = atoi(v);
    return (c >= 64 && c % 64 == 0 && c <= 8192) ? c : 1024;
  }
  if (n_items >= 148) return std::max(1024, (ctx_cap + 63) / 64 * 64);
  return 1024;
}

// prompt tokens per request per prefill forward: a row budget of
// SPECTRE_PREFILL_ROWS (default 512) split over the requests, at most 16
static int prefill_chunk(int n_req) {
  static const int rows = [] {
    const char* v = getenv("SPECTRE_PREFILL_ROWS");
    return v ? std::max(64, atoi(v)) : 512;
  }();
  return std::max(1, std::min(16, rows / std::max(1, n_req)));
}

static int pick_splits(int n_tiles, int k_iters, int ctas = 148) {
  // one wave of CTAs, one split-K job each (two jobs per CTA measured slower)
  int s = ctas / n_tiles;
  if (s > 12) s = 12;     // partial traffic grows with s (consumers unroll <= 12)
  if (s < 1) s = 1;
  while (s > 1 && k_iters / s < 3) --s;
  return s;
}

// ---------------------------------------------------------------- one model
struct ModelRT {
  SpectreModelDims dm{};
  SpectreModelWeights w{};
  // draft decode steps as persistent chains (chain.cu): first = embed + qkv(0) +
  // RoPE; mid[l] = layer l's o .. layer l+1's RoPE; last = layer L-1's o .. final norm
  bool use_chain = false;
  void* ch_first = nullptr;
  std::vector<void*> ch_mid;
  void* ch_last = nullptr;
  unsigned* ch_bar = nullptr;
  unsigned long long* ch_dbg = nullptr;   // SPECTRE_CHAIN_DBG: [L + 1][64] phase stamps
  ModelRT() = default;
  ModelRT(const ModelRT&) = delete;
  ModelRT& operator=(const ModelRT&) = delete;
  ~ModelRT() {
    for (void* p : ch_mid) chain_free(p);
    if (ch_first) chain_free(ch_first);
    if (ch_last) chain_free(ch_last);
  }
  int n_req = 0, rows_cap = 0, ctx_cap = 0, max_new = 1, split_max = 1, rb_cap = 1;
  int sp_qkv = 1, sp_o = 1, sp_d = 1;
  bool down_pu = false;   // split-K GEMMs as (tile, split, token pass) units (layout())
  bool pair_q = false, pair_o = false, pair_d = false;   // ... as CTA-pair units instead
  int tr_qkv = 256, tr_o = 256, tr_d = 256;   // weight rows per tile, per GEMM
  int tile_rows = 256;   // weight rows per GEMM CTA (128 for small-T models)
  bool half_gemm = false; // decode GEMMs in the half-SM config (2 CTAs per SM, 128-row tiles)
  int attn_chunk = 128;
  float* h = nullptr;
  __nv_bfloat16 *x = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
  float *part = nullptr, *att_o = nullptr, *att_ml = nullptr, *amax_v = nullptr;
  int sampling = 0;           // temperature > 0: lm_head writes fp32 logits
  float inv_t = 1.f;
  uint64_t seed = 0;
  float* logits = nullptr;    // [rows_cap][vocab] (sampling)
  float2* lstat = nullptr;    // [rows_cap] (max, sum exp) of logits / T
  int* att_cnt = nullptr;
  int* amax_i = nullptr;
  float2* rope = nullptr;
  CUtensorMap tm_k32{}, tm_v32{};   // whole K / V cache as [L*slots*n_kv*ctx_cap][hd] rows,
                                    // 32-key boxes (warp-per-item attention)
  BatchDev bt{};
  std::vector<GemmPlan> pq, po, pgu, pd;
  // large-T plans (T > 0 sampling only: batch invariance across T is not part
  // of its contract): 128-row tiles as (tile, split, 256-token pass) units, fewer
  // splits -> far less fp32 partial traffic at config 3's ~1,280 verify rows
  std::vector<GemmPlan> pqL, poL, pdL;
  // large-T plans' split counts (config 3, T = 1,280, target ms per round:
  // down 2 / 3 / 4 / 5 splits 18.78 / 18.46-18.57 / 18.70 / 19.21; o 1 best,
  // q/k/v 2 and 3 even)
  static constexpr int kLargeT = 768, kSpLqkv = 2, kSpLo = 1, kSpLd = 3;
  GemmPlan plm{};

  int nqkv() const { return (dm.n_q_heads + 2 * dm.n_kv_heads) * dm.head_dim; }
  int group() const { return dm.n_q_heads / dm.n_kv_heads; }

  void layout(Bump& b) {
    const int d = dm.d_model, R = rows_cap;
    const int qd = dm.n_q_heads * dm.head_dim;
    const int tr = half_gemm ? 128 : tile_rows, ctas = half_gemm ? 296 : 148;
    tr_qkv = tr_o = tr_d = tr;
    if (!half_gemm) {
      // per-GEMM tile height.  q/k/v and o: 128-row tiles halve the split
      // count, and at T=256 the fp32 split-K partials (s*T*N*4 B, written and
      // re-read) cost as much HBM as the weights; measured -0.12 ms/round.
      // down (K = ffn) keeps 256-row tiles (its partials are 0.3x its weights).
      tr_qkv = tr_o = 128;
      if (const char* v = getenv("SPECTRE_QKV_TILE")) tr_qkv = atoi(v) == 128 ? 128 : tr;
      if (const char* v = getenv("SPECTRE_O_TILE")) tr_o = atoi(v) == 128 ? 128 : tr;
      if (const char* v = getenv("SPECTRE_DOWN_TILE")) tr_d = atoi(v) == 128 ? 128 : tr;
    }
    sp_qkv = pick_splits((nqkv() + tr_qkv - 1) / tr_qkv, d / 64, ctas);
    sp_o = pick_splits((d + tr_o - 1) / tr_o, qd / 64, ctas);
    sp_d = pick_splits((d + tr_d - 1) / tr_d, dm.ffn / 64, ctas);
    // large verify batches (rows_cap >= kLargeT: config 5's 128 x 7 rows): the
    // split-K GEMMs as 128-row (tile, split, 256-token pass) units over every
    // SM -- one plan for every T of this engine, so still batch invariant.
    // 128-row one-box units: splits for about `waves` waves of units
    // (measured at Qwen2.5-32B, T=896: down 4 waves, 328 -> 297 us; q/k/v 4
    // waves, 83.4 -> 70.5 us; o 2 waves, 60.0 -> 51.1 us).  Where the 256-row
    // tiles pair up (N % 512 == 0), CTA pairs over (tile pair, split, 256-token
    // chunk) units instead (cta_group::2: 1.5x the MMA rate per SM of one-box
    // tiles); isolated, L2 flushed, vs the one-box units: 32B T=896 down
    // 293.8 -> 238.6 us (3 splits), q/k/v 91.2 -> 70.7 (1), o 76.8 -> 68.8 (1);
    // 8B T=1280 down 175.1 -> 138.2 (3), q/k/v 85.0 -> 62.5 (1), o 76.8 -> 59.6 (1).
    down_pu = !half_gemm && !use_chain && rows_cap >= kLargeT;
    if (down_pu) {
      const int passes = (rows_cap + 255) / 256;
      auto pu_splits = [&](int n, int k, int waves) {
        const int units = ((n + 127) / 128) * passes;
        int sp = std::max(1, std::min(12, (waves * ctas + units / 2) / units));
        while (sp > 1 && k / 64 / sp < 3) --sp;
        return sp;
      };
      // splits: the best wave fill (units / (waves * CTAs)) with >= 48 k blocks
      // (3,072 K) per unit, fewer splits on ties (in context: 32B down 7
      // splits 181 us vs 3 / 5 splits 231 us; 8B T=1,280 down 3 splits
      // 102.5 us vs 5 / 7 splits 106.5 / 112.0 us, where 5+ fall below 48)
      auto pair_splits = [&](int n, int k) {
        const int g2 = ctas & ~1;
        int best = 1;
        double best_fill = 0.0;
        for (int sp = 1; sp <= 8 && (sp == 1 || k / 64 / sp >= 48); ++sp) {
          const int units = (n / 256) * sp * passes;
          const double fill = (double)units / ((double)((units + g2 - 1) / g2) * g2);
          if (fill > best_fill + 1e-9) {
            best_fill = fill;
            best = sp;
          }
        }
        return best;
      };
      static const bool pair_env = [] {   // SPECTRE_PAIR_UNITS=0: one-box units only
        const char* v = getenv("SPECTRE_PAIR_UNITS");
        return v ? atoi(v) != 0 : true;
      }();
      // in context (PDL prologues under the previous kernel) the o projection
      // keeps the one-box units: 32B 50.7 vs 66.6 us, 8B T=1280 37.9 vs 52.1
      pair_q = pair_env && nqkv() % 512 == 0;
      pair_o = false;
      pair_d = pair_env && d % 512 == 0;
      tr_qkv = pair_q ? 256 : 128;
      tr_o = pair_o ? 256 : 128;
      tr_d = pair_d ? 256 : 128;
      sp_qkv = pair_q ? pair_splits(nqkv(), d) : pu_splits(nqkv(), d, 4);
      sp_o = pair_o ? pair_splits(d, qd) : pu_splits(d, qd, 2);
      sp_d = pair_d ? pair_splits(d, dm.ffn) : pu_splits(d, dm.ffn, 4);
    }
    size_t part_n = std::max({(size_t)sp_qkv * nqkv(), (size_t)sp_o * d, (size_t)sp_d * d});
    if (down_pu)   // the large-T plans (sampling engines) share the buffer
      part_n = std::max({part_n, (size_t)kSpLqkv * nqkv(), (size_t)kSpLo * d, (size_t)kSpLd * d});
    if (use_chain)
      part_n = std::max({part_n, (size_t)chain_splits(nqkv(), d) * nqkv(),
                         (size_t)chain_splits(d, qd) * d, (size_t)chain_splits(d, dm.ffn) * d});
    attn_chunk = attn_chunk_default(n_req * dm.n_kv_heads, ctx_cap);
    split_max = (ctx_cap + attn_chunk - 1) / attn_chunk;
    // m-tiles per request, in whole attention row blocks (2 m-tiles at hd 128, 3 at hd 64)
    rb_cap = round_up((max_new * group() + 15) / 16, dm.head_dim == 128 ? 2 : 3);
    h = b.take<float>((size_t)R * d);
    x = b.take<__nv_bfloat16>((size_t)R * d);
    q = b.take<__nv_bfloat16>((size_t)R * qd);
    attn = b.take<__nv_bfloat16>((size_t)R * qd);
    act = b.take<__nv_bfloat16>((size_t)R * dm.ffn);
    part = b.take<float>(part_n * R);
    const size_t att_rows = (size_t)n_req * dm.n_kv_heads * rb_cap * split_max * 16;
    att_o = b.take<float>(att_rows * dm.head_dim);
    att_ml = b.take<float>(att_rows * 2);
    att_cnt = b.take<int>((size_t)n_req * dm.n_kv_heads * rb_cap);
    const int n_blocks = gemm_sk_grid() * 8;   // argmax partials: one per CTA epilogue warp
    if (sampling) {
      logits = b.take<float>((size_t)R * dm.vocab);
      lstat = b.take<float2>(R);
    }
    amax_v = b.take<float>((size_t)n_blocks * R);
    amax_i = b.take<int>((size_t)n_blocks * R);
    rope = b.take<float2>((size_t)ctx_cap * dm.head_dim / 2);
    ch_bar = b.take<unsigned>(64);
    if (use_chain && getenv("SPECTRE_CHAIN_DBG"))
      ch_dbg = b.take<unsigned long long>((size_t)(dm.n_layers + 1) * 64);
    bt.tok = b.take<int>(R);
    bt.pos = b.take<int>(R);
    bt.slot = b.take<int>(R);
    bt.out_tok = b.take<int>(R);
    bt.t_dev = b.take<int>(1);
    bt.q_off = b.take<int>(n_req);
    bt.n_new = b.take<int>(n_req);
    bt.pos0 = b.take<int>(n_req);
    bt.rslot = b.take<int>(n_req);
  }

  int plan() {
    const int d = dm.d_model, L = dm.n_layers, qd = dm.n_q_heads * dm.head_dim, F = dm.ffn;
    auto bf = [](const void* p) { return reinterpret_cast<const __nv_bfloat16*>(p); };
    pq.resize(L);
    po.resize(L);
    pgu.resize(L);
    pd.resize(L);
    const int tr = half_gemm ? 128 : tile_rows;
    for (int l = 0; l < L; ++l) {
      TRY(gemm_plan(&pq[l], bf(w.wqkv) + (size_t)l * nqkv() * d, nqkv(), d, x, rows_cap,
                    kPartial, sp_qkv, 0, 0, tr_qkv));
      TRY(gemm_plan(&po[l], bf(w.wo) + (size_t)l * d * qd, d, qd, attn, rows_cap, kPartial,
                    sp_o, 0, 0, tr_o));
      // SwiGLU needs full K per tile: 128-row tiles when they fit one wave
      // (draft); 256-row tiles as CTA pairs when those fit one wave (8B: 112
      // pair CTAs; two accumulators share every X stage); else 128-row tiles
      // (32B: 432 tiles in 2.9 waves beat 216 256-row tiles in 1.5 waves:
      // T=896 591 -> 461 us, T=128 131 -> 125 us; bit-identical per token)
      static const bool gu_pair = [] {   // CTA pairs (cta_group::2) for the 256-row SwiGLU
        const char* v = getenv("SPECTRE_GU_PAIR");   // tiles: half the token tile per CTA,
        return v ? atoi(v) != 0 : true;              // measured 68.7 -> 66.4 us (bit-identical)
      }();
      // large verify batches (rows_cap >= kLargeT): CTA pairs over (tile pair,
      // 256-token chunk) units on every SM, neighbouring pairs on the same
      // tiles (isolated, L2 flushed: 8B T=1280 279.5 -> 207.9 us, 32B T=896
      // 457.8 (128-row tiles) -> 398.3 us; T=320 109.6 -> 113.6, so not below)
      const bool pair_units = gu_pair && !half_gemm && (2 * F / 256) % 2 == 0 &&
                              down_pu;
      const bool pair_fits = gu_pair && !half_gemm && (2 * F / 256) % 2 == 0 &&
                             2 * F / 256 <= gemm_sk_grid();
      const bool gu128 = !pair_units && ((2 * F) / 128 <= gemm_sk_grid() || !pair_fits);
      TRY(gemm_plan(&pgu[l], bf(w.wgu) + (size_t)l * 2 * F * d, 2 * F, d, x, rows_cap, kSwiGLU,
                    1, 0, 0, gu128 ? 128 : 256));
      TRY(gemm_plan(&pd[l], bf(w.wd) + (size_t)l * d * F, d, F, act, rows_cap, kPartial, sp_d,
                    0, 0, tr_d));
      if (pair_units) TRY(gemm_set_pair_units(&pgu[l]));
      else if (pair_fits && !gu128) TRY(gemm_set_pair(&pgu[l]));
      if (down_pu) {
        TRY(pair_q ? gemm_set_pair_units(&pq[l]) : gemm_set_pass_units(&pq[l], 256));
        TRY(pair_o ? gemm_set_pair_units(&po[l]) : gemm_set_pass_units(&po[l], 256));
        TRY(pair_d ? gemm_set_pair_units(&pd[l]) : gemm_set_pass_units(&pd[l], 256));
      }
      if (half_gemm) {
        // partial GEMMs only: the SwiGLU GEMM measured faster in the full config
        for (GemmPlan* p : {&pq[l], &po[l], &pd[l]}) TRY(gemm_set_half(p));
      }
      for (GemmPlan* p : {&pq[l], &po[l], &pd[l]})
        TRY(gemm_set_outputs(p, part, nullptr, nullptr, nullptr, 0));
      TRY(gemm_set_outputs(&pgu[l], nullptr, nullptr, nullptr, act, F));
      for (GemmPlan* p : {&pq[l], &po[l], &pgu[l], &pd[l]}) p->args.t_dev = bt.t_dev;
    }
    if (sampling && !use_chain && !half_gemm && rows_cap >= kLargeT) {
      pqL.resize(L);
      poL.resize(L);
      pdL.resize(L);
      for (int l = 0; l < L; ++l) {
        TRY(gemm_plan(&pqL[l], bf(w.wqkv) + (size_t)l * nqkv() * d, nqkv(), d, x, rows_cap,
                      kPartial, kSpLqkv, 0, 0, 128));
        TRY(gemm_plan(&poL[l], bf(w.wo) + (size_t)l * d * qd, d, qd, attn, rows_cap, kPartial,
                      kSpLo, 0, 0, 128));
        // down: the normal plan's CTA-pair units where they apply (8B T=1280 in
        // context: 107.4 -> 102.4 us), else 128-row units in kSpLd splits
        TRY(gemm_plan(&pdL[l], bf(w.wd) + (size_t)l * d * F, d, F, act, rows_cap, kPartial,
                      pair_d ? sp_d : kSpLd, 0, 0, pair_d ? 256 : 128));
        TRY(pair_d ? gemm_set_pair_units(&pdL[l]) : gemm_set_pass_units(&pdL[l], 256));
        for (GemmPlan* p : {&pqL[l], &poL[l], &pdL[l]}) {
          if (p != &pdL[l]) TRY(gemm_set_pass_units(p, 256));
          TRY(gemm_set_outputs(p, part, nullptr, nullptr, nullptr, 0));
          p->args.t_dev = bt.t_dev;
        }
      }
    }
    if (sampling) {   // materialise fp32 logits (one split) for the samplers
      // large verify batches (config 3: ~1,280 rows): 128-row tiles balance
      // better (1,490 -> 1,351 us at T = 1,280)
      TRY(gemm_plan(&plm, w.lm_head, dm.vocab, d, x, rows_cap, kPartial, 1, 0, 0,
                    !pqL.empty() ? 128 : 256));
      TRY(gemm_set_outputs(&plm, logits, nullptr, nullptr, nullptr, 0));
    } else {
      // whole tiles per CTA (no stream-K): logits independent of the CTA
      // budget.  256-row tiles (128-row neutral at T=256); for large verify
      // batches CTA-pair units where the 256-row tiles pair up (Qwen2.5-32B,
      // 594 tiles, T=896 isolated: 1,413 -> 1,312 us), else 128-row tiles
      // (1,558 -> 1,427 us); argmax over full-K logits is exact either way
      const bool lm_pair = down_pu && pair_d && (dm.vocab % 512) == 0;
      TRY(gemm_plan(&plm, w.lm_head, dm.vocab, d, x, rows_cap, kArgmax, 1, 0, 0,
                    down_pu && !lm_pair ? 128 : 256));
      if (lm_pair) TRY(gemm_set_pair_units(&plm));
      TRY(gemm_set_outputs(&plm, nullptr, amax_v, amax_i, nullptr, 0));
    }
    const uint64_t kv_rows = (uint64_t)L * n_req * dm.n_kv_heads * ctx_cap;
    TRY(make_tmap_bf16(&tm_k32, w.k_cache, dm.head_dim, kv_rows, 32, 64));
    TRY(make_tmap_bf16(&tm_v32, w.v_cache, dm.head_dim, kv_rows, 32, 64));
    plm.args.t_dev = bt.t_dev;
    if (use_chain) TRY(plan_chains());
    return SPECTRE_OK;
  }

  int plan_chains() {
    const int d = dm.d_model, L = dm.n_layers, qd = dm.n_q_heads * dm.head_dim, F = dm.ffn;
    auto bf = [](const void* p) { return reinterpret_cast<const __nv_bfloat16*>(p); };
    const size_t kv_layer = (size_t)n_req * dm.n_kv_heads * ctx_cap * dm.head_dim;
    auto* kc = reinterpret_cast<__nv_bfloat16*>(w.k_cache);
    auto* vc = reinterpret_cast<__nv_bfloat16*>(w.v_cache);
    int chain_idx = 0;
    auto model = [&](int rope_layer, int pre_wait) {
      ChainModel m{};
      m.dbg = ch_dbg ? ch_dbg + 64 * chain_idx++ : nullptr;
      m.rows_cap = rows_cap;
      m.d = d;
      m.n_q = dm.n_q_heads;
      m.n_kv = dm.n_kv_heads;
      m.hd = dm.head_dim;
      m.ctx_cap = ctx_cap;
      m.eps = dm.rms_eps;
      m.t_dev = bt.t_dev;
      m.tok = bt.tok;
      m.embed = w.embed;
      m.h = h;
      m.x = x;
      m.tok_pos = bt.pos;
      m.tok_slot = bt.slot;
      m.rope = rope;
      m.q = q;
      m.kc = rope_layer >= 0 ? kc + rope_layer * kv_layer : nullptr;
      m.vc = rope_layer >= 0 ? vc + rope_layer * kv_layer : nullptr;
      m.part = part;
      m.bar = ch_bar;
      m.t_pre_wait = pre_wait;
      return m;
    };
    auto add_qkv_rope = [&](void* c, int l) {
      TRY(chain_add_gemm(c, bf(w.wqkv) + (size_t)l * nqkv() * d, nqkv(), d, x, rows_cap,
                         kPhGemmPartial, part, nullptr));
      TRY(chain_add_glue(c, kPhRope, nullptr));
      return SPECTRE_OK;
    };
    auto add_mlp_block = [&](void* c, int l) {
      TRY(chain_add_gemm(c, bf(w.wo) + (size_t)l * d * qd, d, qd, attn, rows_cap, kPhGemmPartial,
                         part, nullptr));
      TRY(chain_add_glue(c, kPhResid, w.mlp_norm + (size_t)l * d));
      TRY(chain_add_gemm(c, bf(w.wgu) + (size_t)l * 2 * F * d, 2 * F, d, x, rows_cap,
                         kPhGemmSwiGLU, nullptr, act));
      TRY(chain_add_gemm(c, bf(w.wd) + (size_t)l * d * F, d, F, act, rows_cap, kPhGemmPartial,
                         part, nullptr));
      TRY(chain_add_glue(c, kPhResid,
                         l + 1 < L ? w.attn_norm + (size_t)(l + 1) * d : w.final_norm));
      return SPECTRE_OK;
    };
    ch_first = chain_alloc();
    TRY(chain_add_glue(ch_first, kPhEmbed, w.attn_norm));
    TRY(add_qkv_rope(ch_first, 0));
    TRY(chain_set_model(ch_first, model(0, 0)));   // follows the batch kernel directly
    for (int l = 0; l + 1 < L; ++l) {
      void* c = chain_alloc();
      ch_mid.push_back(c);
      TRY(add_mlp_block(c, l));
      TRY(add_qkv_rope(c, l + 1));
      TRY(chain_set_model(c, model(l + 1, 1)));
    }
    ch_last = chain_alloc();
    TRY(add_mlp_block(ch_last, L - 1));
    TRY(chain_set_model(ch_last, model(-1, 1)));
    return SPECTRE_OK;
  }

  // One forward pass over the packed batch in `bt`; `new_per_req` bounds
  // n_new[b] (sizes the attention row blocks).
  // sample_rows: in sampling mode also draw a token for every row (target
  // verify / prefill); the draft's decode steps sample per request instead.
  // head = false: stop after the last layer's residual (prefill chunks whose
  // next-token prediction nobody reads)
  // t_typical (> 0): the rows the step usually carries, when far below the
  // bound (the draft's first step of a round: 1-2 catch-up tokens per request,
  // bounded by the longest possible catch-up); picks the chains' MMA pass width
  // (a pass narrower than T stays correct, it streams the weights once per pass)
  int forward(int new_per_req, cudaStream_t s, void* out_x = nullptr, bool sample_rows = true,
              bool head = true, int t_typical = 0) {
    const int d = dm.d_model, L = dm.n_layers, hd = dm.head_dim;
    const float eps = dm.rms_eps;
    const int rows = new_per_req * group();
    AttnArgs a{};
    a.q = q;
    a.q_off = bt.q_off;
    a.n_new = bt.n_new;
    a.pos0 = bt.pos0;
    a.slot = bt.rslot;
    a.n_req = n_req;
    a.n_q = dm.n_q_heads;
    a.n_kv = dm.n_kv_heads;
    a.ctx_cap = ctx_cap;
    a.rb_max = (rows + 15) / 16;
    if (a.rb_max > rb_cap) return arg_fail("forward: rows per request exceed capacity");
    a.split_max = split_max;
    a.chunk = attn_chunk;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
    static const int attn_debug = [] {   // diagnostics (timing only), read once
      const char* v = getenv("SPECTRE_ATTN_DEBUG");
      return v ? atoi(v) : 0;
    }();
    a.debug = attn_debug;
    a.part_o = att_o;
    a.part_ml = att_ml;
    a.done_cnt = att_cnt;
    a.out = attn;
    const size_t kv_layer = (size_t)n_req * dm.n_kv_heads * ctx_cap * hd;
    auto* kc = reinterpret_cast<__nv_bfloat16*>(w.k_cache);
    auto* vc = reinterpret_cast<__nv_bfloat16*>(w.v_cache);
    if (use_chain) {
      int t_bound = std::min(rows_cap, n_req * new_per_req);
      if (t_typical > 0) t_bound = std::min(t_bound, t_typical);
      TRY(chain_launch(ch_first, s, t_bound));
      for (int l = 0; l < L; ++l) {
        a.layer_row0 = l * n_req * dm.n_kv_heads * ctx_cap;
        TRY(launch_attention_w(tm_k32, tm_v32, a, hd, rows, s));
        TRY(chain_launch(l + 1 < L ? ch_mid[l] : ch_last, s, t_bound));
      }
    }
    if (!use_chain) TRY(launch_embed_rmsnorm(bt.tok, bt.t_dev, rows_cap, w.embed, w.attn_norm, h,
                                             x, d, eps, s));
    const bool large = !pqL.empty() && n_req * new_per_req >= kLargeT;
    const int s_qkv = large ? kSpLqkv : sp_qkv, s_o = large ? kSpLo : sp_o,
              s_d = large && !pair_d ? kSpLd : sp_d;
    for (int l = 0; l < L && !use_chain; ++l) {
      TRY(gemm_run(large ? pqL[l] : pq[l], s));
      TRY(launch_qkv_rope_kv(part, s_qkv, rows_cap, bt.t_dev, rows_cap, bt.pos, bt.slot,
                               rope, q, kc + l * kv_layer, vc + l * kv_layer, dm.n_q_heads,
                               dm.n_kv_heads, hd, ctx_cap, s));
      a.layer_row0 = l * n_req * dm.n_kv_heads * ctx_cap;
      TRY(launch_attention_w(tm_k32, tm_v32, a, hd, rows, s));
      TRY(gemm_run(large ? poL[l] : po[l], s));
      TRY(launch_residual_rmsnorm(part, s_o, rows_cap, bt.t_dev, rows_cap,
                                    w.mlp_norm + (size_t)l * d, h, x, d, eps, s));
      TRY(gemm_run(pgu[l], s));
      TRY(gemm_run(large ? pdL[l] : pd[l], s));
      const float* next = (l + 1 < L) ? w.attn_norm + (size_t)(l + 1) * d : w.final_norm;
      TRY(launch_residual_rmsnorm(part, s_d, rows_cap, bt.t_dev, rows_cap, next, h, x, d, eps,
                                    s));
    }
    if (!head) {
      if (out_x)
        SPECTRE_CUDA_TRY(cudaMemcpyAsync(out_x, x, (size_t)rows_cap * d * 2,
                                         cudaMemcpyDeviceToDevice, s));
      return SPECTRE_OK;
    }
    TRY(gemm_run(plm, s));
    if (sampling) {
      if (sample_rows)
        TRY(launch_sample_rows(logits, dm.vocab, bt, rows_cap, inv_t, seed, lstat, s));
    } else {
      TRY(launch_argmax_reduce(amax_v, amax_i, (plm.grid) * 8, rows_cap, bt.t_dev, rows_cap,
                               bt.out_tok, nullptr, s));
    }
    if (out_x)
      SPECTRE_CUDA_TRY(cudaMemcpyAsync(out_x, x, (size_t)rows_cap * d * 2,
                                       cudaMemcpyDeviceToDevice, s));
    return SPECTRE_OK;
  }
};

// ------------------------------------------------------------------- engine
struct Engine {
  SpectreDecodeConfig cfg{};
  ModelRT tgt, drf;
  DecodeStateDev st{};
  int prefill_cs = 1;
  int draft_new_max = 1;
  cudaStream_t s_draft = nullptr, s_cap = nullptr, s_main = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t exec_loop = nullptr;
  cudaGraph_t graph_loop = nullptr;
  int graph_failed = 0;
  int* mode_host = nullptr;  // pinned
  int warmed = 0;
  int device = 0;
  int attached = 0;           // layout-only view of a peer process's engine (IPC)
  cudaStream_t s_cap2 = nullptr;
  // rejection sampling (temperature > 0): draft q-store by output position
  int qwin = 0;               // slots per request (positions mod qwin)
  float* qstore = nullptr;    // [n_req][qwin][vocab] draft logits
  float2* qstat = nullptr;    // [n_req][qwin] (max, sum exp)
  int* dprompts = nullptr;    // [n_req][dprompt_len] compressed prompts (draft side)

  ~Engine() {
    if (exec_loop) cudaGraphExecDestroy(exec_loop);
    if (graph_loop) cudaGraphDestroy(graph_loop);
    if (s_draft) cudaStreamDestroy(s_draft);
    if (s_cap) cudaStreamDestroy(s_cap);
    if (s_cap2) cudaStreamDestroy(s_cap2);
    if (s_main) cudaStreamDestroy(s_main);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (mode_host) cudaFreeHost(mode_host);
  }

  static void sizes(const SpectreModelDims& t, const SpectreModelDims& d,
                    const SpectreDecodeConfig& c, int* rows_t, int* rows_d, int* cs, int* dnew) {
    *cs = prefill_chunk(c.n_req);
    *dnew = 2 * c.gamma + 4;
    *rows_t = round_up(std::max(c.n_req * (c.gamma + 1), c.n_req * *cs), 64);
    const int nd = c.n_req + std::max(0, c.background_requests);   // + background entries
    *rows_d = round_up(std::max(c.n_req * *dnew + nd - c.n_req, nd * *cs), 64);
  }

  void layout(Bump& b) {
    const int n = cfg.n_req, G = cfg.gamma + 1;
    tgt.layout(b);
    drf.layout(b);
    st.pos = b.take<int>(n);
    st.done = b.take<int>(n);
    st.synced = b.take<int>(n);
    st.cached_len = b.take<int>(n);
    st.cached_start = b.take<int>(n);
    st.in_rollback = b.take<int>(n);
    st.hist_len = b.take<int>(n);
    st.kvd = b.take<int>(n);
    st.gen_count = b.take<int>(n);
    st.gen_done = b.take<int>(n);
    st.gen_start = b.take<int>(n);
    st.vkind = b.take<int>(n);
    st.vcand_n = b.take<int>(n);
    st.delta = b.take<int>(n);
    st.rolled = b.take<int>(n);
    st.req_mode = b.take<int>(n);
    st.q_round = b.take<int>(n);
    st.q_serial = b.take<int>(n);
    st.r_round = b.take<int>(n);
    st.r_serial = b.take<int>(n);
    st.committed = b.take<uint64_t>((size_t)n * cfg.output_len);
    st.hist = b.take<uint64_t>((size_t)n * st.hist_cap);
    st.cached_tok = b.take<uint64_t>((size_t)n * G);
    st.cand_tok = b.take<uint64_t>((size_t)n * G);
    if (st.dprompt_len < cfg.prompt_len || st.n_bg > 0)
      dprompts = b.take<int>((size_t)(n + st.n_bg) * st.dprompt_len);
    if (st.n_bg > 0) {
      const int nb = st.n_bg;
      st.bg_remaining = b.take<int>(nb);
      st.bg_ctx = b.take<int>(nb);
      st.bg_last = b.take<int>(nb);
      st.bg_emitted = b.take<int>(nb);
      st.bg_round_left = b.take<int>(nb);
      st.bg_out = b.take<int>((size_t)nb * st.bg_out_len);
    }
    st.ctrl = b.take<CtrlDev>(1);
    const int R = cfg.max_rounds;
    st.trace.mode = b.take<int>(R);
    st.trace.participants = b.take<int>(R);
    st.trace.delta = b.take<int>(R);
    st.trace.n_roll = b.take<int>(R);
    st.trace.content_sum = b.take<int>(R);
    st.trace.content_n = b.take<int>(R);
    st.trace.n_padded = b.take<int>(R);
    st.trace.t_round_ns = b.take<long long>(R);
    st.trace.t_verify_ns = b.take<long long>(R);
    st.trace.t_draft_ns = b.take<long long>(R);
    st.trace.r_hat_ema = b.take<double>(R);
    st.trace.accepted_len_ema = b.take<double>(R);
    st.trace.r_star = b.take<double>(R);
    st.trace.n_stale = b.take<int>(R);
    st.trace.n_regular = b.take<int>(R);
    st.trace.n_forced = b.take<int>(R);
    st.trace.fair_counter = b.take<int>(R);
    st.trace.timeout = b.take<int>(R);
    if (st.sampling) {
      st.samp_a = b.take<int>(n);
      st.samp_bonus = b.take<int>(n);
      qstore = b.take<float>((size_t)n * qwin * drf.dm.vocab);
      qstat = b.take<float2>((size_t)n * qwin);
    }
  }

  void configure(const SpectreModelDims& t, const SpectreModelWeights& tw,
                 const SpectreModelDims& d, const SpectreModelWeights& dw,
                 const SpectreDecodeConfig& c) {
    cfg = c;
    int rt, rd;
    sizes(t, d, c, &rt, &rd, &prefill_cs, &draft_new_max);
    tgt.dm = t;
    tgt.w = tw;
    tgt.n_req = c.n_req;
    tgt.rows_cap = rt;
    tgt.ctx_cap = c.ctx_cap;
    tgt.max_new = std::max(c.gamma + 1, prefill_cs);
    drf.dm = d;
    drf.w = dw;
    drf.n_req = c.n_req + std::max(0, c.background_requests);   // KV slots n_req.. : background
    drf.rows_cap = rd;
    drf.ctx_cap = c.ctx_cap;
    drf.max_new = std::max(draft_new_max, prefill_cs);
    drf.tile_rows = tile_rows_default(256);
    drf.half_gemm = [] {
      const char* v = getenv("SPECTRE_DRAFT_HALF");
      return v ? atoi(v) != 0 : true;
    }();
    // the draft's forwards as persistent chains (SPECTRE_DRAFT_CHAIN=0: per-op kernels)
    drf.use_chain = [&] {
      const char* v = getenv("SPECTRE_DRAFT_CHAIN");
      const bool on = v ? atoi(v) != 0 : true;
      const int qd = d.n_q_heads * d.head_dim, nq = (d.n_q_heads + 2 * d.n_kv_heads) * d.head_dim;
      return on && d.d_model % 128 == 0 && nq % 128 == 0 && (2 * d.ffn) % 128 == 0 &&
             qd % 64 == 0 && d.ffn % 64 == 0 && d.d_model <= 2048;
    }();
    tgt.tile_rows = tile_rows_default(256);
    st.n_req = c.n_req;
    st.gamma = c.gamma;
    st.out_len = c.output_len;
    st.prompt_len = c.prompt_len;
    st.dprompt_len = (c.draft_prompt_keep > 0 && 2 * c.draft_prompt_keep < c.prompt_len)
                         ? 2 * c.draft_prompt_keep : c.prompt_len;
    st.n_bg = std::max(0, c.background_requests);
    st.bg_out_len = c.background_output_len > 0 ? c.background_output_len : 128;
    st.fair_period = c.fairness_period > 0 ? c.fairness_period : 10;
    st.draft_cap = c.draft_capacity > 0 ? c.draft_capacity : 256;
    st.vocab = d.vocab;
    st.variant = c.variant;
    st.controller = c.controller;
    st.r_kind = c.r_kind;
    st.max_rounds = c.max_rounds;
    st.has_fixed_l = c.has_fixed_l;
    st.hist_cap = c.ctx_cap - c.prompt_len;
    st.seed = c.seed;
    st.alpha = c.alpha;
    st.alpha_switch = c.alpha_switch_pos > 0 ? c.alpha_switch_pos : 0x7fffffff;
    st.alpha_late = c.alpha_switch_pos > 0 ? c.alpha_late : c.alpha;
    st.t_target = c.t_target;
    st.t_draft = c.t_draft;
    st.ema_decay = c.ema_decay;
    st.fixed_l = c.fixed_threshold_l;
    st.use_handles = 0;
    st.sampling = c.temperature > 0.0 ? 1 : 0;
    st.breaker_threshold = c.breaker_threshold > 0 ? c.breaker_threshold : 3;
    st.breaker_cooldown = c.breaker_cooldown > 0 ? c.breaker_cooldown : 5;
    st.timeout_lag = c.reply_timeout_rounds > 0 ? c.reply_timeout_rounds - 1 : 1;
    qwin = 4 * c.gamma + 4;   // > every candidate-to-speculation position gap
    for (ModelRT* m : {&tgt, &drf}) {
      m->sampling = st.sampling;
      m->inv_t = st.sampling ? (float)(1.0 / c.temperature) : 1.f;
      m->seed = c.seed;
    }
  }

  // ---- round pieces
  int draft_phase(int which, cudaStream_t s) {
    if (st.n_bg > 0) {   // a forced regular round (regular items only, one step), if due
      TRY(launch_bg_forced_prep(st, drf.bt, which, s));
      TRY(drf.forward(1, s, nullptr, false));
      TRY(launch_bg_forced_append(st, drf.bt, s));
    }
    TRY(launch_draft_prep(st, drf.bt, which, s));
    const int steps = which == 'O' ? cfg.gamma - 1 : cfg.gamma;   // 'M': the longest query
    for (int i = 0; i < steps; ++i) {
      TRY(drf.forward(i == 0 ? draft_new_max : 1, s, nullptr, false, true,
                      i == 0 ? 2 * drf.n_req : 0));
      if (st.sampling)
        TRY(launch_draft_sample(st, drf.bt, drf.logits, drf.dm.vocab, drf.inv_t, qstore, qstat,
                                qwin, s));
      TRY(launch_draft_append(st, drf.bt, which, i == steps - 1, s));
    }
    return SPECTRE_OK;
  }
  int verify_phase(cudaStream_t s) {
    TRY(launch_verify_prep(st, tgt.bt, s));
    TRY(tgt.forward(cfg.gamma + 1, s));
    return SPECTRE_OK;
  }

  int round_eager(cudaStream_t s, int* mode_out) {
    TRY(launch_round_begin(st, s));
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(mode_host, &st.ctrl->mode, sizeof(int),
                                     cudaMemcpyDeviceToHost, s));
    SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
    const int mode = *mode_host;
    *mode_out = mode;
    if (mode == 0) return SPECTRE_OK;
    if (mode == 'O') TRY(draft_phase('O', s));
    if (mode == 'P') {
      TRY(parallel_phase(s, s_draft));
    } else {
      TRY(verify_phase(s));
    }
    TRY(accept(s));
    return SPECTRE_OK;
  }

  // draft speculation on `sd` concurrent with the verify on `s` (disjoint CTA
  // budgets for the two measured slower: both phases share HBM bandwidth)
  int parallel_phase(cudaStream_t s, cudaStream_t sd) {
    SPECTRE_CUDA_TRY(cudaEventRecord(ev_fork, s));
    SPECTRE_CUDA_TRY(cudaStreamWaitEvent(sd, ev_fork, 0));
    TRY(draft_phase('P', sd));
    SPECTRE_CUDA_TRY(cudaEventRecord(ev_join, sd));
    TRY(verify_phase(s));
    SPECTRE_CUDA_TRY(cudaStreamWaitEvent(s, ev_join, 0));
    return SPECTRE_OK;
  }

  int accept(cudaStream_t s) {
    if (st.sampling)
      TRY(launch_accept_sample(st, tgt.bt, tgt.logits, tgt.dm.vocab, tgt.inv_t, tgt.lstat, qstore,
                               qstat, qwin, st.samp_a, st.samp_bonus, s));
    return launch_accept(st, tgt.bt, s);
  }

  // Capture a conditional IF node at the current capture point of `s`, with
  // its body captured from `fn` on the helper capture stream.
  template <class Fn>
  int add_if_node(cudaStream_t s, cudaGraphConditionalHandle hnd, Fn fn, bool update_deps,
                  cudaGraphNode_t* node_out) {
    cudaStreamCaptureStatus status;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    SPECTRE_CUDA_TRY(cudaStreamGetCaptureInfo(s, &status, nullptr, &g, &deps, &ndeps));
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hnd;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    SPECTRE_CUDA_TRY(cudaGraphAddNode(&node, g, deps, ndeps, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    SPECTRE_CUDA_TRY(cudaStreamBeginCaptureToGraph(s_cap, body, nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeRelaxed));
    int r = fn(s_cap);
    cudaGraph_t out;
    cudaError_t e = cudaStreamEndCapture(s_cap, &out);
    if (r) return r;
    SPECTRE_CUDA_TRY(e);
    if (update_deps)
      SPECTRE_CUDA_TRY(
          cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    *node_out = node;
    return SPECTRE_OK;
  }

  int build_loop_graph(cudaStream_t s) {
    cudaGraph_t g = nullptr;
    DecodeStateDev saved = st;
    int r = SPECTRE_OK;
    bool capturing = false;
    auto fail = [&](cudaError_t e, const char* what) {
      if (!r) r = cuda_fail(e, what);
    };
    do {
      cudaError_t e = cudaGraphCreate(&g, 0);
      if (e != cudaSuccess) { fail(e, "cudaGraphCreate"); break; }
      cudaGraphConditionalHandle h_loop, h_ord, h_par, h_ar;
      if ((e = cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault)) ||
          (e = cudaGraphConditionalHandleCreate(&h_ord, g, 0, cudaGraphCondAssignDefault)) ||
          (e = cudaGraphConditionalHandleCreate(&h_par, g, 0, cudaGraphCondAssignDefault)) ||
          (e = cudaGraphConditionalHandleCreate(&h_ar, g, 0, cudaGraphCondAssignDefault))) {
        fail(e, "cudaGraphConditionalHandleCreate");
        break;
      }
      cudaGraphNodeParams wp{};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h_loop;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      cudaGraphNode_t wnode;
      if ((e = cudaGraphAddNode(&wnode, g, nullptr, 0, &wp))) { fail(e, "cudaGraphAddNode(while)"); break; }
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      st.h_loop = h_loop;
      st.h_ord = h_ord;
      st.h_par = h_par;
      st.h_ar = h_ar;
      st.use_handles = 1;
      if ((e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed))) {
        fail(e, "cudaStreamBeginCaptureToGraph");
        break;
      }
      capturing = true;
      if ((r = launch_round_begin(st, s))) break;
      cudaGraphNode_t n_if[3];
      // the three mode bodies hang off round_begin; exactly one runs
      if ((r = add_if_node(s, h_ord, [&](cudaStream_t cs) {
             if (int q = draft_phase('O', cs)) return q;
             return verify_phase(cs);
           }, false, &n_if[0])))
        break;
      if ((r = add_if_node(s, h_par, [&](cudaStream_t cs) { return parallel_phase(cs, s_cap2); },
                           false, &n_if[1])))
        break;
      if ((r = add_if_node(s, h_ar, [&](cudaStream_t cs) { return verify_phase(cs); }, false,
                           &n_if[2])))
        break;
      if ((e = cudaStreamUpdateCaptureDependencies(s, n_if, 3,
                                                   cudaStreamSetCaptureDependencies))) {
        fail(e, "cudaStreamUpdateCaptureDependencies");
        break;
      }
      if ((r = accept(s))) break;
    } while (0);
    if (capturing) {
      cudaGraph_t captured;
      cudaError_t e = cudaStreamEndCapture(s, &captured);
      if (e != cudaSuccess) fail(e, "cudaStreamEndCapture(loop body)");
    }
    if (!r) {
      cudaError_t e = cudaGraphInstantiate(&exec_loop, g, 0);
      if (e != cudaSuccess) fail(e, "cudaGraphInstantiate(loop)");
    }
    if (r) {
      if (g) cudaGraphDestroy(g);
      st = saved;
      exec_loop = nullptr;
      cudaGetLastError();
      return r;
    }
    graph_loop = g;
    // the graph captured its own copy of the state with the conditional
    // handles; eager rounds / host-driven steps launched later from `st`
    // must not call cudaGraphSetConditional outside the graph
    st.use_handles = 0;
    return SPECTRE_OK;
  }
};

}  // namespace spectre

using namespace spectre;

static bool dims_ok(const SpectreModelDims* m) {
  return m && m->d_model % 64 == 0 && m->n_layers > 0 && m->n_kv_heads > 0 &&
         m->n_q_heads % m->n_kv_heads == 0 && (m->head_dim == 64 || m->head_dim == 128) &&
         m->ffn % 64 == 0 && m->vocab > 1 && (m->n_q_heads * m->head_dim) % 64 == 0;
}

extern "C" size_t spectre_engine_workspace_bytes(const SpectreModelDims* target,
                                                 const SpectreModelDims* draft,
                                                 const SpectreDecodeConfig* cfg) {
  if (!dims_ok(target) || !dims_ok(draft) || !cfg) return 0;
  Engine e;
  e.configure(*target, SpectreModelWeights{}, *draft, SpectreModelWeights{}, *cfg);
  Bump b{nullptr};
  e.layout(b);
  return b.off + 1024;
}

extern "C" void* spectre_engine_create(const SpectreModelDims* target,
                                       const SpectreModelWeights* tw,
                                       const SpectreModelDims* draft,
                                       const SpectreModelWeights* dw,
                                       const SpectreDecodeConfig* cfg, void* workspace,
                                       size_t workspace_bytes) {
  if (!dims_ok(target) || !dims_ok(draft) || !tw || !dw || !cfg || !workspace) {
    arg_fail("spectre_engine_create: dims / pointers");
    return nullptr;
  }
  if (cfg->role < SPECTRE_ROLE_BOTH || cfg->role > SPECTRE_ROLE_DRAFT) {
    arg_fail("spectre_engine_create: role");
    return nullptr;
  }
  if (cfg->n_req < 1 || cfg->n_req > 1024 || cfg->gamma < 1 || cfg->gamma > 16 ||
      cfg->output_len < 2 || cfg->prompt_len < 1 || cfg->max_rounds < 1 ||
      cfg->ctx_cap < cfg->prompt_len + cfg->output_len + 4 * cfg->gamma + 16 ||
      target->vocab != draft->vocab) {
    arg_fail("spectre_engine_create: decode config");
    return nullptr;
  }
  if (cfg->background_requests > 0 &&
      (cfg->role != SPECTRE_ROLE_BOTH || cfg->temperature > 0.0 ||
       (cfg->draft_capacity > 0 ? cfg->draft_capacity : 256) < cfg->n_req ||
       cfg->n_req + cfg->background_requests > 1024 ||
       cfg->prompt_len + (cfg->background_output_len > 0 ? cfg->background_output_len : 128) + 8 >
           cfg->ctx_cap)) {
    arg_fail("spectre_engine_create: background tenants need role both, greedy decoding, "
             "draft_capacity >= n_req, n_req + background <= 1024 and KV room for their output");
    return nullptr;
  }
  if (cfg->temperature > 0.0 &&
      (cfg->alpha < 1.0 || (cfg->alpha_switch_pos > 0 && cfg->alpha_late < 1.0))) {
    // rejection sampling tests min(1, p/q) against the draft's q; the alpha
    // noise would replace the proposal by a token not drawn from q
    arg_fail("spectre_engine_create: temperature > 0 needs alpha == 1 (no draft noise)");
    return nullptr;
  }
  auto e = std::make_unique<Engine>();
  e->configure(*target, *tw, *draft, *dw, *cfg);
  Bump b{reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255))};
  e->layout(b);
  if (b.off + 256 > workspace_bytes) {
    arg_fail("spectre_engine_create: workspace too small");
    return nullptr;
  }
  if ((cfg->role != SPECTRE_ROLE_DRAFT && e->tgt.plan()) ||
      (cfg->role != SPECTRE_ROLE_TARGET && e->drf.plan()))
    return nullptr;
  cudaGetDevice(&e->device);
  if (cudaStreamCreateWithFlags(&e->s_draft, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->s_main, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->s_cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->s_cap2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaMallocHost(&e->mode_host, sizeof(int)) != cudaSuccess) {
    cuda_fail(cudaGetLastError(), "spectre_engine_create: streams");
    return nullptr;
  }
  if (launch_rope_table(e->tgt.rope, cfg->ctx_cap, target->head_dim, target->rope_theta,
                        nullptr) ||
      launch_rope_table(e->drf.rope, cfg->ctx_cap, draft->head_dim, draft->rope_theta, nullptr))
    return nullptr;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cuda_fail(cudaGetLastError(), "spectre_engine_create: init");
    return nullptr;
  }
  return e.release();
}

extern "C" int spectre_engine_destroy(void* engine) {
  delete reinterpret_cast<Engine*>(engine);
  return SPECTRE_OK;
}

extern "C" int spectre_engine_prefill(void* engine, const int32_t* prompts, void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || !prompts || e->attached) return arg_fail("spectre_engine_prefill");
  cudaStream_t s = as_stream(stream);
  const int cs = e->prefill_cs;
  for (ModelRT* m : {&e->drf, &e->tgt}) {
    if ((m == &e->drf && e->cfg.role == SPECTRE_ROLE_TARGET) ||
        (m == &e->tgt && e->cfg.role == SPECTRE_ROLE_DRAFT))
      continue;   // disaggregated: this side holds only one model
    // the draft prefills its prompt view: the (possibly compressed) prompts,
    // then the background requests' prompts
    const int* src = prompts;
    int P = e->cfg.prompt_len;
    if (m == &e->drf && e->dprompts) {
      if (e->st.dprompt_len < P)
        TRY(launch_compress_prompts(prompts, P, e->cfg.draft_prompt_keep, e->cfg.n_req,
                                    e->dprompts, s));
      else
        SPECTRE_CUDA_TRY(cudaMemcpyAsync(e->dprompts, prompts, (size_t)e->cfg.n_req * P * 4,
                                         cudaMemcpyDeviceToDevice, s));
      src = e->dprompts;
      P = e->st.dprompt_len;
      TRY(launch_bg_prompts(e->cfg.seed, e->cfg.n_req, e->st.n_bg, P, e->drf.dm.vocab,
                            e->dprompts, s));
    }
    for (int c0 = 0; c0 < P; c0 += cs) {
      TRY(launch_prefill_batch(src, P, m->n_req, c0, cs, m->bt, s));
      // only the target's prediction at the last prompt position is read
      // (admission commits it as output token 0)
      TRY(m->forward(cs, s, nullptr, true, m == &e->tgt && c0 + cs >= P));
    }
  }
  TRY(launch_admit(e->st, e->tgt.bt, s));
  if (e->cfg.role == SPECTRE_ROLE_BOTH) TRY(launch_bg_init(e->st, e->dprompts, e->st.dprompt_len, s));
  return SPECTRE_OK;
}

extern "C" int spectre_engine_run(void* engine, int32_t max_rounds, int32_t use_graph,
                                  int32_t* rounds_run, void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || max_rounds < 0 || e->attached) return arg_fail("spectre_engine_run");
  cudaStream_t caller = as_stream(stream);
  cudaStream_t s = e->s_main;  // capturable stream, ordered after the caller's work
  SPECTRE_CUDA_TRY(cudaEventRecord(e->ev_in, caller));
  SPECTRE_CUDA_TRY(cudaStreamWaitEvent(s, e->ev_in, 0));
  TRY(launch_set_round_limit(e->st, max_rounds, s));  // device-side budget, no host sync
  if (use_graph && !e->graph_failed) {
    if (!e->exec_loop) {
      if (!e->warmed) {
        // one eager round primes every kernel attribute outside capture
        int mode;
        TRY(e->round_eager(s, &mode));
        e->warmed = 1;
      }
      if (e->build_loop_graph(s)) e->graph_failed = 1;  // eager fallback, see last_error
    }
    if (e->exec_loop) SPECTRE_CUDA_TRY(cudaGraphLaunch(e->exec_loop, s));
  }
  if (!use_graph || e->graph_failed) {
    for (int i = 0; i < max_rounds + 1; ++i) {
      int mode;
      TRY(e->round_eager(s, &mode));
      if (mode == 0) break;
    }
  }
  SPECTRE_CUDA_TRY(cudaEventRecord(e->ev_out, s));
  SPECTRE_CUDA_TRY(cudaStreamWaitEvent(caller, e->ev_out, 0));
  if (rounds_run) {
    CtrlDev c;
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(&c, e->st.ctrl, sizeof(c), cudaMemcpyDeviceToHost, s));
    SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
    *rounds_run = c.round - c.round_base;
  }
  return SPECTRE_OK;
}

// Roofline timing (bench.py): launch the draft's mid-layer chains back to back
// `reps` times over the current draft batch (the step's row count; activations
// are whatever the buffers hold — the weight stream and the phase structure are
// those of a decode step).  Returns the number of chain launches issued;
// *weight_bytes = weight bytes one pass over the mid chains streams.
extern "C" int spectre_engine_launch_chains(void* engine, int32_t reps, int64_t* weight_bytes,
                                            void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || reps < 1 || !e->drf.use_chain || e->drf.ch_mid.empty())
    return arg_fail("spectre_engine_launch_chains: no draft chains");
  cudaStream_t s = as_stream(stream);
  const SpectreModelDims& d = e->drf.dm;
  const long long per_layer = (long long)d.d_model * d.n_q_heads * d.head_dim +
                              3ll * d.d_model * d.ffn +
                              (long long)(d.n_q_heads + 2 * d.n_kv_heads) * d.head_dim * d.d_model;
  if (weight_bytes) *weight_bytes = 2 * per_layer * (long long)e->drf.ch_mid.size();
  int n = 0;
  for (int r = 0; r < reps; ++r)
    for (void* c : e->drf.ch_mid) {
      TRY(chain_launch(c, s, e->drf.n_req));   // decode-shaped: one token per request
      ++n;
    }
  return n;
}

// Diagnostics: the draft chains' last per-phase globaltimer stamps (CTA 0),
// [n_layers + 1][64] u64 — only with SPECTRE_CHAIN_DBG set at engine creation.
extern "C" int spectre_engine_chain_stamps(void* engine, uint64_t* out, int32_t n) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || !out || !e->drf.ch_dbg) return arg_fail("spectre_engine_chain_stamps");
  const int have = (e->drf.dm.n_layers + 1) * 64;
  SPECTRE_CUDA_TRY(cudaMemcpy(out, e->drf.ch_dbg, (size_t)std::min(n, have) * 8,
                              cudaMemcpyDeviceToHost));
  return std::min(n, have);
}

extern "C" int spectre_engine_graph_status(void* engine) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e) return -1;
  return e->exec_loop ? 1 : (e->graph_failed ? 2 : 0);
}

extern "C" int spectre_engine_read(void* engine, int64_t* committed, int32_t* committed_pos,
                                   const SpectreRoundTrace* trace, int32_t* n_rounds,
                                   void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e) return arg_fail("spectre_engine_read");
  cudaStream_t s = as_stream(stream);
  const int n = e->cfg.n_req;
  if (committed)
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(committed, e->st.committed,
                                     (size_t)n * e->cfg.output_len * 8,
                                     cudaMemcpyDeviceToDevice, s));
  if (committed_pos)
    SPECTRE_CUDA_TRY(
        cudaMemcpyAsync(committed_pos, e->st.pos, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  CtrlDev c;
  SPECTRE_CUDA_TRY(cudaMemcpyAsync(&c, e->st.ctrl, sizeof(c), cudaMemcpyDeviceToHost, s));
  SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
  const int R = std::min(c.round, e->cfg.max_rounds);
  if (n_rounds) *n_rounds = R;
  if (c.error) {
    set_last_error("device protocol violation code " + std::to_string(c.error) +
                   " (request " + std::to_string(c.error_req) + ")");
    return SPECTRE_EINVAL;
  }
  if (trace && R > 0) {
    const RoundTraceDev& t = e->st.trace;
    auto cp = [&](void* dst, const void* src, size_t bytes) -> int {
      if (!dst) return 0;
      SPECTRE_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
      return 0;
    };
    TRY(cp(trace->mode, t.mode, R * 4));
    TRY(cp(trace->participants, t.participants, R * 4));
    TRY(cp(trace->delta, t.delta, R * 4));
    TRY(cp(trace->n_roll, t.n_roll, R * 4));
    TRY(cp(trace->content_sum, t.content_sum, R * 4));
    TRY(cp(trace->content_n, t.content_n, R * 4));
    TRY(cp(trace->n_padded, t.n_padded, R * 4));
    TRY(cp(trace->t_round_ns, t.t_round_ns, R * 8));
    TRY(cp(trace->t_verify_ns, t.t_verify_ns, R * 8));
    TRY(cp(trace->t_draft_ns, t.t_draft_ns, R * 8));
    TRY(cp(trace->r_hat_ema, t.r_hat_ema, R * 8));
    TRY(cp(trace->accepted_len_ema, t.accepted_len_ema, R * 8));
    TRY(cp(trace->r_star, t.r_star, R * 8));
    TRY(cp(trace->n_stale, t.n_stale, R * 4));
    TRY(cp(trace->n_regular, t.n_regular, R * 4));
    TRY(cp(trace->n_forced, t.n_forced, R * 4));
    TRY(cp(trace->fair_counter, t.fair_counter, R * 4));
    TRY(cp(trace->timeout, t.timeout, R * 4));
  }
  return SPECTRE_OK;
}

extern "C" int spectre_engine_read_background(void* engine, int32_t* tokens, int32_t* emitted,
                                              int32_t* totals, void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || e->st.n_bg <= 0) return arg_fail("spectre_engine_read_background: no background");
  cudaStream_t s = as_stream(stream);
  if (tokens)
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(tokens, e->st.bg_out,
                                     (size_t)e->st.n_bg * e->st.bg_out_len * 4,
                                     cudaMemcpyDeviceToDevice, s));
  if (emitted)
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(emitted, e->st.bg_emitted, (size_t)e->st.n_bg * 4,
                                     cudaMemcpyDeviceToDevice, s));
  CtrlDev c;
  SPECTRE_CUDA_TRY(cudaMemcpyAsync(&c, e->st.ctrl, sizeof(c), cudaMemcpyDeviceToHost, s));
  SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
  if (totals) {
    totals[0] = c.bg_tokens;
    totals[1] = c.bg_completed;
  }
  return SPECTRE_OK;
}

extern "C" int spectre_engine_read_committed(void* engine, int64_t* committed, void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || !committed) return arg_fail("spectre_engine_read_committed");
  SPECTRE_CUDA_TRY(cudaMemcpyAsync(committed, e->st.committed,
                                   (size_t)e->cfg.n_req * e->cfg.output_len * 8,
                                   cudaMemcpyDeviceToDevice, as_stream(stream)));
  return SPECTRE_OK;
}

extern "C" int spectre_engine_forward(void* engine, int32_t which, const int32_t* tok,
                                      const int32_t* pos, const int32_t* slot, int32_t T,
                                      const int32_t* q_off, const int32_t* n_new,
                                      const int32_t* pos0, int32_t* out_tok, void* out_x,
                                      void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || (which != 0 && which != 1)) return arg_fail("spectre_engine_forward");
  ModelRT& m = which == 0 ? e->tgt : e->drf;
  if (T < 0 || T > m.rows_cap) return arg_fail("spectre_engine_forward: T > rows_cap");
  cudaStream_t s = as_stream(stream);
  const int n = e->cfg.n_req;
  auto d2d = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
  };
  if (T > 0) {
    SPECTRE_CUDA_TRY(d2d(m.bt.tok, tok, (size_t)T * 4));
    SPECTRE_CUDA_TRY(d2d(m.bt.pos, pos, (size_t)T * 4));
    SPECTRE_CUDA_TRY(d2d(m.bt.slot, slot, (size_t)T * 4));
  }
  SPECTRE_CUDA_TRY(d2d(m.bt.q_off, q_off, (size_t)n * 4));
  SPECTRE_CUDA_TRY(d2d(m.bt.n_new, n_new, (size_t)n * 4));
  SPECTRE_CUDA_TRY(d2d(m.bt.pos0, pos0, (size_t)n * 4));
  if (m.n_req > n)   // the draft's background entries do not take part
    SPECTRE_CUDA_TRY(cudaMemsetAsync(m.bt.n_new + n, 0, (size_t)(m.n_req - n) * 4, s));
  std::vector<int> ident(m.n_req);
  for (int i = 0; i < m.n_req; ++i) ident[i] = i;
  SPECTRE_CUDA_TRY(cudaMemcpyAsync(m.bt.rslot, ident.data(), (size_t)m.n_req * 4,
                                   cudaMemcpyHostToDevice, s));
  SPECTRE_CUDA_TRY(cudaMemcpyAsync(m.bt.t_dev, &T, 4, cudaMemcpyHostToDevice, s));
  int max_new = 1;
  {
    std::vector<int> nn(n);
    SPECTRE_CUDA_TRY(cudaMemcpyAsync(nn.data(), n_new, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
    for (int v : nn) max_new = std::max(max_new, v);
  }
  TRY(m.forward(max_new, s, out_x));
  if (T > 0) SPECTRE_CUDA_TRY(d2d(out_tok, m.bt.out_tok, (size_t)T * 4));
  SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
  return SPECTRE_OK;
}

extern "C" int spectre_engine_step(void* engine, int32_t step, int32_t mode, void* stream) {
  auto* e = reinterpret_cast<Engine*>(engine);
  if (!e || e->attached) return arg_fail("spectre_engine_step");
  cudaStream_t s = as_stream(stream);
  switch (step) {
    case SPECTRE_STEP_BEGIN: {
      TRY(launch_round_begin(e->st, s));
      SPECTRE_CUDA_TRY(cudaMemcpyAsync(e->mode_host, &e->st.ctrl->mode, sizeof(int),
                                       cudaMemcpyDeviceToHost, s));
      SPECTRE_CUDA_TRY(cudaStreamSynchronize(s));
      return *e->mode_host;
    }
    case SPECTRE_STEP_DRAFT:
      if (mode == 'O' || mode == 'P' || mode == 'M') TRY(e->draft_phase(mode, s));
      return SPECTRE_OK;
    case SPECTRE_STEP_VERIFY:
      TRY(e->verify_phase(s));
      return SPECTRE_OK;
    case SPECTRE_STEP_ACCEPT:
      TRY(e->accept(s));
      return SPECTRE_OK;
    default:
      return arg_fail("spectre_engine_step: step");
  }
}

extern "C" int spectre_engine_exchange(void* src, void* dst, int32_t direction,
                                       int32_t src_req0, int32_t dst_req0, int32_t n,
                                       void* stream) {
  auto* a = reinterpret_cast<Engine*>(src);
  auto* b = reinterpret_cast<Engine*>(dst);
  if (!a || !b || n < 0 || src_req0 < 0 || dst_req0 < 0 || src_req0 + n > a->cfg.n_req ||
      dst_req0 + n > b->cfg.n_req || a->cfg.output_len != b->cfg.output_len ||
      a->st.hist_cap != b->st.hist_cap || a->cfg.gamma != b->cfg.gamma)
    return arg_fail("spectre_engine_exchange");
  cudaStream_t s = as_stream(stream);
  // cudaMemcpyDefault: unified addressing routes peer copies over NVLink
  auto cp = [&](void* d, const void* sp, size_t bytes) {
    return cudaMemcpyAsync(d, sp, bytes, cudaMemcpyDefault, s);
  };
  auto ints = [&](int* d, const int* sp) {
    return cp(d + dst_req0, sp + src_req0, (size_t)n * sizeof(int));
  };
  if (direction == 0) {   // target -> draft: what the draft server's sync needs
    SPECTRE_CUDA_TRY(cp(&b->st.ctrl->mode, &a->st.ctrl->mode, sizeof(int)));
    SPECTRE_CUDA_TRY(ints(b->st.pos, a->st.pos));
    SPECTRE_CUDA_TRY(ints(b->st.done, a->st.done));
    SPECTRE_CUDA_TRY(ints(b->st.cached_len, a->st.cached_len));
    SPECTRE_CUDA_TRY(ints(b->st.in_rollback, a->st.in_rollback));
    SPECTRE_CUDA_TRY(ints(b->st.req_mode, a->st.req_mode));
    SPECTRE_CUDA_TRY(ints(b->st.q_round, a->st.q_round));
    SPECTRE_CUDA_TRY(ints(b->st.q_serial, a->st.q_serial));
    SPECTRE_CUDA_TRY(cp(b->st.committed + (size_t)dst_req0 * b->cfg.output_len,
                        a->st.committed + (size_t)src_req0 * a->cfg.output_len,
                        (size_t)n * a->cfg.output_len * sizeof(uint64_t)));
  } else if (direction == 1) {   // draft -> target: speculation + draft timing
    SPECTRE_CUDA_TRY(cp(b->st.hist + (size_t)dst_req0 * b->st.hist_cap,
                        a->st.hist + (size_t)src_req0 * a->st.hist_cap,
                        (size_t)n * a->st.hist_cap * sizeof(uint64_t)));
    SPECTRE_CUDA_TRY(ints(b->st.hist_len, a->st.hist_len));
    SPECTRE_CUDA_TRY(ints(b->st.gen_count, a->st.gen_count));
    SPECTRE_CUDA_TRY(ints(b->st.gen_done, a->st.gen_done));
    SPECTRE_CUDA_TRY(ints(b->st.gen_start, a->st.gen_start));
    SPECTRE_CUDA_TRY(ints(b->st.r_round, a->st.r_round));
    SPECTRE_CUDA_TRY(ints(b->st.r_serial, a->st.r_serial));
    // draft phase timing only: the target's own clock fields stay untouched
    SPECTRE_CUDA_TRY(cp(&b->st.ctrl->t_draft_begin, &a->st.ctrl->t_draft_begin,
                        2 * sizeof(long long)));
    SPECTRE_CUDA_TRY(cp(&b->st.ctrl->draft_steps, &a->st.ctrl->draft_steps, sizeof(int)));
  } else {
    return arg_fail("spectre_engine_exchange: direction");
  }
  return SPECTRE_OK;
}

// Direct NVLink access between the GPUs of a disaggregated pair (idempotent).
extern "C" int spectre_enable_peer_access(int32_t dev_a, int32_t dev_b) {
  if (dev_a == dev_b) return SPECTRE_OK;
  int can_ab = 0, can_ba = 0;
  SPECTRE_CUDA_TRY(cudaDeviceCanAccessPeer(&can_ab, dev_a, dev_b));
  SPECTRE_CUDA_TRY(cudaDeviceCanAccessPeer(&can_ba, dev_b, dev_a));
  if (!can_ab || !can_ba) return arg_fail("spectre_enable_peer_access: no peer path");
  int cur = 0;
  SPECTRE_CUDA_TRY(cudaGetDevice(&cur));
  for (int k = 0; k < 2; ++k) {
    SPECTRE_CUDA_TRY(cudaSetDevice(k == 0 ? dev_a : dev_b));
    cudaError_t e = cudaDeviceEnablePeerAccess(k == 0 ? dev_b : dev_a, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) {
      cudaSetDevice(cur);
      return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
  }
  SPECTRE_CUDA_TRY(cudaSetDevice(cur));
  return SPECTRE_OK;
}

// ---------------------------------------------------------------------------
// One process per GPU (config 5): a peer process maps this engine's workspace
// through CUDA IPC and attaches a layout-only view of it, so
// spectre_engine_exchange writes straight into the peer's state (NVLink peer
// copies across GPUs; the same device also works).

#include <cuda.h>

extern "C" int spectre_ipc_export(const void* dev_ptr, uint8_t* handle_out, uint64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return arg_fail("spectre_ipc_export");
  // allocation base: the IPC handle names the whole cudaMalloc block
  using AddrRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static AddrRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<AddrRange>(fn);
  }();
  if (!get_range) return arg_fail("spectre_ipc_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return arg_fail("spectre_ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  SPECTRE_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == SPECTRE_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  return SPECTRE_OK;
}

extern "C" int spectre_ipc_open(const uint8_t* handle, uint64_t offset, void** base_out,
                                void** dev_ptr_out) {
  if (!handle || !base_out || !dev_ptr_out) return arg_fail("spectre_ipc_open");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  SPECTRE_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = base;
  *dev_ptr_out = static_cast<char*>(base) + offset;
  return SPECTRE_OK;
}

extern "C" int spectre_ipc_close(void* base) {
  if (!base) return arg_fail("spectre_ipc_close");
  SPECTRE_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return SPECTRE_OK;
}

extern "C" void* spectre_engine_attach(const SpectreModelDims* target,
                                       const SpectreModelDims* draft,
                                       const SpectreDecodeConfig* cfg, void* workspace,
                                       size_t workspace_bytes) {
  if (!dims_ok(target) || !dims_ok(draft) || !cfg || !workspace) {
    arg_fail("spectre_engine_attach");
    return nullptr;
  }
  auto e = std::make_unique<Engine>();
  e->configure(*target, SpectreModelWeights{}, *draft, SpectreModelWeights{}, *cfg);
  Bump b{reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255))};
  e->layout(b);   // same dims + config -> the owner's exact layout
  if (b.off + 256 > workspace_bytes) {
    arg_fail("spectre_engine_attach: workspace too small");
    return nullptr;
  }
  e->attached = 1;
  return e.release();
}
