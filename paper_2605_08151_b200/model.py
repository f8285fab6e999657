"""Model mode: a Llama-shaped bf16 target/draft pair driven by the device round loop.

The reference's model pair is `TokenStreamOracle` (oracle.py:47-113): a hash
stream as the target's greedy output and an alpha-proposer as the draft.
Here the pair is real transformer weights of the BASELINE shapes (random
init, no checkpoints) running on hand-written sm_100a kernels:

* target greedy token at output position q = argmax of the verify forward
  (tcgen05 GEMMs, gamma-query attention, greedy argmax fused into lm_head);
* draft proposal = the draft model's greedy token, kept with probability
  `alpha` and otherwise replaced (the reference's alpha-proposer semantics,
  oracle.py:83-85, applied on top of a real draft: "controlled noise").

Coupling: a 1B-shape draft (d=2048) cannot be a literal layer
truncation of an 8B-shape target (d=4096).  Both models therefore share one
"bigram backbone": the target's embedding and lm_head are the draft's lifted
by a fixed orthonormal map Q (E_T = E_D Q^T, LM_T = LM_D Q^T), so
LM_T . E_T[x] = LM_D . E_D[x]; the transformer branches (o_proj, down_proj)
are damped by `branch_scale`.  The natural agreement alpha_0 is set by the
two branch scales and the sweep knob `alpha` lowers it further.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .decoder import PolicyVariant
from .metrics import MetricsReport


@dataclass(frozen=True)
class ModelSpec:
    """Public HF config.json shapes."""
    name: str
    d_model: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 500000.0

    @property
    def qkv_rows(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim

    def streamed_params(self) -> int:
        """Weights read per forward pass (all layers + lm_head; embedding is a gather)."""
        d, qd = self.d_model, self.n_q_heads * self.head_dim
        per_layer = self.qkv_rows * d + d * qd + 2 * self.ffn * d + d * self.ffn
        return self.n_layers * per_layer + self.vocab * d

    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    def dims(self) -> _native.ModelDims:
        return _native.ModelDims(self.d_model, self.n_layers, self.n_q_heads, self.n_kv_heads,
                                 self.head_dim, self.ffn, self.vocab, self.rms_eps,
                                 self.rope_theta)


LLAMA_31_8B = ModelSpec("llama-3.1-8b", 4096, 32, 32, 8, 128, 14336, 128256)
LLAMA_32_1B = ModelSpec("llama-3.2-1b", 2048, 16, 32, 8, 64, 8192, 128256)
# Qwen2.5 shapes share one padded vocabulary (152064) so target/draft ids agree
QWEN_25_32B = ModelSpec("qwen2.5-32b", 5120, 64, 40, 8, 128, 27648, 152064, 1e-6, 1e6)
QWEN_25_05B = ModelSpec("qwen2.5-0.5b", 896, 24, 14, 2, 64, 4864, 152064, 1e-6, 1e6)
# small shapes for numerics tests (same kernels, seconds to run)
TINY_TARGET = ModelSpec("tiny-target", 256, 2, 4, 2, 64, 512, 1024)
TINY_DRAFT = ModelSpec("tiny-draft", 128, 2, 4, 2, 64, 256, 1024)
SMALL_TARGET = ModelSpec("small-target", 1024, 4, 8, 2, 128, 2048, 32000)
SMALL_DRAFT = ModelSpec("small-draft", 512, 2, 8, 2, 64, 1024, 32000)


class ModelWeights:
    """Device tensors of one model + its KV cache (torch-owned memory)."""

    def __init__(self, spec: ModelSpec, n_req: int, ctx_cap: int, device="cuda"):
        torch = _native.require_cuda()
        self.spec = spec
        L, d, F, V = spec.n_layers, spec.d_model, spec.ffn, spec.vocab
        qd = spec.n_q_heads * spec.head_dim
        bf = torch.bfloat16
        self.embed = torch.empty(V, d, dtype=bf, device=device)
        self.attn_norm = torch.ones(L, d, dtype=torch.float32, device=device)
        self.wqkv = torch.empty(L, spec.qkv_rows, d, dtype=bf, device=device)
        self.wo = torch.empty(L, d, qd, dtype=bf, device=device)
        self.mlp_norm = torch.ones(L, d, dtype=torch.float32, device=device)
        self.wgu = torch.empty(L, 2 * F, d, dtype=bf, device=device)   # rows [g0, u0, g1, u1, ..]
        self.wd = torch.empty(L, d, F, dtype=bf, device=device)
        self.final_norm = torch.ones(d, dtype=torch.float32, device=device)
        self.lm_head = torch.empty(V, d, dtype=bf, device=device)
        kv_shape = (L, n_req, spec.n_kv_heads, ctx_cap, spec.head_dim)
        self.k_cache = torch.zeros(kv_shape, dtype=bf, device=device)
        self.v_cache = torch.zeros(kv_shape, dtype=bf, device=device)

    def init_layers(self, gen, branch_scale: float, std: float = 0.02) -> None:
        torch = _native.require_cuda()
        for l in range(self.spec.n_layers):
            self.wqkv[l].copy_(torch.randn(self.wqkv[l].shape, generator=gen, device="cuda") * std)
            self.wo[l].copy_(torch.randn(self.wo[l].shape, generator=gen, device="cuda")
                             * (std * branch_scale))
            self.wgu[l].copy_(torch.randn(self.wgu[l].shape, generator=gen, device="cuda") * std)
            self.wd[l].copy_(torch.randn(self.wd[l].shape, generator=gen, device="cuda")
                             * (std * branch_scale))

    def gate_up(self, layer: int):
        """De-interleaved (gate [F][d], up [F][d]) views for reference code."""
        F, d = self.spec.ffn, self.spec.d_model
        w = self.wgu[layer].view(F, 2, d)
        return w[:, 0], w[:, 1]

    def struct(self) -> _native.ModelWeights:
        p = lambda t: t.data_ptr()
        return _native.ModelWeights(p(self.embed), p(self.attn_norm), p(self.wqkv), p(self.wo),
                                    p(self.mlp_norm), p(self.wgu), p(self.wd),
                                    p(self.final_norm), p(self.lm_head), p(self.k_cache),
                                    p(self.v_cache))

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (
            self.embed, self.wqkv, self.wo, self.wgu, self.wd, self.lm_head))


@dataclass
class ModelPair:
    target: ModelWeights
    draft: ModelWeights
    n_req: int
    ctx_cap: int
    n_bg: int = 0       # extra draft KV slots for background tenants


def build_pair(target: ModelSpec, draft: ModelSpec, n_req: int, ctx_cap: int, seed: int = 0,
               target_branch: float = 0.08, draft_branch: float = 0.08,
               n_bg: int = 0) -> ModelPair:
    """Random-init target/draft coupled through a shared lifted backbone (H6).
    n_bg: draft KV slots for background (regular) tenants of the draft server."""
    torch = _native.require_cuda()
    if target.vocab != draft.vocab:
        raise ValueError("target and draft must share a vocabulary")
    gen = torch.Generator(device="cuda").manual_seed(seed)
    T = ModelWeights(target, n_req, ctx_cap)
    D = ModelWeights(draft, n_req + n_bg, ctx_cap)
    V, dD, dT = draft.vocab, draft.d_model, target.d_model
    D.embed.copy_(torch.randn(V, dD, generator=gen, device="cuda"))
    D.lm_head.copy_(torch.randn(V, dD, generator=gen, device="cuda") / math.sqrt(dD))
    if dT == dD:
        Q = torch.eye(dD, device="cuda")
    else:
        q, _ = torch.linalg.qr(torch.randn(dT, dD, generator=gen, device="cuda"))
        Q = q[:, :dD]                               # [dT][dD], orthonormal columns
    for r0 in range(0, V, 16384):                   # E_T = E_D Q^T, LM_T = LM_D Q^T
        T.embed[r0:r0 + 16384].copy_(D.embed[r0:r0 + 16384].float() @ Q.t())
        T.lm_head[r0:r0 + 16384].copy_(D.lm_head[r0:r0 + 16384].float() @ Q.t())
    D.init_layers(gen, draft_branch)
    T.init_layers(gen, target_branch)
    torch.cuda.synchronize()
    return ModelPair(T, D, n_req, ctx_cap, n_bg)


CONTROLLERS = {"reference": 0, "measured": 1, "round": 2}


@dataclass
class DecodeSpec:
    """Decode-loop knobs (names follow SimConfig, core.py:63-115)."""
    n_req: int = 64
    gamma: int = 4
    output_len: int = 1024
    prompt_len: int = 128
    alpha: float = 1.0              # draft keep probability (controlled noise)
    seed: int = 0
    controller: str = "round"       # reference | measured | round
    r_kind: int = 0                 # 0: |R|/B (reference r-hat), 1: PADDED fraction
    t_target: float = 0.050
    t_draft: float = 0.005
    ema_decay: float = 0.9
    fixed_threshold_l: float | None = None
    max_rounds: int | None = None
    temperature: float = 0.0        # 0: greedy; > 0: speculative rejection sampling (config 3)
    breaker_threshold: int = 3      # circuit breaker (core.py:93-94, target_engine.py:337-380)
    breaker_cooldown: int = 5
    compression_p: float = 1.0      # draft prompt compression (core.py compression_p,
                                    # draft_engine.py:123-131): keep floor(p*S/2) head and
                                    # tail prompt tokens in the draft's KV cache
    # background (regular) tenants of the draft model + the speculative-priority
    # fairness scheduler (core.py:79-85, draft_engine.py:134-155, 302-394)
    background_requests: int = 0
    background_output_len: int = 128
    fairness_period: int = 10
    draft_capacity: int = 256
    reply_timeout_rounds: int = 2   # reply_timeout = 2 t_target (core.py:123)
    # non-stationary acceptance (config 4 drift workload): from draft output
    # position alpha_switch_pos on the keep probability is alpha_late
    alpha_switch_pos: int = 0
    alpha_late: float = 1.0

    def draft_prompt_keep(self) -> int:
        """compress_prompt (draft_engine.py:123-131): keep = int((p / 2) * S); no
        compression when 2 * keep >= S."""
        if not 0.0 <= self.compression_p <= 1.0:
            raise ValueError(f"compression_p must be in [0, 1], got {self.compression_p}")
        keep = int((self.compression_p / 2.0) * self.prompt_len)
        if 2 * keep >= self.prompt_len:
            return 0
        if keep == 0:
            raise ValueError("compression_p keeps no prompt token for the draft")
        return keep

    def __post_init__(self):
        if self.temperature > 0 and (self.alpha < 1.0 or
                                     (self.alpha_switch_pos > 0 and self.alpha_late < 1.0)):
            raise ValueError("temperature > 0 (rejection sampling) needs alpha == 1: the "
                             "alpha noise would replace proposals not drawn from q")

    def ctx_cap(self) -> int:
        need = self.prompt_len + self.output_len + 4 * self.gamma + 16
        return (need + 63) // 64 * 64


_VAR = {PolicyVariant.AR: 0, PolicyVariant.ORDINARY: 1, PolicyVariant.PARALLEL: 2,
        PolicyVariant.HYBRID: 3}


ROLES = {"both": 0, "target": 1, "draft": 2}


class SpectreEngine:
    """Owns the libspectre engine handle and its workspace.  role "target" /
    "draft" builds one side of a disaggregated pair (config 5, see disagg.py)."""

    def __init__(self, pair: ModelPair, spec: DecodeSpec, variant: PolicyVariant | str,
                 role: str = "both"):
        torch = _native.require_cuda()
        L = _native.lib()
        if isinstance(variant, str):
            variant = PolicyVariant.parse(variant)
        self.pair, self.spec, self.variant = pair, spec, variant
        if spec.ctx_cap() > pair.ctx_cap:
            raise ValueError(f"KV capacity {pair.ctx_cap} < needed {spec.ctx_cap()}")
        if spec.n_req != pair.n_req:
            raise ValueError("n_req must match the KV cache allocation")
        if spec.background_requests != pair.n_bg:
            raise ValueError("background_requests must match the pair's draft background slots")
        self.max_rounds = spec.max_rounds or spec.output_len + 8
        self.cfg = _native.DecodeConfig(
            seed=spec.seed & ((1 << 64) - 1), n_req=spec.n_req, gamma=spec.gamma,
            output_len=spec.output_len, prompt_len=spec.prompt_len, variant=_VAR[variant],
            controller=CONTROLLERS[spec.controller], r_kind=spec.r_kind,
            max_rounds=self.max_rounds, ctx_cap=pair.ctx_cap,
            has_fixed_l=int(spec.fixed_threshold_l is not None), alpha=spec.alpha,
            t_target=spec.t_target, t_draft=spec.t_draft, ema_decay=spec.ema_decay,
            fixed_threshold_l=float(spec.fixed_threshold_l or 0.0),
            temperature=float(spec.temperature), role=ROLES[role],
            breaker_threshold=int(spec.breaker_threshold),
            breaker_cooldown=int(spec.breaker_cooldown),
            draft_prompt_keep=spec.draft_prompt_keep(),
            background_requests=int(spec.background_requests),
            background_output_len=int(spec.background_output_len),
            fairness_period=int(spec.fairness_period), draft_capacity=int(spec.draft_capacity),
            reply_timeout_rounds=int(spec.reply_timeout_rounds),
            alpha_switch_pos=int(spec.alpha_switch_pos), alpha_late=float(spec.alpha_late))
        self.role = role
        self._tdims = pair.target.spec.dims()
        self._ddims = pair.draft.spec.dims()
        self._tw = pair.target.struct()
        self._dw = pair.draft.struct()
        nbytes = L.spectre_engine_workspace_bytes(self._tdims, self._ddims, self.cfg)
        if nbytes == 0:
            raise ValueError("unsupported model / decode shape")
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        h = L.spectre_engine_create(self._tdims, self._tw, self._ddims, self._dw, self.cfg,
                                    self.workspace.data_ptr(), nbytes)
        if not h:
            raise _native.SpectreError("spectre_engine_create: " +
                                       L.spectre_last_error().decode())
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            _native.lib().spectre_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, prompts, stream=None):
        self._prompts = prompts  # keep alive while the stream runs
        _native.check(_native.lib().spectre_engine_prefill(
            self.handle, prompts.data_ptr(), _native.stream_ptr(stream)), "spectre_engine_prefill")

    def run(self, max_rounds: int | None = None, use_graph: bool = True, stream=None,
            sync: bool = False) -> int | None:
        """Decode rounds on the device.  Asynchronous unless sync=True (then the
        number of rounds run is returned)."""
        n = C.c_int32(0)
        _native.check(_native.lib().spectre_engine_run(
            self.handle, int(max_rounds if max_rounds is not None else self.max_rounds),
            int(use_graph), C.byref(n) if sync else None, _native.stream_ptr(stream)),
            "spectre_engine_run")
        return n.value if sync else None

    def step(self, step: int, mode: int = 0, stream=None) -> int:
        """One piece of a host-driven round (disaggregated pairs); BEGIN returns the mode."""
        r = _native.lib().spectre_engine_step(self.handle, step, mode, _native.stream_ptr(stream))
        if r < 0:
            _native.check(r, "spectre_engine_step")
        return r

    def graph_status(self) -> int:
        return _native.lib().spectre_engine_graph_status(self.handle)

    def read(self):
        torch = _native.require_cuda()
        n, OL, R = self.spec.n_req, self.spec.output_len, self.max_rounds
        committed = torch.zeros(n, OL, dtype=torch.int64, device="cuda")
        pos = torch.zeros(n, dtype=torch.int32, device="cuda")
        bufs = {}
        for f in _native.TRACE_FIELDS:
            dt = (torch.float64 if f in ("r_hat_ema", "accepted_len_ema", "r_star")
                  else torch.int64 if f.startswith("t_") else torch.int32)
            bufs[f] = torch.zeros(R, dtype=dt, device="cuda")
        tr = _native.RoundTraceBufs(**{f: bufs[f].data_ptr() for f in _native.TRACE_FIELDS})
        nr = C.c_int32(0)
        _native.check(_native.lib().spectre_engine_read(
            self.handle, committed.data_ptr(), pos.data_ptr(), tr, C.byref(nr),
            _native.stream_ptr()), "spectre_engine_read")
        torch.cuda.synchronize()
        trace = {f: v[:nr.value].cpu().numpy() for f, v in bufs.items()}
        return committed, pos, trace

    def read_background(self):
        """Background tenants: (tokens [n_bg][background_output_len] int32 on the
        device, emitted [n_bg], (tokens generated, requests completed))."""
        torch = _native.require_cuda()
        n, OL = self.spec.background_requests, self.spec.background_output_len
        toks = torch.zeros(n, OL, dtype=torch.int32, device="cuda")
        emitted = torch.zeros(n, dtype=torch.int32, device="cuda")
        totals = (C.c_int32 * 2)()
        _native.check(_native.lib().spectre_engine_read_background(
            self.handle, toks.data_ptr(), emitted.data_ptr(), totals, _native.stream_ptr()),
            "spectre_engine_read_background")
        return toks, emitted, (int(totals[0]), int(totals[1]))

    def read_committed(self, stream=None):
        """Committed tokens [n_req][output_len] int64 on the device (no host sync)."""
        torch = _native.require_cuda()
        out = torch.empty(self.spec.n_req, self.spec.output_len, dtype=torch.int64,
                          device="cuda")
        _native.check(_native.lib().spectre_engine_read_committed(
            self.handle, out.data_ptr(), _native.stream_ptr(stream)),
            "spectre_engine_read_committed")
        return out

    def forward(self, which: int, tok, pos, slot, q_off, n_new, pos0, want_x=False):
        torch = _native.require_cuda()
        T = int(tok.numel())
        d = (self.pair.target if which == 0 else self.pair.draft).spec.d_model
        out_tok = torch.zeros(max(T, 1), dtype=torch.int32, device="cuda")
        rows_cap = 4096
        out_x = torch.zeros(rows_cap, d, dtype=torch.bfloat16, device="cuda") if want_x else None
        i32 = lambda t: t.to(device="cuda", dtype=torch.int32).contiguous()
        keep = [i32(tok), i32(pos), i32(slot), i32(q_off), i32(n_new), i32(pos0)]
        _native.check(_native.lib().spectre_engine_forward(
            self.handle, which, keep[0].data_ptr(), keep[1].data_ptr(), keep[2].data_ptr(), T,
            keep[3].data_ptr(), keep[4].data_ptr(), keep[5].data_ptr(), out_tok.data_ptr(),
            out_x.data_ptr() if want_x else None, _native.stream_ptr()), "spectre_engine_forward")
        return out_tok[:T], (out_x[:T] if want_x else None)


def synthetic_prompts(n_req: int, prompt_len: int, vocab: int, seed: int = 0, req0: int = 0):
    """Prompt ids = TokenStreamOracle(seed).prompt_tokens(req, P) mod V for
    the global requests req0 .. req0 + n_req - 1, computed by the K8 stream kernel."""
    torch = _native.require_cuda()
    req = torch.arange(req0, req0 + n_req, device="cuda",
                       dtype=torch.int64).repeat_interleave(prompt_len)
    pos = torch.arange(prompt_len, device="cuda", dtype=torch.int64).repeat(n_req)
    out = torch.empty_like(req)
    _native.check(_native.lib().spectre_oracle_stream(
        seed & ((1 << 64) - 1), 1, req.data_ptr(), pos.data_ptr(), out.data_ptr(), req.numel(),
        _native.stream_ptr()), "spectre_oracle_stream")
    u = out.view(torch.int64)
    # unsigned 64-bit value mod V (int64 view may be negative)
    vals = (u.remainder(vocab) + (1 << 64) % vocab * (u < 0)).remainder(vocab)
    return vals.to(torch.int32).view(n_req, prompt_len).contiguous()


@dataclass
class ModelRunResult:
    report: MetricsReport
    variant: PolicyVariant
    committed: object            # torch [n_req][output_len] int64
    committed_pos: object
    trace: dict
    rounds: int
    device_seconds: float        # sum of device round spans
    graph: int                   # engine graph status
    extra: dict = field(default_factory=dict)


def report_from_trace(variant: PolicyVariant, seed: int, trace: dict, total: int,
                      device_seconds: float) -> MetricsReport:
    """MetricsReport (metrics.py:61-101) with device wall time as the clock."""
    P = trace["participants"].astype(np.int64)
    n = len(P)
    r_hat = [int(a) / int(b) for a, b in zip(trace["n_roll"], P)] if n else []
    deltas = int(trace["delta"].sum())
    cs, cn = int(trace["content_sum"].sum()), int(trace["content_n"].sum())
    maxp = int(P.max()) if n else 0
    steady = [i for i in range(n) if P[i] == maxp]
    s_time = sum(int(trace["t_round_ns"][i]) for i in steady) * 1e-9
    s_comm = sum(int(trace["delta"][i]) for i in steady)
    s_dn = sum(int(P[i]) for i in steady)
    s_cs = sum(int(trace["content_sum"][i]) for i in steady)
    s_cn = sum(int(trace["content_n"][i]) for i in steady)
    return MetricsReport(
        variant=variant.value, seed=seed,
        target_throughput=total / device_seconds if device_seconds > 0 else 0.0,
        mean_accepted_length=deltas / int(P.sum()) if n else 0.0,
        content_mean_accepted_length=cs / cn if cn else 0.0,
        mean_rollback_ratio=(sum(r_hat) / n) if n else 0.0,
        rollback_ratio_series=tuple(r_hat),
        mode_timeline="".join(chr(int(m)) for m in trace["mode"]),
        steady_rounds=len(steady),
        steady_target_throughput=s_comm / s_time if s_time > 0 else 0.0,
        steady_mean_accepted_length=s_comm / s_dn if s_dn else 0.0,
        steady_content_mean_accepted_length=s_cs / s_cn if s_cn else 0.0,
        steady_mean_rollback_ratio=(sum(r_hat[i] for i in steady) / len(steady)) if steady else 0.0,
        sim_duration=device_seconds, total_committed=total, total_rounds=n,
        requests_completed=0, fallback_rounds=sum(1 for m in trace["mode"] if m == ord("F")),
        breaker_activations=0 if variant == PolicyVariant.AR else sum(
            1 for i, m in enumerate(trace["mode"])
            if m == ord("F") and (i == 0 or trace["mode"][i - 1] != ord("F"))),
        stale_replies=int(trace["n_stale"].sum()) if "n_stale" in trace else 0,
        timeout_rounds=int(trace["timeout"].sum()) if "timeout" in trace else 0,
        draft_tokens_generated=0)


def decode(pair: ModelPair, spec: DecodeSpec, variant, prompts=None, use_graph=True,
           engine: SpectreEngine | None = None) -> ModelRunResult:
    """Prefill + decode every request to output_len on the device."""
    torch = _native.require_cuda()
    if isinstance(variant, str):
        variant = PolicyVariant.parse(variant)
    eng = engine or SpectreEngine(pair, spec, variant)
    if prompts is None:
        prompts = synthetic_prompts(spec.n_req, spec.prompt_len, pair.target.spec.vocab, spec.seed)
    eng.prefill(prompts)
    rounds = eng.run(use_graph=use_graph, sync=True)
    committed, pos, trace = eng.read()
    dev_s = float(trace["t_round_ns"].sum()) * 1e-9
    total = int(pos.sum().item())
    rep = report_from_trace(variant, spec.seed, trace, total, dev_s)
    upd = {"requests_completed": int((pos >= spec.output_len).sum().item())}
    extra = {}
    if spec.background_requests > 0:   # regular tenants of the draft (metrics.py:61-101)
        bg_toks, bg_emitted, (bg_n, bg_done) = eng.read_background()
        upd.update(background_tokens=bg_n, background_completed=bg_done,
                   draft_throughput=bg_n / dev_s if dev_s > 0 else 0.0)
        extra.update(background_tokens=bg_toks, background_emitted=bg_emitted)
    rep = MetricsReport(**{**rep.__dict__, **upd})
    status = eng.graph_status()
    if status == 2:
        extra["graph_error"] = _native.lib().spectre_last_error().decode(errors="replace")
    return ModelRunResult(rep, variant, committed, pos, trace, rounds, dev_s, status, extra)


def smoke() -> None:
    """Tiny model-mode decode on cuda:0: every speculative variant must commit
    exactly the autoregressive greedy stream (losslessness)."""
    pair = build_pair(TINY_TARGET, TINY_DRAFT, n_req=4, ctx_cap=256, seed=1)
    spec = DecodeSpec(n_req=4, gamma=4, output_len=48, prompt_len=16, alpha=0.9, seed=1)
    ref = decode(pair, spec, "ar")
    for v in ("ordinary", "parallel", "hybrid"):
        got = decode(pair, spec, v)
        assert (got.committed == ref.committed).all(), f"{v} diverged from AR"
