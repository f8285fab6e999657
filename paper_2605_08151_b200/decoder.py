"""`run(config, variant)` — the reference's decoder entry point, on a B200.

Drop-in for specsim.run (/root/reference/pkg/src/specsim/sim.py:989-1005) in
the fault-free regime: the whole round loop executes on the device in one
persistent kernel (csrc/oracle_mode.cu: controller, candidate assembly, draft
sync/rebase/propose, verify, commit, suffix reuse, rollback statistics and
the simulated clock).  The host only prepares inputs (arrival schedule, the
draft RNG seed state), launches, and turns the device trace into the
reference's `RunResult` / `MetricsReport` / `RoundTrace` records.
"""

from __future__ import annotations

import dataclasses
import hashlib
import math
import random
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _native
from .core import ConfigError, SimConfig, parse_delay_spec, validate_config
from .metrics import MetricsReport


class PolicyVariant(Enum):
    """sim.py:55-67 — ar / ordinary / parallel / hybrid (= SPECTRE adaptive)."""
    AR = "ar"
    ORDINARY = "ordinary"
    PARALLEL = "parallel"
    HYBRID = "hybrid"

    @classmethod
    def parse(cls, name: str) -> "PolicyVariant":
        try:
            return cls(name.strip().lower())
        except ValueError:
            valid = ", ".join(v.value for v in cls)
            raise ValueError(f"unknown variant {name!r}; expected one of: {valid}")


_VARIANT_CODE = {PolicyVariant.AR: 0, PolicyVariant.ORDINARY: 1,
                 PolicyVariant.PARALLEL: 2, PolicyVariant.HYBRID: 3}


class ProtocolViolation(RuntimeError):
    """An internal invariant of the coordination protocol was broken
    (target_engine.py:19-20)."""


class SimLivelock(RuntimeError):
    """No commit progress (sim.py:70-71)."""


class OutsideDeviceDomain(NotImplementedError):
    """The configuration needs the reference's faulty-transport machinery
    (drops, reorders, timeouts, stale replies), which the on-device decode
    loop deliberately does not model."""


def generate_arrivals(qps: float, n: int, rng: random.Random) -> list[float]:
    """sim.py:74-85 — Poisson arrivals (workload input preparation)."""
    if qps <= 0:
        raise ValueError(f"qps must be > 0, got {qps}")
    if n < 0:
        raise ValueError(f"n must be >= 0, got {n}")
    t, out = 0.0, []
    for _ in range(n):
        t += rng.expovariate(qps)
        out.append(t)
    return out


@dataclass(frozen=True)
class Workload:
    """sim.py:88-140."""
    arrival_times: tuple
    output_len: int
    prompt_len: int = 0
    label: str = "foreground"

    def __post_init__(self):
        if self.output_len < 1:
            raise ValueError(f"output_len must be >= 1, got {self.output_len}")
        if any(t < 0 for t in self.arrival_times):
            raise ValueError("arrival times must be >= 0")
        if list(self.arrival_times) != sorted(self.arrival_times):
            raise ValueError("arrival times must be non-decreasing")

    @classmethod
    def from_config(cls, config: SimConfig, rng: random.Random) -> "Workload":
        return cls(tuple(generate_arrivals(config.qps, config.n_requests, rng)),
                   config.output_len, config.prompt_len)

    @classmethod
    def from_file(cls, path, output_len: int, prompt_len: int = 0) -> "Workload":
        times = [float(ln) for ln in (s.strip() for s in Path(path).read_text().splitlines())
                 if ln and not ln.startswith("#")]
        return cls(tuple(sorted(times)), output_len, prompt_len)


@dataclass(frozen=True)
class RoundTrace:
    """sim.py:166-179."""
    round: int
    started_at: float
    committed_at: float
    mode: str
    participants: int
    committed_delta: int
    r_hat: float
    speculation_on: bool
    timeout: bool
    conservative: bool
    breaker_streak: int
    disabled_until: int


@dataclass(frozen=True)
class DraftRoundRecord:
    """draft_engine.py:167-179."""
    started_at: float
    finished_at: float
    n_speculative: int
    n_regular: int
    regular_pending_at_start: int
    forced_regular: bool
    t_d_mix: float
    steps: int
    counter_after: int


@dataclass
class RequestState:
    """The finished-request record (target_engine.py:85-102 fields)."""
    request: int
    output_len: int
    round: int = 0
    committed_pos: int = 0
    committed_tokens: list = field(default_factory=list)
    pending_bonus: int | None = None
    cached_segment: object = None
    in_rollback: bool = True
    done: bool = True
    synced_pos: int = 0
    prompt_len: int = 0
    arrived_at: float = 0.0
    admitted_at: float = 0.0
    finished_at: float = 0.0


@dataclass
class RunResult:
    """sim.py:182-192, plus the device-side controller trace."""
    report: MetricsReport
    config: SimConfig
    variant: PolicyVariant
    round_trace: list
    draft_records: list
    finished: dict
    breaker_windows: list
    channel_counters: dict
    lossless: bool
    device_trace: dict = field(default_factory=dict)


def draft_latency(cfg: SimConfig):
    """(alpha_eff, all-speculative step base, slope, free batch, the target's
    initial T_D^mix): prompt compression scales the draft's alpha and its
    speculative step latency (draft_engine.py:205-216, 335-338); the target
    starts from mixed_step_latency(1, unscaled) (sim.py:283-288)."""
    p = cfg.compression_p
    if p < 1.0:
        alpha_eff = cfg.alpha * (1.0 - cfg.compression_beta * (1.0 - p))
        factor = cfg.compression_latency_frac + (1.0 - cfg.compression_latency_frac) * p
    else:
        alpha_eff, factor = cfg.alpha, 1.0
    slope, free = cfg.t_draft_slope, cfg.t_draft_free_batch
    return (alpha_eff, cfg.t_draft * factor, slope, free,
            cfg.t_draft + slope * max(0, 1 - free))


def mixed_step_latency(base: float, slope: float, free: int, scheduled: int) -> float:
    """draft_engine.py:158-164."""
    return base + slope * max(0, scheduled - free)


def _check_domain(cfg: SimConfig, variant: PolicyVariant) -> float:
    kind, args = parse_delay_spec(cfg.delay_dist)
    if kind != "constant":
        raise OutsideDeviceDomain("stochastic transport delay")
    d = args[0]
    if cfg.drop_prob or cfg.reorder_prob:
        raise OutsideDeviceDomain("message drops / reorders")
    if cfg.background_qps > 0 and cfg.background_requests > 0:
        raise OutsideDeviceDomain("background draft tenants")
    if d > cfg.stale_timeout or d >= cfg.heartbeat_period or \
            cfg.heartbeat_period + d > cfg.heartbeat_expiry:
        raise OutsideDeviceDomain("liveness / staleness timeouts would fire")
    if variant is not PolicyVariant.AR:
        g = cfg.gamma
        if g < 2:
            raise OutsideDeviceDomain("gamma < 2 (empty repair replies time out)")
        if cfg.max_concurrency > cfg.draft_capacity:
            raise OutsideDeviceDomain("batch larger than draft capacity")
        t_d_max = max(draft_latency(cfg)[4],
                      mixed_step_latency(*draft_latency(cfg)[1:4], cfg.max_concurrency))
        if 2 * d + (g - 1) * t_d_max >= cfg.reply_timeout:
            raise OutsideDeviceDomain("ordinary repairs would time out")
    return d


def draft_rng_key(seed: int) -> list[int]:
    """CPython's str-seed expansion for random.Random(f"{seed}:draft")
    (sim.py:250): int.from_bytes(s + sha512(s), 'big') as LE 32-bit words."""
    s = f"{seed}:draft".encode()
    a = int.from_bytes(s + hashlib.sha512(s).digest(), "big")
    words = []
    while a:
        words.append(a & 0xFFFFFFFF)
        a >>= 32
    return words or [0]


def draft_uniforms(seed: int, n: int, device=None):
    """n genrand_res53 uniforms of Random(f"{seed}:draft"), generated on the GPU."""
    torch = _native.require_cuda()
    L = _native.lib()
    key = np.asarray(draft_rng_key(seed), dtype=np.uint32)
    state = np.zeros(625, dtype=np.uint32)
    _native.check(L.spectre_mt19937_init_by_array(key.ctypes.data, len(key), state.ctypes.data),
                  "spectre_mt19937_init_by_array")
    dev = torch.device(device or "cuda")
    st = torch.from_numpy(state.view(np.int32).copy()).to(dev)
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _native.check(L.spectre_mt19937_uniforms(st.data_ptr(), out.data_ptr(), n,
                                             _native.stream_ptr()), "spectre_mt19937_uniforms")
    return out[:n]


def _heartbeat_counts(h: float, d: float, t_end: float, final_dispatch: float):
    """HEARTBEAT events that fire / deliver before the loop stops at the final
    commit (sim.py:349, 351-353, 879-891; heap ties resolve by push order)."""
    sent = deliv = 0
    prev, t = 0.0, h
    while t < t_end or (t == t_end and prev <= final_dispatch):
        sent += 1
        td = t + d
        if td < t_end or (td == t_end and t <= final_dispatch):
            deliv += 1
        prev, t = t, t + h
    return sent, deliv


def _mean(xs) -> float:
    return sum(xs) / len(xs) if xs else 0.0


def run(config: SimConfig, variant: PolicyVariant | str, workload: Workload | None = None,
        background: Workload | None = None, *, device=None) -> RunResult:
    """Decode every request of the workload; returns the reference's RunResult."""
    if isinstance(variant, str):
        variant = PolicyVariant.parse(variant)
    cfg, _ = validate_config(config)
    if background is not None and background.arrival_times:
        raise OutsideDeviceDomain("background draft tenants")
    d = _check_domain(cfg, variant)
    torch = _native.require_cuda()
    L = _native.lib()
    dev = torch.device(device or "cuda")
    if workload is None:
        workload = Workload.from_config(cfg, random.Random(f"{cfg.seed}:workload"))
    arrivals = list(workload.arrival_times)
    n = len(arrivals)
    if n == 0:
        raise ConfigError(["empty workload"])
    OL, g = workload.output_len, cfg.gamma
    spec = variant is not PolicyVariant.AR
    n_unif = g * n * max(OL - 1, 1) + 1 if spec else 1
    max_rounds = n * max(OL - 1, 1) + 1
    seed64 = cfg.seed & ((1 << 64) - 1)

    dl = draft_latency(cfg)
    c = _native.OracleConfig(
        seed=seed64, n_requests=n, max_concurrency=cfg.max_concurrency, gamma=g,
        output_len=OL, variant=_VARIANT_CODE[variant],
        fairness_period=cfg.fairness_period,
        has_fixed_l=int(cfg.fixed_threshold_l is not None), max_rounds=max_rounds,
        alpha=dl[0], t_target=cfg.t_target, t_draft=dl[1], delay=d,
        t_target_slope=cfg.t_target_slope, ema_decay=cfg.ema_decay,
        fixed_threshold_l=float(cfg.fixed_threshold_l or 0.0),
        t_draft_slope=dl[2], t_draft_init=dl[4], t_draft_free_batch=dl[3],
        reply_timeout=cfg.reply_timeout)
    ws_bytes = L.spectre_oracle_workspace_bytes(c)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    arr = torch.tensor(arrivals, dtype=torch.float64, device=dev)
    unif = draft_uniforms(cfg.seed, n_unif, dev) if spec else torch.zeros(1, dtype=torch.float64,
                                                                          device=dev)
    i32, f64 = torch.int32, torch.float64
    bufs = dict(
        committed=torch.zeros(n * OL, dtype=torch.int64, device=dev),
        committed_pos=torch.zeros(n, dtype=i32, device=dev),
        admitted_at=torch.zeros(n, dtype=f64, device=dev),
        finished_at=torch.zeros(n, dtype=f64, device=dev),
        scalars=torch.zeros(8, dtype=torch.int64, device=dev),
    )
    for name in _native.ORACLE_OUTPUT_FIELDS:
        if name.startswith("round_"):
            dt = f64 if name in ("round_started", "round_dispatch", "round_commit",
                                 "round_draft_start", "round_draft_done", "round_r_hat_ema",
                                 "round_accepted_len_ema", "round_r_star") else i32
            bufs[name] = torch.zeros(max_rounds, dtype=dt, device=dev)
    outs = _native.OracleOutputs(**{k: bufs[k].data_ptr() for k in _native.ORACLE_OUTPUT_FIELDS})
    _native.check(L.spectre_oracle_run(c, arr.data_ptr(), unif.data_ptr(), n_unif,
                                       ws.data_ptr(), outs, _native.stream_ptr()),
                  "spectre_oracle_run")
    # lossless check on device: committed stream vs the reference stream
    req = torch.arange(n, device=dev, dtype=torch.int64).repeat_interleave(OL)
    pos = torch.arange(OL, device=dev, dtype=torch.int64).repeat(n)
    refs = torch.empty(n * OL, dtype=torch.int64, device=dev)
    _native.check(L.spectre_oracle_stream(seed64, 0, req.data_ptr(), pos.data_ptr(),
                                          refs.data_ptr(), n * OL, _native.stream_ptr()),
                  "spectre_oracle_stream")
    torch.cuda.synchronize(dev)
    sc = bufs["scalars"].cpu().numpy()
    n_rounds, draws, err, err_req, n_fin = (int(x) for x in sc[:5])
    if err != 0:
        names = {1: "commit gap", 2: "position regression", 3: "draft history overflow",
                 4: "uniform stream exhausted",
                 5: "parallel reply after the commit / conservative reply after the deadline",
                 6: "round trace overflow", 7: "misanchored segment"}
        msg = names.get(err, f"error {err}")
        if err in (5,):
            raise OutsideDeviceDomain(msg)
        raise ProtocolViolation(f"device decode loop: {msg} (request {err_req})")
    if n_fin != n:
        raise SimLivelock(f"{n - n_fin} requests unfinished after {n_rounds} rounds")
    h = {k: v[:n_rounds].cpu().numpy() for k, v in bufs.items() if k.startswith("round_")}
    cpos = bufs["committed_pos"].cpu().numpy()
    fin_at = bufs["finished_at"].cpu().numpy()
    adm_at = bufs["admitted_at"].cpu().numpy()
    mask = (torch.arange(OL, device=dev).repeat(n) <
            bufs["committed_pos"].to(torch.int64).repeat_interleave(OL))
    lossless = bool(torch.equal(bufs["committed"][mask], refs[mask]))
    committed = bufs["committed"].cpu().numpy().view(np.uint64).reshape(n, OL)
    result = _assemble_result(cfg, variant, workload, d, h, cpos, fin_at, adm_at, committed,
                              lossless, draws)
    if not result.lossless:                      # sim.py:1000-1004
        raise ProtocolViolation(
            f"losslessness violated: a committed sequence diverged from the reference "
            f"stream (variant={variant.value}, seed={cfg.seed})")
    return result


def _assemble_result(cfg, variant, workload, d, h, cpos, fin_at, adm_at, committed, lossless,
                     draws) -> RunResult:
    spec = variant is not PolicyVariant.AR
    n_rounds = len(h["round_mode"])
    trace, steady_rows = [], []
    r_hats, deltas_all_sum, deltas_all_n = [], 0, 0
    content_sum, content_n = 0, 0
    timeline, draft_records = [], []
    counter = 0
    n_queries = 0
    draft_tokens = 0
    # conservative_mode_check (sim.py:143-146, 599-602) on the T_D^mix the target
    # last received (sim.py:283-288, 833-834), exactly as the device loop did
    lat = draft_latency(cfg)
    last_tdm = lat[4]
    n_conservative = 0
    commit_push = []        # when the event that committed each round was pushed
    for k in range(n_rounds):
        mode = chr(int(h["round_mode"][k]))
        P = int(h["round_participants"][k])
        rh = int(h["round_n_roll"][k]) / P
        r_hats.append(rh)
        timeline.append(mode)
        started, commit = float(h["round_started"][k]), float(h["round_commit"][k])
        cons = mode == "P" and cfg.gamma * last_tdm > cfg.t_target
        n_conservative += cons
        push = float(h["round_dispatch"][k])
        if cons:
            t_t = cfg.t_target + cfg.t_target_slope * (P - 1)
            if float(h["round_draft_done"][k]) + d > push + t_t:
                push = float(h["round_draft_done"][k])   # committed by the reply DELIVERY
        commit_push.append(push)
        trace.append(RoundTrace(round=k + 1, started_at=started, committed_at=commit,
                                mode=mode, participants=P,
                                committed_delta=int(h["round_delta"][k]), r_hat=rh,
                                speculation_on=spec, timeout=False, conservative=cons,
                                breaker_streak=0, disabled_until=0))
        deltas_all_sum += int(h["round_delta"][k])
        deltas_all_n += P
        content_sum += int(h["round_content_sum"][k])
        content_n += int(h["round_content_n"][k])
        steady_rows.append((P, started, commit, int(h["round_delta"][k]),
                            int(h["round_content_sum"][k]), int(h["round_content_n"][k]), rh))
        q = int(h["round_queries"][k])
        if q > 0:
            counter = min(counter + 1, cfg.fairness_period)
            steps = cfg.gamma - 1 if mode == "O" else cfg.gamma
            draft_records.append(DraftRoundRecord(
                started_at=float(h["round_draft_start"][k]),
                finished_at=float(h["round_draft_done"][k]), n_speculative=q, n_regular=0,
                regular_pending_at_start=0, forced_regular=False,
                t_d_mix=mixed_step_latency(*lat[1:4], q),
                steps=steps, counter_after=counter))
            last_tdm = mixed_step_latency(*lat[1:4], q)
            n_queries += q
            draft_tokens += int(h["round_draft_tokens"][k])
    n = len(cpos)
    finished = {}
    for r in range(n):
        toks = [int(t) for t in committed[r, :int(cpos[r])]]
        finished[r] = RequestState(
            request=r, output_len=workload.output_len, committed_pos=int(cpos[r]),
            committed_tokens=toks, pending_bonus=toks[-1] if toks else None,
            prompt_len=workload.prompt_len, arrived_at=float(workload.arrival_times[r]),
            admitted_at=float(adm_at[r]), finished_at=float(fin_at[r]))
    t_end = float(h["round_commit"][-1]) if n_rounds else 0.0
    last_finish = max(fin_at.tolist()) if n else 0.0
    duration = last_finish if last_finish > 0 else t_end
    total = int(sum(int(x) for x in cpos))
    maxp = max((r[0] for r in steady_rows), default=0)
    steady = [r for r in steady_rows if r[0] == maxp]
    s_committed = sum(r[3] for r in steady)
    s_time = sum(r[2] - r[1] for r in steady)
    s_dn = sum(r[0] for r in steady)
    s_cs, s_cn = sum(r[4] for r in steady), sum(r[5] for r in steady)
    final_dispatch = commit_push[-1] if n_rounds else t_end
    hb_sent, hb_deliv = _heartbeat_counts(cfg.heartbeat_period, d, t_end, final_dispatch)
    closes = [float(t) for t in fin_at] if spec else []
    td_sent = 2 * n_queries + len(closes)
    td_deliv = 2 * n_queries + sum(1 for t in closes if t + d < t_end)
    tt_sent, tt_deliv = n_queries + hb_sent, n_queries + hb_deliv
    counters = {
        "to_draft": dict(sent=td_sent, delivered=td_deliv, dropped=0, stale=0, rejected=0),
        "to_target": dict(sent=tt_sent, delivered=tt_deliv, dropped=0, stale=0, rejected=0),
    }
    report = MetricsReport(
        variant=variant.value, seed=cfg.seed,
        target_throughput=(total / duration) if duration > 0 else 0.0,
        draft_throughput=(0 / duration) if duration > 0 else 0.0,
        mean_accepted_length=deltas_all_sum / deltas_all_n if deltas_all_n else 0.0,
        content_mean_accepted_length=content_sum / content_n if content_n else 0.0,
        mean_rollback_ratio=_mean(r_hats),
        rollback_ratio_series=tuple(r_hats),
        mode_timeline="".join(timeline),
        steady_rounds=len(steady),
        steady_target_throughput=(s_committed / s_time) if s_time > 0 else 0.0,
        steady_mean_accepted_length=s_committed / s_dn if s_dn else 0.0,
        steady_content_mean_accepted_length=s_cs / s_cn if s_cn else 0.0,
        steady_mean_rollback_ratio=_mean([r[6] for r in steady]),
        sim_duration=duration, total_committed=total, total_rounds=n_rounds,
        requests_completed=n, breaker_activations=0,
        fallback_rounds=sum(1 for m in timeline if m == "F"), timeout_rounds=0,
        conservative_rounds=n_conservative, transport_sent=td_sent + tt_sent,
        transport_delivered=td_deliv + tt_deliv, transport_dropped=0, transport_stale=0,
        transport_rejected=0, stale_replies=0, draft_tokens_generated=draft_tokens,
        background_tokens=0, background_completed=0)
    device_trace = dict(
        r_hat_ema=h["round_r_hat_ema"], accepted_len_ema=h["round_accepted_len_ema"],
        r_star=h["round_r_star"], n_padded=h["round_n_padded"], rng_draws=draws)
    return RunResult(report=report, config=cfg, variant=variant, round_trace=trace,
                     draft_records=draft_records, finished=finished, breaker_windows=[],
                     channel_counters=counters, lossless=lossless, device_trace=device_trace)


@dataclass(frozen=True)
class SweepEntry:
    variant: str
    axis: str
    axis_value: str
    replicate: int
    report: MetricsReport


def run_sweep(config: SimConfig, variants: Sequence, axis: str, points: Sequence,
              replicates: int = 1) -> list:
    """sim.py:1017-1046 — matched seeds across variants."""
    entries = []
    for label, overrides in points:
        for rep in range(replicates):
            point_cfg = config.with_overrides({**overrides, "seed": config.seed + rep})
            for v in variants:
                pv = PolicyVariant.parse(v) if isinstance(v, str) else v
                res = run(point_cfg, pv)
                report = dataclasses.replace(res.report, axis=axis, axis_value=label)
                entries.append(SweepEntry(pv.value, axis, label, rep, report))
    return entries
