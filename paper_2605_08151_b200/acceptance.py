"""Acceptance battery, criteria 1-5 of the reference's `specsim verify`
(acceptance.py:40-232), run against this package: criteria 1-2 check the
closed-form model (`analytics`), criteria 3-5 drive the CUDA decode loop
(`run` / `run_sweep`, oracle mode) on B200.  Tolerances are the reference's:

  1 formula fidelity        thr_ord 1476.92, thr_par 1664.0, r* 0.34615 (rel 1e-6)
  2 crossover identity      1000 random draws: |thr_par(r*) - thr_ord| <= 1e-9 rel,
                            sign flip across r*
  3 sim-model agreement     B in {1,16,32,64,128}, alpha=1, zero delay: steady
                            ordinary throughput within 2 % of the model,
                            parallel within 5 %
  4 hybrid dominance        crossover sweep (9 alphas x 5 replicates):
                            hybrid >= 0.97 x max(ordinary, parallel)
  5 accepted-length order   per alpha: ordinary >= hybrid >= parallel, strict
                            somewhere

Detail lines use the reference's wording, so a run here can be compared with
the reference's own `specsim verify` output line for line
(`tests/golden/acceptance.json`, made by `scripts/make_golden_acceptance.py`).
Criteria 6-11 exercise subsystems outside the device path (transport chaos,
the multi-tenant draft scheduler, prompt compression, pricing) and are not
restated.

  python -m paper_2605_08151_b200.acceptance [--criteria 1 2 3 4 5]
"""

from __future__ import annotations

import argparse
import functools
import random
from dataclasses import dataclass

from . import analytics
from .core import SimConfig
from .decoder import PolicyVariant, Workload, run, run_sweep


@dataclass(frozen=True)
class CriterionResult:
    cid: int
    name: str
    passed: bool
    detail: str


def _rel_err(value: float, expected: float) -> float:
    return abs(value) if expected == 0 else abs(value - expected) / abs(expected)


def criterion_1_formula_fidelity() -> CriterionResult:
    """acceptance.py:40-65: the model at B=32, L=3, gamma=4, T_T=50 ms, T_D=5 ms."""
    base = dict(batch_size=32, accepted_len=3.0, gamma=4, t_target=0.050, t_draft=0.005)
    thr_ord = analytics.ordinary_throughput(analytics.ThroughputParams(**base))
    thr_par = analytics.parallel_throughput(
        analytics.ThroughputParams(**base, fallback_ratio=0.2))
    r_star = analytics.critical_fallback_ratio(analytics.ThroughputParams(**base))
    ok = (_rel_err(thr_ord, 96.0 / 0.065) <= 1e-6 and round(thr_ord, 2) == 1476.92 and
          _rel_err(thr_par, 1664.0) <= 1e-6 and
          _rel_err(r_star, 0.045 / 0.13) <= 1e-6 and round(r_star, 5) == 0.34615)
    return CriterionResult(1, "formula-fidelity", ok,
                           f"thr_ord={thr_ord:.6f} (expect 1476.92...), thr_par={thr_par:.6f} "
                           f"(expect 1664.0), r*={r_star:.6f} (expect 0.34615...)")


def criterion_2_crossover_identity(draws_wanted: int = 1000) -> CriterionResult:
    """acceptance.py:71-119: at r = r* parallel and ordinary throughput agree,
    and the preference flips sign across it (seeded random parameter draws)."""
    rng = random.Random(20240817)
    worst, flips_ok, draws, attempts = 0.0, True, 0, 0
    while draws < draws_wanted and attempts < 100_000:
        attempts += 1
        batch = rng.randint(1, 256)
        acc = rng.uniform(1.01, 8.0)
        gamma = rng.randint(2, 8)
        t_t = rng.uniform(0.001, 0.2)
        t_d = rng.uniform(1e-5, t_t)
        p = analytics.ThroughputParams(batch_size=batch, accepted_len=acc, gamma=gamma,
                                       t_target=t_t, t_draft=t_d)
        r_star = analytics.critical_fallback_ratio(p)
        if not 1e-9 < r_star < 0.999:
            continue
        draws += 1
        thr_ord = analytics.ordinary_throughput(p)

        def par(r):
            return analytics.parallel_throughput(analytics.ThroughputParams(
                batch_size=batch, accepted_len=acc, gamma=gamma, t_target=t_t, t_draft=t_d,
                fallback_ratio=r))

        worst = max(worst, _rel_err(par(r_star), thr_ord))
        lo, hi = r_star * (1.0 - 1e-3), r_star + (1.0 - r_star) * 1e-3
        if not (par(lo) > thr_ord and par(hi) < thr_ord):
            flips_ok = False
    ok = draws == draws_wanted and worst <= 1e-9 and flips_ok
    return CriterionResult(2, "crossover-identity", ok,
                           f"{draws} draws, worst |thr_par(r*) - thr_ord| relative gap "
                           f"{worst:.3e} (<= 1e-9), sign flip at r*: {flips_ok}")


def criterion_3_sim_model_agreement(batches=(1, 16, 32, 64, 128)) -> CriterionResult:
    """acceptance.py:125-176: alpha = 1, zero transport delay, all requests at
    t=0; the device loop's steady throughput vs the closed-form model."""
    ok, lines = True, []
    for b in batches:
        cfg = SimConfig(batch_size=b, n_requests=b, alpha=1.0, output_len=256, qps=1e6,
                        delay_dist="constant:0", seed=0)
        wl = Workload((0.0,) * b, output_len=cfg.output_len)
        rep_o = run(cfg, PolicyVariant.ORDINARY, workload=wl).report
        model_o = analytics.ordinary_throughput(analytics.ThroughputParams(
            batch_size=b, accepted_len=rep_o.steady_content_mean_accepted_length,
            gamma=cfg.gamma, t_target=cfg.t_target, t_draft=cfg.t_draft))
        rep_p = run(cfg, PolicyVariant.PARALLEL, workload=wl).report
        model_p = analytics.parallel_throughput(analytics.ThroughputParams(
            batch_size=b, accepted_len=rep_p.steady_content_mean_accepted_length,
            gamma=cfg.gamma, t_target=cfg.t_target, t_draft=cfg.t_draft,
            fallback_ratio=min(1.0, rep_p.steady_mean_rollback_ratio)))
        e_o = _rel_err(rep_o.steady_target_throughput, model_o)
        e_p = _rel_err(rep_p.steady_target_throughput, model_p)
        ok = ok and e_o <= 0.02 and e_p <= 0.05
        lines.append(f"B={b}: ord err {e_o:.4f} (<=0.02), par err {e_p:.4f} (<=0.05)")
    return CriterionResult(3, "sim-model-agreement", ok, "; ".join(lines))


# the `crossover` preset (presets.py:30-43, 64-81): alphas chosen so the
# zero-reuse rollback estimate 1 - alpha^gamma lands on these r-hat targets
CROSSOVER_TARGETS = (0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.8, 0.95)
CROSSOVER_BASE = dict(batch_size=32, n_requests=32, output_len=256, qps=1e6, gamma=4)


def crossover_points(gamma: int = 4) -> list[tuple[str, dict]]:
    pts = []
    for r_hat in CROSSOVER_TARGETS:
        alpha = round((1.0 - r_hat) ** (1.0 / gamma), 5)
        pts.append((f"{alpha:.5f}", {"alpha": alpha}))
    return pts


@functools.lru_cache(maxsize=1)
def _crossover_entries():
    cfg = SimConfig().with_overrides(dict(CROSSOVER_BASE))
    return tuple(run_sweep(cfg, ["ar", "ordinary", "parallel", "hybrid"], "alpha",
                           crossover_points(), replicates=5))


def _by_point(entries, metric: str) -> dict:
    sums: dict = {}
    for e in entries:
        sums.setdefault(e.axis_value, {}).setdefault(e.variant, []).append(
            getattr(e.report, metric))
    return {lab: {v: sum(xs) / len(xs) for v, xs in per.items()} for lab, per in sums.items()}


def criterion_4_hybrid_dominance() -> CriterionResult:
    """acceptance.py:206-216: hybrid >= 0.97 x the better fixed mode per alpha."""
    ok, lines = True, []
    for lab, m in _by_point(_crossover_entries(), "target_throughput").items():
        ratio = m["hybrid"] / max(m["ordinary"], m["parallel"])
        ok = ok and ratio >= 0.97
        lines.append(f"alpha={lab}: hybrid/max={ratio:.4f}")
    return CriterionResult(4, "hybrid-dominance", ok,
                           "; ".join(lines) + " (threshold 0.97, 5 replicates)")


def criterion_5_accepted_length_ordering() -> CriterionResult:
    """acceptance.py:219-232: mean accepted length ordinary >= hybrid >= parallel
    at every alpha, strictly somewhere."""
    ok, strict, lines = True, False, []
    for lab, m in _by_point(_crossover_entries(), "mean_accepted_length").items():
        o, h, p = m["ordinary"], m["hybrid"], m["parallel"]
        ok = ok and o >= h - 1e-9 and h >= p - 1e-9
        strict = strict or o > h + 1e-6 or h > p + 1e-6
        lines.append(f"alpha={lab}: O={o:.3f} H={h:.3f} P={p:.3f}")
    return CriterionResult(5, "accepted-length-ordering", ok and strict, "; ".join(lines))


CRITERIA = {
    1: criterion_1_formula_fidelity,
    2: criterion_2_crossover_identity,
    3: criterion_3_sim_model_agreement,
    4: criterion_4_hybrid_dominance,
    5: criterion_5_accepted_length_ordering,
}


def run_all(ids=tuple(CRITERIA)) -> list[CriterionResult]:
    return [CRITERIA[i]() for i in ids]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--criteria", type=int, nargs="+", default=list(CRITERIA))
    args = ap.parse_args(argv)
    results = run_all(args.criteria)
    for r in results:
        print(f"[{'PASS' if r.passed else 'FAIL'}] {r.cid:2d} {r.name}: {r.detail}")
    return 0 if all(r.passed for r in results) else 1


if __name__ == "__main__":
    raise SystemExit(main())
