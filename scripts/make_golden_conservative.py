"""Generate tests/golden/runs_conservative.json from the UNMODIFIED reference:
conservative parallel rounds (gamma * T_D^mix > T_T, sim.py:143-146, 599-606)
whose replies land before the reply deadline — the commit waits for them.

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden_conservative.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import REF, OUT  # noqa: E402


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import hashlib

    import specsim  # noqa: E402
    from specsim.metrics import export_report  # noqa: E402

    cases = []

    def add(name, variant, cfg):
        res = specsim.run(specsim.SimConfig(**cfg), variant)
        csv = export_report(res.report, "csv")
        committed = {str(r): [str(t) for t in s.committed_tokens]
                     for r, s in sorted(res.finished.items())}
        digest = hashlib.sha256(json.dumps(committed, sort_keys=True).encode()).hexdigest()
        cases.append(dict(
            name=name, variant=variant, config=cfg, arrivals=None, report_csv=csv,
            round_trace=[vars(t) for t in res.round_trace],
            draft_records=[vars(r) for r in res.draft_records],
            channel_counters=res.channel_counters, committed=committed,
            committed_sha256=digest, lossless=res.lossless,
            conservative_rounds=res.report.conservative_rounds))

    # gamma * T_D > T_T with default latencies (gamma >= 11), slow drafts at
    # gamma 4 / 6, a contention slope, trickling arrivals, a batch-dependent T_T
    grid = [
        ("g12", dict(gamma=12)),
        ("g16", dict(gamma=16, alpha=0.9)),
        ("td15", dict(gamma=4, t_draft=0.015)),
        ("td20_g4", dict(gamma=4, t_draft=0.02, alpha=0.7)),
        ("td12_g6", dict(gamma=6, t_draft=0.012)),
        ("slope", dict(gamma=10, t_draft=0.0052, t_draft_slope=0.0001, t_draft_free_batch=4)),
        ("tslope", dict(gamma=8, t_draft=0.0075, t_target_slope=0.001)),
        ("trickle", dict(gamma=12, qps=40.0, n_requests=12, batch_size=6)),
    ]
    for tag, over in grid:
        cfg = dict(batch_size=8, n_requests=8, output_len=64, alpha=0.8, qps=1e6, seed=2)
        cfg.update(over)
        for v in ("ordinary", "parallel", "hybrid"):
            add(f"cons_{tag}_{v}", v, cfg)
    assert all(c["conservative_rounds"] > 0 for c in cases if c["variant"] != "ordinary")
    (OUT / "runs_conservative.json").write_text(json.dumps({"cases": cases}))
    print(f"wrote {len(cases)} conservative runs")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
