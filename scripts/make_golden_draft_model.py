"""Generate tests/golden/runs_draft_model.json from the UNMODIFIED reference:
runs with draft-side prompt compression (draft_engine.py:123-131, 205-216) and
the draft contention model (mixed_step_latency, draft_engine.py:158-164) —
the §8f rows 2-3 parts that stay inside the fault-free lockstep domain (no
background tenants).  Same schema as runs.json (scripts/make_golden.py).

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden_draft_model.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "runs_draft_model.json"


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
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
            report_sha16=hashlib.sha256(csv.encode()).hexdigest()[:16],
            round_trace=[vars(t) for t in res.round_trace],
            draft_records=[vars(r) for r in res.draft_records],
            channel_counters=res.channel_counters, committed=None,
            committed_sha256=digest, lossless=res.lossless))

    variants = ("ordinary", "parallel", "hybrid")
    for p in (0.5, 0.8):                         # compression: alpha_eff, latency factor
        cfg = dict(batch_size=8, n_requests=8, output_len=64, alpha=0.8, qps=1e6, seed=13,
                   compression_p=p)
        for v in variants:
            add(f"compress_p{p}_{v}", v, cfg)
    cfg = dict(batch_size=16, n_requests=16, output_len=64, alpha=0.8, qps=1e6, seed=14,
               t_draft_slope=0.0002, t_draft_free_batch=4)     # contention model
    for v in variants:
        add(f"contention_{v}", v, cfg)
    cfg = dict(batch_size=12, n_requests=20, output_len=48, alpha=0.75, qps=40.0, seed=15,
               compression_p=0.6, compression_beta=0.2, compression_latency_frac=0.4,
               t_draft_slope=0.0003, t_draft_free_batch=2)     # both, trickling arrivals
    for v in variants:
        add(f"both_{v}", v, cfg)
    for seed in (0, 1):                          # crossover region: T_D^mix moves r*
        cfg = dict(batch_size=32, n_requests=32, gamma=4, output_len=256, alpha=0.79,
                   qps=1e6, seed=seed, t_draft_slope=0.00008, t_draft_free_batch=8,
                   compression_p=0.7)
        add(f"xover_dm_s{seed}_hybrid", "hybrid", cfg)
    OUT.write_text(json.dumps({"cases": cases}))
    print(f"wrote {len(cases)} runs to {OUT}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
