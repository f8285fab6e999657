"""Generate tests/golden/*.json from the UNMODIFIED reference package.

Runs only in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden.py

The fixtures pin (a) the oracle restatement in oracle/lockstep.py and (b) the
CUDA product path, on the GPU box where the reference is absent.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    import specsim  # noqa: E402
    from specsim.metrics import export_report  # noqa: E402
    from specsim.oracle import TokenStreamOracle  # noqa: E402
    from specsim.sim import Workload  # noqa: E402

    OUT.mkdir(parents=True, exist_ok=True)

    # (1) known-answer vectors for the token streams (tests/test_oracle.py:15-34
    # pins the first five; we add more coordinates and the prompt stream).
    kat = []
    for seed in (0, 7, 123456789, 2**63 + 5):
        o = TokenStreamOracle(seed=seed)
        for req in (0, 1, 63, 255, 100000):
            for pos in (0, 1, 2, 17, 1023, 1151):
                kat.append([seed, 0, req, pos, str(o.reference_token(req, pos))])
                kat.append([seed, 1, req, pos, str(o.prompt_token(req, pos))])
    # (2) MT19937 uniforms of the draft stream, random.Random("{seed}:draft").
    mt = {}
    for seed in (0, 1, 7, 42):
        r = random.Random(f"{seed}:draft")
        mt[str(seed)] = [repr(r.random()) for _ in range(2000)]
    (OUT / "streams.json").write_text(json.dumps({"kat": kat, "draft_uniforms": mt}))

    # (3) full runs.
    cases = []

    def add(name, variant, cfg, workload=None, full_tokens=True):
        res = specsim.run(specsim.SimConfig(**cfg), variant, workload=workload)
        csv = export_report(res.report, "csv")
        committed = {str(r): [str(t) for t in s.committed_tokens]
                     for r, s in sorted(res.finished.items())}
        digest = hashlib.sha256(json.dumps(committed, sort_keys=True).encode()).hexdigest()
        cases.append(dict(
            name=name, variant=variant, config=cfg,
            arrivals=list(workload.arrival_times) if workload is not None else None,
            report_csv=csv,
            report_sha16=hashlib.sha256(csv.encode()).hexdigest()[:16],
            round_trace=[vars(t) for t in res.round_trace],
            draft_records=[vars(r) for r in res.draft_records],
            channel_counters=res.channel_counters,
            committed=committed if full_tokens else None,
            committed_sha256=digest,
            lossless=res.lossless,
        ))

    variants = ("ar", "ordinary", "parallel", "hybrid")
    golden = dict(batch_size=4, n_requests=4, output_len=32, alpha=0.8, qps=1e6, seed=7)
    for v in variants:                                   # cli.py:248-255 goldens
        add(f"cli_golden_{v}", v, golden)
    for seed in (0, 1):                                  # BASELINE config 1
        for alpha in (0.6, 0.8):
            cfg = dict(batch_size=8, n_requests=8, gamma=4, output_len=64,
                       alpha=alpha, qps=1e6, seed=seed)
            for v in variants:
                add(f"c1_s{seed}_a{alpha}_{v}", v, cfg)
    for gamma in (2, 8):
        cfg = dict(batch_size=8, n_requests=8, gamma=gamma, output_len=48,
                   alpha=0.7, qps=1e6, seed=3)
        for v in variants:
            add(f"g{gamma}_{v}", v, cfg)
    # trickling arrivals + admission cap (queueing)
    cfg = dict(batch_size=4, n_requests=12, output_len=40, alpha=0.8, qps=8.0, seed=5)
    for v in variants:
        add(f"trickle_{v}", v, cfg)
    # all-zero arrivals (exact time ties with the heartbeat chain)
    cfg = dict(batch_size=8, n_requests=8, output_len=32, alpha=0.8, qps=1e6, seed=0)
    wl = Workload((0.0,) * 8, output_len=32)
    for v in variants:
        add(f"zero_{v}", v, cfg, workload=wl)
    # crossover-region hybrid (the controller switches both ways)
    for seed in (0, 1, 2):
        cfg = dict(batch_size=32, n_requests=32, gamma=4, output_len=256,
                   alpha=0.79, qps=1e6, seed=seed)
        for v in ("ordinary", "parallel", "hybrid"):
            add(f"xover_s{seed}_{v}", v, cfg, full_tokens=False)
    # batch-dependent T_T, fixed L threshold, short outputs
    add("slope_hybrid", "hybrid", dict(batch_size=16, n_requests=16, output_len=64,
                                       alpha=0.75, qps=1e6, seed=9,
                                       t_target_slope=0.001))
    add("fixedL_hybrid", "hybrid", dict(batch_size=16, n_requests=16, output_len=64,
                                        alpha=0.7, qps=1e6, seed=4,
                                        fixed_threshold_l=2.5))
    add("short_parallel", "parallel", dict(batch_size=8, n_requests=8, output_len=2,
                                           alpha=0.9, qps=1e6, seed=2))
    # BASELINE C2 protocol shape (B=64, gamma=4) in oracle mode
    for v in ("ordinary", "parallel", "hybrid"):
        add(f"c2shape_{v}", v, dict(batch_size=64, n_requests=64, gamma=4,
                                    output_len=128, alpha=0.8, qps=1e6, seed=11),
            full_tokens=False)
    (OUT / "runs.json").write_text(json.dumps({"cases": cases}))
    print(f"wrote {len(kat)} KATs, {len(cases)} runs to {OUT}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
