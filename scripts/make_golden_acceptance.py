"""Generate tests/golden/acceptance.json: the UNMODIFIED reference's
`specsim verify` criteria 1-5 (acceptance.py) — pass flags and detail lines.

Runs only in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden_acceptance.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "acceptance.json"


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF))
    from specsim import acceptance  # noqa: E402
    out = {}
    for fn in (acceptance.criterion_1_formula_fidelity, acceptance.criterion_2_crossover_identity,
               acceptance.criterion_3_sim_model_agreement, acceptance.criterion_4_hybrid_dominance,
               acceptance.criterion_5_accepted_length_ordering):
        t0 = time.time()
        r = fn()
        out[str(r.cid)] = dict(name=r.name, passed=r.passed, detail=r.detail)
        print(f"{r.cid} {r.name} {r.passed} ({time.time() - t0:.1f}s)", flush=True)
    OUT.write_text(json.dumps(out, indent=1))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
