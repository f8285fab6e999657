"""Host-side logic of the product package, on CPU (no compute calls).

* libspectre.so loads and exports every symbol include/spectre.h declares
* the MT19937 seeding entry point reproduces CPython's random.Random state
* config validation and the report schema round-trip reference CSVs byte-exact
* the host accounting that turns the device round trace into the reference's
  RunResult reproduces every golden report when fed the oracle's per-round rows
"""

import random
import re

import numpy as np
import pytest

from oracle import lockstep as L
from paper_2605_08151_b200 import (REPORT_COLUMNS, ConfigError, SimConfig, export_report,
                                   import_report, validate_config)
from paper_2605_08151_b200 import _native
from paper_2605_08151_b200.decoder import (PolicyVariant, Workload, _assemble_result,
                                           draft_rng_key)
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    text = "\n".join(p.read_text() for p in (ROOT / "include").glob("*.h"))
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spectre_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = _declared_symbols()
    assert len(syms) >= 9
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert _native.version().startswith("spectre-b200")


@pytest.mark.parametrize("seed", [0, 1, 7, 42, 2**40 + 3, -5])
def test_mt19937_seed_state_matches_cpython(seed):
    lib = _native.lib()
    key = np.asarray(draft_rng_key(seed), dtype=np.uint32)
    st = np.zeros(625, dtype=np.uint32)
    _native.check(lib.spectre_mt19937_init_by_array(key.ctypes.data, len(key), st.ctypes.data),
                  "init")
    assert list(st) == list(random.Random(f"{seed}:draft").getstate()[1])


def test_config_validation_messages():
    with pytest.raises(ConfigError, match="gamma must be >= 1"):
        validate_config(SimConfig(gamma=0))
    cfg, warnings = validate_config(SimConfig(gamma=20))
    assert warnings and "overlap assumption violated" in warnings[0]
    assert cfg.reply_timeout == 2 * cfg.t_target
    assert SimConfig().with_overrides({"batch_size": "7"}).batch_size == 7
    with pytest.raises(ConfigError):
        SimConfig().with_overrides({"nope": 1})


def test_report_roundtrip_reference_csv(golden_runs):
    assert len(REPORT_COLUMNS) == 33
    for case in golden_runs:
        rep = import_report(case["report_csv"])
        assert export_report(rep) == case["report_csv"]
        assert import_report(export_report(rep, "json"), "json") == rep


@pytest.mark.parametrize("idx", range(51))
def test_host_accounting_reproduces_reference_reports(golden_runs, idx):
    """Feed _assemble_result the per-round rows the device kernel emits (here
    taken from the oracle) and require the reference's report bytes."""
    case = golden_runs[idx]
    lr = L.run(case["config"], case["variant"], arrivals=case["arrivals"])
    cfg, _ = validate_config(SimConfig(**case["config"]))
    arrivals = case["arrivals"] or L.generate_arrivals(cfg.qps, cfg.n_requests,
                                                       random.Random(f"{cfg.seed}:workload"))
    wl = Workload(tuple(arrivals), cfg.output_len, cfg.prompt_len)
    rows = lr.rounds
    h = {
        "round_mode": np.array([ord(r["mode"]) for r in rows]),
        "round_participants": np.array([r["participants"] for r in rows]),
        "round_delta": np.array([r["delta"] for r in rows]),
        "round_n_roll": np.array([r["n_roll"] for r in rows]),
        "round_content_sum": np.array([r["content_sum"] for r in rows]),
        "round_content_n": np.array([r["content_n"] for r in rows]),
        "round_queries": np.array([r["queries"] for r in rows]),
        "round_draft_tokens": np.array([r["draft_tokens"] for r in rows]),
        "round_n_padded": np.array([r["n_padded"] for r in rows]),
        "round_started": np.array([r["started"] for r in rows]),
        "round_dispatch": np.array([r["dispatch"] for r in rows]),
        "round_commit": np.array([r["commit"] for r in rows]),
        "round_draft_start": np.array([r["draft_start"] for r in rows]),
        "round_draft_done": np.array([r["draft_done"] for r in rows]),
        "round_r_hat_ema": np.array([r["r_hat_ema"] for r in rows]),
        "round_accepted_len_ema": np.array([r["accepted_len_ema"] for r in rows]),
        "round_r_star": np.zeros(len(rows)),
    }
    n = len(arrivals)
    OL = cfg.output_len
    cpos = np.array([len(lr.committed[r]) for r in range(n)])
    committed = np.zeros((n, OL), dtype=np.uint64)
    for r in range(n):
        committed[r, :cpos[r]] = np.array(lr.committed[r], dtype=np.uint64)
    adm = np.array([lr.times[r][0] for r in range(n)])
    fin = np.array([lr.times[r][1] for r in range(n)])
    d = L.constant_delay(L.resolve(case["config"]))
    res = _assemble_result(cfg, PolicyVariant.parse(case["variant"]), wl, d, h, cpos, fin, adm,
                           committed, True, lr.rng_draws)
    assert export_report(res.report) == case["report_csv"], case["name"]
    assert [vars(t) for t in res.round_trace] == case["round_trace"]
    assert [vars(t) for t in res.draft_records] == case["draft_records"]
    assert res.channel_counters == case["channel_counters"]


def test_bench_round_roofline_matches_survey_figures():
    """bench.py's whole-round roofline uses SURVEY §8d's algorithmic bytes:
    P_T = 7,504,658,432, P_D = 1,235,746,816, KV 131,072 / 32,768 B per token,
    C2 ordinary round (ctx 640) = 20.38 + 3 x 3.81 GB."""
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench
    from paper_2605_08151_b200 import model as M
    t, d = M.LLAMA_31_8B, M.LLAMA_32_1B
    assert bench.linear_params(t) == 7_504_658_432
    assert bench.linear_params(d) == 1_235_746_816
    assert bench.kv_bytes_per_token(t) == 131_072
    assert bench.kv_bytes_per_token(d) == 32_768
    bt = 2 * bench.linear_params(t) + 64 * 640 * bench.kv_bytes_per_token(t)
    bd = 2 * bench.linear_params(d) + 64 * 640 * bench.kv_bytes_per_token(d)
    assert abs(bt / 1e9 - 20.38) < 0.01 and abs(bd / 1e9 - 3.81) < 0.01


def test_acceptance_criteria_1_2_closed_form():
    """The reference's `specsim verify` criteria 1-2 (acceptance.py:40-119)
    against this package's closed-form model."""
    import json
    from paper_2605_08151_b200 import acceptance as A
    golden = json.loads((Path(__file__).parent / "golden" / "acceptance.json").read_text())
    for r in A.run_all((1, 2)):
        assert r.passed, r
        assert (r.name, r.detail) == (golden[str(r.cid)]["name"], golden[str(r.cid)]["detail"])
