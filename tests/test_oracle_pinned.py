"""Pin the CPU oracle (oracle/lockstep.py) to the reference's own vectors.

* frozen hash values from the reference test suite (tests/test_oracle.py:15-34)
* 240 extra stream KATs + draft-RNG uniforms generated from the reference
* 51 complete reference runs (reports, round traces, draft records, transport
  counters, committed tokens), including the four CLI goldens whose sha256
  fingerprints SURVEY §4 lists.
"""

import hashlib
import json
import random

import pytest

from oracle import lockstep as L


def test_frozen_values_from_reference_suite():
    # /root/reference/pkg/tests/test_oracle.py:15-34
    assert [L.reference_token(0, 0, i) for i in range(5)] == [
        10749833864783185041, 6642847197101178724, 7036274279819827101,
        16062445039872724754, 3348389343249159457]
    assert [L.reference_token(7, 0, i) for i in range(3)] == [
        4115426874723844861, 1025521192397269246, 773058809683055316]
    assert [L.prompt_token(0, 0, i) for i in range(3)] == [
        7741979081032095418, 5817724158014739623, 2388804026663013211]


def test_stream_kats(golden_streams):
    for seed, stream, req, pos, val in golden_streams["kat"]:
        fn = L.reference_token if stream == 0 else L.prompt_token
        assert fn(seed, req, pos) == int(val)


def test_draft_uniform_fixture(golden_streams):
    for seed, vals in golden_streams["draft_uniforms"].items():
        r = random.Random(f"{seed}:draft")
        assert [repr(r.random()) for _ in range(len(vals))] == vals


def test_cli_golden_fingerprints(golden_runs):
    # sha256[:16] of the four `specsim verify --write-golden` reports
    want = {"ar": "18080d98ce9603aa", "ordinary": "e61993ec62047313",
            "parallel": "9203ae75a68fd6b2", "hybrid": "e489748d0793d6af"}
    for case in golden_runs:
        if case["name"].startswith("cli_golden_"):
            v = case["variant"]
            r = L.run(case["config"], v, arrivals=case["arrivals"])
            csv = L.export_csv(r.report)
            assert hashlib.sha256(csv.encode()).hexdigest()[:16] == want[v]


def _committed_json(committed):
    return {str(k): [str(t) for t in v] for k, v in sorted(committed.items())}


@pytest.mark.parametrize("idx", range(51))
def test_lockstep_matches_reference_run(golden_runs, idx):
    case = golden_runs[idx]
    r = L.run(case["config"], case["variant"], arrivals=case["arrivals"])
    assert L.export_csv(r.report) == case["report_csv"], case["name"]
    assert r.round_trace == case["round_trace"]
    assert r.draft_records == case["draft_records"]
    assert r.channel_counters == case["channel_counters"]
    assert r.lossless and case["lossless"]
    cj = _committed_json(r.committed)
    if case["committed"] is not None:
        assert cj == case["committed"]
    digest = hashlib.sha256(json.dumps(cj, sort_keys=True).encode()).hexdigest()
    assert digest == case["committed_sha256"]


@pytest.mark.parametrize("idx", range(14))
def test_lockstep_matches_reference_draft_model(golden_runs_draft_model, idx):
    """Draft prompt compression and the contention latency model (§8f rows 2-3,
    fault-free part): reports, round traces and draft records equal the
    reference's, including every round's T_D^mix."""
    test_lockstep_matches_reference_run(golden_runs_draft_model, idx)


@pytest.mark.parametrize("idx", range(24))
def test_lockstep_matches_reference_conservative(golden_runs_conservative, idx):
    """a10: conservative parallel rounds (gamma * T_D^mix > T_T, sim.py:143-146,
    599-606) — the commit waits for the replies; conservative flags in the
    trace and the report's conservative_rounds equal the reference's."""
    test_lockstep_matches_reference_run(golden_runs_conservative, idx)


def test_verify_semantics():
    # /root/reference/pkg/tests/test_oracle.py:119-178
    cand = [L.reference_token(0, 1, i) for i in range(4)]
    assert L.verify(0, 1, 0, cand) == (4, tuple(L.reference_token(0, 1, i) for i in range(5)),
                                       L.reference_token(0, 1, 4), 5)
    bad = [L.reference_token(0, 1, 0), L.reference_token(0, 1, 1) ^ 1, L.reference_token(0, 1, 2)]
    acc, committed, bonus, newpos = L.verify(0, 1, 0, bad)
    assert (acc, newpos, bonus) == (1, 2, L.reference_token(0, 1, 1))
    assert L.verify(0, 0, 0, (L.PAD, L.PAD, L.PAD))[0] == 0
    assert L.verify(0, 6, 0, (12345,))[:2] == (0, (L.reference_token(0, 6, 0),))


def test_out_of_domain_is_refused():
    with pytest.raises(L.OutOfDomain):
        L.run(dict(batch_size=4, n_requests=4, output_len=8, drop_prob=0.1), "hybrid")
    with pytest.raises(L.OutOfDomain):
        L.run(dict(batch_size=4, n_requests=4, output_len=8, gamma=1), "ordinary")
    # contention makes this round's T_D^mix exceed the last reply's: the
    # (non-conservative) parallel replies would land after the commit
    with pytest.raises(L.OutOfDomain):
        L.run(dict(batch_size=8, n_requests=8, output_len=16, gamma=8, qps=1e6,
                   t_draft_slope=0.0002), "parallel")
    # conservative round whose replies miss the reply deadline (timeouts)
    with pytest.raises(L.OutOfDomain):
        L.run(dict(batch_size=4, n_requests=4, output_len=8, t_draft=0.03), "parallel")


def test_scheduler_restatement_matches_reference():
    """oracle/scheduler.py:schedule_round == the reference's schedule_round
    (draft_engine.py:134-155) on 400 random queues (tests/golden/scheduler.json)."""
    from pathlib import Path

    from oracle import scheduler as S
    golden = Path(__file__).resolve().parent / "golden" / "scheduler.json"
    for c in json.loads(golden.read_text())["cases"]:
        spec, reg, counter, forced = S.schedule_round(list(range(c["n_spec"])),
                                                      list(range(c["n_reg"])), c["counter"],
                                                      c["period"], c["capacity"])
        assert (spec, reg, counter, forced) == (c["spec"], c["reg"], c["counter_after"],
                                                c["forced"]), c
