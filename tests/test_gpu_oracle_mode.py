"""Oracle-mode parity on the B200: the device decode loop vs the reference.

Every golden case (generated from the unmodified reference by
scripts/make_golden.py) must come out of `paper_2605_08151_b200.run` with
identical report bytes, round traces, draft-round records, transport counters
and committed tokens — and the device K8 kernels must reproduce the stream
KATs, the draft RNG and the oracle's verify/propose semantics.
"""

import hashlib
import json
import random

import numpy as np
import pytest

from oracle import lockstep as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2605_08151_b200 as P
    return P


def test_stream_kats_on_device(pkg, golden_streams):
    kat = golden_streams["kat"]
    for seed in sorted({k[0] for k in kat}):
        for stream in (0, 1):
            rows = [k for k in kat if k[0] == seed and k[1] == stream]
            got = pkg.TokenStreamOracle(seed).reference_tokens(
                [r[2] for r in rows], [r[3] for r in rows], stream_id=stream)
            assert [int(x) for x in got] == [int(r[4]) for r in rows]


def test_draft_uniforms_on_device(pkg, golden_streams):
    from paper_2605_08151_b200.decoder import draft_uniforms
    for seed, vals in golden_streams["draft_uniforms"].items():
        got = draft_uniforms(int(seed), len(vals)).cpu().numpy()
        assert [repr(float(x)) for x in got] == vals
    # long stream crosses many twists
    r = random.Random("3:draft")
    want = np.array([r.random() for _ in range(50_000)])
    got = draft_uniforms(3, 50_000).cpu().numpy()
    assert np.array_equal(got, want)


def test_verify_and_propose_batches(pkg):
    rng = random.Random(11)
    o = pkg.TokenStreamOracle(5)
    reqs, starts, cands, lens = [], [], [], []
    for _ in range(300):
        req, start, cnt = rng.randrange(64), rng.randrange(0, 900), rng.randrange(1, 9)
        seg = L.draft_propose(5, req, start, cnt, 0.6, rng)
        if rng.random() < 0.2:
            seg = seg[:1] + [L.PAD] * (cnt - 1)
        reqs.append(req), starts.append(start), lens.append(cnt)
        cands.append(seg + [L.PAD] * (8 - cnt))
    acc, bonus = o.verify_batch(reqs, starts, np.array(cands, dtype=np.uint64), lens)
    for i in range(len(reqs)):
        a, _, b, _ = L.verify(5, reqs[i], starts[i], cands[i][:lens[i]])
        assert (int(acc[i]), int(bonus[i])) == (a, b)
    u = [rng.random() for _ in range(sum(lens))]
    got = o.propose_batch(reqs, starts, lens, 0.7, u)
    off = 0
    for i in range(len(reqs)):
        want = [L.reference_token(5, reqs[i], starts[i] + j) if u[off + j] < 0.7
                else L.reference_token(5, reqs[i], starts[i] + j) ^ L.DISAGREE
                for j in range(lens[i])]
        assert [int(x) for x in got[i, :lens[i]]] == want
        off += lens[i]
    # scalar duck type used by reference code
    assert o.reference_prefix(1, 5) == [L.reference_token(5, 1, i) for i in range(5)]
    out = o.verify(1, 0, [L.reference_token(5, 1, 0), 7])
    assert (out.accepted_count, out.new_position) == (1, 2)


@pytest.mark.parametrize("idx", range(51))
def test_device_decode_loop_matches_reference(pkg, golden_runs, idx):
    case = golden_runs[idx]
    cfg = pkg.SimConfig(**case["config"])
    wl = None
    if case["arrivals"] is not None:
        wl = pkg.Workload(tuple(case["arrivals"]), cfg.output_len, cfg.prompt_len)
    res = pkg.run(cfg, case["variant"], workload=wl)
    assert pkg.export_report(res.report) == case["report_csv"], case["name"]
    assert [vars(t) for t in res.round_trace] == case["round_trace"]
    assert [vars(t) for t in res.draft_records] == case["draft_records"]
    assert res.channel_counters == case["channel_counters"]
    assert res.lossless
    committed = {str(r): [str(t) for t in s.committed_tokens]
                 for r, s in sorted(res.finished.items())}
    if case["committed"] is not None:
        assert committed == case["committed"]
    digest = hashlib.sha256(json.dumps(committed, sort_keys=True).encode()).hexdigest()
    assert digest == case["committed_sha256"]


@pytest.mark.parametrize("idx", range(14))
def test_device_loop_draft_model_matches_reference(pkg, golden_runs_draft_model, idx):
    """Prompt compression + draft contention model (§8f rows 2-3, fault-free
    part): the CUDA loop reproduces the reference's reports, traces and every
    draft round's T_D^mix."""
    test_device_decode_loop_matches_reference(pkg, golden_runs_draft_model, idx)


@pytest.mark.parametrize("idx", range(24))
def test_device_loop_conservative_matches_reference(pkg, golden_runs_conservative, idx):
    """a10: conservative parallel rounds on the device loop (the commit waits
    for the replies; simulated clock in IEEE doubles, no FMA)."""
    test_device_decode_loop_matches_reference(pkg, golden_runs_conservative, idx)


def test_device_loop_outside_domain_refused(pkg):
    with pytest.raises(pkg.OutsideDeviceDomain):
        pkg.run(pkg.SimConfig(batch_size=4, n_requests=4, output_len=8, drop_prob=0.1), "hybrid")
    with pytest.raises(pkg.OutsideDeviceDomain):   # conservative replies miss the deadline
        pkg.run(pkg.SimConfig(batch_size=4, n_requests=4, output_len=8, t_draft=0.03), "parallel")


def test_device_loop_large_batch_against_oracle(pkg):
    # C3-shaped protocol (B=256) with trickling admission, checked against the oracle
    cfg = dict(batch_size=256, n_requests=300, gamma=4, output_len=96, alpha=0.78,
               qps=2000.0, seed=21)
    for v in ("ordinary", "parallel", "hybrid"):
        want = L.run(cfg, v)
        got = pkg.run(pkg.SimConfig(**cfg), v)
        assert pkg.export_report(got.report) == L.export_csv(want.report)
