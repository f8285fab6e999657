"""Background (regular) tenants on the draft model and the speculative-priority
fairness scheduler (draft_engine.py:134-155, 302-394).

* speculative decoding stays lossless under background load;
* the device's per-round schedule (regular items served with the speculation,
  forced regular rounds, FairnessCounter) equals a replay through the CPU
  restatement of the reference's schedule_round (oracle/scheduler.py, pinned
  to the reference by tests/golden/scheduler.json);
* a background request's tokens are the draft model's own greedy stream:
  identical whatever the speculative traffic around it (batch invariance) and
  equal to the fp32 restatement's argmax where its margin is clear.
"""

import pytest

pytestmark = pytest.mark.gpu

N_REQ, N_BG, BG_LEN = 8, 6, 40


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_08151_b200 import model
    return model


@pytest.fixture(scope="module")
def pair(M):
    return M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=N_REQ, ctx_cap=256, seed=19,
                        n_bg=N_BG)


def _spec(M, **kw):
    base = dict(n_req=N_REQ, gamma=4, output_len=64, prompt_len=16, alpha=0.8, seed=19,
                background_requests=N_BG, background_output_len=BG_LEN, fairness_period=3,
                draft_capacity=N_REQ + 2)
    base.update(kw)
    return M.DecodeSpec(**base)


def test_lossless_under_background_load(M, pair):
    import torch
    spec = _spec(M)
    ar = M.decode(pair, spec, "ar")
    for v in ("ordinary", "parallel", "hybrid"):
        got = M.decode(pair, spec, v)
        assert torch.equal(got.committed, ar.committed), v
        assert got.report.background_tokens > 0, v


@pytest.mark.parametrize("variant,cap", [("ordinary", N_REQ + 2), ("parallel", N_REQ + 2),
                                         ("ordinary", N_REQ)])
def test_schedule_matches_reference_scheduler(M, pair, variant, cap):
    from oracle.scheduler import replay_phases
    spec = _spec(M, draft_capacity=cap)
    res = M.decode(pair, spec, variant)
    tr = res.trace
    steps = spec.gamma - 1 if variant == "ordinary" else spec.gamma
    n = len(tr["mode"])
    # every active request is queried in these pure modes (parallel: all; ordinary:
    # the cache-less ones, which is all of them after the first round)
    got = list(zip(tr["n_forced"].tolist(), tr["n_regular"].tolist(),
                   tr["fair_counter"].tolist()))
    want, remaining = replay_phases(tr["participants"].tolist(), N_BG, BG_LEN, [steps] * n,
                                    spec.fairness_period, cap)
    assert got == want
    emitted = res.extra["background_emitted"]
    n_tok, n_done = res.report.background_tokens, res.report.background_completed
    assert emitted.cpu().tolist() == [BG_LEN - r for r in remaining]
    assert n_tok == sum(BG_LEN - r for r in remaining)
    assert n_done == sum(1 for r in remaining if r == 0)
    if cap == N_REQ:
        # no capacity beside the speculation while every request is active:
        # regular work moves only in forced rounds; between two of them exactly
        # fairness_period speculative draft rounds run (criterion 7's bound on
        # the speculative streak with regular work pending, acceptance.py:270-334)
        full = [i for i, p in enumerate(tr["participants"].tolist()) if p == N_REQ]
        assert all(got[i][1] == 0 for i in full)
        forced_rounds = [i for i in full if got[i][0] > 0]
        assert len(forced_rounds) >= 2 and all(
            b - a == spec.fairness_period for a, b in zip(forced_rounds, forced_rounds[1:]))


def test_background_tokens_are_the_drafts_greedy_stream(M, pair):
    import torch
    from oracle.model_ref import reference_forward
    a = M.decode(pair, _spec(M), "ordinary")
    b = M.decode(pair, _spec(M, draft_capacity=N_REQ + 5), "parallel")
    ta, ea = a.extra["background_tokens"], a.extra["background_emitted"]
    tb, eb = b.extra["background_tokens"], b.extra["background_emitted"]
    for j in range(N_BG):
        k = int(min(ea[j], eb[j]))
        assert k > 0
        assert torch.equal(ta[j, :k], tb[j, :k]), j   # independent of the traffic around it
    prompts = M.synthetic_prompts(N_BG, 16, M.SMALL_DRAFT.vocab, seed=19, req0=1_000_000)
    for j in range(N_BG):
        k = int(ea[j])
        seq = torch.cat([prompts[j].long(), ta[j, :k].long()])
        _, logits = reference_forward(pair.draft, seq)
        pred = logits[15:15 + k]                         # next-token predictions
        top2 = pred.topk(2, -1).values
        clear = (top2[:, 0] - top2[:, 1]) > 0.05
        assert torch.equal(ta[j, :k][clear].long(), pred.argmax(-1)[clear]), j
