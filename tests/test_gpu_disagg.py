"""Config 5 (disaggregated draft server + target shards) against the
single-engine decode loop: same prompts, seeds and (deterministic) controller
-> bit-identical committed streams and round modes.  Here both sides share
cuda:0; on a multi-GPU box the same exchanges are NVLink peer copies."""

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_08151_b200 import model
    return model


def _spec(M, n, **kw):
    base = dict(n_req=n, gamma=4, output_len=64, prompt_len=16, alpha=0.8, seed=21,
                controller="reference")
    base.update(kw)
    return M.DecodeSpec(**base)


@pytest.mark.parametrize("variant", ["ordinary", "parallel", "hybrid", "ar"])
def test_single_shard_matches_engine(M, variant):
    import torch
    from paper_2605_08151_b200.disagg import DisaggregatedDecoder
    n = 8
    pair = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=n, ctx_cap=256, seed=21)
    spec = _spec(M, n)
    ref = M.decode(pair, spec, variant, use_graph=False)
    dd = DisaggregatedDecoder(pair, [(pair, n)], spec, variant)
    dd.prefill(M.synthetic_prompts(n, spec.prompt_len, M.TINY_TARGET.vocab, spec.seed))
    dd.run()
    committed, pos, traces = dd.read()
    assert (pos == spec.output_len).all()
    assert torch.equal(committed, ref.committed.cpu())
    assert (traces[0]["mode"] == ref.trace["mode"]).all()


@pytest.mark.parametrize("variant", ["ordinary", "parallel"])
def test_two_target_shards_match_engine(M, variant):
    import torch
    from paper_2605_08151_b200.disagg import DisaggregatedDecoder
    n = 8
    pair = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=n, ctx_cap=256, seed=22)
    spec = _spec(M, n, seed=22)
    ref = M.decode(pair, spec, variant, use_graph=False)
    # separate target replicas (own KV) for shards of 3 and 5 requests
    t1 = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=3, ctx_cap=256, seed=22)
    t2 = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=5, ctx_cap=256, seed=22)
    dd = DisaggregatedDecoder(pair, [(t1, 3), (t2, 5)], spec, variant)
    dd.prefill(M.synthetic_prompts(n, spec.prompt_len, M.TINY_TARGET.vocab, spec.seed))
    dd.run()
    committed, pos, _ = dd.read()
    assert (pos == spec.output_len).all()
    assert torch.equal(committed, ref.committed.cpu())
