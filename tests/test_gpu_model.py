"""Model-mode parity on the B200.

* forward numerics vs the fp32 PyTorch restatement (oracle/model_ref.py):
  final hidden state within bf16 tolerance; greedy tokens identical wherever
  the reference's top-2 logit margin exceeds 0.05 (tolerance stated here)
* batch invariance: a request's outputs are bit-identical whatever else
  shares the batch (what makes speculative decoding lossless here)
* losslessness end to end: ordinary / parallel / hybrid (SPECTRE) commit
  exactly the autoregressive greedy stream, for several draft-noise levels
"""

import pytest

pytestmark = pytest.mark.gpu

MARGIN = 0.05       # logit margin above which argmax must agree with fp32
X_RTOL = 3e-2       # final hidden state: |dx| <= X_RTOL * rms(x) (bf16 storage)


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_08151_b200 import model
    return model


def _forward_chunks(eng, which, prompts, chunk):
    import torch
    n, P = prompts.shape
    outs, xs = [], []
    for c0 in range(0, P, chunk):
        cs = min(chunk, P - c0)
        tok = prompts[:, c0:c0 + cs].reshape(-1)
        pos = torch.arange(c0, c0 + cs, device="cuda").repeat(n)
        slot = torch.arange(n, device="cuda").repeat_interleave(cs)
        q_off = torch.arange(n, device="cuda") * cs
        n_new = torch.full((n,), cs, device="cuda")
        pos0 = torch.full((n,), c0, device="cuda")
        o, x = eng.forward(which, tok, pos, slot, q_off, n_new, pos0, want_x=True)
        outs.append(o.view(n, cs))
        xs.append(x.view(n, cs, -1))
    return torch.cat(outs, 1), torch.cat(xs, 1)


@pytest.mark.parametrize("shapes", ["tiny", "small"])
def test_forward_vs_fp32_reference(M, shapes):
    import torch
    from oracle.model_ref import reference_forward
    tgt, drf = (M.TINY_TARGET, M.TINY_DRAFT) if shapes == "tiny" else (M.SMALL_TARGET,
                                                                        M.SMALL_DRAFT)
    n, P = 4, 40
    pair = M.build_pair(tgt, drf, n_req=n, ctx_cap=256, seed=3, target_branch=1.0,
                        draft_branch=1.0)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=P, seed=3)
    eng = M.SpectreEngine(pair, spec, "hybrid")
    prompts = M.synthetic_prompts(n, P, tgt.vocab, seed=3)
    for which, w in ((0, pair.target), (1, pair.draft)):
        toks, xs = _forward_chunks(eng, which, prompts, 8)
        for r in range(n):
            x_ref, logits = reference_forward(w, prompts[r])
            dx = (xs[r].float() - x_ref).abs()
            assert dx.max().item() <= X_RTOL * x_ref.pow(2).mean().sqrt().item() * 8
            assert dx.mean().item() <= X_RTOL * x_ref.abs().mean().item()
            top2 = logits.topk(2, -1).values
            clear = (top2[:, 0] - top2[:, 1]) > MARGIN
            assert torch.equal(toks[r][clear].long(), logits.argmax(-1)[clear])
            assert clear.float().mean().item() > 0.5


def test_forward_batch_invariance(M):
    import torch
    n, P = 6, 24
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=256, seed=5)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=P, seed=5)
    eng = M.SpectreEngine(pair, spec, "ar")
    prompts = M.synthetic_prompts(n, P, M.SMALL_TARGET.vocab, seed=5)
    full_tok, full_x = _forward_chunks(eng, 0, prompts, 8)
    # same requests, one token at a time (autoregressive shape), fresh KV
    toks, xs = _forward_chunks(eng, 0, prompts, 1)
    assert torch.equal(toks, full_tok)
    assert torch.equal(xs, full_x)
    # ragged: only request 2 participates, chunk of 3
    tok2, x2 = [], []
    for c0 in range(0, P, 3):
        cs = min(3, P - c0)
        tok = prompts[2, c0:c0 + cs]
        z = torch.zeros(n, dtype=torch.int32, device="cuda")
        n_new = z.clone()
        n_new[2] = cs
        pos0 = z.clone()
        pos0[2] = c0
        o, x = eng.forward(0, tok, torch.arange(c0, c0 + cs, device="cuda"),
                           torch.full((cs,), 2, device="cuda"), z, n_new, pos0, want_x=True)
        tok2.append(o)
        x2.append(x)
    assert torch.equal(torch.cat(tok2), full_tok[2])
    assert torch.equal(torch.cat(x2), full_x[2])


@pytest.mark.parametrize("alpha", [1.0, 0.7])
@pytest.mark.parametrize("shapes", ["tiny", "small"])
def test_speculative_decoding_is_lossless(M, shapes, alpha):
    import torch
    tgt, drf = (M.TINY_TARGET, M.TINY_DRAFT) if shapes == "tiny" else (M.SMALL_TARGET,
                                                                        M.SMALL_DRAFT)
    n = 8
    pair = M.build_pair(tgt, drf, n_req=n, ctx_cap=256, seed=7)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=96, prompt_len=32, alpha=alpha, seed=7)
    ar = M.decode(pair, spec, "ar")
    assert (ar.committed_pos == spec.output_len).all()
    for v in ("ordinary", "parallel", "hybrid"):
        for use_graph in (False, True):
            got = M.decode(pair, spec, v, use_graph=use_graph)
            assert (got.committed_pos == spec.output_len).all()
            assert torch.equal(got.committed, ar.committed), (v, use_graph)
            assert got.report.total_committed == n * spec.output_len


@pytest.mark.parametrize("chain", ["0", "1"])
def test_draft_per_op_and_chain_paths_agree(M, chain, monkeypatch):
    """The draft's decode step as persistent chains (default) and as per-op
    kernels (SPECTRE_DRAFT_CHAIN=0: split-K GEMMs in the half-SM config, RoPE /
    residual kernels) both give a lossless decode, and the draft's own
    forward matches the fp32 restatement either way."""
    import torch
    from oracle.model_ref import reference_forward
    monkeypatch.setenv("SPECTRE_DRAFT_CHAIN", chain)
    n = 8
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=256, seed=17)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=16, alpha=0.8, seed=17)
    ar = M.decode(pair, spec, "ar")
    got = M.decode(pair, spec, "hybrid")
    assert torch.equal(got.committed, ar.committed)
    eng = M.SpectreEngine(pair, spec, "hybrid")
    prompts = M.synthetic_prompts(n, 16, M.SMALL_TARGET.vocab, seed=17)
    cs = 4
    xs = []
    for c0 in range(0, 16, cs):
        tok = prompts[:, c0:c0 + cs].reshape(-1)
        pos = torch.arange(c0, c0 + cs, device="cuda").repeat(n)
        slot = torch.arange(n, device="cuda").repeat_interleave(cs)
        q_off = torch.arange(n, device="cuda") * cs
        _, x = eng.forward(1, tok, pos, slot, q_off, torch.full((n,), cs, device="cuda"),
                           torch.full((n,), c0, device="cuda"), want_x=True)
        xs.append(x.view(n, cs, -1))
    xs = torch.cat(xs, 1)
    for r in range(n):
        x_ref, _ = reference_forward(pair.draft, prompts[r])
        assert (xs[r].float() - x_ref).abs().mean().item() <= 3e-2 * x_ref.abs().mean().item()
    eng.close()


def test_device_graph_is_used(M):
    n = 4
    pair = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=n, ctx_cap=256, seed=2)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=16, seed=2)
    res = M.decode(pair, spec, "hybrid", use_graph=True)
    assert res.graph == 1, f"conditional WHILE/IF round graph was not used: {res.extra}"


def test_draft_noise_controls_acceptance(M):
    n = 16
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=512, seed=9)
    Ls = []
    for alpha in (1.0, 0.6, 0.2):
        spec = M.DecodeSpec(n_req=n, gamma=4, output_len=200, prompt_len=32, alpha=alpha, seed=9)
        res = M.decode(pair, spec, "ordinary")
        Ls.append(res.report.content_mean_accepted_length)
    assert Ls[0] > Ls[1] > Ls[2] >= 1.0


@pytest.mark.parametrize("chunk", [8, 12])
@pytest.mark.parametrize("attn_split", [128, 1024])
def test_long_context_forward_vs_fp32_reference(M, chunk, attn_split, monkeypatch):
    """Contexts past several attention key splits, 1-3 m-tiles per item."""
    import torch
    monkeypatch.setenv("SPECTRE_ATTN_CHUNK", str(attn_split))
    from oracle.model_ref import reference_forward
    n, P = 3, 600
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=704, seed=11,
                        target_branch=1.0, draft_branch=1.0)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=32, prompt_len=P, seed=11)
    eng = M.SpectreEngine(pair, spec, "hybrid")
    prompts = M.synthetic_prompts(n, P, M.SMALL_TARGET.vocab, seed=11)
    # the target's packed batch holds <= 8 new tokens per request, the draft's 12
    models = ((0, pair.target), (1, pair.draft)) if chunk <= 8 else ((1, pair.draft),)
    for which, w in models:
        toks, xs = _forward_chunks(eng, which, prompts, chunk)
        for r in range(n):
            x_ref, logits = reference_forward(w, prompts[r])
            dx = (xs[r].float() - x_ref).abs()
            assert dx.max().item() <= X_RTOL * x_ref.pow(2).mean().sqrt().item() * 8
            assert dx.mean().item() <= X_RTOL * x_ref.abs().mean().item()
            top2 = logits.topk(2, -1).values
            clear = (top2[:, 0] - top2[:, 1]) > MARGIN
            assert torch.equal(toks[r][clear].long(), logits.argmax(-1)[clear])


@pytest.mark.parametrize("which", [0, 1])
@pytest.mark.parametrize("attn_split", [128, 1024])
def test_long_context_batch_invariance(M, which, attn_split, monkeypatch):
    """Verify-shaped (5 / 12 new tokens) and one-token passes agree bit for bit
    across attention split boundaries."""
    import torch
    monkeypatch.setenv("SPECTRE_ATTN_CHUNK", str(attn_split))
    n, P = 4, 300
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=384, seed=13)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=32, prompt_len=P, seed=13)
    eng = M.SpectreEngine(pair, spec, "ar")
    prompts = M.synthetic_prompts(n, P, M.SMALL_TARGET.vocab, seed=13)
    ref_tok, ref_x = _forward_chunks(eng, which, prompts, 1)
    for chunk in ((5, 8) if which == 0 else (5, 12)):
        tok, x = _forward_chunks(eng, which, prompts, chunk)
        assert torch.equal(tok, ref_tok), chunk
        assert torch.equal(x, ref_x), chunk


def test_draft_prompt_compression_kv_and_losslessness(M):
    """Model-mode draft prompt compression (draft_engine.py:123-131, StreamingLLM
    head/tail retention): the draft's KV cache after prefill is exactly that of
    the compressed prompt (first and last keep tokens, re-indexed to positions
    0 .. 2 keep - 1), the target is untouched, and speculative decoding stays
    lossless."""
    import torch
    n, P = 8, 40
    pair = M.build_pair(M.SMALL_TARGET, M.SMALL_DRAFT, n_req=n, ctx_cap=256, seed=17)
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=P, seed=17,
                        compression_p=0.5)
    keep = spec.draft_prompt_keep()
    assert keep == 10
    prompts = M.synthetic_prompts(n, P, M.SMALL_TARGET.vocab, seed=17)
    eng = M.SpectreEngine(pair, spec, "ordinary")
    eng.prefill(prompts)
    torch.cuda.synchronize()
    kd = pair.draft.k_cache[:, :, :, :2 * keep].clone()
    vd = pair.draft.v_cache[:, :, :, :2 * keep].clone()
    kt = pair.target.k_cache[:, :, :, :P].clone()
    eng.close()
    comp = torch.cat([prompts[:, :keep], prompts[:, P - keep:]], 1).contiguous()
    ref_spec = M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=2 * keep, seed=17)
    ref = M.SpectreEngine(pair, ref_spec, "ordinary")
    ref.prefill(comp)
    torch.cuda.synchronize()
    assert torch.equal(pair.draft.k_cache[:, :, :, :2 * keep], kd)
    assert torch.equal(pair.draft.v_cache[:, :, :, :2 * keep], vd)
    ref.close()
    # the target saw the whole prompt
    full = M.SpectreEngine(pair, M.DecodeSpec(n_req=n, gamma=4, output_len=64, prompt_len=P,
                                              seed=17), "ordinary")
    full.prefill(prompts)
    torch.cuda.synchronize()
    assert torch.equal(pair.target.k_cache[:, :, :, :P], kt)
    full.close()
    ar = M.decode(pair, spec, "ar", prompts=prompts)
    for v in ("ordinary", "parallel", "hybrid"):
        got = M.decode(pair, spec, v, prompts=prompts)
        assert torch.equal(got.committed, ar.committed), v
