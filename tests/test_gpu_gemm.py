"""tcgen05 weight-streaming GEMM vs a plain PyTorch fp32 reference.

Tolerance: inputs are bf16, accumulation fp32 on both sides; only the
summation order differs, so |err| <= 2e-3 * (|x|.|w| row norm) suffices.
Batch invariance (row t identical for any token count T) is checked bit-exact:
it is what makes the speculative stream equal the autoregressive one.
"""

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu

PARTIAL, ARGMAX, SWIGLU = 0, 1, 2


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_08151_b200 import _native
    L = _native.lib()
    fn = L.spectre_gemm_bf16
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p] * 3 + [C.c_int32] * 6 + [C.c_void_p] * 4 + [C.c_int32] * 2 + \
        [C.c_void_p]
    return torch, _native, fn


def _run(env, X, W, T, rows_cap, splits=1, epi=PARTIAL, t_dev=None, max_stages=0):
    torch, _native, fn = env
    N, K = W.shape
    dev = X.device
    part = torch.zeros(splits, rows_cap, N, dtype=torch.float32, device=dev)
    n_blocks = _native.lib().spectre_gemm_argmax_blocks(N, W.shape[1])
    av = torch.zeros(n_blocks, rows_cap, dtype=torch.float32, device=dev)
    ai = torch.zeros(n_blocks, rows_cap, dtype=torch.int32, device=dev)
    act = torch.zeros(rows_cap, max(N // 2, 1), dtype=torch.bfloat16, device=dev)
    st = fn(X.data_ptr(), W.data_ptr(), t_dev.data_ptr() if t_dev is not None else None, T,
            rows_cap, N, K, splits, epi, part.data_ptr(), av.data_ptr(), ai.data_ptr(),
            act.data_ptr(), act.shape[1], max_stages, _native.stream_ptr())
    _native.check(st, "spectre_gemm_bf16")
    torch.cuda.synchronize()
    return part, av, ai, act


def _ref(torch, X, W, T):
    return X[:T].float() @ W.float().t()


@pytest.mark.parametrize("T,rows_cap,N,K,splits", [
    (1, 64, 256, 64, 1), (16, 64, 384, 512, 1), (64, 64, 1024, 2048, 2),
    (37, 64, 640, 1024, 3), (256, 256, 6144, 4096, 3), (200, 256, 512, 4096, 4),
    (320, 320, 1024, 4096, 4), (512, 512, 256, 256, 1), (130, 192, 768, 1024, 1),
    (700, 768, 384, 512, 2), (1280, 1280, 256, 1024, 1), (300, 320, 640, 2048, 3),
    (256, 256, 28672 // 8, 4096, 1), (77, 128, 1000, 640, 2)])
# 0: defaults (BK=64, 256-row tiles); -8: BK=32 (64B swizzle); 1000: 128-row tiles;
# 3000: half-SM config (128-row tiles, 4 epilogue warps, 2 CTAs per SM)
@pytest.mark.parametrize("bk_flag", [0, -8, 1000, 3000])
def test_partial_matches_fp32(env, T, rows_cap, N, K, splits, bk_flag):
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(T * 7 + N)
    X = torch.randn(rows_cap, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    part, *_ = _run(env, X, W, T, rows_cap, splits, max_stages=bk_flag)
    got = part.sum(0)[:T]
    want = _ref(torch, X, W, T)
    scale = (X[:T].float().abs() @ W.float().abs().t()) + 1e-3
    assert ((got - want).abs() / scale).max().item() < 2e-3


def test_runtime_token_count_and_stage_variants(env):
    torch = env[0]
    X = torch.randn(256, 1024, device="cuda").bfloat16()
    W = (torch.randn(512, 1024, device="cuda") * 0.05).bfloat16()
    want = _ref(torch, X, W, 96)
    for stages in (1, 2, 3, 8, 1002):
        t_dev = torch.tensor([96], dtype=torch.int32, device="cuda")
        part, *_ = _run(env, X, W, 0, 256, 2, t_dev=t_dev, max_stages=stages)
        got = part.sum(0)[:96]
        assert torch.allclose(got, want, atol=5e-2, rtol=1e-2)


def test_batch_invariance_bitwise(env):
    """Row t of Y must be bit-identical whatever the number of tokens T."""
    torch = env[0]
    X = torch.randn(320, 2048, device="cuda").bfloat16()
    W = (torch.randn(1024, 2048, device="cuda") * 0.05).bfloat16()
    outs = {}
    for T in (1, 5, 16, 64, 100, 256, 320):
        part, *_ = _run(env, X, W, T, 320, 2)
        outs[T] = part[:, :T].clone()
    for T, o in outs.items():
        assert torch.equal(o[:, :1], outs[320][:, :1])
        assert torch.equal(o, outs[320][:, :T])


def test_argmax_epilogue(env):
    torch = env[0]
    V, K, T = 128256 - 96, 2048, 70
    torch.manual_seed(5)
    X = torch.randn(128, K, device="cuda").bfloat16()
    W = (torch.randn(V, K, device="cuda") * 0.02).bfloat16()
    _, av, ai, _ = _run(env, X, W, T, 128, 1, ARGMAX)
    best = av[:, :T].argmax(0)
    idx = ai[:, :T].gather(0, best[None]).squeeze(0).long()
    logits = _ref(torch, X, W, T)
    want = logits.argmax(1)
    top2 = logits.topk(2, dim=1).values
    margin = (top2[:, 0] - top2[:, 1])
    clear = margin > 1e-2
    assert torch.equal(idx[clear], want[clear])
    assert clear.float().mean().item() > 0.8   # top-2 gaps of 128k random logits: ~5 % < 1e-2
    # the reported max equals the fp32 logit at the chosen index (within tolerance)
    got_max = av[:, :T].max(0).values
    assert torch.allclose(got_max, logits.gather(1, idx[:, None]).squeeze(1), atol=2e-3, rtol=1e-3)


def test_multipass_argmax_and_swiglu(env):
    torch = env[0]
    X = torch.randn(1024, 512, device="cuda").bfloat16()
    W = (torch.randn(1024, 512, device="cuda") * 0.05).bfloat16()
    T = 900
    _, av, ai, _ = _run(env, X, W, T, 1024, 1, ARGMAX)
    best = av[:, :T].argmax(0)
    idx = ai[:, :T].gather(0, best[None]).squeeze(0).long()
    logits = _ref(torch, X, W, T)
    top2 = logits.topk(2, dim=1).values
    clear = (top2[:, 0] - top2[:, 1]) > 1e-2
    assert torch.equal(idx[clear], logits.argmax(1)[clear])
    _, _, _, act = _run(env, X, W, T, 1024, 1, SWIGLU)
    g = _ref(torch, X, W.view(512, 2, 512)[:, 0], T)   # rows [g0, u0, g1, u1, ...]
    u = _ref(torch, X, W.view(512, 2, 512)[:, 1], T)
    assert torch.allclose(act[:T].float(), torch.nn.functional.silu(g) * u, atol=3e-2, rtol=2e-2)


def test_swiglu_epilogue(env):
    torch = env[0]
    F, K, T = 512, 1024, 48
    X = torch.randn(64, K, device="cuda").bfloat16()
    Wg = (torch.randn(F, K, device="cuda") * 0.05).bfloat16()
    Wu = (torch.randn(F, K, device="cuda") * 0.05).bfloat16()
    # interleave per row pair: [g0, u0, g1, u1, ...]
    W = torch.stack([Wg, Wu], 1).reshape(2 * F, K)
    _, _, _, act = _run(env, X, W.contiguous(), T, 64, 1, SWIGLU)          # stream-K
    _, _, _, act256 = _run(env, X, W.contiguous(), T, 64, 1, SWIGLU, max_stages=2000)
    _, _, _, act128 = _run(env, X, W.contiguous(), T, 64, 1, SWIGLU, max_stages=1000)
    _, _, _, acth = _run(env, X, W.contiguous(), T, 64, 1, SWIGLU, max_stages=3000)
    # rows >= T are unread padding (the 32-token store boxes may write them)
    assert torch.equal(act256[:T], act128[:T])   # same full-K order, different tiling
    assert torch.equal(acth[:T], act128[:T])     # half-SM config: same arithmetic
    assert torch.allclose(act[:T].float(), act256[:T].float(), atol=1e-2, rtol=1e-2)
    g = _ref(torch, X, Wg, T)
    u = _ref(torch, X, Wu, T)
    want = torch.nn.functional.silu(g) * u
    assert torch.allclose(act[:T, :F].float(), want, atol=3e-2, rtol=2e-2)


@pytest.mark.parametrize("epi", [ARGMAX, SWIGLU])
@pytest.mark.parametrize("N,K", [(28672 // 4, 4096), (128256 // 8 - 4, 2048), (1024, 1024)])
def test_stream_k_batch_invariance_bitwise(env, epi, N, K):
    if epi == SWIGLU and N % 128:
        N -= N % 128
    """Stream-K cut points depend on (N, K, grid) only: a token's result is
    bit-identical for any token count, and matches the fp32 reference."""
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(N + K + epi)
    X = torch.randn(256, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.03).bfloat16()
    outs = {}
    for T in (1, 7, 64, 130, 256):
        _, av, ai, act = _run(env, X, W, T, 256, 1, epi)
        outs[T] = (av[:, :T].clone(), ai[:, :T].clone()) if epi == ARGMAX else act[:T].clone()
    for T in (1, 7, 64, 130):
        if epi == ARGMAX:
            assert torch.equal(outs[T][0], outs[256][0][:, :T])
            assert torch.equal(outs[T][1], outs[256][1][:, :T])
        else:
            assert torch.equal(outs[T], outs[256][:T])
    logits = _ref(torch, X, W, 256)
    if epi == ARGMAX:
        av, ai = outs[256]
        idx = ai.gather(0, av.argmax(0)[None]).squeeze(0).long()
        top2 = logits.topk(2, dim=1).values
        clear = (top2[:, 0] - top2[:, 1]) > 1e-2
        assert torch.equal(idx[clear], logits.argmax(1)[clear])
    else:
        Wv = W.view(N // 2, 2, K)
        gt = _ref(torch, X, Wv[:, 0], 256)
        ut = _ref(torch, X, Wv[:, 1], 256)
        want = torch.nn.functional.silu(gt) * ut
        assert torch.allclose(outs[256].float()[:, :N // 2], want, atol=3e-2, rtol=2e-2)


def test_argmax_no_stale_partials(env):
    """Back-to-back launches with different inputs (stream-K contributor CTAs
    write no argmax slot of their own): every result must be fresh."""
    torch = env[0]
    V, K = 32000, 1024
    W = (torch.randn(V, K, device="cuda") * 0.03).bfloat16()
    for seed in range(3):
        g = torch.Generator(device="cuda").manual_seed(seed)
        X = torch.randn(64, K, device="cuda", generator=g).bfloat16()
        for T in (32, 5, 64):
            _, av, ai, _ = _run(env, X, W, T, 64, 1, ARGMAX)
            idx = ai[:, :T].gather(0, av[:, :T].argmax(0)[None]).squeeze(0).long()
            logits = _ref(torch, X, W, T)
            top2 = logits.topk(2, dim=1).values
            clear = (top2[:, 0] - top2[:, 1]) > 1e-2
            assert torch.equal(idx[clear], logits.argmax(1)[clear]), (seed, T)


@pytest.mark.parametrize("T", [16, 100, 256, 300, 512])
def test_cta_pair_swiglu_at_8b_gate_up(env, T):
    """The verify gate/up GEMM exactly as the engine launches it at the 8B
    shape (N = 2*14336, K = 4096): CTA pairs (cta_group::2, flag 4000; past 256
    tokens in 256-token chunks: config 3's verify, prefill) must be
    bit-identical to the single-CTA 256-row kernel (flag 2000: same per-row
    k order) and within bf16 tolerance of the fp32 reference."""
    torch = env[0]
    N, K = 2 * 14336, 4096
    g = torch.Generator(device="cuda").manual_seed(T)
    X = torch.randn(512, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    _, _, _, single = _run(env, X, W, T, 512, 1, SWIGLU, max_stages=2000)
    _, _, _, pair = _run(env, X, W, T, 512, 1, SWIGLU, max_stages=4000)
    assert torch.equal(pair[:T], single[:T])
    Wv = W.view(N // 2, 2, K)
    gt = _ref(torch, X, Wv[:, 0], T)
    ut = _ref(torch, X, Wv[:, 1], T)
    want = torch.nn.functional.silu(gt) * ut
    # bf16 output: 2^-8 relative, plus tanh.approx SiLU (~2^-11)
    assert torch.allclose(pair[:T].float(), want, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("N,K,T", [(2 * 14336, 4096, 100), (2 * 14336, 4096, 300),
                                   (2 * 14336, 4096, 1000), (2 * 27648, 5120, 128),
                                   (2 * 27648, 5120, 896)])
def test_cta_pair_units_swiglu(env, N, K, T):
    """CTA pairs scheduled as (tile pair, 256-token chunk) units over every SM
    (flag 9000: config 3's and config 5's verify gate/up, 112 and 216 tiles of
    256 rows) are bit-identical to the single-CTA 256-row kernel and within
    bf16 tolerance of the fp32 reference."""
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(T + N)
    X = torch.randn(1024, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    _, _, _, single = _run(env, X, W, T, 1024, 1, SWIGLU, max_stages=2000)
    _, _, _, pair = _run(env, X, W, T, 1024, 1, SWIGLU, max_stages=9000)
    assert torch.equal(pair[:T], single[:T])
    Wv = W.view(N // 2, 2, K)
    want = torch.nn.functional.silu(_ref(torch, X, Wv[:, 0], T)) * _ref(torch, X, Wv[:, 1], T)
    assert torch.allclose(pair[:T].float(), want, atol=2e-2, rtol=1e-2)


@pytest.mark.parametrize("N,K,T,S", [(4096, 14336, 1280, 3), (4096, 4096, 300, 2),
                                     (5120, 27648, 896, 4), (7168, 5120, 896, 3)])
def test_cta_pair_units_partial(env, N, K, T, S):
    """Split-K partial GEMMs as CTA pairs over (tile pair, split, 256-token
    chunk) units (flag 9000): every split's partial bit-identical to the
    single-CTA 256-row kernel with the same split ranges, and the split sum
    within fp32-accumulation tolerance of the reference."""
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(T + N + S)
    RC = (T + 63) // 64 * 64
    X = torch.randn(RC, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    single, _, _, _ = _run(env, X, W, T, RC, S, PARTIAL, max_stages=2000)
    pair, _, _, _ = _run(env, X, W, T, RC, S, PARTIAL, max_stages=9000)
    assert torch.equal(pair[:, :T], single[:, :T])
    want = _ref(torch, X, W, T)
    assert torch.allclose(pair[:, :T].sum(0), want, atol=1e-2, rtol=1e-3)


def _argmax_of_slots(torch, av, ai, T):
    """(max, lowest index) over the per-(CTA, warp) partial slots of T tokens."""
    v, i = av[:, :T], ai[:, :T]
    m = v.max(0).values
    big = torch.full_like(i, 2 ** 31 - 1)
    return m, torch.where(v == m[None], i, big).min(0).values


@pytest.mark.parametrize("T", [128, 300, 896])
def test_cta_pair_units_argmax_at_152k_vocab(env, T):
    """Greedy lm_head as CTA pairs over (tile pair, 256-token chunk) units
    (flag 9000; Qwen2.5-32B's head: V = 152064 = 594 tiles of 256 rows, each CTA
    covering scattered chunks): the (max, lowest index) of every token equals the
    single-CTA 256-row kernel's, and the fp32 argmax where the top-2 margin is
    clear."""
    torch = env[0]
    V, K = 152064, 5120
    g = torch.Generator(device="cuda").manual_seed(V + T)
    RC = (T + 63) // 64 * 64
    X = torch.randn(RC, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, K, device="cuda", generator=g) * 0.02).bfloat16()
    _, av1, ai1, _ = _run(env, X, W, T, RC, 1, ARGMAX, max_stages=2000)
    _, av2, ai2, _ = _run(env, X, W, T, RC, 1, ARGMAX, max_stages=9000)
    m1, i1 = _argmax_of_slots(torch, av1, ai1, T)
    m2, i2 = _argmax_of_slots(torch, av2, ai2, T)
    assert torch.equal(m1, m2) and torch.equal(i1, i2)
    logits = _ref(torch, X, W, T)
    top2 = logits.topk(2, dim=1).values
    clear = (top2[:, 0] - top2[:, 1]) > 1e-2
    assert torch.equal(i2[clear].long(), logits.argmax(1)[clear])


@pytest.mark.parametrize("T", [20, 256])
def test_lm_head_argmax_at_128k_vocab(env, T):
    """Greedy lm_head at V = 128256, K = 4096 (the 8B target's head: several
    256-row tiles per CTA) against the fp32 argmax."""
    torch = env[0]
    V, K = 128256, 4096
    g = torch.Generator(device="cuda").manual_seed(V + T)
    X = torch.randn(256, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, K, device="cuda", generator=g) * 0.02).bfloat16()
    _, av, ai, _ = _run(env, X, W, T, 256, 1, ARGMAX, max_stages=2000)
    idx = ai[:, :T].gather(0, av[:, :T].argmax(0)[None]).squeeze(0).long()
    logits = _ref(torch, X, W, T)
    top2 = logits.topk(2, dim=1).values
    clear = (top2[:, 0] - top2[:, 1]) > 1e-2
    assert torch.equal(idx[clear], logits.argmax(1)[clear])
    assert clear.float().mean().item() > 0.8
