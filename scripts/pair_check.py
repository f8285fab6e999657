"""CTA-pair (cta_group::2) GEMM vs the single-CTA kernel and an fp32 reference."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
torch.manual_seed(0)
for N, K in ((1024, 512), (28672, 4096)):
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    X = torch.randn(512, K, device="cuda").bfloat16()
    for T in (16, 100, 256):
        outs = {}
        for flags in (2000, 4000):
            act = torch.zeros(512, N // 2, dtype=torch.bfloat16, device="cuda")
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K, 1, 2,
                                              None, None, None, act.data_ptr(), N // 2, flags,
                                              _native.stream_ptr()), "gemm")
            torch.cuda.synchronize()
            outs[flags] = act[:T].float()
        ref = (X[:T].float() @ W.float().t()).view(T, N // 2, 2)
        ref = torch.nn.functional.silu(ref[..., 0]) * ref[..., 1]
        err = lambda o: ((o - ref).abs().max() / ref.abs().max()).item()
        same = torch.equal(outs[2000], outs[4000])
        print(f"N={N} K={K} T={T}: single err {err(outs[2000]):.2e} pair err {err(outs[4000]):.2e} "
              f"bit-identical {same}", flush=True)
