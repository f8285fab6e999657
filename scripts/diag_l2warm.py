"""Split-K GEMM time with weights L2-warm (same matrix back to back) vs cold
(rotated past L2): is the launch weight-stream bound?  diag_l2warm.py"""
import statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
for name, N, K, splits, flags in (("down", 4096, 14336, 9, 0), ("qkv", 6144, 4096, 3, 1000),
                                  ("o", 4096, 4096, 4, 1000), ("down_half", 4096, 7168, 9, 0)):
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(512, K, device="cuda").bfloat16()
    part = torch.empty(splits, 512, N, device="cuda")
    s = torch.cuda.Stream()
    for mode in ("cold", "warm"):
        ts = []
        for it in range(40):
            W = Ws[it % copies] if mode == "cold" else Ws[0]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, 256, 512, N, K,
                                              splits, 0, part.data_ptr(), None, None, None, 0,
                                              flags, int(s.cuda_stream)), "gemm")
            e1.record(s)
            e1.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        t = statistics.median(ts)
        print(f"{name} N={N} K={K} splits={splits} {mode}: {t:.2f} us  {N*K*2/t/1e3:.0f} GB/s", flush=True)
