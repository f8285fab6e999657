"""GEMM time vs token count for fixed weight shapes (CUDA events, weights rotated past L2)."""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
for name, N, K, epi, splits in (("gate_up 8B", 28672, 4096, 2, 1), ("lm_head 1B", 128256, 2048, 1, 1),
                                ("down 8B", 4096, 14336, 0, 9)):
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(512, K, device="cuda").bfloat16()
    part = torch.empty(splits, 512, N, device="cuda")
    av = torch.empty((N + 31) // 32, 512, device="cuda")
    ai = torch.empty((N + 31) // 32, 512, dtype=torch.int32, device="cuda")
    act = torch.empty(512, N // 2, dtype=torch.bfloat16, device="cuda")
    for T in (16, 64, 128, 256):
        row = []
        for flag in ((0, 2000) if epi else (0,)):
            ts = []
            for it in range(20):
                W = Ws[it % copies]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K,
                                                  splits, epi, part.data_ptr(), av.data_ptr(),
                                                  ai.data_ptr(), act.data_ptr(), N // 2, flag,
                                                  _native.stream_ptr()), "g")
                e1.record(); e1.synchronize()
                if it >= 4: ts.append(e0.elapsed_time(e1) * 1e3)
            t = statistics.median(ts)
            row.append(f"{'sk' if flag == 0 and epi else 'plain'} {t:7.1f} us {N*K*2/t/1e3:6.0f} GB/s")
        print(f"{name:11s} T={T:3d}: " + " | ".join(row), flush=True)
    del Ws
    torch.cuda.empty_cache()
