"""Draft-step GEMMs (Llama-3.2-1B shapes, T = 64 tokens) launched back to back
over 16 distinct weight matrices (one per layer, > L2 in total), CUDA events
on the launching stream: the per-launch floor of the split-K weight streamers
without the glue kernels between them.

    python scripts/time_draft_gemms.py
"""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native

L = _native.lib()
T, NL = 64, 16
s = torch.cuda.Stream()
X = torch.randn(512, 8192, device="cuda").bfloat16()
for name, N, K, splits, flags in (("qkv", 3072, 2048, 12, 3000), ("o", 2048, 2048, 10, 3000),
                                  ("down", 2048, 8192, 12, 3000), ("gate_up", 16384, 2048, 1, 1000)):
    W = torch.randn(NL, N, K, device="cuda").mul_(0.02).bfloat16()
    Xk = X[:, :K].contiguous()
    part = torch.empty(splits, 512, N, device="cuda")
    act = torch.empty(512, max(N // 2, 1), dtype=torch.bfloat16, device="cuda")
    epi = 2 if name == "gate_up" else 0

    def launch(l):
        _native.check(L.spectre_gemm_bf16(Xk.data_ptr(), W[l].data_ptr(), None, T, 512, N, K,
                                          splits, epi, part.data_ptr(), None, None,
                                          act.data_ptr(), max(N // 2, 1), flags,
                                          int(s.cuda_stream)), "gemm")
    times = []
    with torch.cuda.stream(s):
        for l in range(NL):
            launch(l)
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for l in range(NL):
                launch(l)
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / NL)
    t = statistics.median(times)
    mb = N * K * 2 / 1e6
    print(f"{name:8s} N={N} K={K} splits={splits}: {t:6.2f} us/launch  {mb:5.1f} MB  "
          f"{mb / t:5.2f} TB/s", flush=True)
