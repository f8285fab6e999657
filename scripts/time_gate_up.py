"""Time the target verify gate/up + SwiGLU GEMM (8B shape, T = B*gamma) for each
launch mode: single CTAs (2000), CTA pairs with 256 rows per CTA (4000), CTA
pairs with 128 rows per CTA and double-buffered TMEM (5000).  32 distinct
weight matrices (> L2) back to back, CUDA events on the launching stream.

    python scripts/time_gate_up.py [T ...]
"""
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native

L = _native.lib()
F, K, NL = 14336, 4096, 32
W = torch.randn(NL, 2 * F, K, device="cuda").mul_(0.02).bfloat16()
X = torch.randn(1024, K, device="cuda").bfloat16()
act = torch.empty(1024, F, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.Stream()
for T in [int(a) for a in sys.argv[1:]] or [256, 128, 64]:
    for flags in (2000, 4000):
        def launch(l):
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), W[l].data_ptr(), None, T, 1024, 2 * F,
                                              K, 1, 2, None, None, None, act.data_ptr(), F,
                                              flags, int(s.cuda_stream)), "gemm")
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
        byt = 2 * F * K * 2 + T * K * 2 + T * F * 2
        print(f"T={T} flags={flags}: {t:.2f} us  {byt / t / 1e3:.0f} GB/s  "
              f"{2 * T * 2 * F * K / t / 1e6:.0f} TF/s", flush=True)
