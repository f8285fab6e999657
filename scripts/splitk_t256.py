"""Target split-K GEMMs at T=256: 256-row tiles x s splits vs 128-row tiles x
fewer splits (less fp32 partial traffic, more activation re-reads).  Kernel
durations from CUPTI (torch.profiler); weights rotated past L2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2605_08151_b200 import _native
L = _native.lib()
CASES = [  # name, N, K, T, [(flags, splits), ...]
    ("t.qkv", 6144, 4096, 256, [(0, 6), (1000, 3), (1000, 2), (0, 3)]),
    ("t.o", 4096, 4096, 256, [(0, 9), (1000, 4), (1000, 5), (1000, 3)]),
    ("t.down", 4096, 14336, 256, [(0, 9), (1000, 4), (1000, 5), (1000, 3)]),
    ("d.qkv", 3072, 2048, 64, [(1000, 6), (3000, 12), (3000, 6)]),
]
for name, N, K, T, vs in CASES:
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(512, K, device="cuda").bfloat16()
    part = torch.empty(12, 512, N, device="cuda")
    for flags, s in vs:
        def go(it):
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), Ws[it % copies].data_ptr(), None, T, 512,
                                              N, K, s, 0, part.data_ptr(), None, None, None, 0,
                                              flags, _native.stream_ptr()), "g")
        for it in range(5):
            go(it)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for it in range(20):
                go(it)
            torch.cuda.synchronize()
        ds = [e.device_time for e in prof.events() if "gemm" in e.name]
        us = sorted(ds)[len(ds) // 2]
        part_mb = s * T * N * 4 / 1e6
        print(f"{name} flags {flags:4d} splits {s:2d}: {us:7.2f} us  W {N*K*2/us/1e3:6.0f} GB/s  "
              f"partials {part_mb:5.1f} MB (+read back ~{part_mb/6.0:4.1f} us)", flush=True)
    del Ws
    torch.cuda.empty_cache()
