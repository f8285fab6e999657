"""Target gate_up (SwiGLU, T=256): stream-K over all SMs vs plain 256-row
tiles (112 CTAs).  CUPTI kernel durations, weights rotated past L2."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2605_08151_b200 import _native
L = _native.lib()
for name, N, K, T in (("t.gate_up", 28672, 4096, 256), ("d.gate_up", 16384, 2048, 64)):
    copies = max(2, int(400e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(512, K, device="cuda").bfloat16()
    act = torch.empty(512, N // 2, dtype=torch.bfloat16, device="cuda")
    for flags, label in ((0, "stream-K"), (2000, "plain 256"), (1000, "plain 128")):
        def go(it):
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), Ws[it % copies].data_ptr(), None, T,
                                              512, N, K, 1, 2, None, None, None, act.data_ptr(),
                                              N // 2, flags, _native.stream_ptr()), "g")
        for it in range(5):
            go(it)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for it in range(20):
                go(it)
            torch.cuda.synchronize()
        ds = sorted(e.device_time for e in prof.events() if "gemm" in e.name)
        us = ds[len(ds) // 2]
        print(f"{name} {label:10s}: {us:7.2f} us  {N*K*2/us/1e3:6.0f} GB/s", flush=True)
    del Ws
    torch.cuda.empty_cache()
