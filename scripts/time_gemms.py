"""Time the C2 GEMM shapes (CUDA events, weights rotated past L2): BK=32 vs 64."""
import json, sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
SHAPES = [  # name, N, K, epi, splits, T
    ("t.qkv", 6144, 4096, 0, 6, 256), ("t.o", 4096, 4096, 0, 9, 256),
    ("t.gate_up", 28672, 4096, 2, 1, 256), ("t.down", 4096, 14336, 0, 9, 256),
    ("t.lm_head", 128256, 4096, 1, 1, 256),
    ("d.qkv", 3072, 2048, 0, 12, 64), ("d.o", 2048, 2048, 0, 10, 64),
    ("d.gate_up", 16384, 2048, 2, 1, 64), ("d.down", 2048, 8192, 0, 12, 64),
    ("d.lm_head", 128256, 2048, 1, 1, 64),
]
out = {}
for name, N, K, epi, splits, T in SHAPES:
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(512, K, device="cuda").bfloat16()
    part = torch.empty(splits, 512, N, device="cuda")
    av = torch.empty((N + 31) // 32, 512, device="cuda")
    ai = torch.empty((N + 31) // 32, 512, dtype=torch.int32, device="cuda")
    act = torch.empty(512, N // 2, dtype=torch.bfloat16, device="cuda")
    variants = (("sk", 0), ("nosk", 2000)) if epi != 0 else (("256rows", 0),)
    for bk, ms in variants:
        ts = []
        for it in range(30):
            W = Ws[it % copies]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K, splits,
                                              epi, part.data_ptr(), av.data_ptr(), ai.data_ptr(),
                                              act.data_ptr(), N // 2, ms, _native.stream_ptr()), "g")
            e1.record(); e1.synchronize()
            if it >= 5: ts.append(e0.elapsed_time(e1) * 1e3)
        t = statistics.median(ts)
        out[f"{name}.bk{bk}"] = dict(us=round(t, 2), gbs=round(N * K * 2 / t / 1e3, 1))
        print(name, bk, out[f"{name}.bk{bk}"], flush=True)
    del Ws
    torch.cuda.empty_cache()
print(json.dumps(out))
