"""Config 5 target GEMM shapes (Qwen2.5-32B) at the verify row count: tile
height variants (diagnostics).   python scripts/diag_c5_gemm.py [T]"""
import statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 896
RC = 1024
# flags: 2000 256-row tiles, 1000 128-row tiles, 8000 128-row (tile, split, pass) units
CASES = [("gate/up", 55296, 5120, 2, 1, (2000, 1000)), ("lm_head", 152064, 5120, 1, 1, (2000, 1000)),
         ("down s7 256r", 5120, 27648, 0, 7, (2000,)), ("down s3 128r", 5120, 27648, 0, 3, (1000, 8000)),
         ("down s4 128r", 5120, 27648, 0, 4, (1000, 8000)), ("down s2 128r", 5120, 27648, 0, 2, (8000,)),
         ("qkv s3 256r", 7168, 5120, 0, 3, (2000,)), ("qkv s2 128r", 7168, 5120, 0, 2, (1000, 8000)),
         ("o s4 256r", 5120, 5120, 0, 7, (2000,)), ("o s3 128r", 5120, 5120, 0, 3, (1000, 8000)),
         ("o s1 128r", 5120, 5120, 0, 1, (8000,))]
for name, N, K, epi, splits, flagset in CASES:
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    X = torch.randn(RC, K, device="cuda").bfloat16()
    nb = L.spectre_gemm_argmax_blocks(N, K)
    part = torch.zeros(splits, RC, N, device="cuda") if epi == 0 else torch.zeros(1, device="cuda")
    av = torch.zeros(nb, RC, device="cuda")
    ai = torch.zeros(nb, RC, dtype=torch.int32, device="cuda")
    act = torch.zeros(RC, max(1, N // 2), dtype=torch.bfloat16, device="cuda")
    for flags in flagset:
        def run():
            _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, RC, N, K, splits,
                                              epi, part.data_ptr(), av.data_ptr(), ai.data_ptr(),
                                              act.data_ptr(), max(1, N // 2), flags,
                                              _native.stream_ptr()), "gemm")
        run()
        ts = []
        for it in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            e1.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        tile = {2000: "256", 1000: "128", 8000: "128pu"}[flags]
        print(f"{name:14s} T={T} tile={tile}: {statistics.median(ts):8.2f} us  "
              f"{2 * T * N * K / statistics.median(ts) / 1e6:6.0f} TF/s", flush=True)
    del W, part
    torch.cuda.empty_cache()
