"""Target GEMMs at prefill shapes (T = 512 rows): tile height x split-K
(diagnostics).  CUDA events, weights rotated past L2.
    python scripts/diag_prefill_gemm.py [T]"""
import statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
CASES = [("down", 4096, 14336, [(9, 0), (4, 0), (2, 0), (9, 1000), (4, 1000), (2, 1000)]),
         ("qkv", 6144, 4096, [(3, 1000), (2, 1000), (1, 1000), (6, 0), (3, 0), (2, 0)]),
         ("o", 4096, 4096, [(4, 1000), (2, 1000), (1, 1000), (4, 0), (2, 0)])]
for name, N, K, cfgs in CASES:
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    Ws = [(torch.randn(N, K, device="cuda") * 0.02).bfloat16() for _ in range(copies)]
    X = torch.randn(T, K, device="cuda").bfloat16()
    part = torch.empty(12, T, N, device="cuda")
    s = torch.cuda.Stream()
    for splits, flags in cfgs:
        ts = []
        for it in range(25):
            W = Ws[it % copies]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(4):
                _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, T, N, K,
                                                  splits, 0, part.data_ptr(), None, None, None, 0,
                                                  flags, int(s.cuda_stream)), "gemm")
            e1.record(s)
            e1.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3 / 4)
        t = statistics.median(ts)
        tile = 128 if flags >= 1000 else 256
        print(f"{name} T={T} tile={tile} splits={splits}: {t:7.2f} us  "
              f"{2 * T * N * K / t / 1e6:6.0f} TF/s", flush=True)
    del Ws
    torch.cuda.empty_cache()
