"""Standalone target-shape GEMMs for ncu --set full (gate_up SwiGLU, down split-K)."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
def run(N, K, epi, splits, reps=3):
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    X = torch.randn(512, K, device="cuda").bfloat16()
    part = torch.empty(splits, 512, N, device="cuda")
    act = torch.empty(512, max(N // 2, 1), dtype=torch.bfloat16, device="cuda")
    for _ in range(reps):
        _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K, splits, epi,
                                          part.data_ptr(), None, None, act.data_ptr(), N // 2, 0,
                                          _native.stream_ptr()), "gemm")
    torch.cuda.synchronize()
run(28672, 4096, 2, 1)      # target gate_up (SwiGLU)
run(4096, 14336, 0, 9)      # target down (split-K 9)
run(16384, 2048, 2, 1)      # draft gate_up
