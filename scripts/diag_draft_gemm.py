"""Per-CTA timeline / stall counters of one draft split-K GEMM (T=64), via the
GEMM's diagnostics hooks (SPECTRE_GEMM_DBG / SPECTRE_GEMM_STALL printed by the
C-ABI entry point).  python scripts/diag_draft_gemm.py N K splits flags"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
N, K, splits, flags = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (3072, 2048, 12, 3000)))
T = 64
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
X = torch.randn(512, K, device="cuda").bfloat16()
part = torch.empty(splits, 512, N, device="cuda")
for _ in range(3):
    _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K, splits, 0,
                                      part.data_ptr(), None, None, None, 1, flags,
                                      _native.stream_ptr()), "gemm")
    torch.cuda.synchronize()
