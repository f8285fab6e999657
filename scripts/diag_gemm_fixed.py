"""Fixed cost of the GEMM kernel: draft o_proj shape at T = 0, 1, 16, 64."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
N, K, S = 2048, 2048, 10
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
X = torch.randn(512, K, device="cuda").bfloat16()
part = torch.empty(S, 512, N, device="cuda")
for T in (0, 1, 16, 64, 64, 64):
    for s_ in (1, 10):
        _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, 512, N, K, s_, 0,
                                          part.data_ptr(), None, None, None, 0, 0,
                                          _native.stream_ptr()), "g")
torch.cuda.synchronize()
