"""Launch one GEMM shape a few times (for ncu captures): one_gemm.py N K epi T [flags]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
N, K, epi, T = (int(v) for v in sys.argv[1:5])
flags = int(sys.argv[5]) if len(sys.argv) > 5 else 0
splits = int(sys.argv[6]) if len(sys.argv) > 6 else 1
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
RC = max(512, (T + 63) // 64 * 64)   # buffer rows (the kernel clamps T to them)
X = torch.randn(RC, K, device="cuda").bfloat16()
part = torch.empty(12, RC, N, device="cuda") if epi == 0 else torch.empty(1, device="cuda")
av = torch.empty(L.spectre_gemm_argmax_blocks(N, K), RC, device="cuda")
ai = torch.empty(L.spectre_gemm_argmax_blocks(N, K), RC, dtype=torch.int32, device="cuda")
act = torch.empty(RC, N // 2, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, RC, N, K, splits, epi,
                                      part.data_ptr(), av.data_ptr(), ai.data_ptr(), act.data_ptr(),
                                      N // 2, flags, _native.stream_ptr()), "gemm")
torch.cuda.synchronize()
print("ok")
