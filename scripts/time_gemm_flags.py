"""Time one SwiGLU / partial GEMM shape under several C-ABI plan flags
(diagnostics): time_gemm_flags.py N K epi T flag[,flag...] [splits]
(flags: 1000 128-row tiles, 2000 256-row single CTA, 4000 CTA pairs, 9000 CTA
pairs over (tile pair, chunk) units; see spectre_gemm_bf16)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
L = _native.lib()
N, K, epi, T = (int(v) for v in sys.argv[1:5])
flags = [int(f) for f in sys.argv[5].split(",")]
S = int(sys.argv[6]) if len(sys.argv) > 6 else 1
RC = max(512, (T + 63) // 64 * 64)
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
X = torch.randn(RC, K, device="cuda").bfloat16()
part = torch.empty(S, RC, N, device="cuda") if epi == 0 else torch.empty(1, device="cuda")
av = torch.empty(L.spectre_gemm_argmax_blocks(N, K), RC, device="cuda")
ai = torch.empty(L.spectre_gemm_argmax_blocks(N, K), RC, dtype=torch.int32, device="cuda")
act = torch.empty(RC, N // 2, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = _native.stream_ptr()
for f in flags:
    def run():
        _native.check(L.spectre_gemm_bf16(X.data_ptr(), W.data_ptr(), None, T, RC, N, K, S, epi,
                                          part.data_ptr(), av.data_ptr(), ai.data_ptr(),
                                          act.data_ptr(), N // 2, f, s), "gemm")
    for _ in range(3):
        run()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    fl = 2.0 * T * N * K
    print(f"N={N} K={K} T={T} S={S} flag={f}: median {ts[5]:.1f} us min {ts[0]:.1f} us "
          f"({fl / ts[5] / 1e6:.0f} TFLOP/s)", flush=True)
