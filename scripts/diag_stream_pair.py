"""Premise check for 2-CTA verify GEMMs: per-SM weight streaming rate with a
full activation tile per stage (3 x [32 KB W + 32 KB X]) vs the half tile a
CTA pair would hold (4 x [32 KB W + 16 KB X]) vs weights alone."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
from diagnostics import lib as _diag_lib  # noqa: E402
L = _diag_lib()
K = 4096
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
X = torch.randn(256, K, device="cuda").bfloat16()
for grid in (112, 148):
    per = (buf.numel() // grid) // (K * 2 * 256) * (K * 2 * 256)
    for mode, stages, sb, xb, label in ((2, 3, 65536, 4, "3 x (W32+X32)  [today, T=256]"),
                                        (2, 4, 65536, 2, "4 x (W32+X16)  [CTA pair]"),
                                        (2, 6, 65536, 0, "6 x W32        [no X]")):
        # mode 2: 256-row boxes; stage_bytes counts W only (X boxes added on top)
        ms = C.c_float(0)
        for _ in range(3):
            _native.check(L.spectre_diag_stream(C.c_void_p(buf.data_ptr()), C.c_int64(per), grid,
                                                mode, stages, 32768 * 2 // 2, K, xb, 0,
                                                C.c_void_p(X.data_ptr()), C.byref(ms), None), "d")
        gbs = per * grid / (ms.value * 1e-3) / 1e9
        print(f"grid {grid} {label}: W {gbs:7.1f} GB/s ({gbs / grid:5.1f}/SM)", flush=True)
