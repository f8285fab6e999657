"""Per-SM streaming rate: TMA weight boxes alone, and with the shared
activation (X) boxes every GEMM stage also loads (diagnostics)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
from diagnostics import lib as _diag_lib  # noqa: E402
L = _diag_lib()
K = 2048
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
X = torch.randn(256, K, device="cuda").bfloat16()
grid = 148
per = (buf.numel() // grid) // (K * 2 * 256) * (K * 2 * 256)
cfgs = [  # mode, stages, stage bytes, x boxes (64 rows each), stagger
    (0, 5, 32768, 0, 0), (1, 5, 32768, 0, 0),
    (0, 5, 32768, 1, 0), (0, 5, 32768, 1, 1),     # draft-like: T=64
    (0, 3, 32768, 4, 0), (0, 3, 32768, 4, 1),     # target-like: T=256
]
for mode, stages, sb, xb, stag in cfgs:
    ms = C.c_float(0)
    for _ in range(3):
        st = L.spectre_diag_stream(C.c_void_p(buf.data_ptr()), C.c_int64(per), grid, mode, stages,
                                   sb, K, xb, stag, C.c_void_p(X.data_ptr()), C.byref(ms), None)
        _native.check(st, "diag")
    gbs = per * grid / (ms.value * 1e-3) / 1e9
    print(f"mode {mode} stages {stages} x {sb//1024} KB  x_boxes {xb} stagger {stag}: "
          f"W {gbs:7.1f} GB/s ({gbs/grid:5.1f}/SM)", flush=True)
