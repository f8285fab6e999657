import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native
from diagnostics import lib as _diag_lib  # noqa: E402
L = _diag_lib()
out = torch.zeros(8, dtype=torch.int64, device="cuda")
for iters in (1, 8, 64):
    L.spectre_diag_tmem(iters, C.c_void_p(out.data_ptr()), None)
    torch.cuda.synchronize()
    print(iters, "cycles per warp:", out.tolist(), "per load:", [v / iters for v in out.tolist()])
