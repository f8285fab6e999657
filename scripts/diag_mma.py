"""tcgen05.mma issue -> commit -> mbarrier round trip (diagnostics).
depth >= 1: commit per iteration and wait `depth` commits back (the GEMM ring);
0: commit per iteration, never wait; -1: no per-iteration commit.
  python scripts/diag_mma.py"""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: F401
from paper_2605_08151_b200 import _native
from diagnostics import lib as _diag_lib  # noqa: E402
L = _diag_lib()
L.spectre_diag_mma.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_uint64), C.c_void_p]
for n in (64, 256):
    for nmma in (1, 4, 8, 16):
        for depth in (-1, 0, 1, 8):
            cyc = (C.c_uint64 * 2)()
            _native.check(L.spectre_diag_mma(1, 2000, nmma, n, depth, cyc, None), "d")
            print(f"N {n:3d} mma/iter {nmma:2d} depth {depth:2d}: total {cyc[0]:6d} "
                  f"issue {cyc[1]:6d} cycles/iter ({cyc[0] / nmma:7.1f}/mma)", flush=True)
L.spectre_diag_mma_unrolled.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_uint64)]
for n in (64, 128, 256):
    for nm in (1, 4, 8, 16):
        cyc = C.c_uint64(0)
        _native.check(L.spectre_diag_mma_unrolled(nm, n, C.byref(cyc)), "u")
        print(f"unrolled N {n:3d} mma/iter {nm:2d} depth 8: {cyc.value:6d} cycles/iter "
              f"({cyc.value / nm:7.1f}/mma)", flush=True)
