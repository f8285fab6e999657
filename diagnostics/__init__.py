"""Microbenchmarks kept OUT of the product library (libspectre.so).

`diag_stream.cu` holds the round-1 measurement kernels (HBM stream rates,
tcgen05 issue costs, TMEM load latency) that sized the GEMM design; they are
built into their own `diagnostics/libspectre_diag.so` on demand:

    from diagnostics import lib; L = lib()
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent / "paper_2605_08151_b200"
LIB = HERE / "libspectre_diag.so"


def build() -> Path:
    from paper_2605_08151_b200 import _build
    product = _build.build()
    src = HERE / "diag_stream.cu"
    if LIB.exists() and LIB.stat().st_mtime >= max(src.stat().st_mtime, product.stat().st_mtime):
        return LIB
    cmd = [_build.nvcc(), *_build.ARCH, *_build.BASE_FLAGS, "-I", str(PKG.parent / "include"),
           "-I", str(PKG / "csrc"), "-shared", str(src), "-o", str(LIB),
           "-L", str(PKG), "-lspectre", f"-Xlinker=-rpath,{PKG}", "-lcuda"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"diagnostics build failed:\n{out.stdout}\n{out.stderr}")
    return LIB


def lib():
    from paper_2605_08151_b200 import _native
    _native.lib()                       # the product library (GEMM plans) first
    return ctypes.CDLL(str(build()))
