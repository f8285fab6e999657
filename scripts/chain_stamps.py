"""Per-phase timeline of the draft chains (diagnostics): CTA 0's globaltimer
stamps of the last draft step, relative to each chain's start.
    SPECTRE_CHAIN_DBG=1 python scripts/chain_stamps.py"""
import ctypes as C
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("SPECTRE_CHAIN_DBG", "1")
import numpy as np
import torch
from paper_2605_08151_b200 import _native, model as M

L = _native.lib()
L.spectre_engine_chain_stamps.restype = C.c_int
L.spectre_engine_chain_stamps.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
spec = M.DecodeSpec(n_req=64, gamma=4, output_len=256, prompt_len=128, seed=0)
pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=64, ctx_cap=spec.ctx_cap(), seed=0,
                    target_branch=0.004, draft_branch=0.004)
eng = M.SpectreEngine(pair, spec, "ordinary")
prompts = M.synthetic_prompts(64, 128, M.LLAMA_31_8B.vocab, seed=0)
eng.prefill(prompts)
eng.run(max_rounds=20, use_graph=False, sync=True)
n = (M.LLAMA_32_1B.n_layers + 1) * 64
buf = np.zeros(n, dtype=np.uint64)
got = L.spectre_engine_chain_stamps(eng.handle, buf.ctypes.data, n)
st = buf[:got].reshape(-1, 64).astype(np.int64)
names = {0: "first: embed | qkv | rope", 16: "last: o | resid | gu | down | resid"}
kinds = {0: ["embed", "qkv", "rope"], 16: ["o", "resid", "gu", "down", "resid"]}
for i, row in enumerate(st):
    t0 = int(row[0])
    rel = lambda v: (int(v) - t0) / 1e3 if v else float("nan")
    ph = kinds.get(i, ["o", "resid", "gu", "down", "resid", "qkv", "rope"])
    cells = []
    for p, name in enumerate(ph):
        start = 0.0 if p == 0 else rel(row[1 + 2 * p])
        cell = f"{name}[{start:5.2f}"
        if row[32 + p]:
            cell += f" x{rel(row[32 + p]):5.2f}"
        if row[16 + 2 * p]:
            cell += f" acc{rel(row[16 + 2 * p]):5.2f} st{rel(row[17 + 2 * p]):5.2f}"
        cell += f" ->{rel(row[2 + 2 * p]):5.2f}]"
        cells.append(cell)
    print(f"chain {i:2d}: " + " ".join(cells))
