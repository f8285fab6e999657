"""Draft-chain timing sweep (diagnostics): the mid-layer chains back to back
(as bench.py's roofline leg) and ordinary C2 rounds in context, for each value
of an environment knob (default SPECTRE_CHAIN_PF), one process per value.
    python scripts/time_chain.py [--knob SPECTRE_CHAIN_PF] [--values 0,8,16,32]"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import _native, model as M

ap = argparse.ArgumentParser()
ap.add_argument("--knob", default="SPECTRE_CHAIN_PF")
ap.add_argument("--values", default="0,8,16,32")
ap.add_argument("--out-len", type=int, default=384)
ap.add_argument("--variant", default="ordinary")
args = ap.parse_args()
if "," in args.values:
    # one process per value: the library reads most knobs once per process
    import subprocess
    for v in args.values.split(","):
        subprocess.run([sys.executable, __file__, "--knob", args.knob, "--values", v,
                        "--out-len", str(args.out_len), "--variant", args.variant],
                       env={**os.environ, args.knob: v}, check=True)
    sys.exit(0)

L = _native.lib()
B, G = 64, 4
spec = M.DecodeSpec(n_req=B, gamma=G, output_len=args.out_len, prompt_len=128, seed=0)
pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=B, ctx_cap=spec.ctx_cap(), seed=0,
                    target_branch=0.004, draft_branch=0.004)
prompts = M.synthetic_prompts(B, 128, M.LLAMA_31_8B.vocab, seed=0)
V = pair.draft.spec.vocab
out = []
ref_sha = None
for v in args.values.split(","):
    os.environ[args.knob] = v
    eng = M.SpectreEngine(pair, spec, args.variant)
    # chains back to back at mid context
    pos = torch.full((B,), 128 + 512, dtype=torch.int32, device="cuda")
    ar = torch.arange(B, dtype=torch.int32, device="cuda")
    tok = (ar * 7919 + 11) % V
    eng.forward(1, tok, pos, ar, ar, torch.ones(B, dtype=torch.int32, device="cuda"), pos)
    s = torch.cuda.Stream()
    wb = C.c_int64(0)
    L.spectre_engine_launch_chains(eng.handle, 1, C.byref(wb), int(s.cuda_stream))
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        n = L.spectre_engine_launch_chains(eng.handle, 4, C.byref(wb), int(s.cuda_stream))
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    chain_us = statistics.median(ts)
    # in context: a full decode
    eng.prefill(prompts)
    torch.cuda.synchronize()
    eng.run(use_graph=True, sync=True)
    committed, p, trace = eng.read()
    import hashlib
    sha = hashlib.sha256(committed.cpu().numpy().tobytes()).hexdigest()[:16]
    ref_sha = ref_sha or sha
    tr = trace["t_round_ns"].astype("f8") * 1e-6
    td = trace["t_draft_ns"].astype("f8") * 1e-6 if "t_draft_ns" in trace else None
    tv = trace["t_verify_ns"].astype("f8") * 1e-6 if "t_verify_ns" in trace else None
    k = len(tr)
    mid = slice(k // 4, 3 * k // 4)
    row = {"knob": args.knob, "value": v, "chain_us": round(chain_us, 2),
           "round_ms": round(float(tr[mid].mean()), 3),
           "draft_ms": round(float(td[mid].mean()), 3) if td is not None else None,
           "verify_ms": round(float(tv[mid].mean()), 3) if tv is not None else None,
           "tok_s": round(float(p.sum().item()) / float(tr.sum() * 1e-3), 1),
           "sha": sha, "same_tokens": sha == ref_sha}
    print(json.dumps(row), flush=True)
    out.append(row)
    eng.close()
    del eng
    torch.cuda.empty_cache()
