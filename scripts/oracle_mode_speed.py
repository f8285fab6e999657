"""Like-for-like: the reference's decode loop (hash-stream model pair) as the
CUDA oracle-mode loop vs its CPU restatement, C2 protocol shape (B=64, gamma=4,
output 1024, alpha 0.8).  Committed tokens per wall second, one run each
after a warm-up; reports must be byte-identical.

  python scripts/oracle_mode_speed.py
"""
import json
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2605_08151_b200 as P
from oracle import lockstep as L   # checker / CPU baseline only

cfg = dict(batch_size=64, n_requests=64, gamma=4, output_len=1024, alpha=0.8, qps=1e6, seed=0)
out = {}
for v in ("ordinary", "parallel", "hybrid"):
    P.run(P.SimConfig(**cfg), v)            # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    got = P.run(P.SimConfig(**cfg), v)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = L.run(cfg, v)
    t_cpu = time.perf_counter() - t0
    same = P.export_report(got.report) == L.export_csv(want.report)
    tok = 64 * 1024
    out[v] = dict(gpu_s=round(t_gpu, 4), cpu_1core_s=round(t_cpu, 3),
                  gpu_tok_s=round(tok / t_gpu), cpu_1core_tok_s=round(tok / t_cpu),
                  identical_report=same)
    print(v, out[v], flush=True)
Path("gpurun_out/oracle_mode_speed.json").write_text(json.dumps(out, indent=1))
