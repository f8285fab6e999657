"""Run one eager decode round of C2 between cudaProfilerStart/Stop (for ncu).

ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --csv --log-file gpurun_out/round_launches.csv python scripts/profile_round.py
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_08151_b200 import model as M


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="ordinary")
    ap.add_argument("--warm-rounds", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--branch", type=float, default=0.005)
    ap.add_argument("--n-req", type=int, default=64)
    args = ap.parse_args()
    spec = M.DecodeSpec(n_req=args.n_req, gamma=4, output_len=1024, prompt_len=128, seed=0)
    pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=args.n_req,
                        ctx_cap=spec.ctx_cap(), seed=0, target_branch=args.branch,
                        draft_branch=args.branch)
    eng = M.SpectreEngine(pair, spec, args.variant)
    eng.prefill(M.synthetic_prompts(spec.n_req, spec.prompt_len, M.LLAMA_31_8B.vocab))
    eng.run(max_rounds=args.warm_rounds, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.run(max_rounds=args.rounds, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    _, pos, tr = eng.read()
    print("rounds", len(tr["mode"]), "mean pos", float(pos.float().mean()))


if __name__ == "__main__":
    main()
