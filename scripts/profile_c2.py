"""Exploration: C2 (8B-shape target / 1B-shape draft, B=64, gamma=4) on one B200.

Prints per-variant device tok/s, mean round / verify / draft-step times and
acceptance, for a few draft-coupling strengths.  Not part of the bench.
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

from paper_2605_08151_b200 import model as M


def summarize(res, spec):
    tr = res.trace
    n = len(tr["mode"])
    out = dict(variant=res.variant.value, rounds=n, graph=res.graph,
               tok_s=round(res.report.target_throughput, 1),
               mean_L=round(res.report.mean_accepted_length, 3),
               content_L=round(res.report.content_mean_accepted_length, 3),
               r_hat=round(res.report.mean_rollback_ratio, 3),
               pad_frac=round(float(tr["n_padded"].sum() / max(1, tr["participants"].sum())), 3),
               t_round_ms=round(float(tr["t_round_ns"].mean()) * 1e-6, 3),
               t_verify_ms=round(float(tr["t_verify_ns"].mean()) * 1e-6, 3),
               timeline=res.report.mode_timeline[:60])
    for m in "OP":
        sel = tr["mode"] == ord(m)
        if sel.any():
            out[f"t_round_{m}_ms"] = round(float(tr["t_round_ns"][sel].mean()) * 1e-6, 3)
            out[f"t_verify_{m}_ms"] = round(float(tr["t_verify_ns"][sel].mean()) * 1e-6, 3)
            out[f"t_draft_{m}_ms"] = round(float(tr["t_draft_ns"][sel].mean()) * 1e-6, 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-len", type=int, default=1024)
    ap.add_argument("--calib-len", type=int, default=160)
    ap.add_argument("--branches", default="0.02,0.05,0.1")
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--calib-only", action="store_true")
    args = ap.parse_args()
    spec = M.DecodeSpec(n_req=64, gamma=4, output_len=args.out_len, prompt_len=128,
                        alpha=args.alpha, seed=0)
    t0 = time.time()
    results = []
    for br in [float(x) for x in args.branches.split(",")]:
        pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=64, ctx_cap=spec.ctx_cap(),
                            seed=0, target_branch=br, draft_branch=br)
        print(f"# built pair branch={br} in {time.time() - t0:.1f}s", flush=True)
        cal = M.DecodeSpec(**{**spec.__dict__, "output_len": args.calib_len})
        r = M.decode(pair, cal, "ordinary")
        L = r.report.content_mean_accepted_length
        print(json.dumps(dict(branch=br, calib=summarize(r, cal))), flush=True)
        if args.calib_only:
            del pair
            torch.cuda.empty_cache()
            continue
        for v in ("ordinary", "parallel", "hybrid"):
            r = M.decode(pair, spec, v)
            s = summarize(r, spec)
            s["branch"] = br
            results.append(s)
            print(json.dumps(s), flush=True)
        del pair
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
