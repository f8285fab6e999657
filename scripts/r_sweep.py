"""Config 4: fallback-ratio sweep and the r* switch point.

For gamma in {2, 4, 8} and a grid of draft keep-probabilities (controlled
noise; lower alpha -> more fallbacks), decode the C2 pair with ordinary,
parallel and SPECTRE (hybrid, `round` controller) and record device tok/s,
the reference's r-hat (|R|/B), the paper's r (PADDED fraction of parallel
rounds), accepted lengths, the measured round times T_ord / T_par and the
controller's predicted r* = L (1 - T_par/T_ord) / (L - 1).

The empirical crossover is where parallel tok/s overtakes ordinary; the
check is that the hybrid's switch (its predicted r*) lands on it and that
SPECTRE tracks max(ordinary, parallel) across the sweep.

  python scripts/r_sweep.py --out profiles/r01/r_sweep.json [--gammas 2 4 8]
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
from paper_2605_08151_b200.decoder import PolicyVariant


def one(pair, prompts, gamma, alpha, variant, out_len, seed, alpha_late=None, switch=0):
    spec = M.DecodeSpec(n_req=prompts.shape[0], gamma=gamma, output_len=out_len,
                        prompt_len=prompts.shape[1], alpha=alpha, seed=seed, controller="round",
                        alpha_switch_pos=switch if alpha_late is not None else 0,
                        alpha_late=alpha if alpha_late is None else alpha_late)
    eng = M.SpectreEngine(pair, spec, variant)
    eng.prefill(prompts)
    eng.run(use_graph=True)           # warm (graph build)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.prefill(prompts)
    e0.record()
    eng.run(use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    committed, pos, tr = eng.read()
    assert int((pos == out_len).sum()) == prompts.shape[0], "unfinished requests"
    P = tr["participants"].astype(np.float64)
    modes = "".join(chr(int(m)) for m in tr["mode"])
    par = np.array([m == "P" for m in modes])
    ordm = np.array([m == "O" for m in modes])
    t = tr["t_round_ns"].astype(np.float64) * 1e-9
    res = dict(variant=variant, gamma=gamma, alpha=alpha, ms=ms,
               tok_s=prompts.shape[0] * out_len / (ms * 1e-3),
               rounds=len(modes), ordinary_share=float(ordm.mean()),
               r_hat=float((tr["n_roll"] / np.maximum(P, 1)).mean()),
               r_pad_parallel=float(tr["n_padded"][par].sum() / max(1.0, P[par].sum())),
               mean_L=float(tr["delta"].sum() / P.sum()),
               content_L=float(tr["content_sum"].sum() / max(1, tr["content_n"].sum())),
               t_ord_ms=float(t[ordm].mean() * 1e3) if ordm.any() else None,
               t_par_ms=float(t[par].mean() * 1e3) if par.any() else None,
               r_star_last=float(tr["r_star"][-1]) if len(modes) else None,
               r_star_median=float(np.median(tr["r_star"][np.isfinite(tr["r_star"])]))
               if np.isfinite(tr["r_star"]).any() else None,
               timeline_head=modes[:48], timeline=modes)
    del eng
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gammas", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--alphas", type=float, nargs="+",
                    default=[1.0, 0.97, 0.94, 0.9, 0.85, 0.75, 0.6, 0.4])
    ap.add_argument("--branch", type=float, default=0.0015,
                    help="transformer-branch scale: small -> natural agreement near 1")
    ap.add_argument("--out-len", type=int, default=512)
    ap.add_argument("--n-req", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/r_sweep.json")
    ap.add_argument("--drift", type=float, nargs=2, default=[1.0, 0.1],
                    help="drift workload: alpha for the first half of the output, then alpha_late")
    ap.add_argument("--drift-gammas", type=int, nargs="*", default=[8, 4])
    args = ap.parse_args()
    gmax = max(args.gammas)
    ctx = M.DecodeSpec(n_req=args.n_req, gamma=gmax, output_len=args.out_len,
                       prompt_len=128).ctx_cap()
    pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=args.n_req, ctx_cap=ctx, seed=0,
                        target_branch=args.branch, draft_branch=args.branch)
    prompts = M.synthetic_prompts(args.n_req, 128, M.LLAMA_31_8B.vocab, seed=0)
    rows = []
    t0 = time.time()
    for g in args.gammas:
        for a in args.alphas:
            for v in ("ordinary", "parallel", "hybrid"):
                r = one(pair, prompts, g, a, v, args.out_len, seed=0)
                rows.append(r)
                print(json.dumps({k: (round(x, 4) if isinstance(x, float) else x)
                                  for k, x in r.items() if k not in ("timeline_head", "timeline")}),
                      flush=True)
    # crossover analysis per gamma.  Measured switch: where parallel minus
    # ordinary tok/s changes sign along the sweep (either direction), and the
    # paper's r (PADDED fraction of parallel rounds) there.  Predicted switch:
    # the model's fixed point r = r*(L, T_par/T_ord) along the same sweep (the
    # hybrid's r* per point against the parallel run's r), i.e. where the
    # controller's rule "parallel iff r <= r*" flips.
    def sign_change(alphas, f):
        for i in range(len(alphas) - 1):
            a, b = f[i], f[i + 1]
            if a == 0 or (a > 0) != (b > 0):
                t = 0.0 if a == b else a / (a - b)
                return i, t
        return None

    summary = []
    for g in args.gammas:
        pts = sorted([r for r in rows if r["gamma"] == g], key=lambda r: -r["alpha"])
        by = {(r["alpha"], r["variant"]): r for r in pts}
        alphas = sorted({r["alpha"] for r in pts}, reverse=True)
        diff = [by[(a, "parallel")]["tok_s"] - by[(a, "ordinary")]["tok_s"] for a in alphas]
        rpad = [by[(a, "parallel")]["r_pad_parallel"] for a in alphas]
        rstar = [by[(a, "hybrid")]["r_star_median"] for a in alphas]

        def lerp(v, i, t):
            return v[i] + t * (v[i + 1] - v[i])

        cross = None
        m = sign_change(alphas, diff)
        if m is not None:
            i, t = m
            cross = dict(alpha=lerp(alphas, i, t), r_switch=lerp(rpad, i, t),
                         r_star_there=None if None in rstar[i:i + 2] else lerp(rstar, i, t),
                         parallel_wins_below=diff[i + 1] > 0)
            if None not in rstar:
                p = sign_change(alphas, [rs - rp for rs, rp in zip(rstar, rpad)])
                if p is not None:
                    j, u = p
                    cross.update(predicted_alpha=lerp(alphas, j, u),
                                 predicted_r_switch=lerp(rpad, j, u))
                    cross["rel_err"] = (abs(cross["r_switch"] - cross["predicted_r_switch"])
                                        / cross["predicted_r_switch"])
        best = [max(by[(a, "parallel")]["tok_s"], by[(a, "ordinary")]["tok_s"]) for a in alphas]
        hyb = [by[(a, "hybrid")]["tok_s"] for a in alphas]
        summary.append(dict(gamma=g, alphas=alphas, parallel_minus_ordinary=diff,
                            r_pad_parallel=rpad, r_star_hybrid=rstar, crossover=cross,
                            hybrid_over_best=[h / b for h, b in zip(hyb, best)]))
        print(json.dumps(summary[-1]), flush=True)
    drift = []
    for g in args.drift_gammas:
        res = {}
        for v in ("ordinary", "parallel", "hybrid"):
            res[v] = one(pair, prompts, g, args.drift[0], v, args.out_len, seed=0,
                         alpha_late=args.drift[1], switch=args.out_len // 2)
            print(json.dumps({k: (round(x, 4) if isinstance(x, float) else x)
                              for k, x in res[v].items() if k not in ("timeline_head", "timeline")}),
                  flush=True)
        best = max(res["ordinary"]["tok_s"], res["parallel"]["tok_s"])
        drift.append(dict(gamma=g, alpha=args.drift[0], alpha_late=args.drift[1],
                          switch_pos=args.out_len // 2,
                          tok_s={v: r["tok_s"] for v, r in res.items()},
                          hybrid_over_ordinary=res["hybrid"]["tok_s"] / res["ordinary"]["tok_s"],
                          hybrid_over_parallel=res["hybrid"]["tok_s"] / res["parallel"]["tok_s"],
                          hybrid_over_best=res["hybrid"]["tok_s"] / best,
                          timeline=res["hybrid"]["timeline"], points=list(res.values())))
        print(json.dumps({k: v for k, v in drift[-1].items() if k != "points"}), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(dict(points=rows, summary=summary, drift=drift,
                                              branch=args.branch, out_len=args.out_len,
                                              n_req=args.n_req, seconds=time.time() - t0),
                                         indent=1))


if __name__ == "__main__":
    main()
