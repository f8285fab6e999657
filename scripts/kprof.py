"""Per-kernel device times of eager C2 rounds in their real context (PDL overlap,
warm L2), via torch.profiler (CUPTI).  Kernels are attributed to phases by the
protocol kernels that bracket them: draft steps end at k_draft_append, the
target forward runs between k_verify_prep and k_accept.

  python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 3
"""

import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_08151_b200 import model as M


def short(name):
    name = name.replace("void ", "").replace("spectre::", "")
    return name.split("(")[0][:48]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="ordinary")
    ap.add_argument("--warm-rounds", type=int, default=160)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--branch", type=float, default=0.004)
    ap.add_argument("--n-req", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/kprof.json")
    ap.add_argument("--temperature", type=float, default=0.0)
    ap.add_argument("--out-len", type=int, default=1024)
    ap.add_argument("--pair", default="c2", choices=("c2", "c5"),
                    help="c2: Llama-3.1-8B / 3.2-1B shapes; c5: Qwen2.5-32B / 0.5B")
    ap.add_argument("--gamma", type=int, default=4)
    args = ap.parse_args()
    spec = M.DecodeSpec(n_req=args.n_req, gamma=args.gamma, output_len=args.out_len,
                        prompt_len=128, seed=0, temperature=args.temperature)
    tgt, drf = ((M.LLAMA_31_8B, M.LLAMA_32_1B) if args.pair == "c2" else
                (M.QWEN_25_32B, M.QWEN_25_05B))
    pair = M.build_pair(tgt, drf, n_req=args.n_req,
                        ctx_cap=spec.ctx_cap(), seed=0, target_branch=args.branch,
                        draft_branch=args.branch)
    eng = M.SpectreEngine(pair, spec, args.variant)
    eng.prefill(M.synthetic_prompts(spec.n_req, spec.prompt_len, tgt.vocab))
    eng.run(max_rounds=args.warm_rounds, use_graph=False)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.run(max_rounds=args.rounds, use_graph=False)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ks = sorted(((e.time_range.start, e.time_range.end, short(e.name)) for e in evs
                 if "Memcpy" not in e.name and "Memset" not in e.name), key=lambda x: x[0])
    phase = "other"
    tcount = 0
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    spans = defaultdict(float)
    first = {}
    prev_end = None
    for t0, t1, n in ks:
        # marginal (exclusive) time: PDL lets a kernel start while its
        # predecessor runs, so its own duration double-counts the overlap
        excl = t1 - t0 if prev_end is None else max(0.0, t1 - max(t0, prev_end))
        prev_end = t1 if prev_end is None else max(prev_end, t1)
        if n.startswith("k_draft_prep"):
            phase = "draft"
        elif n.startswith("k_verify_prep"):
            phase = "target"
        elif n.startswith("k_accept") or n.startswith("k_round_begin"):
            phase = "other"
        if phase == "target" and n.startswith("k_verify_prep"):
            tcount = 0
        if phase == "target" and n.startswith("gemm_bf16_swapab<0"):
            # target layer order: q/k/v, o, down (split-K partial GEMMs)
            n = n + " " + ("qkv", "o", "down")[tcount % 3]
            tcount += 1
        key = (phase, n)
        agg[key][0] += 1
        agg[key][1] += excl
        agg[key][2] += (t1 - t0)
        spans[phase] += 0
        if phase not in first:
            first[phase] = t0
    # phase wall spans (start of first to end of last kernel per contiguous phase run)
    wall = defaultdict(float)
    cur, s0, last_end = None, None, None
    for t0, t1, n in ks:
        ph = ("draft" if n.startswith("k_draft_prep") else "target" if n.startswith(
            "k_verify_prep") else "other" if n.startswith(("k_accept", "k_round_begin")) else cur)
        if ph != cur:
            if cur is not None:
                wall[cur] += last_end - s0
            cur, s0 = ph, t0
        last_end = t1
    if cur is not None:
        wall[cur] += last_end - s0
    total = ks[-1][1] - ks[0][0] if ks else 0
    busy = sum(t1 - t0 for t0, t1, _ in ks)
    print(f"{len(ks)} kernels over {args.rounds} rounds: span {total/1e3:.3f} ms, "
          f"busy {busy/1e3:.3f} ms")
    for ph in ("draft", "target", "other"):
        print(f"  phase {ph}: wall {wall[ph]/1e3/args.rounds:.3f} ms/round")
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    out = []
    print("  phase  excl ms/round  launches  avg excl us  avg dur us  kernel")
    for (ph, n), (c, us, dur) in rows:
        print(f"  {ph:6s} {us/1e3/args.rounds:8.3f}  n={c/args.rounds:6.1f}  "
              f"{us/c:8.2f}  {dur/c:8.2f}  {n}")
        out.append(dict(phase=ph, kernel=n, per_round_ms=us / 1e3 / args.rounds,
                        launches_per_round=c / args.rounds, avg_excl_us=us / c,
                        avg_dur_us=dur / c))
    _, pos, tr = eng.read()
    ctx = float(pos.float().mean()) + 128
    print("mean ctx", ctx)
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(dict(variant=args.variant, rounds=args.rounds,
                                              mean_ctx=ctx, span_ms=total / 1e3 / args.rounds,
                                              phase_wall_ms={k: v / 1e3 / args.rounds
                                                             for k, v in wall.items()},
                                              kernels=out), indent=1))




def timeline(argv=None):
    """Print the kernel sequence (start/end, us) of one eager ordinary round."""
    import argparse as _a
    ap = _a.ArgumentParser()
    ap.add_argument("--warm-rounds", type=int, default=160)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--count", type=int, default=40)
    args = ap.parse_args(argv)
    spec = M.DecodeSpec(n_req=64, gamma=4, output_len=1024, prompt_len=128, seed=0)
    pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=64, ctx_cap=spec.ctx_cap(), seed=0,
                        target_branch=0.004, draft_branch=0.004)
    eng = M.SpectreEngine(pair, spec, "ordinary")
    eng.prefill(M.synthetic_prompts(64, 128, M.LLAMA_31_8B.vocab))
    eng.run(max_rounds=args.warm_rounds, use_graph=False)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.run(max_rounds=1, use_graph=False)
        torch.cuda.synchronize()
    evs = sorted(((e.time_range.start, e.time_range.end, short(e.name)) for e in prof.events()
                  if e.device_type.name == "CUDA" and "Memcpy" not in e.name
                  and "Memset" not in e.name), key=lambda x: x[0])
    t0 = evs[0][0]
    prev = None
    for i, (a, b, n) in enumerate(evs[args.first:args.first + args.count]):
        gap = (a - prev) if prev is not None else 0.0
        print(f"{i + args.first:4d} start {a - t0:9.2f} end {b - t0:9.2f} dur {b - a:7.2f} "
              f"gap_after_prev_end {gap:7.2f}  {n}")
        prev = b


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "timeline":
        timeline(sys.argv[2:])
    else:
        main()
