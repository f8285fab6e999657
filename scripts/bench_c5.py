"""Config 5 on one GPU: Qwen2.5-32B-shape target + Qwen2.5-0.5B-shape draft,
B=128, gamma=6, greedy — the single-engine loop vs the disaggregated draft
server + target shard (paper_2605_08151_b200/disagg.py) on the same device.
On an 8-GPU box the draft server would sit on GPU 0 and target replicas on
GPUs 1-7 with the same exchanges running as NVLink peer copies; here the
run measures the protocol split's cost and checks the streams agree.

  python scripts/bench_c5.py [--out-len 256] [--variant ordinary]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2605_08151_b200 import model as M
from paper_2605_08151_b200.disagg import DisaggregatedDecoder


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-req", type=int, default=128)
    ap.add_argument("--gamma", type=int, default=6)
    ap.add_argument("--out-len", type=int, default=256)
    ap.add_argument("--variant", default="ordinary")
    ap.add_argument("--branch", type=float, default=0.004)
    ap.add_argument("--out", default="gpurun_out/bench_c5.json")
    args = ap.parse_args()
    spec = M.DecodeSpec(n_req=args.n_req, gamma=args.gamma, output_len=args.out_len,
                        prompt_len=128, seed=0, controller="reference")
    t0 = time.time()
    pair = M.build_pair(M.QWEN_25_32B, M.QWEN_25_05B, n_req=args.n_req, ctx_cap=spec.ctx_cap(),
                        seed=0, target_branch=args.branch, draft_branch=args.branch)
    build_s = time.time() - t0
    prompts = M.synthetic_prompts(args.n_req, 128, M.QWEN_25_32B.vocab, seed=0)
    res = {"workload": f"C5 shapes: qwen2.5-32b target / qwen2.5-0.5b draft, B={args.n_req}, "
                       f"gamma={args.gamma}, output {args.out_len}, greedy, one GPU",
           "variant": args.variant, "weights_build_s": round(build_s, 1)}

    # single engine (device round loop, CUDA graph)
    eng = M.SpectreEngine(pair, spec, args.variant)
    eng.prefill(prompts)
    eng.run(use_graph=True)
    torch.cuda.synchronize()
    eng.prefill(prompts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.run(use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    committed, pos, tr = eng.read()
    assert int((pos == args.out_len).sum()) == args.n_req
    res["engine"] = dict(ms=round(ms, 1), tok_s=round(args.n_req * args.out_len / ms * 1e3, 1),
                         rounds=len(tr["mode"]),
                         mean_L=round(float(tr["delta"].sum() / tr["participants"].sum()), 4))
    ref_committed = committed.cpu()
    del eng
    torch.cuda.empty_cache()

    # disaggregated: draft server + one target shard (same GPU here)
    dd = DisaggregatedDecoder(pair, [(pair, args.n_req)], spec, args.variant)
    dd.prefill(prompts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rounds = dd.run()
    dt = time.perf_counter() - t0
    c2, p2, _ = dd.read()
    res["disaggregated"] = dict(s=round(dt, 3), tok_s=round(args.n_req * args.out_len / dt, 1),
                                rounds=rounds, host_driven=True,
                                identical_to_engine=bool(torch.equal(c2, ref_committed)))
    print(json.dumps(res))
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
