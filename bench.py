"""SPECTRE decode-loop benchmark (BASELINE config 2) on B200.

Metric: committed output tokens/s of the SPECTRE-adaptive (hybrid) decode
loop, Llama-3.1-8B-shape target / Llama-3.2-1B-shape draft (random init,
bf16), B=64 requests per GPU, gamma=4, prompt 128, output 1024 (greedy).
A "step" is one complete pass of the hot path over one batch: prefill the
64 prompts and decode every request to 1024 output tokens.  Inputs are
synthetic; the KV cache (>L2) and weights (15 GB) are streamed every round,
so no explicit L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (one process per GPU): requests are independent, so each rank
decodes its own batch of 64 (weak scaling, default) or its shard of a global
batch (`--shard`: --batch is the job's total, split by dist.shard_requests —
strong scaling); NCCL only gathers counters.  Under torchrun the ranks come
from the environment; `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks.
--impl reference times the reference's own decode loop — stock `specsim.run`
from baseline/_ref (the unmodified reference package, installed there) or, if
that is absent, its CPU restatement oracle/lockstep.py — on every host core.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_DEFAULT = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
# draft/target agreement of the C2 pair (branch 0.004, alpha 1): the alpha_measured
# the GPU arm reports (it inverts the content accepted length); the reference arm,
# launched separately, runs the reference loop at this agreement rate
ALPHA_MEAS_C2 = 0.8709
METRIC = "SPECTRE output tok/s (8B target, B=64, gamma=4) vs ordinary/parallel SD; r* crossover"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_DEFAULT, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------- helpers
def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return ws, rank, local


def allreduce_max(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def allreduce_min(x: float, ws: int) -> float:
    return -allreduce_max(-x, ws)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


KERNELS_PER_LAYER = 8   # qkv GEMM, RoPE/KV write, attention, o GEMM, residual+norm,
#                          gate/up GEMM (SwiGLU), down GEMM, residual+norm


def forward_kernels(n_layers: int, sampling: bool, chain: bool = False) -> int:
    """embed + layers + lm_head + (argmax reduce | row sampler).  chain: the
    draft's persistent chains (chain.cu) — first chain + (attention + chain)
    per layer + lm_head + reduce."""
    if chain:
        return 1 + 2 * n_layers + 2
    return 1 + KERNELS_PER_LAYER * n_layers + 2


def kernels_per_round(mode: str, gamma: int, tL: int, dL: int, sampling: bool = False) -> int:
    """Our kernels launched by one device round (the graph body that runs)."""
    fwd_t = forward_kernels(tL, sampling)
    fwd_d = forward_kernels(dL, sampling, chain=True) - (1 if sampling else 0)   # per-request sampler
    step_d = fwd_d + 1 + (1 if sampling else 0)                       # + append (+ draft sampler)
    n = 2 + (1 if sampling else 0)  # round_begin + accept (+ accept sampler)
    n += 1 + fwd_t  # verify_prep + target forward
    if mode == "O":
        n += 1 + (gamma - 1) * step_d
    elif mode == "P":
        n += 1 + gamma * step_d
    return n


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    from paper_2605_08151_b200 import model as M
    from paper_2605_08151_b200 import _native

    ws, rank, local = dist_setup()
    dev_index = local
    g = args.gamma
    if args.shard:   # strong scaling: --batch requests in total, one contiguous shard per rank
        from paper_2605_08151_b200.dist import shard_requests
        sh = shard_requests(args.batch, ws, rank)
        B, req0, seed = sh.count, sh.start, args.seed
        if B < 1:
            raise SystemExit(f"--shard: {args.batch} requests over {ws} ranks leaves rank {rank} empty")
    else:            # weak scaling: --batch requests per rank
        B, req0, seed = args.batch, 0, args.seed + rank
    spec_kw = dict(n_req=B, gamma=g, output_len=args.out_len, prompt_len=args.prompt_len,
                   alpha=args.alpha, seed=seed, controller=args.controller,
                   temperature=args.temperature)
    base = M.DecodeSpec(**spec_kw)
    pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=B, ctx_cap=base.ctx_cap(),
                        seed=args.seed, target_branch=args.branch, draft_branch=args.branch)
    prompts = M.synthetic_prompts(B, args.prompt_len, M.LLAMA_31_8B.vocab, seed=seed, req0=req0)
    variants = [args.variant] + [v for v in ("ordinary", "parallel") if v != args.variant and
                                 not args.headline_only]
    engines = {v: M.SpectreEngine(pair, base, v) for v in variants}
    stream = torch.cuda.Stream()
    tokens_per_step = B * args.out_len

    def one_step(eng):
        eng.prefill(prompts, stream=stream)
        eng.run(use_graph=True, stream=stream)

    results = {}
    for v in variants:
        eng = engines[v]
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                one_step(eng)
        torch.cuda.synchronize()
        barrier(ws)
        clocks = ClockSampler(dev_index)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            torch.cuda.synchronize()
            barrier(ws)
            ev0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(args.steps):
                    one_step(eng)
            ev1.record(stream)
            torch.cuda.synchronize()
        barrier(ws)
        ms = ev0.elapsed_time(ev1)
        ms_max = allreduce_max(ms, ws)
        committed, pos, trace = eng.read()
        done = int((pos == args.out_len).sum().item())
        if done != B:
            raise RuntimeError(f"{v}: only {done}/{B} requests finished")
        digest = hashlib.sha256(committed.cpu().numpy().tobytes()).hexdigest()[:16]
        total_tokens = allreduce_sum(tokens_per_step * args.steps, ws)
        rep = M.report_from_trace(__import__("paper_2605_08151_b200").PolicyVariant.parse(v),
                                  args.seed, trace, tokens_per_step,
                                  float(trace["t_round_ns"].sum()) * 1e-9)
        modes = "".join(chr(int(m)) for m in trace["mode"])
        samp = args.temperature > 0
        launches = sum(kernels_per_round(m, g, M.LLAMA_31_8B.n_layers, M.LLAMA_32_1B.n_layers,
                                         samp) for m in modes) + 1   # + set_round_limit
        cs = max(1, min(16, 512 // B))         # engine prefill chunk (engine.cu:prefill_chunk)
        chunks = (args.prompt_len + cs - 1) // cs
        prefill_launches = 2 * chunks + 1  # batch kernels + admit
        prefill_launches += chunks * (forward_kernels(32, samp) + forward_kernels(16, samp, True))
        prefill_launches -= 2 * (2 * chunks - 1)   # lm_head + reduce: target's last chunk only
        results[v] = dict(
            ms_per_step=ms_max / args.steps, value=total_tokens / (ms_max / 1e3),
            rounds=len(modes), timeline=modes, clocks=clocks.summary(),
            mean_L=rep.mean_accepted_length, content_L=rep.content_mean_accepted_length,
            r_hat=rep.mean_rollback_ratio,
            pad_frac=float(trace["n_padded"].sum() / max(1, trace["participants"].sum())),
            t_round_ms=float(trace["t_round_ns"].mean()) * 1e-6,
            t_verify_ms=float(trace["t_verify_ns"].mean()) * 1e-6,
            t_draft_ms=float(trace["t_draft_ns"][trace["t_draft_ns"] > 0].mean() * 1e-6)
            if (trace["t_draft_ns"] > 0).any() else 0.0,
            gpu_launches=(launches + prefill_launches) * args.steps,
            ordinary_share=modes.count("O") / max(1, len(modes)), committed_sha256=digest)

    head = results[args.variant]
    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        eng = engines[args.variant]
        host_prompts = prompts.cpu().pin_memory()
        out_host = torch.empty(B, args.out_len, dtype=torch.int64).pin_memory()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev_prompts = torch.empty_like(prompts)
        torch.cuda.synchronize()
        barrier(ws)
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                dev_prompts.copy_(host_prompts, non_blocking=True)
                eng.prefill(dev_prompts, stream=stream)
                eng.run(use_graph=True, stream=stream)
                committed = eng.read_committed(stream=stream)
                out_host.copy_(committed, non_blocking=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = allreduce_max(ev0.elapsed_time(ev1), ws)
        e2e = {"value": allreduce_sum(tokens_per_step * args.steps, ws) / (ms / 1e3),
               "unit": "tok/s", "h2d_bytes_per_step": int(host_prompts.numel() * 4),
               "d2h_bytes_per_step": int(out_host.numel() * 8)}
        e2e_digest = hashlib.sha256(out_host.numpy().tobytes()).hexdigest()[:16]

    # ---- parity: greedy speculative decoding is lossless, so every mode (and the
    # end-to-end pass through the public API) must commit the same token stream
    digests = {v: r["committed_sha256"] for v, r in results.items()}
    if e2e is not None:
        digests["e2e"] = e2e_digest
    parity = {"committed_sha256": digests,
              "identical": len(set(digests.values())) == 1,
              "rule": ("greedy: all modes commit the autoregressive stream (bit-exact)"
                       if args.temperature <= 0 else
                       "T>0: distributional (per-position uniforms differ by mode)")}
    if ws > 1:
        parity["identical"] = bool(allreduce_min(float(parity["identical"]), ws))

    # ---- roofline of the dominant kernel, timed live (CUDA events, its own stream):
    # the draft's chain kernel (largest exclusive time per round, profiles/r02
    # kprof), with the verify gate/up GEMM (the round-1 headline kernel) beside it
    roof = roof_gu = None
    if not args.no_roofline and rank == 0:
        roof = roofline_chain(engines[args.variant], pair, args)
        roof_gu = roofline_gate_up(pair, args)
    # ---- whole-round roofline: algorithmic HBM bytes of one ordinary
    # round at the run's mean context vs the measured ordinary round time
    round_roof = None
    if "ordinary" in results and args.temperature <= 0:
        peaks, src = load_peaks()
        r = results["ordinary"]
        ctx = args.prompt_len + args.out_len / 2.0
        tgt, drf = M.LLAMA_31_8B, M.LLAMA_32_1B
        bytes_t = 2 * linear_params(tgt) + B * ctx * kv_bytes_per_token(tgt)
        bytes_d = 2 * linear_params(drf) + B * ctx * kv_bytes_per_token(drf)
        rbytes = bytes_t + (g - 1) * bytes_d
        ideal_ms = rbytes / (peaks["hbm_gbs"] * 1e9) * 1e3
        committed_per_round = tokens_per_step / max(1, r["rounds"])
        round_roof = {"mode": "ordinary", "bytes": int(rbytes), "mean_ctx": ctx,
                      "ms_at_hbm_peak": round(ideal_ms, 3), "measured_ms": round(r["t_round_ms"], 3),
                      "frac": round(ideal_ms / r["t_round_ms"], 4),
                      "tok_s_at_roofline": round(committed_per_round / ideal_ms * 1e3, 1),
                      "peak_source": src}
    alpha_meas = alpha_from_L(head["content_L"], g)
    # ---- like-for-like: the reference's own decode loop and model pair (hash
    # stream + alpha-proposer) as the device-resident oracle-mode kernel
    omode = None
    if not args.no_oracle_mode and rank == 0:
        omode = oracle_mode_speed(args, alpha_meas)
    # ---- CPU baseline (stock reference loop, or its port), rank 0, N=1 only
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and ws == 1:
        cpu = cpu_baseline(args, alpha_meas=alpha_meas, omode=omode)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(head["value"], 2), "unit": "tok/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(head["ms_per_step"], 3), "higher_is_better": True,
            "scaling": "strong" if args.shard else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic prompts (TokenStreamOracle prompt stream mod V), random-init "
                    "coupled weights",
            "config": {"workload": (f"C2: llama-3.1-8b-shape target / llama-3.2-1b-shape draft, "
                                    f"B={B}/GPU, gamma={g}, prompt {args.prompt_len}, output "
                                    f"{args.out_len}, greedy" if args.temperature <= 0 else
                                    f"C3: llama-3.1-8b-shape target / llama-3.2-1b-shape draft, "
                                    f"B={B}/GPU, gamma={g}, prompt {args.prompt_len}, output "
                                    f"{args.out_len}, T={args.temperature} rejection sampling"),
                       "temperature": args.temperature,
                       "variant": args.variant, "batch_per_gpu": B, "gamma": g,
                       "output_len": args.out_len, "prompt_len": args.prompt_len,
                       "draft_alpha": args.alpha, "branch_scale": args.branch,
                       "controller": args.controller,
                       "parallelism": f"dp{ws} ({'shards of ' + str(args.batch) + ' requests' if args.shard else 'request batches'})",
                       "l2": "inputs > L2 (15 GB weights + KV streamed per round)"},
            "e2e": e2e, "roofline": roof, "roofline_gate_up": roof_gu,
            "round_roofline": round_roof, "cpu_baseline": cpu,
            "parity": parity, "oracle_mode": omode, "alpha_measured": alpha_meas,
            "clocks": head["clocks"], "gpu_launches": head["gpu_launches"],
            "modes": {v: {k: (round(x, 4) if isinstance(x, float) else x)
                          for k, x in r.items() if k not in ("clocks", "timeline")}
                      for v, r in results.items()},
            "timeline_head": head["timeline"][:80],
        }
        print(json.dumps(line), flush=True)
        if not parity["identical"] and args.temperature <= 0:
            raise SystemExit("parity: modes committed different greedy streams")


def linear_params(spec) -> int:
    """Weights streamed by one forward pass: every layer's linears + lm_head
    (SURVEY §8d P_T / P_D; embeddings are row lookups, norms negligible)."""
    d, hd = spec.d_model, spec.head_dim
    per_layer = (d * (spec.n_q_heads + 2 * spec.n_kv_heads) * hd + spec.n_q_heads * hd * d +
                 3 * d * spec.ffn)
    return spec.n_layers * per_layer + spec.vocab * d


def kv_bytes_per_token(spec) -> int:
    return spec.n_layers * spec.n_kv_heads * spec.head_dim * 2 * 2


def alpha_from_L(L: float, gamma: int) -> float:
    """Invert E[delta] = (1 - a^gamma)/(1 - a) for a REPAIRED candidate."""
    lo, hi = 0.0, 0.999999
    for _ in range(60):
        mid = (lo + hi) / 2
        val = (1 - mid ** gamma) / (1 - mid)
        if val < L:
            lo = mid
        else:
            hi = mid
    return round((lo + hi) / 2, 4)


def _traffic(name):
    tf = ROOT / "profiles" / "r02" / "ncu_traffic.json"
    return json.loads(tf.read_text()).get(name) if tf.exists() else None


def roofline_chain(eng, pair, args):
    """The draft decode step's chain kernel (chain.cu: o, residual + norm,
    gate/up, down, residual + norm, next q/k/v, RoPE in one launch), T = B rows
    at mid context: the mid-layer chains launched back to back (PDL-chained, one
    pass = 15 launches over distinct weights, > L2), CUDA events on the
    launching stream.  Algorithmic bytes = the weights a chain streams."""
    import ctypes as C
    import torch
    from paper_2605_08151_b200 import _native
    peaks, src = load_peaks()
    L = _native.lib()
    B = args.batch
    V = pair.draft.spec.vocab
    pos = torch.full((B,), args.prompt_len + args.out_len // 2, dtype=torch.int32, device="cuda")
    ar = torch.arange(B, dtype=torch.int32, device="cuda")
    tok = (ar * 7919 + 11) % V
    # one decode-shaped draft forward leaves the draft batch at T = B rows
    eng.forward(1, tok, pos, ar, ar, torch.ones(B, dtype=torch.int32, device="cuda"), pos)
    s = torch.cuda.Stream()
    wb = C.c_int64(0)
    reps = 4
    n = L.spectre_engine_launch_chains(eng.handle, 1, C.byref(wb), int(s.cuda_stream))   # warm
    if n < 0:
        _native.check(n, "spectre_engine_launch_chains")
    times = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        n = L.spectre_engine_launch_chains(eng.handle, reps, C.byref(wb), int(s.cuda_stream))
        e1.record(s)
        e1.synchronize()
        if n < 0:
            _native.check(n, "spectre_engine_launch_chains")
        times.append(e0.elapsed_time(e1) * 1e-3 / n)
    t = statistics.median(times)
    n_mid = pair.draft.spec.n_layers - 1
    bytes_ = wb.value / n_mid
    gbs = bytes_ / t / 1e9
    hbm = peaks["hbm_gbs"]
    return {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(gbs / hbm, 4),
            "traffic": _traffic("k_chain draft mid-layer chain (o, resid, gate/up, down, resid, "
                                "qkv, rope; T=64)"),
            "kernel": f"k_chain draft mid-layer chain, T={B}",
            "bytes_per_launch": int(bytes_), "us_per_launch": round(t * 1e6, 2),
            "peak_source": src + " (MEASURED_PEAKS.json)"}


def roofline_gate_up(pair, args):
    """Target verify-pass gate/up GEMM (SwiGLU epilogue) at T = B*gamma rows."""
    import torch
    from paper_2605_08151_b200 import _native
    peaks, src = load_peaks()
    L = _native.lib()
    T = args.batch * args.gamma
    W = pair.target.wgu[0]
    F2, K = W.shape
    rows = max(512, (T + 63) // 64 * 64)   # the kernel clamps T to the buffer's rows
    X = torch.randn(rows, K, device="cuda").bfloat16()
    act = torch.empty(rows, F2 // 2, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    times = []
    n_layers = pair.target.spec.n_layers

    # the engine's launch shape: CTA pairs (cta_group::2) unless SPECTRE_GU_PAIR=0,
    # one 256-row tile per CTA (no stream-K); engines with >= 768 verify rows
    # (config 3) schedule the pairs over (tile pair, 256-token chunk) units
    large = args.batch * (args.gamma + 1) >= 768
    flags = (9000 if large else 4000) if os.environ.get("SPECTRE_GU_PAIR", "1") != "0" else 2000

    def launch(layer):
        _native.check(L.spectre_gemm_bf16(X.data_ptr(), pair.target.wgu[layer].data_ptr(), None, T,
                                          rows, F2, K, 1, 2, None, None, None, act.data_ptr(),
                                          F2 // 2, flags, int(s.cuda_stream)), "gemm")

    # back-to-back launches over every layer's weights (> L2, PDL-chained as in
    # the verify pass), CUDA events on the launching stream; repeated 4 times
    with torch.cuda.stream(s):
        for layer in range(n_layers):   # warm
            launch(layer)
        for rep in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for layer in range(n_layers):
                launch(layer)
            e1.record(s)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3 / n_layers)
    t = statistics.median(times)
    bytes_ = F2 * K * 2 + T * K * 2 + T * (F2 // 2) * 2
    flops = 2.0 * T * F2 * K
    gbs = bytes_ / t / 1e9
    tfs = flops / t / 1e12
    hbm = peaks["hbm_gbs"]
    tc = peaks["bf16_tflops"]
    # bound = whichever roof is closer to binding at this intensity
    bound = "hbm" if bytes_ / (hbm * 1e9) >= flops / (tc * 1e12) else "tensor"
    ach, peak, unit = (gbs, hbm, "GB/s") if bound == "hbm" else (tfs, tc, "TFLOP/s")
    kname = f"gemm_bf16_swapab<SwiGLU> target gate_up T={T} N={F2} K={K}"
    traffic = _traffic(kname)   # ncu capture of the same launch shape
    return {"bound": bound, "achieved": round(ach, 1), "peak": peak, "unit": unit,
            "frac": round(ach / peak, 4), "traffic": traffic,
            "kernel": f"gemm_bf16_swapab<SwiGLU> target gate_up T={T} N={F2} K={K}",
            "us_per_launch": round(t * 1e6, 2), "tflops": round(tfs, 1), "gbs": round(gbs, 1),
            "peak_source": src + " (MEASURED_PEAKS.json burst)"}


# ----------------------------------------------------------------- the reference loop on CPU
REF_DIR = ROOT / "baseline" / "_ref"


def reference_kind() -> str:
    """'reference': stock specsim from baseline/_ref (the unmodified package);
    'port': oracle/lockstep.py, its CPU restatement (pinned to 65 reference runs)."""
    return "reference" if (REF_DIR / "specsim" / "__init__.py").exists() else "port"


def _ref_worker(job):
    """One CPU worker: one decode of the reference loop for one seed."""
    cfg, variant, kind = job
    t0 = time.perf_counter()
    if kind == "reference":
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import specsim
        from specsim.metrics import export_report
        r = specsim.run(specsim.SimConfig(**cfg), variant)
        return r.report.total_committed, time.perf_counter() - t0, export_report(r.report, "csv")
    from oracle import lockstep as L
    r = L.run(cfg, variant)
    return r.report["total_committed"], time.perf_counter() - t0, L.export_csv(r.report)


def _pool_run(cfgs, variant, procs, kind):
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        return pool.map(_ref_worker, [(c, variant, kind) for c in cfgs])


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _ref_cfg(args, alpha):
    return dict(batch_size=args.batch, n_requests=args.batch, gamma=args.gamma,
                output_len=args.out_len, alpha=alpha, qps=1e6, seed=args.seed)


def cpu_baseline(args, alpha_meas: float, omode=None):
    """The reference's decode loop on CPU (stock specsim when installed in
    baseline/_ref, else oracle/lockstep.py), one process per host core, one seed
    per process, about one decode per core.  Also checks that the
    device oracle-mode run reproduced the reference's report byte for byte."""
    procs = os.cpu_count() or 1
    kind = reference_kind()
    cfg = _ref_cfg(args, alpha_meas)
    t0 = time.perf_counter()
    res = _pool_run([{**cfg, "seed": args.seed + i} for i in range(procs)], "hybrid", procs, kind)
    dt = time.perf_counter() - t0
    toks = sum(r[0] for r in res)
    if omode is not None and "report_csv" in omode:
        omode["report_identical_to_reference"] = omode.pop("report_csv") == res[0][2]
        omode["checked_against"] = kind
    return {"value": round(toks / dt, 1), "unit": "tok/s", "cores": procs, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"{procs} x {'specsim.run' if kind == 'reference' else 'oracle/lockstep.run'}"
                      f"(hybrid, B={args.batch}, gamma={args.gamma}, output_len={args.out_len}, "
                      f"alpha={alpha_meas} = the GPU run's measured agreement), one process per "
                      f"host core (multiprocessing); per-core "
                      f"{toks / sum(r[1] for r in res):.0f} tok/s; {dt:.1f} s wall"}


def oracle_mode_speed(args, alpha):
    """The reference's protocol AND model pair (hash stream + alpha-proposer),
    decoded by the device-resident oracle-mode loop through the public API
    (host config in, host report out): the like-for-like figure against the
    reference arm.  Wall time per decode, CUDA-synchronised on both sides."""
    import torch
    import paper_2605_08151_b200 as P
    cfg = _ref_cfg(args, alpha)
    P.run(P.SimConfig(**cfg), "hybrid")   # warm (allocations, module load)
    torch.cuda.synchronize()
    n = max(3, args.steps)
    t0 = time.perf_counter()
    for _ in range(n):
        got = P.run(P.SimConfig(**cfg), "hybrid")
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    tok = got.report.total_committed
    return {"value": round(tok / dt, 1), "unit": "tok/s", "ms_per_decode": round(dt * 1e3, 3),
            "decodes": n, "config": f"hybrid, B={args.batch}, gamma={args.gamma}, output_len="
                                    f"{args.out_len}, alpha={alpha}, seed={args.seed}",
            "report_csv": P.export_report(got.report)}


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    alpha = args.alpha_meas
    procs = os.cpu_count() or 1
    kind = reference_kind()
    cfg = _ref_cfg(args, alpha)
    _pool_run([{**cfg, "seed": args.seed + 1000 + i} for i in range(min(procs, args.warmup))],
              args.variant, procs, kind)
    t0 = time.perf_counter()
    toks = 0
    for step in range(args.steps):   # a step = one B=64 decode per host core
        res = _pool_run([{**cfg, "seed": args.seed + step * procs + i} for i in range(procs)],
                        args.variant, procs, kind)
        toks += sum(r[0] for r in res)
    dt = time.perf_counter() - t0
    v = toks / dt
    what = ("stock specsim.run from baseline/_ref (the unmodified reference package)"
            if kind == "reference" else "oracle/lockstep.run (CPU restatement; baseline/_ref "
                                        "absent)")
    sample = (f"{args.steps} steps x {procs} processes x {what}({args.variant}, B={args.batch}, "
              f"gamma={args.gamma}, output_len={args.out_len}, alpha={alpha}); one decode per "
              f"host core per step")
    print(json.dumps({
        "metric": METRIC, "value": round(v, 2), "unit": "tok/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (reference TokenStreamOracle model pair)", "impl": "reference",
        "config": {"workload": "C2 protocol shape on the reference's synthetic model pair "
                               "(the reference has no neural model)",
                   "variant": args.variant, "batch": args.batch, "gamma": args.gamma,
                   "output_len": args.out_len, "alpha": alpha},
        "cpu_baseline": {"value": round(v, 2), "unit": "tok/s", "cores": procs, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(v, 2), "unit": "tok/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int, argv: list[str], script: str | None = None) -> int:
    """`--gpus N` without torchrun: re-launch under torch.distributed.run, one
    process per GPU (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           script or str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--variant", default="hybrid")
    ap.add_argument("--batch", type=int, default=64,
                    help="requests per GPU (weak scaling) or in total with --shard")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: split --batch requests over the ranks")
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--out-len", type=int, default=1024)
    ap.add_argument("--prompt-len", type=int, default=128)
    ap.add_argument("--alpha", type=float, default=1.0, help="draft keep probability")
    ap.add_argument("--alpha-meas", type=float, default=ALPHA_MEAS_C2,
                    help="reference arm: agreement rate of the synthetic pair (the GPU run's "
                         "measured draft/target agreement at C2)")
    ap.add_argument("--branch", type=float, default=0.004)
    ap.add_argument("--controller", default="round")
    ap.add_argument("--temperature", type=float, default=0.0,
                    help="0: greedy (C2); > 0: speculative rejection sampling (C3)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-oracle-mode", action="store_true")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None and int(ws_env) != args.gpus and int(ws_env) > 1:
        raise SystemExit(f"--gpus {args.gpus} disagrees with WORLD_SIZE={ws_env}")
    if args.impl == "reference":
        run_reference(args)      # rank 0 only; CPU work, no GPU needed
        return 0
    if args.gpus > 1 and ws_env is None:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"--gpus {args.gpus}: only {have} CUDA device(s) visible")
        return spawn_ranks(args.gpus, argv)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
