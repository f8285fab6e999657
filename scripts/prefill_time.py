"""Share of the C2 bench step spent in prefill (64 x 128 prompt tokens through
both models, chunks of 8 tokens per request)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import model as M
spec = M.DecodeSpec(n_req=64, gamma=4, output_len=1024, prompt_len=128, seed=0)
pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=64, ctx_cap=spec.ctx_cap(), seed=0,
                    target_branch=0.004, draft_branch=0.004)
eng = M.SpectreEngine(pair, spec, "hybrid")
prompts = M.synthetic_prompts(64, 128, M.LLAMA_31_8B.vocab, seed=0)
s = torch.cuda.Stream()
for _ in range(3):
    eng.prefill(prompts, stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(5):
    eng.prefill(prompts, stream=s)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"prefill {ms:.2f} ms per step; 8192 prompt tokens -> {8192 / ms * 1e3:.0f} tok/s; "
      f"share of a 3.67 s bench step {ms / 3670:.1%}")

from torch.profiler import profile, ProfilerActivity
from collections import defaultdict
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.prefill(prompts, stream=s)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA" and "Memcpy" not in e.name and "Memset" not in e.name:
        k = e.name.split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += e.device_time
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{t / 1e3:8.2f} ms  n={n:5d}  {t / n:8.1f} us  {k}")
