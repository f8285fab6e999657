"""Diagnostic: time isolated target (T=256) / draft (T=64) forward passes,
eager vs CUDA graph, to separate kernel time from launch gaps."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2605_08151_b200 import model as M

n = 64
spec = M.DecodeSpec(n_req=n, gamma=4, output_len=1024, prompt_len=128, seed=0)
pair = M.build_pair(M.LLAMA_31_8B, M.LLAMA_32_1B, n_req=n, ctx_cap=spec.ctx_cap(), seed=0,
                    target_branch=0.004, draft_branch=0.004)
eng = M.SpectreEngine(pair, spec, "ordinary")
prompts = M.synthetic_prompts(n, 128, M.LLAMA_31_8B.vocab)
eng.prefill(prompts)
torch.cuda.synchronize()
for which, per in ((0, 4), (1, 1)):
    T = n * per
    tok = prompts[:, :per].reshape(-1).contiguous()
    pos = (torch.arange(per, device="cuda") + 500).repeat(n)
    slot = torch.arange(n, device="cuda").repeat_interleave(per)
    q_off = torch.arange(n, device="cuda") * per
    n_new = torch.full((n,), per, device="cuda")
    pos0 = torch.full((n,), 500, device="cuda")
    for _ in range(3):
        eng.forward(which, tok, pos, slot, q_off, n_new, pos0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        eng.forward(which, tok, pos, slot, q_off, n_new, pos0)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"model={'target' if which == 0 else 'draft'} T={T} eager forward (incl host sync+memcpy) "
          f"median {ts[len(ts)//2]*1e3:.3f} ms min {ts[0]*1e3:.3f} ms", flush=True)
