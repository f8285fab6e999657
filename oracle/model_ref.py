"""fp32 PyTorch restatement of the model-mode forward pass (TEST INFRASTRUCTURE).

The reference package has no model (model-path parity is
unpinned), so this module is the numerics oracle for the CUDA forward: a plain
full-sequence causal transformer in fp32 that rounds to bf16 at exactly the
points the kernels store bf16 (GEMM inputs, q/k/v after RoPE, attention
output, SwiGLU activation).  Accumulation order differs, so tests compare
with a stated tolerance and compare argmax tokens only where the top-2
logit margin exceeds it.  Only tests/ and smoke() may import this module.
"""

from __future__ import annotations

import math


def rope_table(torch, positions, head_dim: int, theta: float):
    """cos/sin exactly as k_rope_table: double precision, rounded to float."""
    half = head_dim // 2
    i = torch.arange(half, dtype=torch.float64, device=positions.device)
    inv = theta ** (-2.0 * i / head_dim)
    ang = positions.to(torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def _rms(torch, h, w, eps):
    return (h * torch.rsqrt((h * h).mean(-1, keepdim=True) + eps) * w).bfloat16().float()


def reference_forward(weights, tokens, theta=None):
    """tokens: int tensor [S] (one sequence, positions 0..S-1).
    Returns (x_final [S][d] fp32 (bf16-rounded), logits [S][V] fp32)."""
    import torch
    spec = weights.spec
    d, L, hd = spec.d_model, spec.n_layers, spec.head_dim
    nq, nkv = spec.n_q_heads, spec.n_kv_heads
    grp = nq // nkv
    theta = theta or spec.rope_theta
    S = tokens.numel()
    pos = torch.arange(S, device=tokens.device)
    cos, sin = rope_table(torch, pos, hd, theta)
    half = hd // 2

    def rope(x):  # x: [S][H][hd]
        a, b = x[..., :half], x[..., half:]
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.cat([a * c - b * s, b * c + a * s], -1)

    h = weights.embed[tokens.long()].float()
    x = _rms(torch, h, weights.attn_norm[0], spec.rms_eps)
    mask = torch.ones(S, S, dtype=torch.bool, device=tokens.device).tril()
    for l in range(L):
        qkv = x @ weights.wqkv[l].float().t()
        q = qkv[:, :nq * hd].view(S, nq, hd)
        k = qkv[:, nq * hd:(nq + nkv) * hd].view(S, nkv, hd)
        v = qkv[:, (nq + nkv) * hd:].view(S, nkv, hd)
        q = rope(q).bfloat16().float()
        k = rope(k).bfloat16().float()
        v = v.bfloat16().float()
        k = k.repeat_interleave(grp, dim=1)
        v = v.repeat_interleave(grp, dim=1)
        s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(hd)
        s = s.masked_fill(~mask[None], float("-inf"))
        m = s.amax(-1, keepdim=True)
        p = torch.exp(s - m)
        l_ = p.sum(-1, keepdim=True)
        o = torch.einsum("hqk,khd->qhd", p.bfloat16().float(), v) / l_.permute(1, 0, 2)
        o = o.reshape(S, nq * hd).bfloat16().float()
        h = h + o @ weights.wo[l].float().t()
        x = _rms(torch, h, weights.mlp_norm[l], spec.rms_eps)
        wg, wu = weights.gate_up(l)
        g = x @ wg.float().t()
        u = x @ wu.float().t()
        act = (torch.nn.functional.silu(g) * u).bfloat16().float()
        h = h + act @ weights.wd[l].float().t()
        nxt = weights.attn_norm[l + 1] if l + 1 < L else weights.final_norm
        x = _rms(torch, h, nxt, spec.rms_eps)
    logits = x @ weights.lm_head.float().t()
    return x, logits
