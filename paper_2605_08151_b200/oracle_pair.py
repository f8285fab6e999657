"""GPU-backed synthetic model pair — the reference's `TokenStreamOracle` plug-in.

Same duck type as /root/reference/pkg/src/specsim/oracle.py:47-113
(reference_token, reference_prefix, prompt_token(s), draft_propose, verify),
computed by the K8 kernels in csrc/oracle_mode.cu.  Batch forms
(`reference_tokens`, `verify_batch`, `propose_batch`) are the efficient entry
points; the scalar methods exist so reference code can call it unchanged.
The caller owns `rng` exactly as in the reference: uniforms are
drawn from it on the host, in order, one per proposed token.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import PAD, SpeculativeSegment

_MASK = (1 << 64) - 1


@dataclass(frozen=True)
class VerifyOutcome:
    accepted_count: int
    committed: tuple
    bonus: int
    new_position: int


@dataclass(frozen=True)
class TokenStreamOracle:
    seed: int = 0

    # -- batch device entry points ------------------------------------------
    def reference_tokens(self, requests, positions, stream_id: int = 0) -> np.ndarray:
        torch = _native.require_cuda()
        L = _native.lib()
        req = torch.as_tensor(np.asarray(requests, dtype=np.int64)).cuda()
        pos = torch.as_tensor(np.asarray(positions, dtype=np.int64)).cuda()
        if (pos < 0).any():
            raise ValueError("position must be >= 0")
        out = torch.empty_like(req)
        _native.check(L.spectre_oracle_stream(self.seed & _MASK, stream_id, req.data_ptr(),
                                              pos.data_ptr(), out.data_ptr(), req.numel(),
                                              _native.stream_ptr()), "spectre_oracle_stream")
        return out.cpu().numpy().view(np.uint64)

    def verify_batch(self, requests, starts, candidates, lengths):
        """candidates: [n, width] uint64 (PAD-padded).  Returns (accepted, bonus)."""
        torch = _native.require_cuda()
        L = _native.lib()
        cand = np.ascontiguousarray(np.asarray(candidates, dtype=np.uint64))
        n, width = cand.shape
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=dt))).cuda()
        req, st = t(requests, np.int64), t(starts, np.int64)
        cnd = torch.as_tensor(cand.view(np.int64)).cuda()
        ln = t(lengths, np.int32)
        acc = torch.empty(n, dtype=torch.int32, device="cuda")
        bonus = torch.empty(n, dtype=torch.int64, device="cuda")
        _native.check(L.spectre_oracle_verify(self.seed & _MASK, req.data_ptr(), st.data_ptr(),
                                              cnd.data_ptr(), ln.data_ptr(), width,
                                              acc.data_ptr(), bonus.data_ptr(), n,
                                              _native.stream_ptr()), "spectre_oracle_verify")
        return acc.cpu().numpy(), bonus.cpu().numpy().view(np.uint64)

    def propose_batch(self, requests, starts, counts, alpha: float, uniforms) -> np.ndarray:
        torch = _native.require_cuda()
        L = _native.lib()
        counts = np.asarray(counts, dtype=np.int32)
        off = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
        maxc = int(counts.max()) if len(counts) else 0
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=dt))).cuda()
        out = torch.empty(len(counts) * max(maxc, 1), dtype=torch.int64, device="cuda")
        u = t(uniforms, np.float64) if len(uniforms) else torch.zeros(1, dtype=torch.float64,
                                                                      device="cuda")
        keep = [t(requests, np.int64), t(starts, np.int64), t(counts, np.int32),
                t(off, np.int64)]                      # alive until the kernel ran
        _native.check(L.spectre_oracle_propose(
            self.seed & _MASK, float(alpha), keep[0].data_ptr(), keep[1].data_ptr(),
            keep[2].data_ptr(), keep[3].data_ptr(), u.data_ptr(), out.data_ptr(), maxc,
            len(counts),
            _native.stream_ptr()), "spectre_oracle_propose")
        res = out.cpu().numpy().view(np.uint64).reshape(len(counts), max(maxc, 1))
        del keep
        return res

    # -- reference duck type (oracle.py:53-113) ---------------------------------
    def reference_token(self, request: int, position: int) -> int:
        if position < 0:
            raise ValueError(f"position must be >= 0, got {position}")
        return int(self.reference_tokens([request], [position])[0])

    def reference_prefix(self, request: int, length: int) -> list:
        if length <= 0:
            return []
        return [int(x) for x in self.reference_tokens([request] * length, range(length))]

    def prompt_token(self, request: int, index: int) -> int:
        return int(self.reference_tokens([request], [index], stream_id=1)[0])

    def prompt_tokens(self, request: int, length: int) -> list:
        if length <= 0:
            return []
        return [int(x) for x in self.reference_tokens([request] * length, range(length), 1)]

    def draft_propose(self, request: int, start: int, count: int, alpha: float,
                      rng: random.Random, origin_round: int = -1) -> SpeculativeSegment:
        if count < 0:
            raise ValueError(f"count must be >= 0, got {count}")
        if count == 0:
            return SpeculativeSegment((), start, origin_round)
        u = [rng.random() for _ in range(count)]
        toks = self.propose_batch([request], [start], [count], alpha, u)[0]
        return SpeculativeSegment(tuple(int(x) for x in toks), start, origin_round)

    def verify(self, request: int, start: int, candidate) -> VerifyOutcome:
        cand = list(candidate)
        if not cand:
            cand_arr = np.full((1, 1), PAD, dtype=np.uint64)
            ln = [0]
        else:
            cand_arr = np.asarray([cand], dtype=np.uint64)
            ln = [len(cand)]
        acc, bonus = self.verify_batch([request], [start], cand_arr, ln)
        a = int(acc[0])
        committed = tuple(self.reference_prefix_from(request, start, a)) + (int(bonus[0]),)
        return VerifyOutcome(a, committed, int(bonus[0]), start + a + 1)

    def reference_prefix_from(self, request: int, start: int, length: int) -> list:
        if length <= 0:
            return []
        return [int(x) for x in self.reference_tokens([request] * length,
                                                       range(start, start + length))]
