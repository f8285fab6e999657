"""Config 5 with one process per GPU: rank 0 is the draft
server, ranks 1..W-1 each own a target shard.

The state the two sides exchange lives in each engine's workspace.  Every
rank exports its workspace as a CUDA IPC handle; the draft rank attaches a
layout-only view of every target engine and each target attaches a view of
the draft engine (`spectre_engine_attach`), so `spectre_engine_exchange`
writes straight into the peer process's device memory — NVLink peer copies
when the ranks sit on different GPUs, no staging through the host.

Per round the host side carries only two small messages over the
`torch.distributed` group (gloo: CPU tensors, no device sync of its own):

  target  BEGIN (controller -> mode); push target -> draft state; [P: VERIFY]
  all     all_gather(modes)                     <- the reference's query
  draft   DRAFT (mode, or 'M' when shards differ); push draft -> target
  all     barrier                               <- the reference's reply
  target  [O / F: VERIFY]; ACCEPT

Every push is stream-synchronised before the message that announces it, so
the receiver's next launch sees the data.  The reply carries the (round,
serial) tags (target_engine.py:314-331): a push that never happens
(`run(drop=...)`) is a lost reply and trips the circuit breaker exactly as
in the single-process `disagg.DisaggregatedDecoder`, whose results this
class reproduces bit for bit.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native
from .model import DecodeSpec, ModelPair, SpectreEngine, report_from_trace

STEP_BEGIN, STEP_DRAFT, STEP_VERIFY, STEP_ACCEPT = 0, 1, 2, 3
TO_DRAFT, TO_TARGET = 0, 1
O, P, M = ord("O"), ord("P"), ord("M")


@dataclass
class _Peer:
    rank: int
    req0: int
    n: int
    handle: int          # attached view (spectre_engine_attach)
    base: int            # IPC mapping base (spectre_ipc_close)


def _export(engine: SpectreEngine) -> dict:
    L = _native.lib()
    h = (C.c_uint8 * 64)()
    off = C.c_uint64(0)
    _native.check(L.spectre_ipc_export(engine.workspace.data_ptr(), h, C.byref(off)),
                  "spectre_ipc_export")
    return dict(handle=bytes(h), offset=off.value, nbytes=engine.workspace.numel(),
                cfg=bytes(engine.cfg), tdims=bytes(engine._tdims), ddims=bytes(engine._ddims))


def _attach(info: dict) -> tuple[int, int]:
    L = _native.lib()
    base, ptr = C.c_void_p(), C.c_void_p()
    h = (C.c_uint8 * 64).from_buffer_copy(info["handle"])
    _native.check(L.spectre_ipc_open(h, info["offset"], C.byref(base), C.byref(ptr)),
                  "spectre_ipc_open")
    cfg = _native.DecodeConfig.from_buffer_copy(info["cfg"])
    tdims = _native.ModelDims.from_buffer_copy(info["tdims"])
    ddims = _native.ModelDims.from_buffer_copy(info["ddims"])
    view = L.spectre_engine_attach(C.byref(tdims), C.byref(ddims), C.byref(cfg), ptr,
                                   info["nbytes"])
    if not view:
        raise _native.SpectreError("spectre_engine_attach: " + L.spectre_last_error().decode())
    return view, base.value


class ProcessDisaggregatedDecoder:
    """Construct on every rank of an initialised process group (any backend
    that moves CPU tensors; gloo in the tests).  `shards[k]` is the request
    count of target rank k+1, or (count, spec_overrides).  `pair` is this
    rank's model pair (the draft rank uses its draft model, target ranks
    their target model)."""

    def __init__(self, pair: ModelPair, spec: DecodeSpec, variant, shards, group=None):
        torch = _native.require_cuda()
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        shards = [s if isinstance(s, tuple) else (s, {}) for s in shards]
        if len(shards) != self.world - 1:
            raise ValueError("one target shard per rank 1..W-1")
        if sum(n for n, _ in shards) != spec.n_req:
            raise ValueError("shard sizes must add up to spec.n_req")
        self.spec = spec
        self.shards = []
        r0 = 0
        for k, (n, over) in enumerate(shards):
            self.shards.append((k + 1, r0, n, over))
            r0 += n
        self.is_draft = self.rank == 0
        if self.is_draft:
            self.engine = SpectreEngine(pair, spec, variant, role="draft")
        else:
            _, self.req0, self.n, over = self.shards[self.rank - 1]
            sub = DecodeSpec(**{**spec.__dict__, **over, "n_req": self.n})
            self.engine = SpectreEngine(pair, sub, variant, role="target")
        self.variant = self.engine.variant
        self.stream = torch.cuda.Stream()
        infos = [None] * self.world
        dist.all_gather_object(infos, _export(self.engine), group=group)
        self.peers: list[_Peer] = []
        if self.is_draft:
            for rank, req0, n, _ in self.shards:
                view, base = _attach(infos[rank])
                self.peers.append(_Peer(rank, req0, n, view, base))
        else:
            view, base = _attach(infos[0])
            self.peers.append(_Peer(0, 0, spec.n_req, view, base))
        dist.barrier(group=group)

    def close(self):
        L = _native.lib()
        for p in self.peers:
            L.spectre_engine_destroy(p.handle)
            L.spectre_ipc_close(p.base)
        self.peers = []

    def _xchg(self, src, dst, direction, src0, dst0, n):
        _native.check(_native.lib().spectre_engine_exchange(
            src, dst, direction, src0, dst0, n, _native.stream_ptr(self.stream)),
            "spectre_engine_exchange")

    def prefill(self, prompts):
        """prompts [n_req][prompt_len] (all requests) on this rank's device."""
        mine = prompts if self.is_draft else prompts[self.req0:self.req0 + self.n].contiguous()
        self.engine.prefill(mine.cuda(), stream=self.stream)
        self.stream.synchronize()
        self.dist.barrier(group=self.group)

    def run(self, max_rounds: int | None = None, drop=None) -> int:
        """Decode to completion on every rank; returns the number of rounds.
        `drop(round, shard) -> bool` (evaluated on the draft rank) loses that
        shard's reply for the round."""
        torch = _native.require_cuda()
        dist, g = self.dist, self.group
        limit = max_rounds if max_rounds is not None else self.engine.max_rounds
        me = self.engine.handle
        rounds = 0
        while rounds < limit:
            mode = 0
            if not self.is_draft:
                mode = self.engine.step(STEP_BEGIN, stream=self.stream)
                if mode:
                    self._xchg(me, self.peers[0].handle, TO_DRAFT, 0, self.req0, self.n)
                    pushed = torch.cuda.Event()
                    pushed.record(self.stream)
                    if mode == P:   # overlaps the draft phase on the draft GPU
                        self.engine.step(STEP_VERIFY, stream=self.stream)
                    pushed.synchronize()   # the push, not the verify
            mine = torch.tensor([mode], dtype=torch.int64)
            gathered = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
            dist.all_gather(gathered, mine, group=g)
            modes = [int(t.item()) for t in gathered[1:]]
            if all(m == 0 for m in modes):
                break
            if self.is_draft:
                live = {m for m in modes if m}
                draft_mode = (next(iter(live)) if live in ({O}, {P})
                              else M if live & {O, P} else 0)
                if draft_mode:
                    self.engine.step(STEP_DRAFT, draft_mode, stream=self.stream)
                    for k, (p, m) in enumerate(zip(self.peers, modes)):
                        if m in (O, P) and (drop is None or not drop(rounds, k)):
                            self._xchg(me, p.handle, TO_TARGET, p.req0, 0, p.n)
                    self.stream.synchronize()
            dist.barrier(group=g)
            if not self.is_draft and mode:
                if mode != P:
                    self.engine.step(STEP_VERIFY, stream=self.stream)
                self.engine.step(STEP_ACCEPT, stream=self.stream)
            rounds += 1
        self.stream.synchronize()
        return rounds

    def gather(self):
        """(committed [n_req][out] int64, pos [n_req], per-shard traces) on
        every rank (CPU tensors)."""
        torch = _native.require_cuda()
        if self.is_draft:
            mine = None
        else:
            c, p, tr = self.engine.read()
            mine = (c.cpu(), p.cpu(), tr)
        outs = [None] * self.world
        self.dist.all_gather_object(outs, mine, group=self.group)
        outs = outs[1:]
        return (torch.cat([o[0] for o in outs]), torch.cat([o[1] for o in outs]),
                [o[2] for o in outs])

    def report(self, shard: int = 0):
        committed, pos, traces = self.gather()
        _, req0, n, _ = self.shards[shard]
        tr = traces[shard]
        return report_from_trace(self.variant, self.spec.seed, tr,
                                 int(pos[req0:req0 + n].sum().item()),
                                 float(tr["t_round_ns"].sum()) * 1e-9)
