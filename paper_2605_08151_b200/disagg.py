"""Config 5: disaggregated draft / target.

The reference's topology is a draft server and a target endpoint joined by
channels (`draft_engine.py:DraftServer`, `target_engine.py`, `sim.py:235-236`);
the paper ran the drafter on its own GPUs.  Here one
draft-role engine serves every request and one or more target-role engines
each own a shard.  A round is host-driven:

  target BEGIN (controller -> mode)
  exchange target -> draft  (mode, committed tokens, positions, cache flags)
  ordinary:  draft DRAFT ; exchange draft -> target ; target VERIFY ; ACCEPT
  parallel:  draft DRAFT  ∥  target VERIFY ; join ; exchange draft -> target ; ACCEPT
  ar:        target VERIFY ; ACCEPT

Each target shard runs its own controller and may pick its own mode; one
draft phase serves all speculating shards (mode 'M' when they differ: the
draft reads each request's mode from the exchange).  Every query carries a
(round, serial) tag the draft's reply must echo (target_engine.py:314-331):
a reply that never arrives (`run(drop=...)`) degrades its requests to
FALLBACK / PADDED candidates, counts as a timeout for that shard's circuit
breaker (target_engine.py:337-380) and never costs losslessness.

Exchanges are device-to-device copies of a few KB per request
(`spectre_engine_exchange`, cudaMemcpyDefault: NVLink peer copies when the
engines sit on different GPUs); the cross-device ordering is CUDA events.
With the same seeds and a deterministic controller the committed streams are
bit-identical to the single-engine loop (tests/test_gpu_disagg.py).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native
from .decoder import PolicyVariant  # noqa: F401  (re-exported for callers)
from .model import DecodeSpec, ModelPair, SpectreEngine, report_from_trace

STEP_BEGIN, STEP_DRAFT, STEP_VERIFY, STEP_ACCEPT = 0, 1, 2, 3
TO_DRAFT, TO_TARGET = 0, 1


@dataclass
class Shard:
    engine: SpectreEngine
    req0: int          # first request of this shard in the draft server's numbering
    n: int
    stream: object
    device: int        # GPU holding this target replica


def _device_of(pair: ModelPair) -> int:
    return pair.target.embed.device.index or 0


class DisaggregatedDecoder:
    """One draft server + target shards.  `shards` is a list of
    (target_pair, n_requests) or (target_pair, n_requests, spec_overrides);
    the draft pair serves their concatenation.  Overrides (e.g. a replica's
    own t_target / t_draft latency model) apply to that shard's controller."""

    def __init__(self, draft_pair: ModelPair, target_pairs: list[tuple[ModelPair, int]],
                 spec: DecodeSpec, variant: PolicyVariant | str):
        torch = _native.require_cuda()
        target_pairs = [tuple(t) + ({},) * (3 - len(t)) for t in target_pairs]
        n_total = sum(t[1] for t in target_pairs)
        if n_total != spec.n_req:
            raise ValueError("shard sizes must add up to spec.n_req")
        self.spec = spec
        self.draft_device = _device_of(draft_pair)
        with torch.cuda.device(self.draft_device):
            self.draft = SpectreEngine(draft_pair, spec, variant, role="draft")
            self.draft_stream = torch.cuda.Stream()
        self.shards = []
        r0 = 0
        for pair, n, over in target_pairs:
            dev = _device_of(pair)
            _native.check(_native.lib().spectre_enable_peer_access(self.draft_device, dev),
                          "spectre_enable_peer_access")
            sub = DecodeSpec(**{**spec.__dict__, **over, "n_req": n})
            with torch.cuda.device(dev):
                eng = SpectreEngine(pair, sub, variant, role="target")
                self.shards.append(Shard(eng, r0, n, torch.cuda.Stream(), dev))
            r0 += n
        self.variant = self.draft.variant

    def _on(self, sh):
        torch = _native.require_cuda()
        return torch.cuda.device(sh.device if sh is not None else self.draft_device)

    def _xchg(self, src, dst, direction, src0, dst0, n, stream):
        _native.check(_native.lib().spectre_engine_exchange(
            src.handle, dst.handle, direction, src0, dst0, n, _native.stream_ptr(stream)),
            "spectre_engine_exchange")

    def prefill(self, prompts):
        """prompts [n_req][prompt_len] on the device."""
        torch = _native.require_cuda()
        with self._on(None):
            self.draft.prefill(prompts.to(f"cuda:{self.draft_device}"), stream=self.draft_stream)
        for sh in self.shards:
            with self._on(sh):
                sh.engine.prefill(prompts[sh.req0:sh.req0 + sh.n].to(f"cuda:{sh.device}")
                                  .contiguous(), stream=sh.stream)
        for dev in {self.draft_device, *(sh.device for sh in self.shards)}:
            torch.cuda.synchronize(dev)

    def run(self, max_rounds: int | None = None, drop=None) -> int:
        """Decode to completion (or `max_rounds`).  `drop(round, shard) -> bool`
        (fault injection) loses that shard's draft reply: its draft -> target
        exchange is skipped, as a lost DRAFT_REPLY would be (sim.py:816-844)."""
        torch = _native.require_cuda()
        rounds = 0
        limit = max_rounds if max_rounds is not None else self.shards[0].engine.max_rounds
        ds = self.draft_stream
        O, P = ord("O"), ord("P")
        while rounds < limit:
            # every shard runs its own controller (the paper decides per batch)
            modes = []
            for sh in self.shards:
                with self._on(sh):
                    modes.append(sh.engine.step(STEP_BEGIN, stream=sh.stream))
            if all(m == 0 for m in modes):
                break
            live = {m for m in modes if m}
            # one draft phase serves every speculating shard; shards that chose
            # different modes get a mixed phase (per-request mode, 'M')
            draft_mode = (next(iter(live)) if live in ({O}, {P})
                          else ord("M") if live & {O, P} else 0)
            for sh, m in zip(self.shards, modes):
                if not m:
                    continue
                with self._on(sh):
                    self._xchg(sh.engine, self.draft, TO_DRAFT, 0, sh.req0, sh.n, sh.stream)
                    ev = torch.cuda.Event()
                    ev.record(sh.stream)
                ds.wait_event(ev)
            ev_draft = None
            if draft_mode:
                with self._on(None):
                    self.draft.step(STEP_DRAFT, draft_mode, stream=ds)
                    ev_draft = torch.cuda.Event()
                    ev_draft.record(ds)
            # parallel shards verify while the draft speculates
            for sh, m in zip(self.shards, modes):
                if m == P:
                    with self._on(sh):
                        sh.engine.step(STEP_VERIFY, stream=sh.stream)
            for sh, m in zip(self.shards, modes):
                if not m:
                    continue
                k = self.shards.index(sh)
                with self._on(sh):
                    if m in (O, P):
                        sh.stream.wait_event(ev_draft)
                        if drop is None or not drop(rounds, k):
                            self._xchg(self.draft, sh.engine, TO_TARGET, sh.req0, 0, sh.n,
                                       sh.stream)
                    if m != P:
                        sh.engine.step(STEP_VERIFY, stream=sh.stream)
                    sh.engine.step(STEP_ACCEPT, stream=sh.stream)
            for sh in self.shards:   # next round's draft sync starts after this accept
                with self._on(sh):
                    ev = torch.cuda.Event()
                    ev.record(sh.stream)
                ds.wait_event(ev)
            rounds += 1
        for dev in {self.draft_device, *(sh.device for sh in self.shards)}:
            torch.cuda.synchronize(dev)
        return rounds

    def read(self):
        """(committed [n_req][out], pos [n_req], per-shard traces)."""
        torch = _native.require_cuda()
        outs = []
        for sh in self.shards:
            with self._on(sh):
                outs.append(sh.engine.read())
        committed = torch.cat([o[0].cpu() for o in outs])
        pos = torch.cat([o[1].cpu() for o in outs])
        return committed, pos, [o[2] for o in outs]

    def report(self, shard: int = 0):
        _, pos, traces = self.read()
        tr = traces[shard]
        total = int(pos[self.shards[shard].req0:self.shards[shard].req0 +
                        self.shards[shard].n].sum().item())
        return report_from_trace(self.variant, self.spec.seed, tr, total,
                                 float(tr["t_round_ns"].sum()) * 1e-9)
