"""CPU restatement of the draft server's fairness scheduler (TEST INFRASTRUCTURE).

Only tests/ may import this module.  It restates
`schedule_round` (/root/reference/pkg/src/specsim/draft_engine.py:134-155) and
the per-round regular-token accounting of `DraftServer.finish_round`
(draft_engine.py:355-394), and replays the model-mode draft phase the device
engine runs (csrc/model_protocol.cu: k_bg_schedule / k_draft_prep): an
optional forced regular round (1 step), then the round that serves this
phase's speculative queries.  Pinned against the reference's own
schedule_round by tests/golden/scheduler.json (scripts/make_golden_scheduler.py).
"""

from __future__ import annotations


def schedule_round(spec: list, regular: list, counter: int, period: int, capacity: int):
    """draft_engine.py:134-155.  `spec` / `regular`: ready items in FIFO order.
    Returns (scheduled spec, scheduled regular, new counter, forced)."""
    if capacity < 1:
        raise ValueError(f"capacity must be >= 1, got {capacity}")
    if counter >= period and regular:
        return [], list(regular[:capacity]), 0, True
    s = list(spec[:capacity])
    r = list(regular[:capacity - len(s)])
    counter = min(counter + 1, period) if s else 0
    return s, r, counter, False


def replay_phases(n_spec_per_phase, n_bg: int, bg_len: int, steps_per_phase, period: int,
                  capacity: int):
    """The device's model-mode draft phases: per phase, a forced regular round
    (steps 1) when the counter is due and regular work waits, then the round
    serving the phase's speculative queries (steps = the phase's draft steps).
    Regular items: background requests 0..n_bg-1 in FIFO order, bg_len tokens
    each; a scheduled item emits min(remaining, steps) tokens per round
    (draft_engine.py:389-394).  Returns per phase (n_forced_regular,
    n_regular, counter_after) and the final remaining counts."""
    remaining = [bg_len] * n_bg
    counter = 0
    out = []
    for n_spec, steps in zip(n_spec_per_phase, steps_per_phase):
        ready_reg = [j for j in range(n_bg) if remaining[j] > 0]
        n_forced = 0
        if counter >= period and ready_reg:
            _, reg, counter, _ = schedule_round([], ready_reg, counter, period, capacity)
            n_forced = len(reg)
            for j in reg:
                remaining[j] -= min(remaining[j], 1)
            ready_reg = [j for j in range(n_bg) if remaining[j] > 0]
        spec, reg, counter, _ = schedule_round(list(range(n_spec)), ready_reg, counter, period,
                                               capacity)
        eff_steps = steps if spec else 1
        for j in reg:
            remaining[j] -= min(remaining[j], eff_steps)
        out.append((n_forced, len(reg), counter))
    return out, remaining
