"""tests/golden/scheduler.json: schedule_round (draft_engine.py:134-155) of the
UNMODIFIED reference on random ready queues / counters / capacities.
    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden_scheduler.py"""
import json
import random
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from specsim.draft_engine import (DraftQueueItem, FairnessCounter, QueueClass,  # noqa: E402
                                  schedule_round)

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "scheduler.json"
rng = random.Random(2605)
cases = []
for _ in range(400):
    ns, nr = rng.randint(0, 40), rng.randint(0, 40)
    period, cap = rng.randint(1, 12), rng.randint(1, 64)
    counter = rng.randint(0, period)
    items = ([DraftQueueItem(QueueClass.SPECULATIVE, i, 0.0, count=4) for i in range(ns)] +
             [DraftQueueItem(QueueClass.REGULAR, 1000 + i, 0.0, remaining=5) for i in range(nr)])
    sched, fc, forced = schedule_round(items, FairnessCounter(counter, period), cap)
    cases.append(dict(n_spec=ns, n_reg=nr, counter=counter, period=period, capacity=cap,
                      spec=[it.request for it in sched if it.queue_class is QueueClass.SPECULATIVE],
                      reg=[it.request - 1000 for it in sched if it.queue_class is QueueClass.REGULAR],
                      counter_after=fc.consecutive_speculative, forced=forced))
OUT.write_text(json.dumps({"cases": cases}))
print(f"wrote {len(cases)} schedule_round cases")
