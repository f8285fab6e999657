"""World-size-2 (gloo, CPU) coverage of the multi-GPU host path.

Each rank decodes its own request shard (here with the CPU oracle standing in
for the device loop, which needs a GPU) and the ranks aggregate only counters:
max time, total tokens, gathered reports.  SURVEY §8e: multi-GPU results must
equal the union of per-shard single-process runs on the same shards/seeds.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2605_08151_b200.dist import shard_requests


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_cfg(shard, base):
    return dict(base, batch_size=max(shard.count, 1), n_requests=shard.count,
                seed=base["seed"] + shard.rank)


def _worker(rank, world, port, base, q):
    import torch.distributed as dist
    from oracle import lockstep as L
    from paper_2605_08151_b200.dist import aggregate, gather_objects, shard_requests
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = shard_requests(base["n_requests"], world, rank)
        r = L.run(_shard_cfg(shard, base), "hybrid")
        secs, toks = aggregate(r.report["sim_duration"], r.report["total_committed"])
        reports = gather_objects((rank, L.export_csv(r.report)))
        q.put((rank, secs, toks, reports))
    finally:
        dist.destroy_process_group()


def test_sharding_is_a_partition():
    for n in (1, 7, 64, 256, 257):
        for world in (1, 2, 3, 8):
            shards = [shard_requests(n, world, r) for r in range(world)]
            ids = [i for s in shards for i in s.global_ids()]
            assert ids == list(range(n))
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1


@pytest.mark.timeout(180)
def test_two_rank_gloo_aggregation_matches_per_shard_runs():
    from oracle import lockstep as L
    base = dict(n_requests=16, output_len=48, gamma=4, alpha=0.8, qps=1e6, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, base, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=150) for _ in procs]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    out.sort()
    # the same shards run alone in this process
    single = [L.run(_shard_cfg(shard_requests(16, 2, r), base), "hybrid") for r in range(2)]
    want_secs = max(s.report["sim_duration"] for s in single)
    want_toks = sum(s.report["total_committed"] for s in single)
    for rank, secs, toks, reports in out:
        assert secs == want_secs
        assert toks == want_toks == 16 * 48
        assert [csv for _, csv in sorted(reports)] == [L.export_csv(s.report) for s in single]
