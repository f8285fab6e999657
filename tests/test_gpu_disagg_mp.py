"""Config 5 with one process per GPU (paper_2605_08151_b200/disagg_mp.py):
a draft-server process and two target-shard processes exchange state through
CUDA IPC-mapped workspaces, host messages over gloo.  Only one GPU exists
here, so all three processes share cuda:0 (IPC between processes on one
device); results must equal the single-process decode bit for bit."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_08151_b200 import model as M
    from paper_2605_08151_b200.disagg_mp import ProcessDisaggregatedDecoder
    n, na = 8, 3
    variant = case["variant"]
    spec = M.DecodeSpec(n_req=n, gamma=4, output_len=case.get("out", 64), prompt_len=16,
                        alpha=case.get("alpha", 0.8), seed=31, controller="reference")
    shards = [(na, case.get("over_a", {})), (n - na, case.get("over_b", {}))]
    sizes = [n] + [na, n - na]
    pair = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=sizes[rank], ctx_cap=256, seed=31)
    prompts = M.synthetic_prompts(n, spec.prompt_len, M.TINY_TARGET.vocab, spec.seed)
    dd = ProcessDisaggregatedDecoder(pair, spec, variant, shards)
    dd.prefill(prompts)
    drop = (lambda r, k: True) if case.get("drop_all") else None
    dd.run(drop=drop)
    committed, pos, traces = dd.gather()
    dd.close()
    if rank == 0:   # the checker: single-process decodes on the same device
        assert (pos == spec.output_len).all()
        full = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=n, ctx_cap=256, seed=31)
        if case.get("drop_all"):
            ref = M.decode(full, spec, "ar", use_graph=False)
            assert torch.equal(committed, ref.committed.cpu())
            tl = "".join(chr(int(m)) for m in traces[0]["mode"])
            # the reference's windows (5, 9), (14, 18): timeouts detected at the
            # next round's commit (reply_timeout = 2 T_T)
            assert tl[4:9] == "FFFFF" and tl[13:18] == "FFFFF", tl
            assert int(traces[0]["n_stale"].sum()) > 0
        elif case.get("over_a"):
            refs = []
            for lo, hi, over in ((0, na, case["over_a"]), (na, n, case["over_b"])):
                sub = M.DecodeSpec(**{**spec.__dict__, **over, "n_req": hi - lo})
                p1 = M.build_pair(M.TINY_TARGET, M.TINY_DRAFT, n_req=hi - lo, ctx_cap=256,
                                  seed=31)
                refs.append(M.decode(p1, sub, variant, prompts=prompts[lo:hi].contiguous(),
                                     use_graph=False))
            assert torch.equal(committed, torch.cat([r.committed.cpu() for r in refs]))
            for tr, r in zip(traces, refs):
                assert (tr["mode"] == r.trace["mode"]).all()
        else:
            ref = M.decode(full, spec, variant, use_graph=False)
            assert torch.equal(committed, ref.committed.cpu())
            for tr in traces:
                assert (tr["n_stale"] == 0).all()
    dist.barrier()
    dist.destroy_process_group()


CASES = {
    "ordinary": dict(variant="ordinary"),
    "parallel": dict(variant="parallel"),
    "hybrid_mixed": dict(variant="hybrid", alpha=1.0, over_a=dict(t_draft=1e-9),
                         over_b=dict(t_draft=1.0)),
    "lost_replies": dict(variant="ordinary", drop_all=True, out=48),
}


@pytest.mark.parametrize("name", list(CASES))
def test_process_per_gpu_matches_single_process(name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(3, _free_port(), CASES[name]), nprocs=3, join=True)
