"""bench.py host logic on CPU: the multi-GPU launch contract and the
reference arm (no GPU needed)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_gpus_without_devices_fails_clearly(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs present")
    with pytest.raises(SystemExit, match="CUDA device"):
        bench.main(["--gpus", "2"])


def test_gpus_disagreeing_with_world_size(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(SystemExit, match="disagrees"):
        bench.main(["--gpus", "2"])


def test_spawn_launches_one_process_per_rank(tmp_path):
    """spawn_ranks re-launches a script under torch.distributed.run: every rank
    sees RANK / LOCAL_RANK / WORLD_SIZE and the 127.0.0.1 rendezvous, and a
    gloo all-reduce across them works (the path bench.py --gpus N takes)."""
    probe = tmp_path / "probe.py"
    probe.write_text(
        "import os, sys, json, torch, torch.distributed as dist\n"
        "dist.init_process_group('gloo')\n"
        "t = torch.tensor([float(os.environ['RANK']) + 1])\n"
        "dist.all_reduce(t)\n"
        "out = sys.argv[1]\n"
        "open(os.path.join(out, os.environ['RANK']), 'w').write(json.dumps(\n"
        "    dict(rank=int(os.environ['RANK']), local=int(os.environ['LOCAL_RANK']),\n"
        "         world=int(os.environ['WORLD_SIZE']), addr=os.environ['MASTER_ADDR'],\n"
        "         total=t.item())))\n"
        "dist.destroy_process_group()\n")
    rc = bench.spawn_ranks(2, [str(tmp_path)], script=str(probe))
    assert rc == 0
    recs = sorted((json.loads((tmp_path / r).read_text()) for r in ("0", "1")),
                  key=lambda r: r["rank"])
    assert [r["rank"] for r in recs] == [0, 1]
    assert all(r["world"] == 2 and r["addr"] == "127.0.0.1" and r["total"] == 3.0 for r in recs)


def test_reference_arm_runs_the_reference_loop(tmp_path):
    """--impl reference prints one JSON line for the reference's own decode loop
    (stock specsim when baseline/_ref is installed, else the CPU port)."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--out-len", "32", "--batch", "8"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == bench.reference_kind()
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["alpha"] == bench.ALPHA_MEAS_C2


def test_reference_and_port_agree_on_reports():
    """The two CPU legs (stock reference / oracle port) produce the same report
    bytes for the same config (the port is pinned to the reference)."""
    if bench.reference_kind() != "reference":
        pytest.skip("baseline/_ref not installed")
    cfg = dict(batch_size=8, n_requests=8, gamma=4, output_len=48, alpha=0.8, qps=1e6, seed=3)
    for v in ("ordinary", "parallel", "hybrid"):
        ref = bench._ref_worker((cfg, v, "reference"))
        port = bench._ref_worker((cfg, v, "port"))
        assert ref[0] == port[0] and ref[2] == port[2], v
