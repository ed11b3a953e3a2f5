"""bench.py's host-side contract, on CPU: the reference arm stays off the product package,
the multi-GPU shard plan (configs[4]), and the NCCL process-group construction."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

GiB, MiB = 1 << 30, 1 << 20


def test_shard_plan_strong_and_weak():
    assert bench.shard_plan(None, 16.0, 1) == (None, "weak", 16 * GiB)
    for n, per in ((2, 32 * GiB), (4, 16 * GiB), (8, 8 * GiB)):  # configs[4]: 64 GiB over N GPUs
        assert bench.shard_plan(None, 16.0, n) == (64.0, "strong", per)
    assert bench.shard_plan(6.0, 16.0, 4)[2] % (64 * MiB) == 0


def test_nccl_process_group_construction(monkeypatch):
    """N > 1 on distinct GPUs: NCCL bound to this rank's device (the collective is the
    optional 8-byte checksum all-reduce and the max-over-ranks timing)."""
    import torch
    import torch.distributed as dist
    calls = {}
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("LOCAL_RANK", "1")
    monkeypatch.delenv("GFS_BENCH_SHARE_GPU", raising=False)
    monkeypatch.setattr(torch.cuda, "set_device", lambda d: calls.setdefault("device", d))
    monkeypatch.setattr(dist, "init_process_group",
                        lambda backend, **kw: calls.update(backend=backend, **kw))
    d = bench.Dist(2)
    assert calls["backend"] == "nccl" and calls["device_id"] == torch.device("cuda", 1)
    assert calls["device"] == 1 and d.tdev == "cuda:1" and d.rank == 1 and d.world == 2


@pytest.mark.timeout(600)
def test_reference_arm_never_imports_the_product(tmp_path):
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--size-gib', '0.25', "
            f"'--steps', '1', '--warmup', '0', '--dir', {str(tmp_path)!r}]; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "bad = [m for m in sys.modules if m.startswith('paper_2109_05366_b200')]; "
            "assert not bad, bad")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and "decomposition" in line["config"]
    py = line["python_reference"]
    if "unavailable" not in py:  # baseline/_ref holds the reference package
        assert py["arms"]["prefetch_per_tb_lra"]["rpc_count"] == 4096  # the C1 RPC law
        assert py["cores_used"] == 1
