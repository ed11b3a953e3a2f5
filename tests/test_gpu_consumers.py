"""Fused streaming consumers against plain references over the same bytes.

sum64 and nn_f32 are integer / IEEE-exact and compared bit for bit; gemv_f32 accumulates in
fp32 in a different order than the float64 reference, tolerance rtol 1e-4 (stated here)."""

import os

import numpy as np
import pytest

from paper_2109_05366_b200 import rng as grng
from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided

pytestmark = pytest.mark.gpu
KiB, MiB = 1 << 10, 1 << 20
GEMV_RTOL = 1e-4


@pytest.fixture(scope="module")
def setup():
    import torch
    from paper_2109_05366_b200.runtime import GpuFS, ensure_synthetic
    d = "/dev/shm/gfs_test"
    os.makedirs(d, exist_ok=True)
    size = 24 * MiB
    path = ensure_synthetic(d, 3, size)
    cfg = ExperimentConfig({"gpufs.cache_bytes": 8 * MiB, "gpufs.prefetch_bytes": 60 * KiB,
                            "gpufs.policy": "per-tb-lra", "gpu.sm_count": 8,
                            "io.readahead": "adaptive", "io.dir": d})
    wl = gen_sequential_strided([size], 48, size, 64 * KiB, 4096)
    table = ProgramTable.from_programs(wl.programs)
    fs = GpuFS(cfg)
    fs.gopen(path, content_id=3)
    dst = torch.empty(size, dtype=torch.uint8, device="cuda")
    host = np.frombuffer(grng.content(3, 0, size), dtype=np.uint8)
    yield fs, table, dst, host, size
    fs.close()


def decode(u32):
    return (u32 >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def test_sum64_consumer_equals_file_checksum(setup):
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    r = fs.run(table, 64 * KiB, dst, consumer=Consumer("sum64", out=out))
    assert r.stats["user_bytes"] == size
    assert int(out.item()) & ((1 << 64) - 1) == grng.checksum(host)


def test_nn_consumer_matches_numpy_float32(setup):
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    out = torch.full((1,), -1, dtype=torch.int64, device="cuda")  # all ones = +inf key
    qx, qy = 12.5, -77.25
    fs.run(table, 64 * KiB, dst, consumer=Consumer("nn_f32", out=out, qx=qx, qy=qy))
    key = int(out.item()) & ((1 << 64) - 1)
    u = host.view("<u4").reshape(-1, 2)
    lat = decode(u[:, 0]) * np.float32(180) - np.float32(90)
    lng = decode(u[:, 1]) * np.float32(360) - np.float32(180)
    dx, dy = lat - np.float32(qx), lng - np.float32(qy)
    d2 = dx * dx + dy * dy
    best = int(np.argmin(d2))
    assert key & 0xFFFFFFFF == best
    assert np.float32(d2[best]).view(np.uint32) == key >> 32


def test_gemv_consumer_matches_float64_reference(setup):
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    cols = 4096
    rows = size // 4 // cols
    x = torch.linspace(-1, 1, cols, dtype=torch.float32, device="cuda")
    y = torch.zeros(rows, dtype=torch.float32, device="cuda")
    fs.run(table, 64 * KiB, dst, consumer=Consumer("gemv_f32", x=x, y=y, cols=cols))
    A = decode(host.view("<u4")).astype(np.float64).reshape(rows, cols)
    ref = A @ x.cpu().numpy().astype(np.float64)
    got = y.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=GEMV_RTOL, atol=GEMV_RTOL * np.abs(ref).max())
