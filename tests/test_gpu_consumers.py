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


def _matrix(host, cols):
    return decode(host.view("<u4")).astype(np.float64).reshape(-1, cols)


@pytest.mark.parametrize("cols", [1024, 16384])  # shared-memory and global accumulators
def test_gemvt_consumer_matches_float64_reference(setup, cols):
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    rows = size // 4 // cols
    x2 = torch.cos(torch.arange(rows, dtype=torch.float32, device="cuda") * 0.01)
    y2 = torch.zeros(cols, dtype=torch.float32, device="cuda")
    fs.run(table, 64 * KiB, dst, consumer=Consumer("gemvt_f32", x2=x2, y2=y2, cols=cols))
    ref = _matrix(host, cols).T @ x2.cpu().numpy().astype(np.float64)
    got = y2.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=GEMV_RTOL, atol=GEMV_RTOL * np.abs(ref).max())


def test_bicg_consumer_both_products_in_one_pass(setup):
    """POLYBENCH bicg (q = A p, s = A^T r) — also mvt's two products — from one gread pass."""
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    cols = 2048
    rows = size // 4 // cols
    p = torch.linspace(-1, 1, cols, dtype=torch.float32, device="cuda")
    r = torch.sin(torch.arange(rows, dtype=torch.float32, device="cuda") * 0.1)
    q = torch.zeros(rows, dtype=torch.float32, device="cuda")
    s = torch.zeros(cols, dtype=torch.float32, device="cuda")
    fs.run(table, 64 * KiB, dst, consumer=Consumer("bicg_f32", x=p, y=q, x2=r, y2=s, cols=cols))
    A = _matrix(host, cols)
    for got, ref in ((q, A @ p.cpu().numpy().astype(np.float64)),
                     (s, A.T @ r.cpu().numpy().astype(np.float64))):
        got = got.cpu().numpy().astype(np.float64)
        assert np.allclose(got, ref, rtol=GEMV_RTOL, atol=GEMV_RTOL * np.abs(ref).max())


def test_atax_two_gread_passes(setup):
    """POLYBENCH atax y = A^T (A x): pass 1 GEMV, pass 2 GEMVT over a second gread pass."""
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    cols = 4096
    rows = size // 4 // cols
    x = torch.linspace(0, 1, cols, dtype=torch.float32, device="cuda")
    tmp = torch.zeros(rows, dtype=torch.float32, device="cuda")
    y = torch.zeros(cols, dtype=torch.float32, device="cuda")
    fs.run(table, 64 * KiB, dst, consumer=Consumer("gemv_f32", x=x, y=tmp, cols=cols))
    fs.run(table, 64 * KiB, dst, consumer=Consumer("gemvt_f32", x2=tmp, y2=y, cols=cols))
    A = _matrix(host, cols)
    ref = A.T @ (A @ x.cpu().numpy().astype(np.float64))
    got = y.cpu().numpy().astype(np.float64)
    assert np.allclose(got, ref, rtol=2 * GEMV_RTOL, atol=2 * GEMV_RTOL * np.abs(ref).max())


@pytest.mark.parametrize("D,K", [(16, 5), (32, 8), (64, 3)])  # shared-atomic / per-warp accumulators
def test_kmeans_consumer_assignment_exact(setup, D, K):
    """Rodinia kmeans assignment step: per-centroid counts are exact (fp32 distances summed
    over the features in order, as the float32 reference below does); per-centroid feature
    sums within rtol 1e-4 (fp32 accumulation order differs)."""
    import torch
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    P = decode(host.view("<u4")).reshape(-1, D)
    cent = P[np.linspace(0, P.shape[0] - 1, K).astype(np.int64)].copy()
    C = torch.from_numpy(cent).cuda()
    sums = torch.zeros(K, D, dtype=torch.float32, device="cuda")
    counts = torch.zeros(K, dtype=torch.int64, device="cuda")
    fs.run(table, 64 * KiB, dst, consumer=Consumer("kmeans_f32", x=C, y=sums, out=counts, cols=D, k=K))
    d = np.zeros((K, P.shape[0]), dtype=np.float32)
    for c in range(K):
        for j in range(D):
            df = P[:, j] - cent[c, j]
            d[c] = d[c] + df * df
    assign = np.argmin(d, axis=0)
    want_counts = np.bincount(assign, minlength=K)
    assert counts.cpu().numpy().tolist() == want_counts.tolist()
    want_sums = np.stack([P[assign == c].astype(np.float64).sum(0) for c in range(K)])
    assert np.allclose(sums.cpu().numpy(), want_sums, rtol=1e-4)


def test_consumer_validation_is_loud(setup):
    import torch
    from paper_2109_05366_b200.errors import GfsError
    from paper_2109_05366_b200.runtime import Consumer
    fs, table, dst, host, size = setup
    C = torch.zeros(17, 16, device="cuda")
    with pytest.raises(GfsError):  # too many centroids
        fs.run(table, 64 * KiB, dst, consumer=Consumer("kmeans_f32", x=C, y=C, out=C, cols=16, k=17))
    with pytest.raises(GfsError):  # points of 12 features do not tile 64 KiB requests
        fs.run(table, 64 * KiB, dst, consumer=Consumer("kmeans_f32", x=C, y=C, out=C, cols=12, k=2))
    with pytest.raises(GfsError):  # GEMVT without its vectors
        fs.run(table, 64 * KiB, dst, consumer=Consumer("gemvt_f32", cols=1024))


@pytest.mark.parametrize("cta_threads", [128, 256, 512])
@pytest.mark.parametrize("D,K", [(16, 5), (32, 8)])
def test_kmeans_staged_and_direct_paths_agree(setup, D, K, cta_threads):
    """The kmeans consumer runs through the per-warp shared-memory stage (K1 ring, TMA K1) or
    straight from the user buffer (LDG K1, or a stage that does not fit): counts exact
    against numpy on both, sums within rtol 1e-4 of each other (CTAs flush their partial sums
    with global float atomics, so the cross-CTA order is free)."""
    import torch
    from paper_2109_05366_b200.runtime import Consumer, GpuFS
    _fs, table, _dst, host, size = setup
    P = decode(host.view("<u4")).reshape(-1, D)
    cent = P[np.linspace(0, P.shape[0] - 1, K).astype(np.int64)].copy()
    d = np.zeros((K, P.shape[0]), dtype=np.float32)
    for c in range(K):
        for j in range(D):
            df = P[:, j] - cent[c, j]
            d[c] = d[c] + df * df
    want_counts = np.bincount(np.argmin(d, axis=0), minlength=K).tolist()
    got = {}
    for k1 in ("tma", "ldg"):
        cfg = ExperimentConfig({"gpufs.cache_bytes": 8 * MiB, "gpufs.prefetch_bytes": 60 * KiB,
                                "gpufs.policy": "per-tb-lra", "gpu.sm_count": 8,
                                "io.readahead": "adaptive", "io.dir": "/dev/shm/gfs_test",
                                "gpu.k1_copy": k1, "gpu.cta_threads": cta_threads})
        with GpuFS(cfg) as fs:
            fs.gopen(_synth_path(size), content_id=3)
            dst = torch.empty(size, dtype=torch.uint8, device="cuda")
            sums = torch.zeros(K, D, dtype=torch.float32, device="cuda")
            counts = torch.zeros(K, dtype=torch.int64, device="cuda")
            fs.run(table, 64 * KiB, dst, consumer=Consumer("kmeans_f32", x=torch.from_numpy(cent).cuda(),
                                                           y=sums, out=counts, cols=D, k=K))
            assert counts.cpu().numpy().tolist() == want_counts, (k1, cta_threads)
            got[k1] = sums.cpu().numpy()
    assert np.allclose(got["tma"], got["ldg"], rtol=1e-4)


def _synth_path(size):
    from paper_2109_05366_b200.runtime import ensure_synthetic
    return ensure_synthetic("/dev/shm/gfs_test", 3, size)
