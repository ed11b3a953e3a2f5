"""A user kernel reading through the public device-side gread (include/gfs_device.cuh,
SURVEY §8(b)): csrc/user_gemv.cu, built like an application into libgfs_user.so and run
with gfs_run_kernel.  Its TBs read the strided program of gen_sequential_strided
(workloads.py:66-81) one gread at a time, so the delivered bytes, counters, per-TB
delivery and RPC logs must equal the CPU oracle's for that workload; its GEMV output is
checked against float64 numpy (fp32 accumulation in another order: rtol 1e-4, stated here)."""

import os

import numpy as np
import pytest

import golden_util as gu
import oracle as orc
from paper_2109_05366_b200 import native
from paper_2109_05366_b200 import rng as grng
from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided

pytestmark = pytest.mark.gpu
KiB, MiB = 1 << 10, 1 << 20
GEMV_RTOL = 1e-4
COUNTERS = ("user_bytes", "greads", "pc_lookups", "pc_misses", "pc_hits", "pb_hits", "pb_misses",
            "rpc_count", "rpc_requested_bytes", "pc_allocs", "pc_evictions", "pc_remaps", "victims",
            "pb_filled_bytes", "pb_discarded_bytes", "pcie_bytes")


@pytest.fixture(scope="module")
def synth():
    from paper_2109_05366_b200.runtime import ensure_synthetic
    d = "/dev/shm/gfs_test"
    os.makedirs(d, exist_ok=True)
    size = 16 * MiB
    return d, ensure_synthetic(d, 5, size), size


def decode(u32):
    return (u32 >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def user_run(d, path, size, over, n_tb, cols, request, order=None, hint=1):
    import torch
    from paper_2109_05366_b200.runtime import GpuFS
    cfg = ExperimentConfig({**over, "io.dir": d, "mode.deterministic": True, "io.workers": 8,
                            "workload.request_bytes": request})
    U = native.load_user()
    rows = size // 4 // cols
    x = torch.linspace(-1, 1, cols, dtype=torch.float32, device="cuda")
    y = torch.full((rows,), float("nan"), dtype=torch.float32, device="cuda")
    dst = torch.zeros(size, dtype=torch.uint8, device="cuda")
    with GpuFS(cfg, max_request_bytes=request) as fs:
        fid = fs.gopen(path, content_id=5)
        r = fs.run_user(U.gfs_example_gemv, fid, size, n_tb, request, cols, x.data_ptr(), y.data_ptr(),
                        dst.data_ptr(), hint, order=order)
        csum = fs.checksum(dst, size)
    torch.cuda.synchronize()
    return cfg, r, x, y, dst, csum


def oracle_of(cfg, size, n_tb, request):
    wl = gen_sequential_strided([size], n_tb, size, request, cfg["gpufs.page_size"])
    cfg = cfg.copy_with({"workload.file_bytes": size, "workload.n_tb": n_tb})
    return orc.run_oracle(cfg, wl, source=orc.SRC_SYNTH, materialize_dst=True, log=True)


@pytest.mark.parametrize("readahead", ["static", "adaptive"])
@pytest.mark.parametrize("policy,cache", [("per-tb-lra", 64 * MiB), ("per-tb-lra", 4 * MiB),
                                          ("global-lru-dealloc", 64 * MiB)])
def test_user_gemv_matches_oracle(synth, readahead, policy, cache):
    d, path, size = synth
    n_tb, cols, request = 32, 1024, 64 * KiB
    over = {"gpufs.page_size": 4 * KiB, "gpufs.prefetch_bytes": 60 * KiB, "gpufs.cache_bytes": cache,
            "gpufs.policy": policy, "gpu.sm_count": 4, "gpu.threads_per_tb": 512,
            "io.readahead": readahead, "io.ra_max_bytes": 256 * KiB}
    cfg, r, x, y, dst, csum = user_run(d, path, size, over, n_tb, cols, request)
    ref = oracle_of(cfg, size, n_tb, request)
    st = r.stats
    assert st["word_mismatches"] == 0
    host = np.frombuffer(grng.content(5, 0, size), dtype=np.uint8)
    assert csum == grng.checksum(host)  # (the oracle's synthetic source is content id = file id)
    for k in COUNTERS:
        if policy == "global-lru-dealloc" and k in ("pc_evictions", "victims"):
            continue
        assert st[k] == ref.stats[k], (k, st[k], ref.stats[k])
    assert np.array_equal(gu.by_tb(r.deliveries), gu.by_tb(ref.deliveries))
    assert np.array_equal(gu.by_tb(r.rpcs), gu.by_tb(ref.rpcs))
    A = decode(host.view("<u4")).astype(np.float64).reshape(-1, cols)
    want = A @ x.cpu().numpy().astype(np.float64)
    got = y.cpu().numpy().astype(np.float64)
    assert np.allclose(got, want, rtol=GEMV_RTOL, atol=GEMV_RTOL * np.abs(want).max())


def test_user_gemv_shuffled_order_and_whole_file_stream(synth):
    """Dispatch order is the run's (gpu_exec.py:242-265); without the stream hint the
    readahead law sees the whole file (windows end at EOF): bytes are still exact."""
    d, path, size = synth
    n_tb, cols, request = 64, 512, 16 * KiB
    over = {"gpufs.cache_bytes": 8 * MiB, "gpu.sm_count": 8, "io.readahead": "adaptive"}
    order = np.random.default_rng(3).permutation(n_tb).astype(np.int32)
    cfg, r, x, y, dst, csum = user_run(d, path, size, over, n_tb, cols, request, order=order, hint=0)
    assert r.stats["user_bytes"] == size and r.stats["word_mismatches"] == 0
    assert r.stats["greads"] == size // request
    host = np.frombuffer(grng.content(5, 0, size), dtype=np.uint8)
    assert csum == grng.checksum(host)
    assert sorted(set(int(t) for t in r.deliveries[:, 0])) == list(range(n_tb))


def test_user_kernel_errors_are_reported(synth):
    """Arguments the user entry point refuses fail loudly; the context stays usable."""
    import torch
    from paper_2109_05366_b200.errors import GfsError
    from paper_2109_05366_b200.runtime import GpuFS
    d, path, size = synth
    cfg = ExperimentConfig({"io.dir": d, "gpu.cta_threads": 512, "gpu.sm_count": 2})
    U = native.load_user()
    x = torch.zeros(1024, dtype=torch.float32, device="cuda")
    y = torch.zeros(size // 4096, dtype=torch.float32, device="cuda")
    dst = torch.zeros(size, dtype=torch.uint8, device="cuda")
    with GpuFS(cfg) as fs:
        fid = fs.gopen(path, content_id=5)
        with pytest.raises(GfsError):  # cols not a multiple of 4: the entry point refuses
            fs.run_user(U.gfs_example_gemv, fid, size, 16, 64 * KiB, 1022, x.data_ptr(), y.data_ptr(),
                        dst.data_ptr(), 1)
        r = fs.run_user(U.gfs_example_gemv, fid, size, 16, 64 * KiB, 1024, x.data_ptr(), y.data_ptr(),
                        dst.data_ptr(), 1)  # the context is still usable
        assert r.stats["user_bytes"] == size
