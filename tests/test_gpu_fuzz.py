"""Randomised device-vs-oracle parity: seeded random small configurations (odd file
sizes, unaligned strides and requests, several files, tiny caches, both policies, both
readahead modes, every transfer) at resident_limit 1, where the reference's behaviour is
fully deterministic, so every log must match the oracle exactly — global delivery order,
RPC trace, victim sequence, adaptive windows — plus counters and the user-buffer bytes."""

import os

import numpy as np
import pytest

import oracle as orc
from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.rng import SeededRng
from paper_2109_05366_b200.workloads import build_workload

pytestmark = pytest.mark.gpu

N_CASES = 40
TRANSFERS = ["zerocopy", "bounce", "dma", "mapped", "mapped_dma", "mapped_hybrid", "pread_hybrid"]
COUNTERS = ["greads", "user_bytes", "cache_hit_user_bytes", "pc_lookups", "pc_hits",
            "pc_hit_pending", "pc_misses", "pc_allocs", "pc_evictions", "pc_remaps", "pb_hits",
            "pb_misses", "pb_filled_bytes", "pb_consumed_bytes", "pb_discarded_bytes", "rpc_count",
            "rpc_requested_bytes", "preads", "pread_bytes", "pcie_bytes", "pcie_transfers", "victims"]


def random_case(k: int) -> dict:
    r = SeededRng(1000 + k)
    page = [4096, 8192, 16384][r.below(3)]
    n_files = 1 + r.below(3)
    n_tb = 1 + r.below(12)
    stride = page * (1 + r.below(24)) + (r.below(2) * r.below(page))  # maybe unaligned
    total = n_tb * stride
    file_bytes = -(-total // n_files) + r.below(3 * page)
    request = max(16, page * (1 + r.below(4)) - r.below(2) * r.below(page // 2))
    request = min(request, stride)
    frames = 4 + r.below(60)
    return {
        "workload.n_tb": n_tb, "workload.n_files": n_files, "workload.file_bytes": file_bytes,
        "workload.total_bytes": total, "workload.request_bytes": request,
        "gpufs.page_size": page, "gpufs.prefetch_bytes": page * r.below(8),
        "gpufs.cache_bytes": frames * page,
        "gpufs.policy": ["global-lru-dealloc", "per-tb-lra"][r.below(2)],
        "io.readahead": ["static", "adaptive", "doubling"][r.below(3)],
        "io.ra_max_bytes": page * (1 << (2 + r.below(4))),
        "gpu.dispatch_order": ["round-robin", "shuffled", "reverse"][r.below(3)],
        "gpu.sm_count": 1, "gpu.max_threads_per_sm": 2048, "gpu.threads_per_tb": 2048,
        "io.transfer": TRANSFERS[k % len(TRANSFERS)], "seed": 7 + k,
        "io.ra_init_bytes": page * r.below(6),
        "gpu.k1_copy": ("tma", "ldg")[k % 2],
        "gpu.cta_threads": (256, 128, 512)[k % 3],
    }


@pytest.mark.parametrize("k", range(N_CASES))
def test_random_config_matches_oracle_exactly(k):
    from paper_2109_05366_b200.runtime import Simulation
    over = random_case(k)
    d = "/dev/shm/gfs_fuzz"
    os.makedirs(d, exist_ok=True)
    cfg = ExperimentConfig({**over, "io.dir": d, "mode.deterministic": True, "io.workers": 4})
    sim = Simulation(cfg, over["seed"])
    sim.run(keep_output=True)
    st = sim.result.stats
    ref_cfg = ExperimentConfig(over)
    ref = orc.run_oracle(ref_cfg, build_workload(ref_cfg), source=orc.SRC_SYNTH, materialize_dst=True,
                         order=None)
    for c in COUNTERS:
        assert st[c] == ref.stats[c], (k, c, st[c], ref.stats[c], over)
    assert np.array_equal(sim.result.deliveries, ref.deliveries), (k, over)
    assert np.array_equal(sim.result.rpcs, ref.rpcs), (k, over)
    assert np.array_equal(sim.result.victims, ref.victims), (k, over)
    assert np.array_equal(sim.result.windows, ref.windows), (k, over)
    got = sim.output[:len(ref.dst)].cpu().numpy()
    assert np.array_equal(got, ref.dst), (k, over)
    assert st["word_mismatches"] == 0
