"""Generate golden fixtures by running the REFERENCE simulator in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (gpuiosim, pure Python) cannot travel to the GPU box, so its
outputs are frozen here as small JSON fixtures: counters, and run-length
encoded delivery / RPC / victim logs.  Logs are canonicalised as the
reference's determinism allows:

* ``order == "global"``  — resident_limit == 1: the whole event order is
  deterministic, logs are kept in the reference's global order;
* ``order == "per_tb"``  — per-TB sequences are schedule-invariant; logs are
  stably sorted by TB (RPC records are recorded at service time, so only the
  per-TB order is meaningful);
* victims are stored only when ``victims`` is "global" or "per_tb"; otherwise
  only their count (order-dependent under interleaving).
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from gpuiosim.config import ExperimentConfig  # noqa: E402
from gpuiosim.simulation import Simulation  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
KiB, MiB = 1024, 1024 ** 2

MICRO = {"workload.kind": "strided", "workload.n_tb": 120,
         "workload.file_bytes": 98_304_000, "workload.n_files": 1}
R1 = {"gpu.sm_count": 1, "gpu.max_threads_per_sm": 2048, "gpu.threads_per_tb": 2048}
TINY = {"workload.kind": "strided", "workload.n_tb": 2, "workload.n_files": 1,
        "workload.file_bytes": 32 * 4096, "workload.request_bytes": 2 * 4096,
        "gpufs.page_size": 4096, "gpufs.cache_bytes": 8 * 4096,
        "gpufs.prefetch_bytes": 3 * 4096, "gpu.sm_count": 1,
        "gpu.max_threads_per_sm": 512, "gpu.threads_per_tb": 512,
        "gpu.start_jitter_ns": 0}
PRESSURE = {**MICRO, "gpufs.cache_bytes": 98_304_000 // 2, "gpufs.page_size": 4 * KiB,
            "workload.request_bytes": 64 * KiB}
C1 = {"workload.kind": "strided", "workload.n_tb": 128, "workload.file_bytes": 256 * MiB,
      "workload.n_files": 1, "workload.request_bytes": 64 * KiB, "gpufs.page_size": 4 * KiB,
      "gpufs.cache_bytes": 512 * MiB}

# name -> (overrides, seed, log order, victims order)
CASES = {
    "tiny_global": ({**TINY, "gpufs.policy": "global-lru-dealloc"}, 1, "global", "global"),
    "tiny_lra": ({**TINY, "gpufs.policy": "per-tb-lra"}, 1, "global", "global"),
    "micro_pf60": ({**MICRO, "gpufs.prefetch_bytes": 60 * KiB}, 42, "per_tb", "global"),
    "micro_nopf": ({**MICRO, "gpufs.prefetch_bytes": 0}, 42, "per_tb", "global"),
    "micro_page64k": ({**MICRO, "gpufs.page_size": 64 * KiB, "gpufs.prefetch_bytes": 0},
                      42, "per_tb", "global"),
    "micro_pf12": ({**MICRO, "gpufs.prefetch_bytes": 12 * KiB}, 42, "per_tb", "global"),
    "micro_pf252": ({**MICRO, "gpufs.prefetch_bytes": 252 * KiB}, 42, "per_tb", "global"),
    "micro_unaligned_req": ({**MICRO, "workload.request_bytes": 10_000,
                             "gpufs.prefetch_bytes": 28 * KiB}, 42, "per_tb", "global"),
    "pressure_lra": ({**PRESSURE, "gpufs.policy": "per-tb-lra",
                      "gpufs.prefetch_bytes": 60 * KiB}, 42, "per_tb", "count"),
    "pressure_global_pf": ({**PRESSURE, "gpufs.policy": "global-lru-dealloc",
                            "gpufs.prefetch_bytes": 60 * KiB}, 42, "per_tb", "count"),
    "pressure_global_nopf": ({**PRESSURE, "gpufs.policy": "global-lru-dealloc",
                              "gpufs.prefetch_bytes": 0}, 42, "per_tb", "count"),
    "pressure_lra_r1": ({**PRESSURE, **R1, "gpufs.policy": "per-tb-lra",
                         "gpufs.prefetch_bytes": 60 * KiB}, 42, "global", "global"),
    "pressure_global_r1": ({**PRESSURE, **R1, "gpufs.policy": "global-lru-dealloc",
                            "gpufs.prefetch_bytes": 60 * KiB}, 42, "global", "global"),
    "pressure_global_r1_shuffled": ({**PRESSURE, **R1, "gpufs.policy": "global-lru-dealloc",
                                     "gpufs.prefetch_bytes": 28 * KiB,
                                     "gpu.dispatch_order": "shuffled"}, 7, "global", "global"),
    "pressure_lra_fit": ({**PRESSURE, "workload.n_tb": 60, "gpufs.policy": "per-tb-lra",
                          "gpufs.prefetch_bytes": 60 * KiB}, 42, "per_tb", "per_tb"),
    "short_tail": ({"workload.n_tb": 1, "workload.file_bytes": 98_304,
                    "gpu.start_jitter_ns": 0}, 1, "global", "global"),
    "eight_mib": ({"workload.n_tb": 1, "workload.file_bytes": 8 * MiB,
                   "gpu.start_jitter_ns": 0, "gpufs.prefetch_bytes": 60 * KiB}, 1, "global", "global"),
    "multi_file_unaligned_r1": ({**R1, "workload.n_tb": 8, "workload.n_files": 2,
                                 "workload.file_bytes": 1_000_000, "workload.request_bytes": 16 * KiB,
                                 "gpufs.prefetch_bytes": 12 * KiB, "gpufs.cache_bytes": 64 * 4096,
                                 "gpufs.policy": "global-lru-dealloc"}, 3, "global", "global"),
    "multi_file_lra_r1": ({**R1, "workload.n_tb": 8, "workload.n_files": 3,
                           "workload.file_bytes": 700_000, "workload.request_bytes": 24 * KiB,
                           "gpufs.prefetch_bytes": 28 * KiB, "gpufs.cache_bytes": 96 * 4096,
                           "gpufs.policy": "per-tb-lra",
                           "gpu.dispatch_order": "reverse"}, 5, "global", "global"),
    "benchmark_nw": ({"workload.kind": "benchmark", "workload.benchmark": "nw",
                      "workload.scale": 0.01, "gpufs.prefetch_bytes": 60 * KiB,
                      "gpufs.policy": "per-tb-lra", "gpufs.cache_bytes": 8 * MiB,
                      "gpu.sm_count": 25}, 42, "per_tb", "count"),
    "benchmark_pathfinder": ({"workload.kind": "benchmark", "workload.benchmark": "pathfinder",
                              "workload.scale": 0.01, "gpufs.prefetch_bytes": 60 * KiB,
                              "gpufs.policy": "global-lru-dealloc",
                              "gpufs.cache_bytes": 4 * MiB}, 42, "per_tb", "count"),
    "raw_mode": ({**MICRO, "workload.n_tb": 8, "workload.file_bytes": 8 * MiB,
                  "mode.gpu_cache_disabled": True, "workload.request_bytes": 256 * KiB},
                 42, "per_tb", "global"),
    "c1_lra_pf60": ({**C1, "gpufs.policy": "per-tb-lra", "gpufs.prefetch_bytes": 60 * KiB},
                    42, "per_tb", "global"),
    "c1_global_pf60": ({**C1, "gpufs.policy": "global-lru-dealloc",
                        "gpufs.prefetch_bytes": 60 * KiB}, 42, "per_tb", "global"),
    "c1_global_nopf": ({**C1, "gpufs.policy": "global-lru-dealloc",
                        "gpufs.prefetch_bytes": 0}, 42, "per_tb", "global"),
    # the Mosaic-style random workload (workloads.py:84-102): requests overlap across TBs,
    # so only residency 1 is schedule-invariant
    "mosaic_4k_r1": ({**R1, "workload.kind": "random", "workload.n_tb": 8,
                      "workload.file_bytes": 8 * MiB, "workload.requests_per_tb": 48,
                      "workload.request_bytes": 4 * KiB, "gpufs.page_size": 4 * KiB,
                      "gpufs.prefetch_bytes": 0, "gpufs.cache_bytes": 256 * 4096,
                      "gpufs.policy": "global-lru-dealloc"}, 11, "global", "global"),
    "mosaic_64k_pf_r1": ({**R1, "workload.kind": "random", "workload.n_tb": 6,
                          "workload.file_bytes": 4 * MiB, "workload.requests_per_tb": 24,
                          "workload.request_bytes": 64 * KiB, "gpufs.page_size": 4 * KiB,
                          "gpufs.prefetch_bytes": 60 * KiB, "gpufs.cache_bytes": 512 * 4096,
                          "gpufs.policy": "per-tb-lra"}, 12, "global", "global"),
    "mosaic_page64k_r1": ({**R1, "workload.kind": "random", "workload.n_tb": 4,
                           "workload.file_bytes": 6 * MiB + 4096, "workload.requests_per_tb": 40,
                           "workload.request_bytes": 8 * KiB, "gpufs.page_size": 64 * KiB,
                           "gpufs.prefetch_bytes": 0, "gpufs.cache_bytes": 24 * 64 * KiB,
                           "gpufs.policy": "global-lru-dealloc"}, 13, "global", "global"),
}

COUNTERS = ["greads", "user_bytes", "cache_hit_user_bytes", "tag_mismatches", "pc_lookups",
            "pc_hits", "pc_hit_pending", "pc_misses", "pc_allocs", "pc_evictions", "pc_remaps",
            "pb_hits", "pb_misses", "pb_filled_bytes", "pb_consumed_bytes",
            "pb_discarded_bytes", "rpc_count", "rpc_requested_bytes", "preads", "pread_bytes"]


def _stable_by_tb(recs):
    return sorted(recs, key=lambda r: r[0]) if recs else recs


def rle_pages(recs):
    """(tb, fid, page) records -> [[tb, fid, first_page, count], ...]."""
    out = []
    for tb, fid, page in recs:
        if out and out[-1][0] == tb and out[-1][1] == fid and out[-1][2] + out[-1][3] == page:
            out[-1][3] += 1
        else:
            out.append([tb, fid, page, 1])
    return out


def rle_rpcs(recs):
    """(tb, fid, off, size) -> [[tb, fid, off0, size, count], ...] with off_k = off0 + k*size."""
    out = []
    for tb, fid, off, size in recs:
        if (out and out[-1][0] == tb and out[-1][1] == fid and out[-1][3] == size
                and out[-1][2] + out[-1][3] * out[-1][4] == off):
            out[-1][4] += 1
        else:
            out.append([tb, fid, off, size, 1])
    return out


def run_case(name, overrides, seed, order, vorder):
    over = dict(overrides)
    trace_path = f"/tmp/golden_trace_{name}.txt"
    over["workload.record_trace"] = trace_path
    over["repetitions"] = 1
    cfg = ExperimentConfig(over)
    sim = Simulation(cfg, seed)
    sim.metrics.log_deliveries = True
    rep = sim.run()
    m = sim.metrics
    deliveries = [tuple(d) for d in m.deliveries]
    rpcs = [(r.tb_id, r.file_id, r.offset, r.size) for r in sim.recorded]
    victims = [tuple(v) for v in sim.cache.victim_log] if sim.cache is not None else []
    if order == "per_tb":
        deliveries = _stable_by_tb(deliveries)
        rpcs = _stable_by_tb(rpcs)
    if vorder == "per_tb":
        victims = _stable_by_tb(victims)
    out = {
        "name": name,
        "overrides": {k: v for k, v in overrides.items()},
        "seed": seed,
        "order": order,
        "victims_order": vorder,
        "counters": {k: getattr(m, k) for k in COUNTERS},
        "pcie_bytes": sim.pcie.bytes_moved,
        "pcie_transfers": sim.pcie.transfers,
        "report": {k: rep[k] for k in ("user_bytes", "rpc_count", "pc_evictions", "pc_remaps",
                                       "pb_hits", "prefetch_waste_bytes", "greads")},
        "n_victims": len(sim.cache.victim_log) if sim.cache is not None else 0,
        "deliveries_rle": rle_pages(deliveries),
        "rpcs_rle": rle_rpcs(rpcs),
        "victims_rle": rle_pages(victims) if vorder != "count" else None,
        "unique_bytes": sim.workload.unique_bytes,
        "total_bytes": sim.workload.total_bytes,
    }
    os.remove(trace_path)
    return out


def fuzz_cases() -> dict:
    """The randomised resident_limit-1 cases of tests/test_gpu_fuzz.py that the reference
    can express (static readahead; the io.* keys are the B200 layer's own)."""
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from test_gpu_fuzz import N_CASES, random_case
    out = {}
    for k in range(N_CASES):
        over = random_case(k)
        if over["io.readahead"] != "static":
            continue
        seed = over.pop("seed")
        over = {kk: v for kk, v in over.items()
                if not kk.startswith("io.") and kk not in ("gpu.k1_copy", "gpu.cta_threads")}
        out[f"fuzz_{k:02d}"] = (over, seed, "global", "global")
    return out


def main():
    only = set(sys.argv[1:])
    for name, (over, seed, order, vorder) in {**CASES, **fuzz_cases()}.items():
        if only and name not in only:
            continue
        res = run_case(name, over, seed, order, vorder)
        with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
            json.dump(res, fh, separators=(",", ":"))
        print(f"{name}: rpc={res['counters']['rpc_count']} deliveries_runs={len(res['deliveries_rle'])}"
              f" victims={res['n_victims']}")


if __name__ == "__main__":
    main()
