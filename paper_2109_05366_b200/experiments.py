"""Repetitions, one-key sweeps and figure presets on real hardware.

Mirrors the reference harness (gpuiosim/experiments.py:21-183): ``run_config`` runs a
configuration ``repetitions`` times (seeds seed, seed+1, ...) and appends the mean row;
``sweep`` varies one key; ``run_preset`` reproduces the paper's figure arms —
fig2 (page-size sweep, whole-stride requests), fig8 (prefetch-size sweep at 4 KiB pages),
fig10micro (file = 2 x cache: per-tb-lra+prefetch vs global+prefetch vs original GPUfs)
and bench (the fourteen application input shapes, three arms each) — writing the same
36-column CSV.  The device-timing keys of the reference are accepted and ignored; every
run is a real pass over real (synthetic, W-law) files.
"""

from __future__ import annotations

import os

from .config import ExperimentConfig
from .errors import GfsError
from .metrics import mean_report, write_csv
from .workloads import BENCHMARKS

KiB, MiB = 1 << 10, 1 << 20

_MICRO = {"workload.kind": "strided", "workload.n_tb": 120,
          "workload.file_bytes": 98_304_000, "workload.n_files": 1}
_STRIDE = 98_304_000 // 120


def run_config(cfg: ExperimentConfig, label: str = "run") -> list:
    from .runtime import Simulation
    reports = [Simulation(cfg, cfg["seed"] + r, label=label, rep=r).run()
               for r in range(cfg["repetitions"])]
    return reports + [mean_report(reports)]


def sweep(cfg: ExperimentConfig, key: str, values: list) -> list:
    rows = []
    for v in values:
        rows.extend(run_config(cfg.copy_with({key: v}), label=f"{key}={v}"))
    return rows


def _arms_fig2(base):
    for size in (4 * KiB, 16 * KiB, 64 * KiB, 256 * KiB, 1024 * KiB):
        yield f"page-{size}", base.copy_with({**_MICRO, "gpufs.page_size": size,
                                              "workload.request_bytes": _STRIDE,
                                              "gpufs.prefetch_bytes": 0})


def _arms_fig8(base):
    for pf in (0, 12 * KiB, 28 * KiB, 60 * KiB, 124 * KiB, 252 * KiB):
        yield f"prefetch-{pf}", base.copy_with({**_MICRO, "gpufs.page_size": 4 * KiB,
                                                "workload.request_bytes": 64 * KiB,
                                                "gpufs.prefetch_bytes": pf})


def _arms_fig10micro(base):
    pressure = {**_MICRO, "gpufs.cache_bytes": 98_304_000 // 2, "gpufs.page_size": 4 * KiB,
                "workload.request_bytes": 64 * KiB}
    yield "lra-prefetch", base.copy_with({**pressure, "gpufs.policy": "per-tb-lra",
                                          "gpufs.prefetch_bytes": 60 * KiB})
    yield "global-prefetch", base.copy_with({**pressure, "gpufs.policy": "global-lru-dealloc",
                                             "gpufs.prefetch_bytes": 60 * KiB})
    yield "baseline-4k", base.copy_with({**pressure, "gpufs.policy": "global-lru-dealloc",
                                         "gpufs.prefetch_bytes": 0})


def _arms_bench(base):
    scale = base["workload.scale"]
    cache = max(int(500_000_000 * scale), 4 * MiB)
    arms = (("baseline-4k", {"gpufs.policy": "global-lru-dealloc", "gpufs.prefetch_bytes": 0}),
            ("prefetch", {"gpufs.policy": "global-lru-dealloc", "gpufs.prefetch_bytes": 60 * KiB}),
            ("lra-prefetch", {"gpufs.policy": "per-tb-lra", "gpufs.prefetch_bytes": 60 * KiB}))
    for name in sorted(BENCHMARKS):
        for arm, over in arms:
            yield f"{name}-{arm}", base.copy_with({
                "workload.kind": "benchmark", "workload.benchmark": name,
                "gpufs.page_size": 4 * KiB, "workload.request_bytes": 64 * KiB,
                "gpufs.cache_bytes": cache, **over})


def _arms_mosaic(base):
    """The Mosaic-style random workload (workloads.py:84-102): page-aligned
    random 4 KiB reads, 4 KiB vs 64 KiB GPU pages, no prefetch (prefetching a random stream
    only wastes transfer)."""
    for page in (4 * KiB, 64 * KiB):
        yield f"random-page-{page}", base.copy_with({
            "workload.kind": "random", "workload.n_tb": 256, "workload.requests_per_tb": 256,
            "workload.file_bytes": 1 << 30, "workload.request_bytes": 4 * KiB,
            "gpufs.page_size": page, "gpufs.prefetch_bytes": 0,
            "gpufs.cache_bytes": 256 * MiB, "gpufs.policy": "per-tb-lra"})


def _run_fig3(base, out_dir):
    """The GPU's access pattern vs its host-only replay (experiments.py:135-156): a raw-mode
    gread run (no GPU page cache) records its RPC trace, then host threads replay it with
    no GPU and no PCIe in the loop."""
    rows = []
    for size in (4 * KiB, 16 * KiB, 64 * KiB, 128 * KiB, 256 * KiB, 800 * KiB):
        trace = os.path.join(out_dir, f"fig3-trace-{size}.txt")
        rows.extend(run_config(base.copy_with({**_MICRO, "repetitions": 1,
                                               "workload.request_bytes": size,
                                               "mode.gpu_cache_disabled": True,
                                               "workload.record_trace": trace}),
                               label=f"gpu-pattern-{size}"))
        rows.extend(run_config(base.copy_with({**_MICRO, "repetitions": 1,
                                               "workload.request_bytes": size,
                                               "mode.replay_trace": trace}),
                               label=f"cpu-replay-{size}"))
    return rows


PRESETS = {"fig2": _arms_fig2, "fig3": _run_fig3, "fig8": _arms_fig8,
           "fig10micro": _arms_fig10micro, "bench": _arms_bench, "mosaic": _arms_mosaic}


def run_preset(name: str, base: ExperimentConfig, out_dir: str) -> str:
    """Run a figure preset; returns the CSV path (same name as the reference's)."""
    if name not in PRESETS:
        raise GfsError(f"unknown preset {name!r}; have {', '.join(PRESETS)} "
                       "(fig5/fig6 reproduce host-model pathologies, out of scope)")
    os.makedirs(out_dir, exist_ok=True)
    rows = []
    if name == "fig3":
        rows = _run_fig3(base, out_dir)
    else:
        for label, cfg in PRESETS[name](base):
            rows.extend(run_config(cfg, label))
    path = os.path.join(out_dir, f"{name}.csv")
    write_csv(path, rows)
    return path
