"""Shared helpers: load reference golden fixtures and compare a run against them.

Used by the oracle tests (CPU) and the device parity tests (GPU), so both
sides are held to the same definition of "matches the reference".
"""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2109_05366_b200.config import ExperimentConfig

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_DIR = os.path.join(HERE, "golden")

# Counters that are schedule-invariant for every golden case (no shared pages).
INVARIANT = ["greads", "user_bytes", "cache_hit_user_bytes", "tag_mismatches", "pc_lookups",
             "pc_hits", "pc_hit_pending", "pc_misses", "pc_allocs", "pc_evictions", "pc_remaps",
             "pb_hits", "pb_misses", "pb_filled_bytes", "pb_consumed_bytes",
             "pb_discarded_bytes", "rpc_count", "rpc_requested_bytes", "preads", "pread_bytes"]
# Cases whose strides share pages across TBs: who fetches a shared page (and
# whether the other TB waits or hits) depends on timing in the reference.
SHARED_PAGE_CASES = {"micro_page64k"}
TIMING_COUNTERS = {"pc_hits", "pc_hit_pending", "pc_lookups", "pb_hits", "pb_misses",
                   "pb_filled_bytes", "pb_consumed_bytes", "pb_discarded_bytes",
                   "cache_hit_user_bytes", "rpc_requested_bytes", "pc_misses", "pc_allocs",
                   "preads", "pread_bytes", "rpc_count"}


def case_names() -> list[str]:
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "*.json")))


def load(name: str) -> dict:
    with open(os.path.join(GOLDEN_DIR, f"{name}.json")) as fh:
        return json.load(fh)


def config_of(g: dict, **extra) -> ExperimentConfig:
    return ExperimentConfig({**g["overrides"], **extra})


def expand_pages(rle) -> np.ndarray:
    rows = []
    for tb, fid, first, count in rle:
        p = np.arange(first, first + count, dtype=np.int64)
        rows.append(np.stack([np.full(count, tb), np.full(count, fid), p], axis=1))
    return np.concatenate(rows) if rows else np.zeros((0, 3), np.int64)


def expand_rpcs(rle) -> np.ndarray:
    rows = []
    for tb, fid, off0, size, count in rle:
        off = off0 + size * np.arange(count, dtype=np.int64)
        rows.append(np.stack([np.full(count, tb), np.full(count, fid), off,
                              np.full(count, size)], axis=1))
    return np.concatenate(rows) if rows else np.zeros((0, 4), np.int64)


def by_tb(a: np.ndarray) -> np.ndarray:
    """Stable sort of log records by their TB column (per-TB order preserved)."""
    if len(a) == 0:
        return a
    return a[np.argsort(a[:, 0], kind="stable")]


def compare(g: dict, stats: dict, deliveries, rpcs, victims, *, exact_victims=True) -> list[str]:
    """Differences between a run and golden case g ('' list = parity)."""
    errs = []
    shared = g["name"] in SHARED_PAGE_CASES
    for k in INVARIANT:
        if shared and k in TIMING_COUNTERS:
            continue
        if stats.get(k) != g["counters"][k]:
            errs.append(f"{k}: got {stats.get(k)} want {g['counters'][k]}")
    if shared:
        # invariants only: every shared page fetched once, total bytes
        for k in ("user_bytes", "greads", "pc_evictions", "pc_remaps"):
            if stats.get(k) != g["counters"][k]:
                errs.append(f"{k}: got {stats.get(k)} want {g['counters'][k]}")
    if stats.get("pcie_bytes") != g["pcie_bytes"] and not shared:
        errs.append(f"pcie_bytes: got {stats.get('pcie_bytes')} want {g['pcie_bytes']}")
    if stats.get("pcie_transfers") != g["pcie_transfers"] and not shared:
        errs.append(f"pcie_transfers: got {stats.get('pcie_transfers')} want {g['pcie_transfers']}")
    if stats.get("victims", g["n_victims"]) != g["n_victims"]:
        errs.append(f"victims: got {stats.get('victims')} want {g['n_victims']}")
    want_d = expand_pages(g["deliveries_rle"])
    got_d = np.asarray(deliveries, dtype=np.int64).reshape(-1, 3)
    if g["order"] == "per_tb":
        got_d = by_tb(got_d)
    if got_d.shape != want_d.shape or not np.array_equal(got_d, want_d):
        errs.append(f"deliveries differ ({len(got_d)} vs {len(want_d)})")
    if not shared:
        want_r = expand_rpcs(g["rpcs_rle"])
        got_r = np.asarray(rpcs, dtype=np.int64).reshape(-1, 4)
        if g["order"] == "per_tb":
            got_r = by_tb(got_r)
        if got_r.shape != want_r.shape or not np.array_equal(got_r, want_r):
            errs.append(f"rpc trace differs ({len(got_r)} vs {len(want_r)})")
    if g["victims_rle"] is not None and exact_victims:
        want_v = expand_pages(g["victims_rle"])
        got_v = np.asarray(victims, dtype=np.int64).reshape(-1, 3)
        if g["victims_order"] == "per_tb":
            got_v = by_tb(got_v)
        if got_v.shape != want_v.shape or not np.array_equal(got_v, want_v):
            errs.append(f"victim log differs ({len(got_v)} vs {len(want_v)})")
    return errs


# ---- readahead-law fixtures (tests/golden/windows, made by make_windows.py) ----

WINDOW_DIR = os.path.join(GOLDEN_DIR, "windows")


def window_case_names() -> list[str]:
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(WINDOW_DIR, "*.json")))


def window_case(name: str, **extra):
    """(fixture, config, workload) replaying a reference HostOs read stream as one TB whose
    program is the read list (one segment = one gread each), ondemand readahead with the
    reference's EOF clamp, a cache larger than the file (the reference host cache never
    evicts here)."""
    from paper_2109_05366_b200.workloads import WorkloadSpec, union_bytes
    with open(os.path.join(WINDOW_DIR, f"{name}.json")) as fh:
        g = json.load(fh)
    reads = [tuple(r) for r in g["reads"]]
    req = max(sz for _, sz in reads)
    fb = g["file_bytes"]
    cache = max(4 << 20, (fb + 2 * g["ra_max"] + (1 << 20)) // (1 << 20) * (1 << 20))
    over = {"gpufs.page_size": g["page"], "gpufs.prefetch_bytes": 0, "gpufs.cache_bytes": cache,
            "gpufs.policy": "per-tb-lra", "io.readahead": "adaptive", "io.ra_clamp": "eof",
            "io.ra_max_bytes": g["ra_max"], "gpu.sm_count": 1, "gpu.threads_per_tb": 2048,
            "mode.deterministic": True, "workload.request_bytes": req}
    over.update(extra)
    cfg = ExperimentConfig(over)
    prog = [(0, off, min(sz, fb - off)) for off, sz in reads if off < fb]
    wl = WorkloadSpec(name=f"window_{name}", files={0: fb}, read_only={0: True}, programs=[prog],
                      request_bytes=req, total_bytes=sum(ln for _, _, ln in prog),
                      unique_bytes=union_bytes([prog]))
    return g, cfg, wl
