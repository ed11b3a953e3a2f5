"""The disk arm against its O_DIRECT roofline probe, alone: 4 GiB synthetic file on /tmp
(block device), probe sweep, one gread pass through the pread daemon (auto -> bounce),
probe again.  Prints one JSON line.  Not a benchmark of record.

    python tools/disk_probe.py [--size-gib 4]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-gib", type=float, default=4.0)
    a = ap.parse_args()
    from paper_2109_05366_b200.runtime import ensure_synthetic
    size = int(a.size_gib * bench.GiB)
    cfg = bench.make_cfg(bench.headline_overrides(size, 1, "/tmp"), [])
    cfg = cfg.copy_with({"io.dir": "/tmp", "mode.ramfs": False})
    path = ensure_synthetic("/tmp", 0, size)
    before, how0 = bench.storage_probe(path, size)
    r = bench.run_arm(cfg, path, 0, 0, 2, 1)
    after, how1 = bench.storage_probe(path, size)
    st = r["stats"][-1]
    g = st["user_bytes"] / st["kernel_ns"]
    best = max(before, after)
    print(json.dumps({"arm_gbps": round(g, 3), "transfer": r["transfer"], "probe_before": round(before, 3),
                      "probe_before_how": how0, "probe_after": round(after, 3), "probe_after_how": how1,
                      "frac": round(g / best, 4), "io_workers": cfg.io_workers(), "ra_max": cfg.ra_max()}))


if __name__ == "__main__":
    main()
