"""One headline gread pass for profilers (ncu application replay re-runs this process).

    python tools/profile_run.py [--size-gib 2] [--set k=v ...]

Creates the synthetic file once (reused across replays), runs exactly one gfs_run with
the headline configuration, prints its device-timed GB/s.  Not a benchmark of record.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-gib", type=float, default=2.0)
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--dir", default="/dev/shm")
    a = ap.parse_args()
    size = int(a.size_gib * bench.GiB)
    cfg = bench.make_cfg(bench.headline_overrides(size, 1, a.dir), a.set)
    path = bench.ensure_file(cfg, bench.Dist(1))
    r = bench.run_arm(cfg, path, 0, 0, 1, 0)
    st = r["stats"][-1]
    print(f"profile_run: {st['user_bytes'] / st['kernel_ns']:.2f} GB/s, kernel {st['kernel_ns'] / 1e6:.1f} ms, "
          f"mismatched words {r['mismatched_words']}", flush=True)


if __name__ == "__main__":
    main()
