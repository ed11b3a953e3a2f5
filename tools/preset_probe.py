"""The reference's figure-preset arms behind acceptance criterion 3 (fig8 prefetch-61440 vs
fig2 page-65536), each with its per-CTA time split.  Not a benchmark of record.

    python tools/preset_probe.py [--set key=value ...] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dir", default="/dev/shm/gfs_test")
    a = ap.parse_args()
    from paper_2109_05366_b200.config import ExperimentConfig
    from paper_2109_05366_b200.experiments import PRESETS
    from paper_2109_05366_b200.runtime import Simulation
    os.makedirs(a.dir, exist_ok=True)
    base = ExperimentConfig({"repetitions": 1, "io.dir": a.dir})
    for kv in a.set:
        k, v = kv.split("=", 1)
        base.set(k, v)
    arms = dict(PRESETS["fig8"](base))
    arms.update(dict(PRESETS["fig2"](base)))
    for name in ("prefetch-61440", "page-65536", "page-4096"):
        cfg = arms[name]
        for r in range(a.reps):
            sim = Simulation(cfg, 42)
            rep = sim.run()
            st = sim.result.stats
            n = max(1, min(st["ctas"], cfg["workload.n_tb"]))
            print(json.dumps({"arm": name, "rep": r, "gbps": round(rep["io_bandwidth_bps"] / 1e9, 3),
                              "rpc_count": st["rpc_count"], "kernel_ms": round(st["kernel_ns"] / 1e6, 3),
                              "per_cta_us": {k: round(st[k] / n / 1e3, 1) for k in
                                             ("wait_ns", "meta_ns", "copy_ns", "install_ns", "lookup_ns", "alloc_ns")},
                              "transfer": cfg.transfer()}), flush=True)


if __name__ == "__main__":
    main()
