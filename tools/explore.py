"""Exploration harness: run the headline workload under config variants, one line each.

    python tools/explore.py [--size-gib 16] [--steps 2] "k=v k=v" "k=v" ...

Prints GB/s (device-timed), and where the CTAs' time went (fraction of CTA-time spent
waiting for RPCs, in metadata, in copies).  Not a benchmark of record (bench.py is).
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-gib", type=float, default=16.0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    import torch
    from paper_2109_05366_b200.build import build
    build()
    size = int(a.size_gib * bench.GiB)
    base = bench.headline_overrides(size, 1, a.dir)
    dist = bench.Dist(1)
    path = None
    dst = None
    for v in a.variants or [""]:
        sets = [x for x in v.split() if x]
        cfg = bench.make_cfg(base, sets)
        if cfg["io.dir"] != a.dir or path is None:
            path = bench.ensure_file(cfg, dist)
        try:
            t0 = time.time()
            if dst is not None and dst.numel() < cfg["workload.total_bytes"]:
                dst = None  # a larger workload than the last variant: fresh user buffer
                torch.cuda.empty_cache()
            r = bench.run_arm(cfg, path, 0, 0, a.steps, 1, dst=dst)
            dst = r["dst"]
            st = r["stats"][-1]
            ns = st["kernel_ns"]
            cta_ns = ns * r["ctas"]
            W = st["io_workers"]
            line = {"variant": v or "headline", "gbps": round(st["user_bytes"] / ns, 2),
                    "rpcs": st["rpc_count"],
                    "cta_wait": round(st["wait_ns"] / cta_ns, 3),
                    "cta_meta": round(st["meta_ns"] / cta_ns, 3),
                    "cta_copy": round(st["copy_ns"] / cta_ns, 3),
                    "us_rpc_wait": round(st["wait_ns"] / max(1, st["rpc_count"]) / 1e3, 1),
                    "greads": st["greads"],
                    "us_gread_meta": round(st["meta_ns"] / max(1, st["greads"]) / 1e3, 2),
                    "us_gread_copy": round(st["copy_ns"] / max(1, st["greads"]) / 1e3, 2),
                    "us_gread_install": round(st["install_ns"] / max(1, st["greads"]) / 1e3, 2),
                    "us_gread_other": round((cta_ns - st["wait_ns"] - st["meta_ns"] - st["copy_ns"]
                                             - st["install_ns"]) / max(1, st["greads"]) / 1e3, 2),
                    "host_pread": round(st["host_pread_ns"] / (W * ns), 3),
                    "host_xfer": round(st["host_xfer_ns"] / (W * ns), 3),
                    "host_idle": round(st["host_idle_ns"] / (W * ns), 3),
                    "us_pread": round(st["host_pread_ns"] / max(1, st["host_requests"]) / 1e3, 1),
                    "mism": r["mismatched_words"], "wall_s": round(time.time() - t0, 1)}
        except Exception as e:
            line = {"variant": v, "error": str(e)[:400]}
        print(json.dumps(line), flush=True)
    del dst
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
