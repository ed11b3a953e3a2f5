"""Cache-hit throughput: every TB reads its stride twice in one program (file < cache); the
second pass is served from the HBM page cache.  Prints the device time of one pass and of
the two-pass program, and the extra time the hit pass adds (it overlaps other TBs' cold
windows, so it is not an isolated hit-copy rate).  Not a benchmark of record.

    python tools/hit_probe.py [--size-gib 4] [--n-tb 1024] [--request-kib 64]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import bench  # noqa: E402


def main():
    import torch
    from paper_2109_05366_b200.runtime import GpuFS
    from paper_2109_05366_b200.workloads import ProgramTable
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-gib", type=float, default=4.0)
    ap.add_argument("--n-tb", type=int, default=1024)
    ap.add_argument("--request-kib", type=int, default=64)
    ap.add_argument("--set", action="append", default=[])
    a = ap.parse_args()
    GiB, KiB = bench.GiB, bench.KiB
    size = int(a.size_gib * GiB)
    req = a.request_kib * KiB
    cfg = bench.make_cfg({**bench.headline_overrides(size, 1, "/dev/shm"), "gpufs.cache_bytes": 2 * size,
                          "workload.request_bytes": req}, a.set)
    path = bench.ensure_file(cfg, bench.Dist(1))
    stride = size // a.n_tb
    once = ProgramTable.from_programs([[(0, t * stride, stride)] for t in range(a.n_tb)])
    twice = ProgramTable.from_programs([[(0, t * stride, stride)] * 2 for t in range(a.n_tb)])
    dst = torch.empty(twice.dst_bytes, dtype=torch.uint8, device="cuda")
    out = {}
    with GpuFS(cfg, max_request_bytes=req) as fs:
        fs.gopen(path, content_id=0)
        for name, table in (("once", once), ("twice", twice)):
            print(f"hit_probe: {name} warm-up", file=sys.stderr, flush=True)
            fs.run(table, req, dst)
            print(f"hit_probe: {name} timed", file=sys.stderr, flush=True)
            r = fs.run(table, req, dst)
            out[name] = {"ms": r.stats["kernel_ns"] / 1e6, "pc_hits": r.stats["pc_hits"],
                         "mism": r.stats["word_mismatches"]}
    # the second pass of early TBs overlaps other TBs' cold windows, so this is the extra
    # device time the hits cost the whole program, not an isolated hit-copy rate
    hit_s = (out["twice"]["ms"] - out["once"]["ms"]) / 1e3
    out["hit_pass_extra_ms"] = round(hit_s * 1e3, 3)
    out["hit_bytes_per_extra_s_gbps"] = round(size / hit_s / 1e9, 1) if hit_s > 0 else None
    out["config"] = {"size": size, "n_tb": a.n_tb, "request": req, "transfer": cfg.transfer()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
