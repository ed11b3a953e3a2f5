"""Device timelines (mode.timeline) of (1) a headline gread pass and (2) the C4 gesummv
shape with the GEMV consumer fused — the overlap evidence nsys would give (PCIe transfers
outstanding while CTAs compute).  Writes a summary JSON and Chrome/Perfetto traces.

    python tools/timeline_run.py [--out gpurun_out] [--size-gib 2]
"""

import argparse
import gzip
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import bench  # noqa: E402


def gz(path):
    with open(path, "rb") as a, gzip.open(path + ".gz", "wb") as b:
        shutil.copyfileobj(a, b)
    os.remove(path)


def main():
    import torch
    from paper_2109_05366_b200 import timeline
    from paper_2109_05366_b200.runtime import Consumer, GpuFS
    from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--size-gib", type=float, default=2.0)
    ap.add_argument("--set", action="append", default=[])
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    KiB, GiB = bench.KiB, bench.GiB
    size = int(a.size_gib * GiB)
    cfg = bench.make_cfg({**bench.headline_overrides(size, 1, "/dev/shm"), "mode.timeline": True}, a.set)
    path = bench.ensure_file(cfg, bench.Dist(1))
    res = {}
    # (1) headline pass
    r = bench.run_arm(cfg, path, 0, 0, 1, 1)
    fs_stats = r["stats"][-1]
    # run_arm does not keep the timeline; repeat the pass on a GpuFS we hold
    wl, table = bench.shard_table(cfg, 0)
    dst = r["dst"]
    with GpuFS(cfg, max_request_bytes=wl.request_bytes) as fs:
        fs.gopen(path, content_id=0)
        fs.run(table, wl.request_bytes, dst)
        rr = fs.run(table, wl.request_bytes, dst)
        s = timeline.summary(rr.timeline)
        s["gbps"] = round(rr.stats["user_bytes"] / rr.stats["kernel_ns"], 3)
        s["transfer"] = cfg.transfer()
        res["headline_pass"] = s
        timeline.chrome_trace(rr.timeline, os.path.join(a.out, "timeline_headline.json"), 100_000)
        gz(os.path.join(a.out, "timeline_headline.json"))
    # (2) gesummv shape with the fused GEMV consumer (and without, for the I/O-only rate)
    n_tb, unit = 128, 128 * 4096
    total = 950_000_000 // unit * unit
    cfg2 = cfg.copy_with({"workload.n_tb": n_tb, "workload.total_bytes": total})
    with GpuFS(cfg2, max_request_bytes=64 * KiB) as fs:
        fs.gopen(path, content_id=0)
        wl2 = gen_sequential_strided([cfg["workload.file_bytes"]], n_tb, total, 64 * KiB, 4096)
        t2 = ProgramTable.from_programs(wl2.programs)
        cols = 4096
        x = torch.rand(cols, device="cuda")
        y = torch.zeros(total // 4 // cols, device="cuda")
        for name, cons in (("gesummv_gread_only", None),
                           ("gesummv_fused_gemv", Consumer("gemv_f32", x=x, y=y, cols=cols)),
                           ("kmeans_fused", Consumer("kmeans_f32", x=torch.rand(8, 32, device="cuda"),
                                                     y=torch.zeros(8, 32, device="cuda"),
                                                     out=torch.zeros(8, dtype=torch.int64, device="cuda"),
                                                     cols=32, k=8))):
            fs.run(t2, 64 * KiB, dst, consumer=cons)
            rr = fs.run(t2, 64 * KiB, dst, consumer=cons)
            s = timeline.summary(rr.timeline)
            s["gbps"] = round(rr.stats["user_bytes"] / rr.stats["kernel_ns"], 3)
            res[name] = s
            if cons is not None and name == "gesummv_fused_gemv":
                timeline.chrome_trace(rr.timeline, os.path.join(a.out, f"timeline_{name}.json"))
                gz(os.path.join(a.out, f"timeline_{name}.json"))
    res["note"] = ("GPU globaltimer intervals per CTA: rpc = request published .. data in HBM; "
                   "consume = fused consumer over a delivered request. consume_overlap_frac = share "
                   "of compute time during which some transfer was outstanding.")
    res["headline_counters"] = {k: fs_stats[k] for k in ("user_bytes", "rpc_count", "kernel_ns")}
    with open(os.path.join(a.out, "timeline_summary.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
