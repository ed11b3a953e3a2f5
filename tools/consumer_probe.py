"""Where fused-consumer time goes: C4 shape (950 MB, 128 TBs) through the timeline, one line
per consumer variant (GB/s, CTA time computing, per-request consume p50).  Not a
benchmark of record.

    python tools/consumer_probe.py [key=value ...]
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import bench  # noqa: E402


def main():
    import numpy as np
    import torch
    from paper_2109_05366_b200 import timeline
    from paper_2109_05366_b200.runtime import Consumer, GpuFS
    from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided
    KiB, GiB = bench.KiB, bench.GiB
    n_tb, unit = 128, 128 * 4096
    total = 950_000_000 // unit * unit
    cfg = bench.make_cfg({**bench.headline_overrides(16 * GiB, 1, "/dev/shm"), "mode.timeline": True,
                          "workload.n_tb": n_tb, "workload.total_bytes": total},
                         [x for x in sys.argv[1:] if "=" in x])
    path = bench.ensure_file(cfg, bench.Dist(1))
    wl = gen_sequential_strided([cfg["workload.file_bytes"]], n_tb, total, 64 * KiB, 4096)
    table = ProgramTable.from_programs(wl.programs)
    dst = torch.empty(total, dtype=torch.uint8, device="cuda")
    variants = {"none": None}
    for D, K in ((32, 8),):
        variants[f"kmeans_D{D}_K{K}"] = Consumer("kmeans_f32", x=torch.rand(K, D, device="cuda"),
                                                 y=torch.zeros(K, D, device="cuda"),
                                                 out=torch.zeros(K, dtype=torch.int64, device="cuda"),
                                                 cols=D, k=K)
    cols = 4096
    variants["gemv"] = Consumer("gemv_f32", x=torch.rand(cols, device="cuda"),
                                y=torch.zeros(total // 4 // cols, device="cuda"), cols=cols)
    variants["gemvt"] = Consumer("gemvt_f32", x2=torch.rand(total // 4 // cols, device="cuda"),
                                 y2=torch.zeros(cols, device="cuda"), cols=cols)
    only = os.environ.get("GFS_PROBE_ONLY")  # one variant (for ncu: warm-up launch, then the timed one)
    if only:
        variants = {only: variants[only]}
    with GpuFS(cfg, max_request_bytes=64 * KiB) as fs:
        fs.gopen(path, content_id=0)
        for name, cons in variants.items():
            fs.run(table, 64 * KiB, dst, consumer=cons)
            r = fs.run(table, 64 * KiB, dst, consumer=cons)
            d = timeline.decode(r.timeline)
            con = d["kind"] == 2
            s = timeline.summary(r.timeline)
            line = {"variant": name, "gbps": round(r.stats["user_bytes"] / r.stats["kernel_ns"], 2),
                    "cta_consume_frac": s.get("cta_consume_frac"),
                    "consume_p50_us": round(float(np.percentile((d["t1"][con] - d["t0"][con]), 50)) / 1e3, 2)
                    if con.any() else None}
            print(json.dumps(line), flush=True)
            if name == "kmeans_D32_K8":  # where a TB's time goes: waits vs compute
                per = {}
                for k in range(len(d["t0"])):
                    cta = int(d["cta"][k])
                    e = per.setdefault(cta, {"rpc_wait": 0, "consume": 0, "gread": 0, "first": None, "last": 0})
                    dur = int(d["t1"][k] - d["t0"][k])
                    kind = int(d["kind"][k])
                    e[("rpc_wait", "gread", "consume")[kind]] += dur
                    e["first"] = int(d["t0"][k]) if e["first"] is None else min(e["first"], int(d["t0"][k]))
                    e["last"] = max(e["last"], int(d["t1"][k]))
                t0 = int(d["t0"].min())
                ends = sorted((v["last"] - t0) / 1e6 for v in per.values())
                avg = {k: round(float(np.mean([v[k] for v in per.values()])) / 1e6, 2) for k in ("rpc_wait", "consume", "gread")}
                print(json.dumps({"kmeans_per_cta_ms": avg, "cta_end_ms_p0_p50_p100": [ends[0], ends[len(ends) // 2], ends[-1]],
                                  "span_ms": (int(d["t1"].max()) - t0) / 1e6}), flush=True)


if __name__ == "__main__":
    main()
