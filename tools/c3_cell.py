"""A few C3 cells (configs[2]) with overrides, each with its per-CTA time split from the
device timeline: where a TB's time goes when there are few TBs.  Not a benchmark of record.

    python tools/c3_cell.py --cell 64x4K --cell 64x16K --arm static [--set key=value ...]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import bench  # noqa: E402
from sweep_c3 import ARMS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cell", action="append", default=[])
    ap.add_argument("--arm", default="prefetch_static")
    ap.add_argument("--size-gib", type=float, default=2.0)
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--timeline", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2109_05366_b200 import timeline
    from paper_2109_05366_b200.runtime import GpuFS
    from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided
    size = int(a.size_gib * bench.GiB)
    base = bench.headline_overrides(size, 1, "/dev/shm")
    base["gpufs.cache_bytes"] = 1 * bench.GiB
    base.update(ARMS[a.arm])
    if a.timeline:
        base["mode.timeline"] = True
    cfg = bench.make_cfg(base, a.set)
    path = bench.ensure_file(cfg, bench.Dist(1))
    dst = torch.empty(size, dtype=torch.uint8, device="cuda")
    with GpuFS(cfg, max_request_bytes=2 * bench.MiB) as fs:
        fs.gopen(path, content_id=0)
        for cell in a.cell or ["64x4K"]:
            n_tb, req = cell.split("x")
            n_tb, req = int(n_tb), int(req.rstrip("K")) * 1024
            wl = gen_sequential_strided([size], n_tb, size, req, cfg["gpufs.page_size"])
            table = ProgramTable.from_programs(wl.programs)
            fs.run(table, req, dst)
            r = fs.run(table, req, dst)
            st = r.stats
            out = {"cell": cell, "arm": a.arm, "set": a.set, "gbps": round(size / st["kernel_ns"], 3),
                   "transfer": fs.transfer, "ctas": st["ctas"], "rpc_count": st["rpc_count"], "early_answers": st.get("early_answers"),
                   "per_cta_ms": {k: round(st[k] / max(1, min(n_tb, st["ctas"])) / 1e6, 2)
                                  for k in ("wait_ns", "meta_ns", "copy_ns", "install_ns", "lookup_ns", "alloc_ns")},
                   "kernel_ms": round(st["kernel_ns"] / 1e6, 2)}
            if a.timeline and r.timeline is not None:
                d = timeline.decode(r.timeline)
                for kind, name in ((0, "rpc"), (1, "gread")):
                    m = d["kind"] == kind
                    if m.any():
                        dur = (d["t1"][m] - d["t0"][m]) / 1e3
                        out[f"{name}_us_p50_p90"] = [round(float(np.percentile(dur, 50)), 1),
                                                    round(float(np.percentile(dur, 90)), 1)]
                m = d["kind"] == 1
                if m.any():  # per TB: first gread start .. last gread end, against the pass
                    t0, t1, tb = d["t0"][m], d["t1"][m], d["tb"][m]
                    g0 = int(t0.min())
                    life = [(int(t0[tb == t].min()) - g0, int(t1[tb == t].max()) - g0) for t in np.unique(tb)]
                    ends = np.array([b for _, b in life]) / 1e6
                    starts = np.array([a for a, _ in life]) / 1e6
                    out["tb_start_ms_max"] = round(float(starts.max()), 2)
                    tbs = np.unique(tb)
                    cta_of = {int(t): int(d["cta"][m][tb == t][0]) for t in tbs}
                    late = np.argsort(ends)[-6:][::-1]
                    out["latest_tbs"] = [(int(tbs[i]), cta_of[int(tbs[i])], round(float(ends[i]), 2)) for i in late]
                    out["tb_end_ms_p10_p50_max"] = [round(float(np.percentile(ends, 10)), 2),
                                                    round(float(np.percentile(ends, 50)), 2),
                                                    round(float(ends.max()), 2)]
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
