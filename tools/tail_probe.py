"""Where the headline pass loses time against the link: device timeline of one 16 GiB
headline pass — ramp before the link is busy, tail after the last transfer lands, and the
outstanding-transfer count over time.  Not a benchmark of record.

    python tools/tail_probe.py [--set k=v ...]
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
    from paper_2109_05366_b200 import timeline
    from paper_2109_05366_b200.runtime import GpuFS
    GiB = bench.GiB
    cfg = bench.make_cfg({**bench.headline_overrides(16 * GiB, 1, "/dev/shm"), "mode.timeline": True},
                         [a.split("=", 1)[0] + "=" + a.split("=", 1)[1] for a in sys.argv[1:] if "=" in a])
    path = bench.ensure_file(cfg, bench.Dist(1))
    r = bench.run_arm(cfg, path, 0, 0, 1, 1)
    wl, table = bench.shard_table(cfg, 0)
    with GpuFS(cfg, max_request_bytes=wl.request_bytes) as fs:
        fs.gopen(path, content_id=0)
        rr = fs.run(table, wl.request_bytes, r["dst"])
    d = timeline.decode(rr.timeline)
    t0 = int(d["t0"].min())
    end = int(d["t1"].max())
    rpc = d["kind"] == 0
    first_done = int(d["t1"][rpc].min())
    last_done = int(d["t1"][rpc].max())
    # outstanding transfers over time (1 ms bins)
    bins = np.arange(t0, end + 1_000_000, 1_000_000)
    out = [int(((d["t0"][rpc] <= b) & (d["t1"][rpc] > b)).sum()) for b in bins]
    res = {"gbps": round(rr.stats["user_bytes"] / rr.stats["kernel_ns"], 3),
           "kernel_ms": rr.stats["kernel_ns"] / 1e6, "span_ms": (end - t0) / 1e6,
           "first_transfer_done_ms": (first_done - t0) / 1e6,
           "last_transfer_done_ms": (last_done - t0) / 1e6,
           "tail_after_last_transfer_ms": (end - last_done) / 1e6,
           "rpcs": int(rpc.sum()), "window_mib": round(float(d["bytes"][rpc].mean()) / (1 << 20), 2),
           "outstanding_per_ms": out, "summary": timeline.summary(rr.timeline)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
