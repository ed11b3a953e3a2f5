"""The Mosaic-style random workload (preset `mosaic`) under a few transfers / TB counts,
with per-request RPC and gread latencies from the device timeline.  Not a benchmark of
record.

    python tools/mosaic_probe.py
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2109_05366_b200 import timeline  # noqa: E402
from paper_2109_05366_b200.experiments import PRESETS  # noqa: E402
from paper_2109_05366_b200.runtime import Simulation  # noqa: E402

base = bench.make_cfg(bench.headline_overrides(16 << 30, 1, "/dev/shm"), [])
bench.ensure_file(base, bench.Dist(1))
for label, mcfg in PRESETS["mosaic"](base):
    extras = [{}, {"io.transfer": "bounce"}, {"workload.n_tb": 512}, {"workload.requests_per_tb": 1024}]
    if os.environ.get("GFS_MOSAIC_EXTRAS"):  # e.g. '[{}, {"gpu.k1_direct": false}]'
        extras = json.loads(os.environ["GFS_MOSAIC_EXTRAS"])
    for extra in extras:
        cfg = mcfg.copy_with({"workload.file_bytes": base["workload.file_bytes"], "mode.timeline": True, **extra})
        sim = Simulation(cfg, 42)
        t0 = time.time(); rep = sim.run(); wall = time.time() - t0
        st = sim.result.stats
        d = timeline.decode(sim.result.timeline)
        rpc = d["kind"] == 0; gr = d["kind"] == 1
        lat = (d["t1"][rpc] - d["t0"][rpc]) / 1e3; gl = (d["t1"][gr] - d["t0"][gr]) / 1e3
        print(json.dumps({"label": label, "extra": extra, "gbps": round(rep["io_bandwidth_bps"] / 1e9, 3),
                          "kernel_ms": st["kernel_ns"] / 1e6, "wall_s": round(wall, 2), "rpcs": st["rpc_count"],
                          "ctas": st["ctas"], "rpc_lat_us_p50_p99": [round(float(np.percentile(lat, q)), 1) for q in (50, 99)],
                          "gread_us_p50_p99": [round(float(np.percentile(gl, q)), 1) for q in (50, 99)],
                          "pc_hit_pending": st["pc_hit_pending"], "transfer": cfg.transfer()}), flush=True)
