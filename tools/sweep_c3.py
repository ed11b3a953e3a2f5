"""configs[2] (C3): request/stride sweep x threadblock count, per arm.

    python tools/sweep_c3.py [--size-gib 2] [--out profiles/r01/c3_sweep.json]

Arms: the paper's prefetcher (4 KiB pages, 60 KiB prefetch, per-tb-lra),
the same with the adaptive window, the original non-prefetching GPUfs (4 KiB pages, no
prefetch, global-lru-dealloc), the 64 KiB-page arm (no prefetch), and CPU
read()+cudaMemcpy with the request size as the read chunk (16 threads).  Each cell is one
cold-cache pass over the file (device-timed), after one warm-up pass.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30
REQUESTS = [4 * KiB, 16 * KiB, 64 * KiB, 256 * KiB, 1 * MiB, 2 * MiB]
N_TBS = [64, 128, 256, 512, 1024]
ARMS = {
    "prefetch_static": {"gpufs.page_size": 4 * KiB, "gpufs.prefetch_bytes": 60 * KiB,
                        "gpufs.policy": "per-tb-lra", "io.readahead": "static"},
    "prefetch_adaptive": {"gpufs.page_size": 4 * KiB, "gpufs.prefetch_bytes": 60 * KiB,
                          "gpufs.policy": "per-tb-lra", "io.readahead": "adaptive"},
    "nonprefetch_gpufs": {"gpufs.page_size": 4 * KiB, "gpufs.prefetch_bytes": 0,
                          "gpufs.policy": "global-lru-dealloc", "io.readahead": "static"},
    "page64k": {"gpufs.page_size": 64 * KiB, "gpufs.prefetch_bytes": 0,
                "gpufs.policy": "global-lru-dealloc", "io.readahead": "static"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-gib", type=float, default=2.0)
    ap.add_argument("--dir", default="/dev/shm")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c3_sweep.json"))
    a = ap.parse_args()
    import torch
    from paper_2109_05366_b200 import native
    from paper_2109_05366_b200.build import build
    from paper_2109_05366_b200.runtime import GpuFS
    from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided
    build()
    size = int(a.size_gib * GiB)
    base = bench.headline_overrides(size, 1, a.dir)
    base["gpufs.cache_bytes"] = 1 * GiB  # file = 2x cache at the default 2 GiB
    cfg0 = bench.make_cfg(base, [])
    path = bench.ensure_file(cfg0, bench.Dist(1))
    dst = torch.empty(size, dtype=torch.uint8, device="cuda")
    results = {"file_bytes": size, "cache_bytes": base["gpufs.cache_bytes"], "arms": {}}
    for arm, over in ARMS.items():
        cfg = bench.make_cfg({**base, **over}, [])
        cells = {}
        with GpuFS(cfg, max_request_bytes=2 * MiB) as fs:
            fs.gopen(path, content_id=0)
            for n_tb in N_TBS:
                for req in REQUESTS:
                    stride = size // n_tb
                    if req > stride:
                        continue
                    wl = gen_sequential_strided([size], n_tb, size, req, cfg["gpufs.page_size"])
                    table = ProgramTable.from_programs(wl.programs)
                    try:
                        fs.run(table, req, dst)
                        r = fs.run(table, req, dst)
                        cells[f"{n_tb}x{req >> 10}K"] = round(size / r.stats["kernel_ns"], 3)
                    except Exception as e:  # recorded, not hidden
                        cells[f"{n_tb}x{req >> 10}K"] = f"error: {str(e)[:120]}"
                    print(arm, n_tb, req, cells[f"{n_tb}x{req >> 10}K"], flush=True)
        results["arms"][arm] = cells
    cpu = {}
    for req in REQUESTS:
        t = native.bench_read_memcpy(path, 0, size, dst.data_ptr(), 0, 16, max(req, 4096), True, False)
        cpu[f"{req >> 10}K"] = round(size / t / 1e9, 3)
        print("cpu_read_memcpy_16t", req, cpu[f"{req >> 10}K"], flush=True)
    results["arms"]["cpu_read_memcpy_16t"] = cpu
    results["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
