"""Re-run stress cases (tests/test_gpu_stress.py random_case) with variants, many reps on one
context, and report word mismatches per rep (GFS_DEBUG_MISMATCH=1 prints the first bad word).

    python tools/stress_repro.py --case 29 --reps 6 [--set key=value ...] [--variants]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("GFS_DEBUG_MISMATCH", "1")

from paper_2109_05366_b200.config import ExperimentConfig  # noqa: E402
from paper_2109_05366_b200.workloads import ProgramTable  # noqa: E402
from test_gpu_stress import FILE_BYTES, random_case  # noqa: E402


def run(k, reps, extra):
    import torch
    from paper_2109_05366_b200.runtime import GpuFS, ensure_synthetic
    over, progs, request = random_case(k)
    over.update(extra)
    d = "/dev/shm/gfs_stress"
    os.makedirs(d, exist_ok=True)
    paths = [ensure_synthetic(d, cid, fb) for cid, fb in enumerate(FILE_BYTES)]
    cfg = ExperimentConfig({**over, "io.dir": d})
    table = ProgramTable.from_programs(progs)
    out = []
    with GpuFS(cfg, max_request_bytes=request) as fs:
        for cid, p in enumerate(paths):
            fs.gopen(p, content_id=cid)
        dst = torch.empty(table.dst_bytes, dtype=torch.uint8, device="cuda")
        for rep in range(reps):
            dst.fill_(0xA5)
            r = fs.run(table, request, dst)
            v = fs.verify(table, dst)
            out.append((r.stats["word_mismatches"], v))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", type=int, action="append", default=[])
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--variants", action="store_true")
    a = ap.parse_args()
    extra = {}
    for kv in a.set:
        key, v = kv.split("=", 1)
        extra[key] = int(v) if v.isdigit() else v
    variants = [{}]
    if a.variants:
        variants = [{}, {"gpu.k1_copy": "ldg"}, {"gpu.cta_threads": 256}, {"io.transfer": "mapped"},
                    {"io.transfer": "bounce"}, {"io.readahead": "doubling"}, {"gpu.lookahead": False}]
    for k in a.case or [29]:
        for v in variants:
            res = run(k, a.reps, {**extra, **v})
            print(json.dumps({"case": k, "variant": {**extra, **v}, "mismatch_per_rep": res}), flush=True)


if __name__ == "__main__":
    main()
