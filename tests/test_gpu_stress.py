"""Stress at full residency (592 CTAs): seeded random multi-segment programs — several files,
unaligned offsets and lengths, segments re-read or jumping backwards, requests that do or do
not divide pages, caches above and below the union — under every transfer and both K1
copies, lookahead on.  Schedules are free here (hundreds of TBs racing for shared pages),
so only schedule-invariant quantities are compared: every delivered byte must satisfy the
file's word law (device check during the pass and `gfs_verify_dst` after it), and
`greads` / `user_bytes` must equal the program's closed form (gpu_exec.py:95-129), and the
page table must pass check_unique_mapping (gpu_cache.py:217-224) after every pass.  Each
case runs three times on one context to shake out races between the passes."""

import os

import pytest

from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.rng import SeededRng
from paper_2109_05366_b200.workloads import ProgramTable

pytestmark = pytest.mark.gpu

KiB, MiB = 1 << 10, 1 << 20
N_CASES = 72
TRANSFERS = ["mapped_dma", "mapped", "bounce", "dma", "zerocopy", "mapped_hybrid", "pread_hybrid"]
FILE_BYTES = [512 * MiB + 12345, 320 * MiB]


def random_case(k: int):
    r = SeededRng(5000 + k)
    n_tb = 100 + r.below(1100)
    page = [4096, 4096, 8192][r.below(3)]
    request = [4 * KiB, 10_000, 64 * KiB, 100_000, 1 * MiB][r.below(5)]
    progs = []
    for _ in range(n_tb):
        segs = []
        for _ in range(1 + r.below(4)):
            if segs and r.below(4) == 0:
                segs.append(segs[r.below(len(segs))])  # re-read an earlier segment
                continue
            fid = r.below(len(FILE_BYTES))
            fs = FILE_BYTES[fid]
            ln = 1 + r.below(2 * MiB)
            off = r.below(fs - ln)
            if r.below(2):
                off -= off % page
            segs.append((fid, off, ln))
        progs.append(segs)
    cfg = {
        "gpufs.page_size": page,
        "gpufs.prefetch_bytes": page * r.below(16),
        "gpufs.cache_bytes": [256 * MiB, 1024 * MiB, 4096 * MiB][r.below(3)],
        "gpufs.policy": "global-lru-dealloc" if r.below(6) == 0 else "per-tb-lra",
        "io.readahead": ["static", "adaptive", "doubling"][r.below(3)],
        "io.ra_max_bytes": page << (4 + r.below(9)),
        "io.transfer": TRANSFERS[k % len(TRANSFERS)],
        "gpu.k1_copy": ("tma", "ldg")[(k // len(TRANSFERS)) % 2],
        "gpu.cta_threads": (256, 512, 128)[k % 3],
        "workload.request_bytes": request,
        "mode.verify": True,
    }
    return cfg, progs, request


def _case_id(k: int) -> str:
    return f"{k}-{TRANSFERS[k % len(TRANSFERS)]}-{('tma', 'ldg')[(k // len(TRANSFERS)) % 2]}"


def eof_case(k: int):
    """EOF-heavy programs: every TB reads to the end of a file from a random point in its last
    48 MiB, so TBs end on short EOF pages and release frames at the same time — under
    global-lru-dealloc, where every release and recycled take goes through the one global
    lock (take_recycled / release_frame), and a cache far smaller than the pages touched."""
    r = SeededRng(9000 + k)
    n_tb = 200 + r.below(300)
    page = 4096
    request = [4 * KiB, 10_000, 64 * KiB][r.below(3)]
    progs = []
    for _ in range(n_tb):
        fid = r.below(len(FILE_BYTES))
        fs = FILE_BYTES[fid]
        ln = 1 + r.below(48 * MiB)
        progs.append([(fid, fs - ln, ln)])
    cfg = {
        "gpufs.page_size": page,
        "gpufs.prefetch_bytes": page * r.below(16),
        "gpufs.cache_bytes": [64 * MiB, 128 * MiB][r.below(2)],
        "gpufs.policy": "global-lru-dealloc" if k % 4 else "per-tb-lra",
        "io.readahead": ["static", "adaptive", "doubling"][k % 3],
        "io.ra_max_bytes": page << (4 + r.below(6)),
        "io.transfer": TRANSFERS[k % len(TRANSFERS)],
        "workload.request_bytes": request,
        "mode.verify": True,
    }
    return cfg, progs, request


@pytest.mark.parametrize("k", range(N_CASES), ids=_case_id)
def test_random_multisegment_programs_full_residency(k):
    _run_case(k, *random_case(k))


@pytest.mark.parametrize("k", range(12), ids=lambda k: f"eof{k}-{TRANSFERS[k % len(TRANSFERS)]}")
def test_eof_heavy_programs_full_residency(k):
    _run_case(k, *eof_case(k))


def _run_case(k, over, progs, request):
    import torch
    from paper_2109_05366_b200.runtime import GpuFS, ensure_synthetic
    d = "/dev/shm/gfs_stress"
    os.makedirs(d, exist_ok=True)
    paths = [ensure_synthetic(d, cid, fb) for cid, fb in enumerate(FILE_BYTES)]
    cfg = ExperimentConfig({**over, "io.dir": d})
    table = ProgramTable.from_programs(progs)
    want_bytes = sum(ln for segs in progs for _, _, ln in segs)
    want_greads = sum(-(-ln // request) for segs in progs for _, _, ln in segs)
    with GpuFS(cfg, max_request_bytes=request) as fs:
        for cid, p in enumerate(paths):
            fs.gopen(p, content_id=cid)
        dst = torch.empty(table.dst_bytes, dtype=torch.uint8, device="cuda")
        for rep in range(3):
            dst.fill_(0xA5)
            r = fs.run(table, request, dst)
            st = r.stats
            assert st["user_bytes"] == want_bytes, (k, rep, st["user_bytes"], want_bytes, over)
            assert st["greads"] == want_greads, (k, rep, st["greads"], want_greads, over)
            assert st["word_mismatches"] == 0, (k, rep, over)
            assert fs.verify(table, dst) == 0, (k, rep, over)
            m = fs.check_unique_mapping()  # raises on a duplicate / stale / lost mapping
            assert m["mapped_pages"] > 0, (k, rep, m)
