"""Multi-rank host logic on CPU (gloo, world_size 2): the sharding bench.py --gpus N uses.

Each rank owns a disjoint contiguous shard of one file and runs the
reference algorithm (the oracle, as the checker) on it; the shards must tile the file,
per-TB RPC traces must be the base-0 traces shifted by the shard base, and the 8-byte
checksum all-reduce must equal the single-process checksum of the whole file.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

KiB, MiB = 1 << 10, 1 << 20
WORLD = 2
SHARD = 2 * MiB


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg():
    from paper_2109_05366_b200.config import ExperimentConfig
    return ExperimentConfig({"workload.n_tb": 8, "workload.file_bytes": SHARD * WORLD,
                             "workload.total_bytes": SHARD, "workload.request_bytes": 64 * KiB,
                             "gpufs.prefetch_bytes": 28 * KiB, "gpufs.cache_bytes": 1 * MiB,
                             "gpufs.policy": "per-tb-lra", "gpu.sm_count": 2})


def _shard(cfg, rank):
    from paper_2109_05366_b200.workloads import gen_sequential_strided
    return gen_sequential_strided([cfg["workload.file_bytes"]], cfg["workload.n_tb"], SHARD,
                                  cfg["workload.request_bytes"], cfg["gpufs.page_size"],
                                  file_base_offset=rank * SHARD)


def _worker(rank, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import torch
    import oracle as orc
    from paper_2109_05366_b200 import rng as grng
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    cfg = _cfg()
    wl = _shard(cfg, rank)
    res = orc.run_oracle(cfg, wl, source=orc.SRC_SYNTH, materialize_dst=True)
    csum = grng.checksum(res.dst.tobytes(), word_base=rank * SHARD // 8)
    t = torch.tensor([csum - (1 << 64) if csum >= (1 << 63) else csum], dtype=torch.int64)
    dist.all_reduce(t)
    lo = min(off for prog in wl.programs for _f, off, _l in prog)
    hi = max(off + ln for prog in wl.programs for _f, off, ln in prog)
    spans = torch.tensor([lo, hi], dtype=torch.int64)
    gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(WORLD)]
    dist.all_gather(gathered, spans)
    if rank == 0:
        out["sum"] = int(t.item()) & ((1 << 64) - 1)
        out["spans"] = [g.tolist() for g in gathered]
    out[f"rpcs{rank}"] = res.rpcs.tolist()
    out[f"bytes{rank}"] = res.stats["user_bytes"]
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_sharded_ranks_tile_the_file_and_reduce_checksums():
    import oracle as orc
    from paper_2109_05366_b200 import rng as grng
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    # shards tile [0, WORLD * SHARD) without overlap
    assert sorted(out["spans"]) == [[r * SHARD, (r + 1) * SHARD] for r in range(WORLD)]
    assert all(out[f"bytes{r}"] == SHARD for r in range(WORLD))
    # all-reduced 8-byte checksum == checksum of the whole file in one process
    whole = grng.content(0, 0, WORLD * SHARD)
    assert out["sum"] == grng.checksum(whole)
    # shift invariance: rank r's per-TB RPC trace = rank 0's shifted by r * SHARD
    r0 = np.asarray(out["rpcs0"])
    r1 = np.asarray(out["rpcs1"])
    shifted = r0.copy()
    shifted[:, 2] += SHARD
    assert np.array_equal(r1, shifted)
    # and the rank-0 shard equals a plain (unsharded-config) run of the same bytes
    cfg = _cfg()
    base = orc.run_oracle(cfg, _shard(cfg, 0))
    assert np.array_equal(base.rpcs, r0)


def _shard_worker(rank, world, d, size, port):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_05366_b200.runtime import ensure_synthetic_shard
    path = ensure_synthetic_shard(d, 7, size, rank, world, dist.barrier)
    dist.barrier()
    dist.destroy_process_group()
    return path


def test_sharded_generation_equals_whole_file(tmp_path):
    """Ranks writing their own shards (gfs_gen_file_range) produce the same bytes as one
    writer (W-law content), and the ready stamp appears only once all shards are done."""
    import torch.multiprocessing as tmp
    from paper_2109_05366_b200 import native
    from paper_2109_05366_b200 import rng as grng
    from paper_2109_05366_b200.runtime import synthetic_path, synthetic_ready
    size = (3 << 20) + 4104  # not a multiple of the shard count: last rank takes the rest
    d = str(tmp_path)
    tmp.spawn(_shard_worker, args=(2, d, size, 29631), nprocs=2, join=True)
    path = synthetic_path(d, 7, size)
    assert synthetic_ready(path, size)
    got = open(path, "rb").read()
    assert got == grng.content(7, 0, size)
    whole = str(tmp_path / "whole.bin")
    native.gen_file(whole, 7, size)
    assert open(whole, "rb").read() == got
