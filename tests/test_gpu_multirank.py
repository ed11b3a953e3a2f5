"""Multi-rank device path (world_size 2, both ranks on cuda:0, gloo for the host-side
collectives): each rank reads its own disjoint contiguous shard of one file through its
own GpuFS — the sharding bench.py --gpus N uses — and must match the
oracle run of the same shard exactly: counters, per-TB RPC traces, user-buffer bytes; the
all-reduced 8-byte checksum must equal the whole file's."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
KiB, MiB = 1 << 10, 1 << 20
WORLD = 2
SHARD = 24 * MiB


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, d, transfer, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import torch
    import oracle as orc
    from paper_2109_05366_b200 import rng as grng
    from paper_2109_05366_b200.config import ExperimentConfig
    from paper_2109_05366_b200.runtime import GpuFS, ensure_synthetic_shard
    from paper_2109_05366_b200.workloads import ProgramTable, gen_sequential_strided
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(WORLD))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        cfg = ExperimentConfig({"workload.n_tb": 24, "workload.file_bytes": SHARD * WORLD,
                                "workload.total_bytes": SHARD, "workload.request_bytes": 64 * KiB,
                                "gpufs.prefetch_bytes": 60 * KiB, "gpufs.cache_bytes": 8 * MiB,
                                "gpufs.policy": "per-tb-lra", "gpu.sm_count": 4, "io.dir": d,
                                "io.readahead": "adaptive", "io.ra_max_bytes": 512 * KiB,
                                "io.transfer": transfer, "mode.deterministic": True, "io.workers": 4})
        path = ensure_synthetic_shard(d, 0, SHARD * WORLD, rank, WORLD, dist.barrier)
        wl = gen_sequential_strided([SHARD * WORLD], 24, SHARD, 64 * KiB, 4096,
                                    file_base_offset=rank * SHARD)
        table = ProgramTable.from_programs(wl.programs)
        with GpuFS(cfg) as fs:
            fs.gopen(path, content_id=0)
            dst = torch.empty(table.dst_bytes, dtype=torch.uint8, device="cuda:0")
            r = fs.run(table, 64 * KiB, dst)
            csum = fs.checksum(dst, word_base=rank * SHARD // 8)
            got = dst.cpu().numpy()
        ref = orc.run_oracle(cfg, wl, source=orc.SRC_SYNTH, materialize_dst=True)
        keys = ("user_bytes", "rpc_count", "pb_hits", "pc_misses", "pc_remaps", "victims")
        out[f"ok{rank}"] = (all(r.stats[k] == ref.stats[k] for k in keys)
                            and np.array_equal(r.rpcs[np.argsort(r.rpcs[:, 0], kind="stable")],
                                               ref.rpcs[np.argsort(ref.rpcs[:, 0], kind="stable")])
                            and np.array_equal(got, ref.dst) and r.stats["word_mismatches"] == 0)
        t = torch.tensor([csum - (1 << 64) if csum >= (1 << 63) else csum], dtype=torch.int64)
        dist.all_reduce(t)
        if rank == 0:
            out["sum"] = int(t.item()) & ((1 << 64) - 1)
            out["whole"] = grng.checksum(grng.content(0, 0, SHARD * WORLD))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("transfer", ["mapped_dma", "bounce"])
def test_two_ranks_read_their_shards_exactly(transfer):
    d = "/dev/shm/gfs_multirank" if os.path.isdir("/dev/shm") else "/tmp/gfs_multirank"
    os.makedirs(d, exist_ok=True)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), d, transfer, out), nprocs=WORLD, join=True)
    assert out["ok0"] and out["ok1"]
    assert out["sum"] == out["whole"]
