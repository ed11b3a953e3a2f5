"""The device's ondemand readahead (io.readahead=adaptive) against the reference's own
HostOs window_history (host_os.py:106-152), stream by stream, and against the oracle in
full (windows, RPC trace, deliveries, counters, bytes), under every transfer.

Fixtures: tests/golden/windows/*.json (tests/golden/make_windows.py ran the reference).
Each stream is one TB whose program is the fixture's read list, io.ra_clamp=eof (the
reference's clamp).  Streams in test_readahead_law.BOUNDED outgrow a TB's readahead state
(two landing halves, four markers); they match the reference up to the documented read and
the oracle everywhere.
"""

import os

import numpy as np
import pytest

import golden_util as gu
import oracle as orc
from test_readahead_law import BOUNDED, _prefix

pytestmark = pytest.mark.gpu

TRANSFERS = ["mapped_dma", "mapped", "bounce", "zerocopy", "dma", "mapped_hybrid", "pread_hybrid"]


def run_device(cfg, wl, transfer):
    import torch
    from paper_2109_05366_b200.runtime import GpuFS, ensure_synthetic
    from paper_2109_05366_b200.workloads import ProgramTable
    d = "/dev/shm/gfs_test" if os.path.isdir("/dev/shm") else "/tmp/gfs_test"
    path = ensure_synthetic(d, 0, wl.files[0])
    table = ProgramTable.from_programs(wl.programs)
    run_cfg = cfg.copy_with({"io.transfer": transfer, "io.dir": d, "io.workers": 4})
    with GpuFS(run_cfg, max_request_bytes=wl.request_bytes) as fs:
        fs.gopen(path, content_id=0)
        dst = torch.empty(max(table.dst_bytes, 1), dtype=torch.uint8, device="cuda")
        res = fs.run(table, wl.request_bytes, dst)
        out = dst[:table.dst_bytes].cpu().numpy()
    return res, out


@pytest.mark.parametrize("transfer", TRANSFERS)
@pytest.mark.parametrize("name", gu.window_case_names())
def test_device_windows_match_reference_and_oracle(name, transfer):
    g, cfg, wl = gu.window_case(name)
    res, out = run_device(cfg, wl, transfer)
    ref = orc.run_oracle(cfg, wl, source=orc.SRC_SYNTH, materialize_dst=True)
    got = res.windows[:, 1].tolist()
    if name in BOUNDED:
        k = BOUNDED[name]
        assert got[:len(_prefix(g, k))] == _prefix(g, k)
    else:
        assert got == g["window_history"]
    assert got == ref.windows[:, 1].tolist()
    assert np.array_equal(res.rpcs, ref.rpcs)
    assert np.array_equal(res.deliveries, ref.deliveries)
    for k in ("user_bytes", "greads", "pc_misses", "pc_hits", "pb_hits", "pb_misses", "rpc_count",
              "rpc_requested_bytes", "pb_filled_bytes", "pb_consumed_bytes", "pb_discarded_bytes",
              "pcie_bytes"):
        assert res.stats[k] == ref.stats[k], (k, res.stats[k], ref.stats[k])
    assert np.array_equal(out, ref.dst)
    assert res.stats["word_mismatches"] == 0
