"""The oracle's restatement of the ondemand readahead law (io.readahead=adaptive) against
the reference's own HostOs window_history (host_os.py:106-152), read stream by read stream.

Fixtures: tests/golden/windows/*.json, produced by running the reference in this container
(tests/golden/make_windows.py).  The device replays the same streams in
tests/test_gpu_readahead.py and must match both.
"""

import numpy as np
import pytest

import golden_util as gu
import oracle as orc


# Streams whose readahead state outgrows a TB's bound — two landing halves (the window
# being read and one pending) and OD_MARKS = 4 markers — while the reference's host page
# cache keeps every window and every marker: they match the reference up to the first read
# that needs the dropped state (a return to an abandoned run's window, a marker four
# decisions old), then follow the bounded law (the device is held to the oracle in full).
BOUNDED = {"two_runs": 80, "random_mix": 47}


def _prefix(g: dict, k: int) -> list:
    return g["window_history"][:g["history_len_after_read"][k - 1]] if k else []


@pytest.mark.parametrize("name", gu.window_case_names())
def test_oracle_window_history_matches_reference(name):
    g, cfg, wl = gu.window_case(name)
    if name in BOUNDED:
        k = BOUNDED[name]
        wl_k = wl.__class__(**{**wl.__dict__, "programs": [wl.programs[0][:k]]})
        assert orc.run_oracle(cfg, wl_k).windows[:, 1].tolist() == _prefix(g, k)
        return
    res = orc.run_oracle(cfg, wl)
    assert res.windows[:, 1].tolist() == g["window_history"]
    assert np.all(res.windows[:, 0] == 0)
    # every byte requested was delivered, each page fetched once (the cache holds the file)
    assert res.stats["user_bytes"] == wl.total_bytes
    assert res.stats["pc_misses"] == len({(off + k) // g["page"] for _, off, ln in wl.programs[0]
                                          for k in range(0, ln, 1)} )


def test_fixture_set_covers_reference_tests():
    names = set(gu.window_case_names())
    # tests/test_host_os.py:51-141 and acceptance criterion 1 (tests/test_acceptance.py:54-74)
    assert {"criterion1_256", "cold_4k", "marker_once", "cached_rewind", "nonsequential_reset",
            "context_recovery", "request_at_ra_max", "eof_clamp"} <= names
    g = gu.window_case("criterion1_256")[0]
    assert g["window_history"][:4] == [16384, 32768, 65536, 131072]
    assert set(g["window_history"][3:]) == {131072}


def test_headline_law_ramp():
    """The bench's stream (64 KiB requests, 16 MiB cap) ramps 256 KiB .. 8 MiB; a TB whose
    stride is the whole file under the segment clamp gets exactly the reference's windows
    (its last one clamped at the stride end = EOF)."""
    g, cfg, wl = gu.window_case("req64k_cap16m")
    one = wl.__class__(**{**wl.__dict__, "programs": [[(0, 0, g["file_bytes"])]]})
    res = orc.run_oracle(cfg.copy_with({"io.ra_clamp": "segment"}), one)
    assert res.windows[:, 1].tolist() == g["window_history"]
    assert res.stats["rpc_count"] == 8  # sync 64K, async 192K, 512K .. 8M, the clamped 256K
    assert res.stats["pcie_bytes"] == g["file_bytes"]  # nothing fetched twice or past the end


def test_stride_streams_under_segment_clamp():
    """Strides of one file as TBs (the bench's shape, scaled): the first request of a stride
    that does not start the file is not sequential (its neighbour's pages are outside the
    stream), so it is fetched alone and the ramp starts one request later; windows end at the
    stride end; no byte crosses PCIe twice."""
    from paper_2109_05366_b200.config import ExperimentConfig
    from paper_2109_05366_b200.workloads import build_workload
    cfg = ExperimentConfig({"workload.file_bytes": 64 << 20, "workload.n_tb": 4,
                            "workload.request_bytes": 64 << 10, "gpufs.page_size": 4096,
                            "gpufs.prefetch_bytes": 60 << 10, "gpufs.cache_bytes": 128 << 20,
                            "gpufs.policy": "per-tb-lra", "io.readahead": "adaptive",
                            "io.ra_max_bytes": 16 << 20, "mode.deterministic": True})
    wl = build_workload(cfg)
    res = orc.run_oracle(cfg, wl)
    KiB, MiB = 1 << 10, 1 << 20
    w0 = [256 * KiB, 512 * KiB, 1 * MiB, 2 * MiB, 4 * MiB, 8 * MiB, 256 * KiB]
    # TB > 0: request 0 alone (64 KiB), the ramp from request 1: 256K .. 8M, then the rest
    wk = [256 * KiB, 512 * KiB, 1 * MiB, 2 * MiB, 4 * MiB, 8 * MiB, 192 * KiB]
    for tb in range(4):
        got = res.windows[res.windows[:, 0] == tb, 1].tolist()
        assert got == (w0 if tb == 0 else wk), (tb, got)
    assert res.stats["pcie_bytes"] == 64 << 20
    assert res.stats["pb_discarded_bytes"] == 0
