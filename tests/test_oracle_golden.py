"""Pin the CPU oracle against the reference's own outputs and known answers.

The golden fixtures were produced by running the reference simulator
(tests/golden/make_golden.py); the closed-form values below are the
reference tests' known answers (file:line cited per test).
"""

import numpy as np
import pytest

import golden_util as gu
import oracle as orc
from paper_2109_05366_b200 import rng as grng
from paper_2109_05366_b200.workloads import build_workload


@pytest.mark.parametrize("name", gu.case_names())
def test_oracle_matches_reference_golden(name):
    g = gu.load(name)
    cfg = gu.config_of(g, seed=g["seed"])
    wl = build_workload(cfg)
    res = orc.run_oracle(cfg, wl)
    errs = gu.compare(g, res.stats, res.deliveries, res.rpcs, res.victims)
    assert not errs, f"{name}: " + "; ".join(errs)
    assert wl.total_bytes == g["total_bytes"] and wl.unique_bytes == g["unique_bytes"]


def test_splitmix_known_vectors():
    # reference tests/test_simcore.py:70-75
    r = grng.SeededRng(0)
    assert [r.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                0x06C45D188009454F]
    L = orc.lib()
    assert L.orc_mix64(0) == 0xE220A8397B1DCDAF


def test_page_tag_matches_python_and_unique():
    # reference tests/test_simcore.py:135-146: tags unique over an 8x512 grid
    L = orc.lib()
    tags = {L.orc_page_tag(f, p) for f in range(8) for p in range(512)}
    assert len(tags) == 8 * 512
    assert all(L.orc_page_tag(f, p) == grng.page_tag(f, p) for f in (0, 3) for p in (0, 1, 999))


def test_word_law_c_vs_numpy():
    L = orc.lib()
    w = grng.words(3, 1000, 2000)
    assert all(int(w[k]) == L.orc_word(3, 1000 + k) for k in range(0, 2000, 97))
    buf = bytearray(777)
    import ctypes
    cbuf = (ctypes.c_uint8 * 777)()
    L.orc_gen_bytes(2, 12345, 777, cbuf)
    assert bytes(cbuf) == grng.content(2, 12345, 777)
    assert len(buf) == 777


def test_checksum_c_vs_numpy():
    L = orc.lib()
    data = grng.content(1, 0, 100_003)
    arr = np.frombuffer(data, dtype=np.uint8).copy()
    assert L.orc_checksum(arr.ctypes.data, len(arr), 0) == grng.checksum(data)
    # position sensitivity: swapping two pages changes the checksum
    sw = bytearray(data)
    sw[0:4096], sw[4096:8192] = data[4096:8192], data[0:4096]
    assert grng.checksum(bytes(sw)) != grng.checksum(data)


def test_rpc_law_criterion_6():
    # reference tests/test_acceptance.py:163-176
    g = gu.load("micro_pf60")
    assert g["counters"]["rpc_count"] == 120 * -(-819200 // (64 * 1024)) == 1560
    assert g["counters"]["pb_hits"] == 22440


def test_tiny_oracle_criterion_8_shapes():
    # reference tests/test_acceptance.py:244-266: 32 deliveries, 8 RPCs, 24 victims
    for name in ("tiny_global", "tiny_lra"):
        g = gu.load(name)
        cfg = gu.config_of(g, seed=1)
        res = orc.run_oracle(cfg, build_workload(cfg))
        assert len(res.deliveries) == 32 and len(res.rpcs) == 8 and len(res.victims) == 24


def test_gread_counts():
    # reference tests/test_gpu_exec.py:89-100
    from paper_2109_05366_b200.config import ExperimentConfig
    for fb, greads in ((8 * 1024 ** 2, 128), (98_304, 2)):
        cfg = ExperimentConfig({"workload.n_tb": 1, "workload.file_bytes": fb})
        res = orc.run_oracle(cfg, build_workload(cfg))
        assert res.stats["greads"] == greads and res.stats["user_bytes"] == fb


def test_materialized_synth_delivers_file_bytes():
    from paper_2109_05366_b200.config import ExperimentConfig
    cfg = ExperimentConfig({"workload.n_tb": 4, "workload.file_bytes": 1_000_000,
                            "workload.n_files": 2, "workload.request_bytes": 10_000,
                            "gpufs.prefetch_bytes": 12 * 1024, "gpufs.cache_bytes": 32 * 4096,
                            "gpu.sm_count": 1, "gpu.threads_per_tb": 2048,
                            "gpufs.policy": "per-tb-lra"})
    wl = build_workload(cfg)
    res = orc.run_oracle(cfg, wl, source=orc.SRC_SYNTH, materialize_dst=True)
    want = grng.content(0, 0, 1_000_000) + grng.content(1, 0, 1_000_000)
    assert res.dst.tobytes() == want
    assert res.checksum == grng.checksum(want)


def test_materialized_files_odirect(tmp_path):
    from paper_2109_05366_b200.config import ExperimentConfig
    size = 3 * 1024 * 1024 + 12_345
    path = tmp_path / "f0.bin"
    path.write_bytes(grng.content(0, 0, size))
    cfg = ExperimentConfig({"workload.n_tb": 3, "workload.file_bytes": size - size % 3,
                            "workload.total_bytes": size - size % 3,
                            "gpufs.prefetch_bytes": 60 * 1024, "gpufs.cache_bytes": 1 << 20})
    wl = build_workload(cfg)
    wl = wl.__class__(wl.name, {0: size}, wl.read_only, wl.programs, wl.request_bytes,
                      wl.total_bytes, wl.unique_bytes)
    for direct in (False, True):
        try:
            res = orc.run_oracle(cfg, wl, source=orc.SRC_FILES, paths=[str(path)],
                                 io_direct=direct, materialize_dst=True)
        except orc.OracleError as e:
            if direct and "Invalid argument" in str(e):
                pytest.skip("filesystem without O_DIRECT")
            raise
        assert res.dst.tobytes() == grng.content(0, 0, wl.total_bytes)


def test_oracle_file_generator_matches_product(tmp_path):
    """The reference arm writes its input with the oracle's generator (no product library);
    the bytes and the version stamp equal the product's synthetic file."""
    from paper_2109_05366_b200 import native
    from paper_2109_05366_b200.runtime import SYNTH_VERSION
    size = 3 * 1048576 + 12344
    a, b = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    orc.gen_file(a, 2, size, threads=3)
    native.gen_file(b, 2, size)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert open(a + ".ok").read().strip() == SYNTH_VERSION == orc.SYNTH_STAMP
