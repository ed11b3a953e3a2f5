"""CPU-side checks of the C ABI: the library loads without a GPU, exports every entry
point include/gfs.h declares, its host-only pieces work, and device calls fail loudly
(no CPU fallback exists)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2109_05366_b200 import build as gbuild
from paper_2109_05366_b200 import native
from paper_2109_05366_b200 import rng as grng
from paper_2109_05366_b200.config import ExperimentConfig
from paper_2109_05366_b200.errors import GfsError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    gbuild.build()
    return native.load()


def header_functions():
    text = open(os.path.join(ROOT, "include", "gfs.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+\**(gfs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_expected_entry_points():
    assert header_functions() == sorted(native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.gfs_abi_version() == 1


def test_stat_names_match_oracle_counters(lib):
    import oracle as orc
    names = native.stat_names()
    for k in orc.stat_names():
        assert k in names
    for k in ("kernel_ns", "wall_ns", "ctas", "word_mismatches"):
        assert k in names


def test_struct_sizes_match_header(lib):
    # gfs_config: 7 int64 + 13 int32 + 3 reserved int32 = 56 + 64 = 120 bytes
    assert C.sizeof(native.GfsConfig) == 120
    assert C.sizeof(native.GfsProgram) == 48


def test_gen_file_matches_content_law(lib, tmp_path):
    path = str(tmp_path / "synth.bin")
    size = 5 * 1024 * 1024 + 123
    native.gen_file(path, 7, size, threads=4)
    data = open(path, "rb").read()
    assert len(data) == size
    assert data == grng.content(7, 0, size)


def test_gen_file_rejects_bad_arguments(lib, tmp_path):
    with pytest.raises(GfsError):
        native.gen_file(str(tmp_path / "x.bin"), -1, 10)
    with pytest.raises(GfsError):
        native.gen_file("/nonexistent-dir/x.bin", 0, 10)


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2109_05366_b200.runtime import GpuFS
    with pytest.raises(GfsError):
        GpuFS(ExperimentConfig({"gpufs.cache_bytes": 1 << 20}))


def test_config_validation_mirrors_reference(lib):
    from paper_2109_05366_b200.runtime import native_config
    cfg = ExperimentConfig({"gpufs.policy": "per-tb-lra", "gpu.sm_count": 148,
                            "gpu.threads_per_tb": 512})
    c = native_config(cfg)
    assert c.resident_limit == 592 and c.policy == 1
    with pytest.raises(GfsError):
        ExperimentConfig({"gpufs.prefetch_bytes": 1000})
    with pytest.raises(GfsError):
        ExperimentConfig({"io.transfer": "carrier-pigeon"})
    with pytest.raises(GfsError):
        ExperimentConfig({"no.such": 1})


def test_checksum_law_python_vs_oracle():
    import oracle as orc
    L = orc.lib()
    buf = np.frombuffer(grng.content(0, 4096, 65536), dtype=np.uint8).copy()
    assert L.orc_checksum(buf.ctypes.data, len(buf), 3) == grng.checksum(buf, 3)
