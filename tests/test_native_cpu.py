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
    assert lib.gfs_abi_version() == native.ABI_VERSION


def test_user_kernel_library_links_against_libgfs(lib):
    """The example user kernel (csrc/user_gemv.cu over include/gfs_device.cuh) is built like
    an application: its own .so, resolving gfs_run_kernel from libgfs.so."""
    U = native.load_user()
    assert hasattr(U, "gfs_example_gemv")
    import subprocess
    out = subprocess.run(["nm", "-D", "--undefined-only", native.USER_LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "gfs_run_kernel" in out


def test_stat_names_match_oracle_counters(lib):
    import oracle as orc
    names = native.stat_names()
    for k in orc.stat_names():
        assert k in names
    for k in ("kernel_ns", "wall_ns", "ctas", "word_mismatches"):
        assert k in names


def test_struct_layouts_match_header(lib, tmp_path):
    """The ctypes mirrors have the C structs' sizes and field offsets (compiled from
    include/gfs.h with the host compiler)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no host C compiler")
    checks = {"gfs_config": native.GfsConfig, "gfs_program": native.GfsProgram,
              "gfs_consumer": native.GfsConsumer, "gfs_launch": native.GfsLaunch,
              "gfs_mapping_check": native.GfsMappingCheck}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gfs.h"', "int main(void) {"]
    for cname, py in checks.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _t in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                  check=True).stdout.splitlines())
    for cname, py in checks.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _t in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


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


def test_auto_transfer_and_first_window_rules(monkeypatch, tmp_path):
    """auto: tmpfs + adaptive -> mapped_hybrid, + doubling -> mapped_dma, + static -> mapped, disk -> bounce,
    never a copy-engine mode under a kernel profiler; the first copy-engine window is the
    whole cap when TBs outnumber resident slots, the largest power of two below a stride otherwise."""
    from paper_2109_05366_b200 import config as gcfg
    monkeypatch.delenv("GFS_PROFILER", raising=False)
    for k in [k for k in os.environ if "INJECTION" in k]:
        monkeypatch.delenv(k, raising=False)
    KiB, MiB = 1 << 10, 1 << 20
    base = {"workload.kind": "strided", "workload.n_tb": 1024, "workload.file_bytes": 16 << 30,
            "gpu.sm_count": 148, "gpu.threads_per_tb": 512, "gpufs.prefetch_bytes": 60 * KiB}
    monkeypatch.setattr(gcfg, "on_tmpfs", lambda p: True)
    c = ExperimentConfig({**base, "io.readahead": "adaptive"})
    assert c.transfer() == "mapped_hybrid" and c.ra_max() == 16 * MiB
    assert c.ra_init() == 0  # the ondemand law has no first-window knob (4 requests, host_os.py:139)
    d = ExperimentConfig({**base, "io.readahead": "doubling"})
    assert d.transfer() == "mapped_dma" and d.ra_init() == d.ra_max() == 16 * MiB
    assert ExperimentConfig({**base, "io.readahead": "static"}).transfer() == "mapped"
    few = ExperimentConfig({**base, "io.readahead": "doubling", "workload.n_tb": 128,
                            "workload.total_bytes": 949485568})
    assert few.ra_init() == 4 * MiB  # largest power of two below a 7.4 MB stride
    four = ExperimentConfig({**base, "io.readahead": "doubling", "workload.n_tb": 256,
                             "workload.file_bytes": 1 << 30})
    assert four.ra_init() == 2 * MiB  # a 4 MiB stride still gets two windows
    assert ExperimentConfig({**base, "io.readahead": "doubling", "io.ra_init_bytes": 64 * KiB}).ra_init() == 64 * KiB
    monkeypatch.setenv("GFS_PROFILER", "1")
    assert ExperimentConfig({**base, "io.readahead": "adaptive"}).transfer() == "mapped"
    monkeypatch.delenv("GFS_PROFILER")
    monkeypatch.setattr(gcfg, "on_tmpfs", lambda p: False)
    assert ExperimentConfig({**base, "io.readahead": "adaptive"}).transfer() == "bounce"


def test_io_workers_split_across_local_ranks(monkeypatch):
    cores = len(os.sched_getaffinity(0))
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    one = ExperimentConfig().io_workers()
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    eight = ExperimentConfig().io_workers()
    assert one == max(4, cores) and eight == max(1, cores // 8)
    assert 8 * eight <= max(8, cores)  # the ranks' daemons together never oversubscribe the host
    assert ExperimentConfig({"io.workers": 3}).io_workers() == 3


def test_gen_file_range_composes_the_whole_file(lib, tmp_path):
    size = (1 << 20) + 808
    a, b = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    native.gen_file(a, 4, size)
    native.gen_file_range(b, 4, size, 520, size - 520, threads=3)  # tail first, then the head
    native.gen_file_range(b, 4, size, 0, 520, threads=1)
    assert open(a, "rb").read() == open(b, "rb").read() == grng.content(4, 0, size)
    with pytest.raises(GfsError):
        native.gen_file_range(b, 4, size, 3, 8)  # offsets are word aligned
