"""ctypes binding of libgfs.so (include/gfs.h).

There is no fallback: if the library is missing or a call fails, a GfsError is
raised.  The binding releases the GIL for every call (ctypes does), so the host
I/O daemon threads inside libgfs and Python threads run concurrently.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import GfsError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "libgfs.so")

POLICY = {"global-lru-dealloc": 0, "per-tb-lra": 1}
READAHEAD = {"static": 0, "doubling": 1, "adaptive": 2}  # adaptive = ondemand law
RA_CLAMP = {"segment": 0, "eof": 1}
TRANSFER = {"zerocopy": 0, "dma": 1, "bounce": 2, "mapped_dma": 3, "mapped": 4,
            "mapped_hybrid": 5, "pread_hybrid": 6}
O_RDONLY, O_RDWR = 0, 2
ABI_VERSION = 9  # include/gfs.h GFS_ABI_VERSION: the struct layouts below
LOG_DELIVERIES, LOG_RPCS, LOG_VICTIMS, LOG_WINDOWS, LOG_TIMELINE = 0, 1, 2, 3, 4
LOG_WIDTH = {LOG_DELIVERIES: 3, LOG_RPCS: 4, LOG_VICTIMS: 3, LOG_WINDOWS: 2, LOG_TIMELINE: 4}
TL_RPC, TL_GREAD, TL_CONSUME = 0, 1, 2

# Every entry point declared in include/gfs.h (tests check the library exports them).
EXPORTS = ["gfs_create", "gfs_destroy", "gfs_gopen", "gfs_gclose", "gfs_file_size", "gfs_run",
           "gfs_run_consume",
           "gfs_log_len", "gfs_log_copy", "gfs_checksum", "gfs_verify_dst", "gfs_gen_file",
           "gfs_last_error", "gfs_abi_version", "gfs_stat_count", "gfs_stat_name",
           "gfs_resident_ctas", "gfs_bench_storage", "gfs_bench_h2d", "gfs_bench_read_memcpy",
           "gfs_replay", "gfs_gen_file_range", "gfs_transfer", "gfs_run_kernel",
           "gfs_check_mapping"]
USER_LIB_PATH = os.path.join(PKG, "_lib", "libgfs_user.so")  # example user kernel (csrc/user_gemv.cu)


class GfsConfig(C.Structure):
    _fields_ = [
        ("page_size", C.c_int64), ("cache_bytes", C.c_int64), ("prefetch_bytes", C.c_int64),
        ("staging_bytes", C.c_int64), ("ra_max_bytes", C.c_int64), ("ra_init_bytes", C.c_int64),
        ("max_request_bytes", C.c_int64),
        ("policy", C.c_int32), ("resident_limit", C.c_int32), ("readahead", C.c_int32),
        ("transfer", C.c_int32), ("io_workers", C.c_int32), ("io_direct", C.c_int32),
        ("device", C.c_int32), ("cta_threads", C.c_int32), ("max_ctas", C.c_int32),
        ("raw_mode", C.c_int32), ("pcie_disabled", C.c_int32), ("log", C.c_int32),
        ("verify", C.c_int32), ("timeline", C.c_int32), ("k1_tma", C.c_int32),
        ("numa_pin", C.c_int32), ("lookahead", C.c_int32), ("ra_clamp", C.c_int32),
        ("rpc_slots", C.c_int32), ("k1_direct", C.c_int32), ("k1_early", C.c_int32),
    ]


CONSUME = {"none": 0, "sum64": 1, "gemv_f32": 2, "nn_f32": 3, "gemvt_f32": 4, "bicg_f32": 5,
           "kmeans_f32": 6}
KMEANS_MAX_K = 16


class GfsConsumer(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("k", C.c_int32), ("cols", C.c_int64),
        ("x", C.c_void_p), ("y", C.c_void_p), ("qx", C.c_float), ("qy", C.c_float),
        ("out", C.c_void_p), ("x2", C.c_void_p), ("y2", C.c_void_p),
    ]


class GfsProgram(C.Structure):
    _fields_ = [
        ("n_tb", C.c_int32), ("reserved", C.c_int32), ("request_bytes", C.c_int64),
        ("segs", C.POINTER(C.c_int64)), ("prog_off", C.POINTER(C.c_int64)),
        ("dst_off", C.POINTER(C.c_int64)), ("order", C.POINTER(C.c_int32)),
    ]


class GfsMappingCheck(C.Structure):
    _fields_ = [("mapped_pages", C.c_int64), ("duplicate_frames", C.c_int64),
                ("key_mismatches", C.c_int64), ("unsettled", C.c_int64), ("lost_frames", C.c_int64)]


class GfsLaunch(C.Structure):
    """gfs_launch: what gfs_run_kernel hands a user kernel's launch callback."""
    _fields_ = [
        ("dev", C.c_void_p), ("dev_bytes", C.c_int64), ("n_ctas", C.c_int32),
        ("cta_threads", C.c_int32), ("smem_bytes", C.c_int64), ("stream", C.c_void_p),
        ("n_tb", C.c_int32), ("reserved", C.c_int32),
    ]


_lib = None
_nstats = None


def load(path: str = LIB_PATH):
    """Load libgfs.so (raises GfsError when it is absent: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GfsError(f"{path} is not built; run `python -m paper_2109_05366_b200.build` "
                       "(the B200 path has no CPU fallback)")
    L = C.CDLL(path)
    vp, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
    L.gfs_create.argtypes = [C.POINTER(GfsConfig), C.POINTER(vp)]
    L.gfs_destroy.argtypes = [vp]
    L.gfs_destroy.restype = None
    L.gfs_gopen.argtypes = [vp, C.c_char_p, i32, i64, C.POINTER(i32)]
    L.gfs_gclose.argtypes = [vp, i32]
    L.gfs_file_size.argtypes = [vp, i32, C.POINTER(i64)]
    L.gfs_run.argtypes = [vp, C.POINTER(GfsProgram), vp, u64, vp]
    L.gfs_run_consume.argtypes = [vp, C.POINTER(GfsProgram), vp, u64, C.POINTER(GfsConsumer), vp]
    L.gfs_run_consume.restype = i32
    L.gfs_log_len.argtypes = [vp, i32, C.POINTER(i64)]
    L.gfs_log_copy.argtypes = [vp, i32, C.POINTER(i64), i64]
    L.gfs_checksum.argtypes = [vp, vp, u64, u64, C.POINTER(u64)]
    L.gfs_verify_dst.argtypes = [vp, C.POINTER(GfsProgram), vp, u64, C.POINTER(i64)]
    L.gfs_gen_file.argtypes = [C.c_char_p, i64, i64, i32]
    L.gfs_gen_file_range.argtypes = [C.c_char_p, i64, i64, i64, i64, i32]
    L.gfs_last_error.restype = C.c_char_p
    L.gfs_stat_name.restype = C.c_char_p
    L.gfs_stat_name.argtypes = [i32]
    L.gfs_resident_ctas.argtypes = [vp]
    L.gfs_transfer.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
    L.gfs_run_kernel.argtypes = [vp, i32, C.POINTER(C.c_int32), vp, vp, vp]
    L.gfs_check_mapping.argtypes = [vp, C.POINTER(GfsMappingCheck)]
    dp = C.POINTER(C.c_double)
    L.gfs_bench_storage.argtypes = [C.c_char_p, i64, i64, i32, i64, i32, dp]
    L.gfs_bench_h2d.argtypes = [i32, i64, i32, dp]
    L.gfs_bench_read_memcpy.argtypes = [C.c_char_p, i64, i64, vp, i32, i32, i64, i32, i32, dp]
    L.gfs_replay.argtypes = [C.POINTER(C.c_char_p), i32, C.POINTER(i64), i64, i32, i32, i32,
                             C.POINTER(i64), C.POINTER(i64), dp]
    for name in ("gfs_create", "gfs_gopen", "gfs_gclose", "gfs_file_size", "gfs_run",
                 "gfs_log_len", "gfs_log_copy", "gfs_checksum", "gfs_verify_dst", "gfs_gen_file",
                 "gfs_bench_storage", "gfs_bench_h2d", "gfs_bench_read_memcpy", "gfs_replay",
                 "gfs_gen_file_range", "gfs_transfer", "gfs_run_kernel", "gfs_check_mapping"):
        getattr(L, name).restype = i32
    if L.gfs_abi_version() != ABI_VERSION:
        raise GfsError(f"{path} has ABI {L.gfs_abi_version()}, this package needs {ABI_VERSION}: rebuild it")
    _lib = L
    return L


_user = None


def load_user(path: str = USER_LIB_PATH):
    """The example user-kernel library (a GEMV written against include/gfs_device.cuh and
    driven by gfs_run_kernel, linked against libgfs.so like an application would be)."""
    global _user
    if _user is not None:
        return _user
    load()  # libgfs.so first: the user library resolves gfs_run_kernel from it
    if not os.path.exists(path):
        raise GfsError(f"{path} is not built; run `python -m paper_2109_05366_b200.build`")
    U = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
    U.gfs_example_gemv.argtypes = [vp, i32, i64, i32, i64, i64, vp, vp, vp, i32, C.POINTER(C.c_int32), vp]
    U.gfs_example_gemv.restype = i32
    _user = U
    return U


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().gfs_last_error().decode(errors="replace")
        raise GfsError(f"{what}: {msg} (code {rc})")


def stat_names() -> list[str]:
    global _nstats
    L = load()
    if _nstats is None:
        _nstats = [L.gfs_stat_name(i).decode() for i in range(L.gfs_stat_count())]
    return _nstats


def gen_file(path: str, content_id: int, size: int, threads: int | None = None) -> None:
    L = load()
    check(L.gfs_gen_file(os.fsencode(path), content_id, size, threads or os.cpu_count() or 4),
          f"gfs_gen_file({path})")


def gen_file_range(path: str, content_id: int, size: int, offset: int, length: int,
                   threads: int | None = None) -> None:
    L = load()
    check(L.gfs_gen_file_range(os.fsencode(path), content_id, size, offset, length,
                               threads or os.cpu_count() or 4), f"gfs_gen_file_range({path})")


def bench_storage(path: str, offset: int, size: int, threads: int, chunk: int, direct: bool) -> float:
    """Seconds to read [offset, offset+size) of path with `threads` parallel readers."""
    L = load()
    sec = C.c_double()
    check(L.gfs_bench_storage(os.fsencode(path), offset, size, threads, chunk, int(direct),
                              C.byref(sec)), "gfs_bench_storage")
    return sec.value


def bench_h2d(device: int, nbytes: int, reps: int = 5) -> float:
    """Best seconds of a pinned host->HBM copy of nbytes."""
    L = load()
    sec = C.c_double()
    check(L.gfs_bench_h2d(device, nbytes, reps, C.byref(sec)), "gfs_bench_h2d")
    return sec.value


def bench_read_memcpy(path: str, offset: int, size: int, dst_ptr: int, device: int, threads: int,
                      chunk: int, direct: bool, sync: bool) -> float:
    """Seconds for the CPU read()+cudaMemcpy baseline over [offset, offset+size)."""
    L = load()
    sec = C.c_double()
    check(L.gfs_bench_read_memcpy(os.fsencode(path), offset, size, dst_ptr, device, threads, chunk,
                                  int(direct), int(sync), C.byref(sec)), "gfs_bench_read_memcpy")
    return sec.value


def replay(paths: list[str], records, n_slots: int, n_workers: int, direct: bool = True):
    """Host-only replay of a recorded RPC trace (include/gfs.h gfs_replay); records is an
    int64 [n, 4] array of (tb, file, offset, size).  Returns (user_bytes, preads, seconds)."""
    import numpy as np
    L = load()
    recs = np.ascontiguousarray(records, dtype=np.int64).reshape(-1, 4)
    arr = (C.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
    ub, npr, sec = C.c_int64(), C.c_int64(), C.c_double()
    check(L.gfs_replay(arr, len(paths), recs.ctypes.data_as(C.POINTER(C.c_int64)), len(recs),
                       n_slots, n_workers, int(direct), C.byref(ub), C.byref(npr), C.byref(sec)),
          "gfs_replay")
    return ub.value, npr.value, sec.value
