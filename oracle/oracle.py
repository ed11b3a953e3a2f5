"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loaded only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs, as the checker — never by the product package
(paper_2109_05366_b200 has no import of this module; tests assert that).

``run_oracle(cfg, workload, ...)`` executes gfs_oracle.c's restatement of the
reference gread path (see that file's header for the file:line map) and
returns counters named like gpuiosim.metrics.Metrics, the delivery / RPC /
victim logs, and — when a data source is attached — the user buffer and its
checksum.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libgfs_oracle.so")

SRC_NONE, SRC_SYNTH, SRC_FILES = 0, 1, 2
LOG_DELIVERIES, LOG_RPCS, LOG_VICTIMS, LOG_WINDOWS = 0, 1, 2, 3
READAHEAD = {"static": 0, "doubling": 1, "adaptive": 2}  # adaptive = the ondemand law


class OrcCfg(C.Structure):
    _fields_ = [
        ("page_size", C.c_int64), ("cache_bytes", C.c_int64), ("prefetch_bytes", C.c_int64),
        ("request_bytes", C.c_int64), ("staging_bytes", C.c_int64), ("ra_max_bytes", C.c_int64),
        ("ra_init_bytes", C.c_int64),
        ("policy", C.c_int32), ("resident_limit", C.c_int32), ("raw_mode", C.c_int32),
        ("readahead", C.c_int32), ("pcie_disabled", C.c_int32), ("log", C.c_int32),
        ("n_files", C.c_int32), ("n_tb", C.c_int32),
        ("ra_clamp", C.c_int32), ("reserved", C.c_int32),
        ("file_sizes", C.POINTER(C.c_int64)), ("read_only", C.POINTER(C.c_uint8)),
        ("prog_off", C.POINTER(C.c_int64)), ("segs", C.POINTER(C.c_int64)),
        ("order", C.POINTER(C.c_int32)), ("dst_off", C.POINTER(C.c_int64)),
        ("dst", C.POINTER(C.c_uint8)), ("checksum_bytes", C.c_int64),
        ("source", C.c_int32), ("io_direct", C.c_int32),
        ("paths", C.POINTER(C.c_char_p)),
    ]


_lib = None


def build() -> str:
    """Compile the oracle (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
                os.path.join(HERE, "gfs_oracle.c")):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(OrcCfg)]
        L.orc_execute.argtypes = [C.c_void_p]
        L.orc_error.restype = C.c_char_p
        L.orc_error.argtypes = [C.c_void_p]
        L.orc_stats_copy.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_log_len.restype = C.c_int64
        L.orc_log_len.argtypes = [C.c_void_p, C.c_int]
        L.orc_log_copy.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64)]
        L.orc_result_checksum.restype = C.c_uint64
        L.orc_result_checksum.argtypes = [C.c_void_p]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_stat_name.restype = C.c_char_p
        L.orc_word.restype = C.c_uint64
        L.orc_word.argtypes = [C.c_int64, C.c_int64]
        L.orc_page_tag.restype = C.c_uint64
        L.orc_page_tag.argtypes = [C.c_int64, C.c_int64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_checksum.restype = C.c_uint64
        L.orc_checksum.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.orc_gen_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        L.orc_gen_file_range.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        L.orc_gen_file_range.restype = C.c_int
        _lib = L
    return _lib


def stat_names() -> list[str]:
    L = lib()
    return [L.orc_stat_name(i).decode() for i in range(L.orc_nstats())]


class OracleError(Exception):
    pass


@dataclass
class OracleResult:
    stats: dict
    deliveries: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int64))
    rpcs: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int64))
    victims: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int64))
    windows: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int64))
    dst: np.ndarray | None = None
    checksum: int | None = None


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def run_oracle(cfg, workload, *, source: int = SRC_NONE, paths=None, io_direct: bool = False,
               materialize_dst: bool = False, log: bool = True, order=None) -> OracleResult:
    """Run the restatement for `cfg` (paper_2109_05366_b200.config.ExperimentConfig)
    over `workload` (WorkloadSpec)."""
    from paper_2109_05366_b200.workloads import ProgramTable, dispatch_order
    table = ProgramTable.from_programs(workload.programs)
    n_files = len(workload.files)
    if order is None:
        order = dispatch_order(table.n_tb, cfg["gpu.dispatch_order"], cfg["seed"])
    params = {"page_size": cfg["gpufs.page_size"], "cache_bytes": cfg["gpufs.cache_bytes"],
              "prefetch_bytes": cfg["gpufs.prefetch_bytes"], "request_bytes": workload.request_bytes,
              "staging_bytes": cfg["rpc.staging_bytes"], "ra_max_bytes": cfg.ra_max(),
              "ra_init_bytes": cfg.ra_init(), "policy": cfg["gpufs.policy"],
              "resident_limit": cfg.resident_limit(), "raw_mode": bool(cfg["mode.gpu_cache_disabled"]),
              "readahead": cfg["io.readahead"], "ra_clamp": cfg["io.ra_clamp"],
              "pcie_disabled": bool(cfg["mode.pcie_disabled"])}
    return run_raw(params, [workload.files[f] for f in range(n_files)],
                   [workload.read_only[f] for f in range(n_files)], table.segs, table.prog_off,
                   table.dst_off, order, source=source, paths=paths, io_direct=io_direct,
                   materialize_dst=materialize_dst, log=log)


def programs_to_arrays(programs):
    """Per-TB programs [(file, offset, length), ...] -> (segs [n, 3], prog_off, dst_off, dst_bytes):
    the flat layout every runner takes (TB t's bytes land at dst_off[t] in program order)."""
    segs = np.asarray([s for prog in programs for s in prog], dtype=np.int64).reshape(-1, 3)
    prog_off = np.zeros(len(programs) + 1, dtype=np.int64)
    prog_off[1:] = np.cumsum([len(p) for p in programs])
    lens = np.asarray([sum(ln for _, _, ln in p) for p in programs], dtype=np.int64)
    dst_off = np.zeros(len(programs), dtype=np.int64)
    if len(programs) > 1:
        dst_off[1:] = np.cumsum(lens)[:-1]
    return segs, prog_off, dst_off, int(lens.sum())


def run_raw(params: dict, file_sizes, read_only, segs, prog_off, dst_off, order, *,
            source: int = SRC_NONE, paths=None, io_direct: bool = False,
            materialize_dst: bool = False, log: bool = True) -> OracleResult:
    """The restatement over plain arrays (no import of the product package): params holds
    page_size, cache_bytes, prefetch_bytes, request_bytes, staging_bytes, ra_max_bytes,
    ra_init_bytes, policy (name), resident_limit, raw_mode, readahead (name), ra_clamp
    (name), pcie_disabled."""
    L = lib()
    n_files = len(file_sizes)
    sizes = np.asarray(file_sizes, dtype=np.int64)
    ro = np.asarray([1 if r else 0 for r in read_only], dtype=np.uint8)
    order = np.ascontiguousarray(order, dtype=np.int32)
    segs = np.ascontiguousarray(np.asarray(segs, dtype=np.int64).reshape(-1))
    if segs.size == 0:
        segs = np.zeros(3, np.int64)
    prog_off = np.ascontiguousarray(prog_off, dtype=np.int64)
    dst_off = np.ascontiguousarray(dst_off, dtype=np.int64)
    n_tb = len(prog_off) - 1
    dst_bytes = 0
    for t in range(n_tb):
        a, b = int(prog_off[t]), int(prog_off[t + 1])
        dst_bytes = max(dst_bytes, int(dst_off[t]) + int(segs.reshape(-1, 3)[a:b, 2].sum()) if b > a else 0)
    dst = np.zeros(max(dst_bytes, 1), dtype=np.uint8) if materialize_dst else None
    c = OrcCfg()
    c.page_size = params["page_size"]
    c.cache_bytes = params["cache_bytes"]
    c.prefetch_bytes = params["prefetch_bytes"]
    c.request_bytes = params["request_bytes"]
    c.staging_bytes = params["staging_bytes"]
    c.ra_max_bytes = params["ra_max_bytes"]
    c.ra_init_bytes = params.get("ra_init_bytes", 0)
    c.policy = 1 if params["policy"] == "per-tb-lra" else 0
    c.resident_limit = params["resident_limit"]
    c.raw_mode = int(bool(params.get("raw_mode", False)))
    c.readahead = READAHEAD[params["readahead"]]
    c.ra_clamp = 1 if params.get("ra_clamp", "segment") == "eof" else 0
    c.pcie_disabled = int(bool(params.get("pcie_disabled", False)))
    c.log = int(log)
    c.n_files = n_files
    c.n_tb = n_tb
    c.file_sizes = _ptr(sizes, C.c_int64)
    c.read_only = _ptr(ro, C.c_uint8)
    c.prog_off = _ptr(prog_off, C.c_int64)
    c.segs = _ptr(segs, C.c_int64)
    c.order = _ptr(order, C.c_int32)
    c.dst_off = _ptr(dst_off, C.c_int64)
    c.dst = _ptr(dst, C.c_uint8) if dst is not None else None
    c.checksum_bytes = dst_bytes if dst is not None else 0
    c.source = source
    c.io_direct = int(io_direct)
    path_arr = None
    if source == SRC_FILES:
        path_arr = (C.c_char_p * n_files)(*[os.fsencode(p) for p in paths])
        c.paths = C.cast(path_arr, C.POINTER(C.c_char_p))
    h = L.orc_create(C.byref(c))
    if not h:
        raise OracleError("orc_create failed")
    try:
        if L.orc_execute(h) != 0:
            raise OracleError(L.orc_error(h).decode())
        names = stat_names()
        buf = (C.c_int64 * len(names))()
        L.orc_stats_copy(h, buf)
        res = OracleResult(stats=dict(zip(names, list(buf))))
        for kind, width, attr in ((LOG_DELIVERIES, 3, "deliveries"), (LOG_RPCS, 4, "rpcs"),
                                  (LOG_VICTIMS, 3, "victims"), (LOG_WINDOWS, 2, "windows")):
            n = L.orc_log_len(h, kind)
            arr = np.zeros((n, width), dtype=np.int64)
            if n:
                L.orc_log_copy(h, kind, _ptr(arr, C.c_int64))
            setattr(res, attr, arr)
        if dst is not None:
            res.dst = dst[:dst_bytes]
            res.checksum = int(L.orc_result_checksum(h))
        return res
    finally:
        L.orc_destroy(h)


SYNTH_STAMP = "W1"  # the content law's version tag, as stamped next to synthetic files


def gen_file(path: str, content_id: int, size: int, threads: int = 0) -> None:
    """Write a synthetic W(content_id, i) file with the oracle's generator (no product
    library): `threads` writers over disjoint ranges, then the version stamp."""
    import threading
    L = lib()
    threads = threads or os.cpu_count() or 1
    with open(path, "wb") as fh:
        fh.truncate(size)
    step = ((size + threads - 1) // threads + 7) // 8 * 8
    errs = []

    def one(k):
        lo = k * step
        n = min(step, size - lo)
        if n > 0 and L.orc_gen_file_range(os.fsencode(path), content_id, size, lo, n) != 0:
            errs.append(k)
    ths = [threading.Thread(target=one, args=(k,)) for k in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise OracleError(f"orc_gen_file_range failed for {path}")
    with open(path + ".ok", "w") as fh:
        fh.write(SYNTH_STAMP)
