"""Python front end of the B200 file layer: gopen / gread / gclose and the drop-in
``Simulation(cfg, seed).run()``.

``GpuFS`` owns one libgfs context (one GPU, its HBM page cache, its pinned RPC ring
and its I/O daemon threads).  ``Simulation`` mirrors the reference's outer API
(gpuiosim/simulation.py:98-242): same constructor, ``run()`` returns a
``MetricsReport`` with the reference's CSV columns, and after the run the object
exposes ``metrics`` (counters, and ``deliveries`` when
``metrics.log_deliveries`` is set before ``run`` — metrics.py:44-46),
``recorded`` (the RPC trace, rpc.py:196-197) and ``cache.victim_log``
(gpu_cache.py:88), so reference-style parity checks run unchanged.

PyTorch is used only for plumbing: user buffers are ``torch.uint8`` CUDA tensors
whose ``data_ptr()`` crosses the C ABI.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import native
from .config import ExperimentConfig
from .errors import GfsError
from .metrics import Metrics, MetricsReport, build_report
from .rng import SeededRng
from .workloads import (ProgramTable, TraceRecord, WorkloadSpec, build_workload,
                        dispatch_order, load_trace, save_trace, trace_workload)

O_RDONLY, O_RDWR = native.O_RDONLY, native.O_RDWR


def native_config(cfg: ExperimentConfig, max_request_bytes: int = 0) -> native.GfsConfig:
    c = native.GfsConfig()
    if cfg["gpufs.policy"] not in native.POLICY:
        raise GfsError(f"unknown gpufs.policy {cfg['gpufs.policy']!r}")
    c.page_size = cfg["gpufs.page_size"]
    c.cache_bytes = cfg["gpufs.cache_bytes"]
    c.prefetch_bytes = cfg["gpufs.prefetch_bytes"]
    c.staging_bytes = cfg["rpc.staging_bytes"]
    c.ra_max_bytes = cfg.ra_max()
    c.ra_init_bytes = cfg.ra_init()
    c.max_request_bytes = max_request_bytes or cfg["workload.request_bytes"]
    c.policy = native.POLICY[cfg["gpufs.policy"]]
    c.resident_limit = cfg.resident_limit()
    c.readahead = native.READAHEAD[cfg["io.readahead"]]
    c.transfer = native.TRANSFER[cfg.transfer()]
    c.io_workers = cfg.io_workers()
    c.io_direct = int(bool(cfg["io.direct"]))
    c.device = cfg["gpu.device"]
    c.cta_threads = cfg["gpu.cta_threads"]
    c.max_ctas = 0
    c.raw_mode = int(bool(cfg["mode.gpu_cache_disabled"]))
    c.pcie_disabled = int(bool(cfg["mode.pcie_disabled"]))
    c.log = int(bool(cfg["mode.deterministic"]))
    c.verify = int(bool(cfg["mode.verify"]))
    c.timeline = int(bool(cfg["mode.timeline"]))
    if cfg["gpu.k1_copy"] not in ("tma", "ldg"):
        raise GfsError(f"gpu.k1_copy must be tma or ldg, not {cfg['gpu.k1_copy']!r}")
    c.k1_tma = int(cfg["gpu.k1_copy"] == "tma")
    c.numa_pin = int(bool(cfg["io.numa_pin"]))
    c.lookahead = int(bool(cfg["gpu.lookahead"]))
    c.ra_clamp = native.RA_CLAMP[cfg["io.ra_clamp"]]
    c.rpc_slots = cfg["rpc.n_slots"]
    c.k1_direct = int(bool(cfg["gpu.k1_direct"]))
    c.k1_early = int(bool(cfg["gpu.k1_early"]))
    return c


@dataclass
class RunResult:
    stats: dict
    deliveries: np.ndarray | None = None
    rpcs: np.ndarray | None = None
    victims: np.ndarray | None = None
    windows: np.ndarray | None = None
    timeline: np.ndarray | None = None  # [n, 4] GFS_LOG_TIMELINE records (mode.timeline)
    extra: dict = field(default_factory=dict)

    @property
    def seconds(self) -> float:
        return self.stats["kernel_ns"] / 1e9

    @property
    def gbps(self) -> float:
        ns = self.stats["kernel_ns"]
        return self.stats["user_bytes"] / ns if ns else 0.0


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


@dataclass
class Consumer:
    """A streaming consumer fused into the gread loop (include/gfs.h gfs_consumer).

    sum64:    out (uint64 CUDA tensor [1]) += sum_i mix64(w_i ^ (i * golden)) over file words
    gemv_f32: y (float32 [rows]) += A x, A = the file as a row-major [rows, cols] matrix of
              f32 = (u32 >> 8) * 2^-24 (the gesummv/mvt/bicg/atax access pattern)
    nn_f32:   out (uint64 [1]) = min over records (lat, lng) of (dist2 bits << 32 | index),
              the Rodinia nn scan
    gemvt_f32: y2 (float32 [cols]) += A^T x2 (x2 float32 [rows]); mvt's second product and
              atax's second pass
    bicg_f32: both products in one pass (bicg: q = A p, s = A^T r; mvt)
    kmeans_f32: Rodinia kmeans assignment step over points of `cols` features: x = centroids
              float32 [k, cols]; y float32 [k, cols] += features of the points nearest to each
              centroid; out uint64 [k] += their count
    """
    kind: str
    out: object = None
    x: object = None
    y: object = None
    cols: int = 0
    qx: float = 0.0
    qy: float = 0.0
    x2: object = None
    y2: object = None
    k: int = 0

    def native(self) -> "native.GfsConsumer":
        k = native.GfsConsumer()
        if self.kind not in native.CONSUME:
            raise GfsError(f"unknown consumer {self.kind!r}")
        k.kind = native.CONSUME[self.kind]
        k.cols = self.cols
        k.x = self.x.data_ptr() if self.x is not None else None
        k.y = self.y.data_ptr() if self.y is not None else None
        k.out = self.out.data_ptr() if self.out is not None else None
        k.x2 = self.x2.data_ptr() if self.x2 is not None else None
        k.y2 = self.y2.data_ptr() if self.y2 is not None else None
        k.k = self.k
        k.qx, k.qy = self.qx, self.qy
        return k


class GpuFS:
    """One GPU's file layer: HBM page cache + RPC ring + host I/O daemon."""

    # pinned page-cache transfers -> the pread daemon transfer moving the same bytes (used
    # when the file's pages cannot be pinned: not memory-resident, or not enough pinnable RAM)
    PIN_FALLBACK = {"mapped_dma": "dma", "mapped_hybrid": "bounce", "mapped": "bounce"}

    def __init__(self, cfg: ExperimentConfig, max_request_bytes: int = 0):
        self.cfg = cfg
        self._lib = native.load()
        self._max_req = max_request_bytes
        self._ncfg = native_config(cfg, max_request_bytes)
        h = C.c_void_p()
        native.check(self._lib.gfs_create(C.byref(self._ncfg), C.byref(h)), "gfs_create")
        self._h = h
        self.files: dict[int, dict] = {}
        self.fallback: str | None = None  # "<from> -> <to>: <why>" after a pin-failure fallback

    # -- lifecycle ----------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.gfs_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def resident_ctas(self) -> int:
        return self._lib.gfs_resident_ctas(self._h)

    @property
    def transfer(self) -> str:
        """The transfer in use (gfs_create may downgrade a copy-engine transfer to its SM-pull
        sibling when copy streams cannot progress beside the persistent kernel)."""
        t, was = C.c_int(), C.c_int()
        native.check(self._lib.gfs_transfer(self._h, C.byref(t), C.byref(was)), "gfs_transfer")
        return {v: k for k, v in native.TRANSFER.items()}[t.value]

    # -- files ----------------------------------------------------------------

    def gopen(self, path: str, flags: int = O_RDONLY, content_id: int = -1) -> int:
        fid = C.c_int()
        native.check(self._lib.gfs_gopen(self._h, os.fsencode(path), flags, content_id,
                                         C.byref(fid)), f"gopen({path})")
        size = C.c_int64()
        native.check(self._lib.gfs_file_size(self._h, fid.value, C.byref(size)), "gfs_file_size")
        self.files[fid.value] = {"path": path, "size": size.value,
                                 "read_only": not (flags & O_RDWR), "content_id": content_id}
        return fid.value

    def gclose(self, fid: int) -> None:
        native.check(self._lib.gfs_gclose(self._h, fid), f"gclose({fid})")
        self.files.pop(fid, None)

    # -- the hot path ---------------------------------------------------------

    def _program(self, table: ProgramTable, request_bytes: int, order: np.ndarray):
        p = native.GfsProgram()
        p.n_tb = table.n_tb
        p.request_bytes = request_bytes
        segs = np.ascontiguousarray(table.segs.reshape(-1), dtype=np.int64)
        if segs.size == 0:
            segs = np.zeros(3, np.int64)
        keep = (segs, np.ascontiguousarray(table.prog_off), np.ascontiguousarray(table.dst_off),
                np.ascontiguousarray(order, dtype=np.int32))
        p.segs = _ptr(keep[0], C.c_int64)
        p.prog_off = _ptr(keep[1], C.c_int64)
        p.dst_off = _ptr(keep[2], C.c_int64)
        p.order = _ptr(keep[3], C.c_int32)
        return p, keep

    def run(self, table: ProgramTable, request_bytes: int, dst=None, order=None,
            consumer: "Consumer | None" = None) -> RunResult:
        """All TBs' gread loops (gpu_exec.py:95-239); dst = uint8 CUDA tensor or None;
        `consumer` runs a fused streaming consumer over every delivered request."""
        if order is None:
            order = np.arange(table.n_tb, dtype=np.int32)
        prog, keep = self._program(table, request_bytes, order)
        dst_ptr, dst_bytes = None, 0
        if dst is not None:
            if not dst.is_cuda or dst.numel() * dst.element_size() < table.dst_bytes:
                raise GfsError("dst must be a CUDA tensor of at least the program's bytes")
            dst_ptr, dst_bytes = dst.data_ptr(), dst.numel() * dst.element_size()
        names = native.stat_names()
        out = (C.c_int64 * len(names))()
        cons = consumer.native() if consumer is not None else None
        rc = self._lib.gfs_run_consume(self._h, C.byref(prog), dst_ptr, dst_bytes,
                                       C.byref(cons) if cons is not None else None, out)
        if rc != 0 and self._pin_failed():
            # the mapped transfers could not pin the file's pages: same run through the
            # pread daemon (O_DIRECT pread -> pinned staging -> HBM), still on the GPU path
            self._reopen_with(self.PIN_FALLBACK[self.transfer])
            rc = self._lib.gfs_run_consume(self._h, C.byref(prog), dst_ptr, dst_bytes,
                                           C.byref(cons) if cons is not None else None, out)
        native.check(rc, "gfs_run")
        del keep
        return self._result(out, names)

    def run_user(self, entry, *args, order=None) -> RunResult:
        """A user kernel over the device-side gread (include/gfs_device.cuh): `entry` is the
        application's C entry point, called as entry(ctx, *args, order, stats_out); it ends in
        gfs_run_kernel, which prepares the run like gfs_run and launches the kernel.  Returns
        the run's counters and logs like run()."""
        names = native.stat_names()
        out = (C.c_int64 * len(names))()
        ordp = None
        if order is not None:
            order = np.ascontiguousarray(order, dtype=np.int32)
            ordp = _ptr(order, C.c_int32)
        native.check(entry(self._h, *args, ordp, out), "gfs_run_kernel")
        return self._result(out, names)

    def _result(self, out, names) -> RunResult:
        res = RunResult(stats=dict(zip(names, list(out))))
        if self._ncfg.timeline:
            res.timeline = self.log(native.LOG_TIMELINE)
        if self._ncfg.log:
            res.deliveries = self.log(native.LOG_DELIVERIES)
            res.rpcs = self.log(native.LOG_RPCS)
            res.victims = self.log(native.LOG_VICTIMS)
            res.windows = self.log(native.LOG_WINDOWS)
        return res

    def _pin_failed(self) -> bool:
        msg = self._lib.gfs_last_error().decode(errors="replace")
        return self.transfer in self.PIN_FALLBACK and "mapped transfers need" in msg

    def _reopen_with(self, transfer: str) -> None:
        why = self._lib.gfs_last_error().decode(errors="replace")
        was = self.transfer
        files = [self.files[f] for f in sorted(self.files)]
        self.close()
        self.cfg = self.cfg.copy_with({"io.transfer": transfer})
        self._ncfg = native_config(self.cfg, self._max_req)
        h = C.c_void_p()
        native.check(self._lib.gfs_create(C.byref(self._ncfg), C.byref(h)), "gfs_create")
        self._h = h
        self.files = {}
        for f in files:
            self.gopen(f["path"], O_RDONLY if f["read_only"] else O_RDWR, f["content_id"])
        self.fallback = f"{was} -> {transfer}: {why[:200]}"

    def gread(self, fid: int, offset: int, size: int, dst=None) -> RunResult:
        """One threadblock's gread of [offset, offset+size) (gpu_exec.py:107-129)."""
        table = ProgramTable.from_programs([[(fid, offset, size)]])
        return self.run(table, size, dst)

    def log(self, kind: int) -> np.ndarray:
        n = C.c_int64()
        native.check(self._lib.gfs_log_len(self._h, kind, C.byref(n)), "gfs_log_len")
        w = native.LOG_WIDTH[kind]
        arr = np.zeros((n.value, w), dtype=np.int64)
        if n.value:
            native.check(self._lib.gfs_log_copy(self._h, kind, _ptr(arr, C.c_int64), n.value),
                         "gfs_log_copy")
        return arr

    # -- consumers ----------------------------------------------------------------

    def checksum(self, buf, nbytes: int | None = None, word_base: int = 0) -> int:
        n = buf.numel() * buf.element_size() if nbytes is None else nbytes
        v = C.c_uint64()
        native.check(self._lib.gfs_checksum(self._h, buf.data_ptr(), n, word_base, C.byref(v)),
                     "gfs_checksum")
        return v.value

    def check_unique_mapping(self) -> dict:
        """GpuPageCache.check_unique_mapping (gpu_cache.py:217-224) on the device page table
        the last run left; raises GfsError on a violation, else returns the counts."""
        v = native.GfsMappingCheck()
        rc = self._lib.gfs_check_mapping(self._h, C.byref(v))
        out = {k: getattr(v, k) for k, _ in native.GfsMappingCheck._fields_}
        native.check(rc, "check_unique_mapping")
        return out

    def verify(self, table: ProgramTable, dst) -> int:
        prog, keep = self._program(table, 1, np.arange(table.n_tb, dtype=np.int32))
        v = C.c_int64()
        native.check(self._lib.gfs_verify_dst(self._h, C.byref(prog), dst.data_ptr(),
                                              dst.numel() * dst.element_size(), C.byref(v)),
                     "gfs_verify_dst")
        del keep
        return v.value


# ----------------------------------------------------------------- synthetic files

SYNTH_VERSION = "W1"  # content law W(f, i) = mix64(page_tag(f, i >> 9) ^ i)


def synth_dir(cfg: ExperimentConfig) -> str:
    if cfg["io.dir"]:
        return cfg["io.dir"]
    return "/dev/shm" if cfg["mode.ramfs"] else "/tmp"


def ensure_synthetic(directory: str, content_id: int, size: int) -> str:
    """Path of synthetic file `content_id` of `size` bytes, generating it if needed."""
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, f"gfs_synth_c{content_id}_{size}.bin")
    stamp = path + ".ok"
    if os.path.exists(path) and os.path.exists(stamp) and os.path.getsize(path) == size:
        with open(stamp) as fh:
            if fh.read().strip() == SYNTH_VERSION:
                return path
    native.gen_file(path, content_id, size)
    with open(stamp, "w") as fh:
        fh.write(SYNTH_VERSION)
    return path


def synthetic_path(directory: str, content_id: int, size: int) -> str:
    return os.path.join(directory, f"gfs_synth_c{content_id}_{size}.bin")


def synthetic_ready(path: str, size: int) -> bool:
    stamp = path + ".ok"
    if not (os.path.exists(path) and os.path.exists(stamp) and os.path.getsize(path) == size):
        return False
    with open(stamp) as fh:
        return fh.read().strip() == SYNTH_VERSION


def gpu_local_cpus(device: int) -> list[int]:
    """Host CPUs on the GPU's PCIe root (sysfs local_cpulist) that this process may use;
    all usable CPUs when that is unknown."""
    allowed = sorted(os.sched_getaffinity(0))
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/local_cpulist") as fh:
            text = fh.read().strip()
    except Exception:
        return allowed
    cpus = set()
    for part in text.split(","):
        a, _, b = part.partition("-")
        if a.strip():
            cpus.update(range(int(a), int(b or a) + 1))
    local = [c for c in allowed if c in cpus]
    return local or allowed


def ensure_synthetic_shard(directory: str, content_id: int, size: int, rank: int, world: int,
                           barrier, device: int | None = None) -> str:
    """Sharded runs: every rank writes its own contiguous 1/world of the file from the CPUs
    local to its GPU, so tmpfs places each shard's pages on the NUMA node that DMAs them
    (first touch).  `barrier` synchronises the ranks."""
    os.makedirs(directory, exist_ok=True)
    path = synthetic_path(directory, content_id, size)
    ready = synthetic_ready(path, size)
    barrier()
    if ready:
        return path
    if rank == 0:
        for p in (path + ".ok", path):
            if os.path.exists(p):
                os.remove(p)
        with open(path, "wb") as fh:
            fh.truncate(size)
    barrier()
    shard = size // world // 8 * 8
    lo = rank * shard
    hi = size if rank == world - 1 else lo + shard
    old = os.sched_getaffinity(0)
    cpus = gpu_local_cpus(device) if device is not None else sorted(old)
    try:
        os.sched_setaffinity(0, cpus)
        native.gen_file_range(path, content_id, size, lo, hi - lo, threads=len(cpus))
    finally:
        os.sched_setaffinity(0, old)
    barrier()
    if rank == 0:
        with open(path + ".ok", "w") as fh:
            fh.write(SYNTH_VERSION)
    barrier()
    return path


def open_workload_files(fs: GpuFS, cfg: ExperimentConfig, workload: WorkloadSpec) -> list[int]:
    """gopen every workload file: real paths from io.paths, else synthetic files."""
    paths = [p for p in cfg["io.paths"].split(",") if p] if cfg["io.paths"] else []
    fids = []
    for f in range(len(workload.files)):
        flags = O_RDONLY if workload.read_only[f] else O_RDWR
        if paths:
            fids.append(fs.gopen(paths[f], flags, -1))
        else:
            path = ensure_synthetic(synth_dir(cfg), f, workload.files[f])
            fids.append(fs.gopen(path, flags, f))
    if fids != list(range(len(fids))):
        raise GfsError("file ids must be assigned densely from 0 on a fresh GpuFS")
    return fids


# ----------------------------------------------------------------- drop-in Simulation

class _CacheView:
    def __init__(self):
        self.victim_log: list = []


class Simulation:
    """Drop-in for gpuiosim.simulation.Simulation on the B200.

    Simulation(cfg, seed, label, rep).run() -> MetricsReport.  Real files (io.paths)
    or synthetic files (io.dir) are read through the GPU page cache into a device
    user buffer; counters, logs and the verified byte checksum are kept on the object.
    """

    def __init__(self, cfg: ExperimentConfig, seed: int, label: str = "run", rep: int = 0):
        self.cfg = cfg
        self.seed = seed
        self.label = label
        self.rep = rep
        self.trace = load_trace(cfg["mode.replay_trace"]) if cfg["mode.replay_trace"] else None
        self.workload = (trace_workload(self.trace, cfg) if self.trace is not None
                         else build_workload(cfg, SeededRng(seed)))
        self.metrics = Metrics()
        self.cache = _CacheView()
        self.recorded: list | None = None
        self.result: RunResult | None = None
        self.checksum: int | None = None
        self.mismatched_words: int | None = None
        self.mapping: dict | None = None  # check_unique_mapping counts of the last run

    def run(self, keep_output: bool = False) -> MetricsReport:
        if self.trace is not None:
            return self._run_replay()
        import torch
        cfg = self.cfg
        wl = self.workload
        log = bool(cfg["mode.deterministic"] or self.metrics.log_deliveries
                   or cfg["workload.record_trace"])
        run_cfg = cfg.copy_with({"mode.deterministic": log}) if log != cfg["mode.deterministic"] else cfg
        table = ProgramTable.from_programs(wl.programs)
        order = dispatch_order(table.n_tb, cfg["gpu.dispatch_order"], self.seed)
        dev = torch.device("cuda", cfg["gpu.device"])
        with GpuFS(run_cfg, max_request_bytes=wl.request_bytes) as fs:
            open_workload_files(fs, cfg, wl)
            dst = torch.empty(max(table.dst_bytes, 1), dtype=torch.uint8, device=dev)
            res = fs.run(table, wl.request_bytes, dst, order)
            if cfg["mode.verify"] and not cfg["io.paths"]:
                self.mismatched_words = fs.verify(table, dst)
                res.stats["tag_mismatches"] += int(self.mismatched_words > 0)
            self.checksum = fs.checksum(dst, table.dst_bytes)
            # simulation.py:252-253: the cache's unique-mapping invariant after every run
            self.mapping = fs.check_unique_mapping() if not cfg["mode.gpu_cache_disabled"] else None
            if keep_output:
                self.output = dst
        self.result = res
        self.metrics = Metrics(res.stats, log_deliveries=self.metrics.log_deliveries)
        if log:
            self.metrics.deliveries = [tuple(r) for r in res.deliveries.tolist()]
            self.cache.victim_log = [tuple(r) for r in res.victims.tolist()]
            self.recorded = [TraceRecord(*r) for r in res.rpcs.tolist()]
            if res.windows is not None:
                self.metrics.window_history = [int(w) for w in res.windows[:, 1]]
            if cfg["workload.record_trace"]:
                save_trace(cfg["workload.record_trace"], self.recorded)
        self._verify(res.stats)
        return build_report(self.label, wl.name, self.seed, self.rep, res.stats,
                            self.metrics.window_history)

    def _run_replay(self) -> MetricsReport:
        """Host-only replay (simulation.py:147-164, HostStream :67-95): the trace's preads
        issued back to back by rpc.n_workers host threads, grouped by the reference's
        slot partitioning; no GPU, no PCIe (the paper's §3.3 methodology)."""
        cfg, wl = self.cfg, self.workload
        paths = [p for p in cfg["io.paths"].split(",") if p] if cfg["io.paths"] else []
        if not paths:
            paths = [ensure_synthetic(synth_dir(cfg), f, wl.files[f]) for f in range(len(wl.files))]
        recs = np.array([(r.tb_id, r.file_id, r.offset, r.size) for r in self.trace], dtype=np.int64)
        user, preads, sec = native.replay(paths, recs, cfg["rpc.n_slots"], cfg["rpc.n_workers"],
                                          cfg["io.direct"])
        st = {k: 0 for k in native.stat_names()}
        st.update(user_bytes=user, preads=preads, pread_bytes=user, storage_bytes=user,
                  kernel_ns=int(sec * 1e9), wall_ns=int(sec * 1e9))
        self.result = RunResult(stats=st)
        self.metrics = Metrics(st)
        if user != wl.total_bytes:
            raise GfsError(f"replay delivered {user} of {wl.total_bytes} bytes")
        return build_report(self.label, wl.name, self.seed, self.rep, st)

    def _verify(self, st: dict) -> None:
        """Post-run invariants of gpuiosim/simulation.py:246-264 on real counters."""
        wl = self.workload
        if st["tag_mismatches"] or st.get("word_mismatches"):
            raise GfsError(f"{st['tag_mismatches']} pages delivered with wrong content")
        in_bounds = all(off + ln <= wl.files[fid] for prog in wl.programs for fid, off, ln in prog)
        if in_bounds and st["user_bytes"] != wl.total_bytes:
            raise GfsError(f"delivered {st['user_bytes']} of {wl.total_bytes} bytes")
        if st["storage_bytes"] < wl.unique_bytes:
            raise GfsError("storage read less than the unique workload bytes")
        if not self.cfg["mode.pcie_disabled"]:
            if st["pcie_bytes"] < st["user_bytes"] - st["cache_hit_user_bytes"]:
                raise GfsError("PCIe moved less than the delivered bytes")
