/*
 * gfs.h — C ABI of libgfs.so, the B200-native GPUfs-style sequential-read layer.
 *
 * Drop-in boundary for the reference's sequential gread path
 * (/root/reference/pkg/src/gpuiosim).  The reference is a Python package;
 * its outer API is Simulation(cfg, seed).run() -> MetricsReport
 * (simulation.py:98-242) and its inner contract is ThreadBlock._gread
 * (gpu_exec.py:107-129) over GpuPageCache (gpu_cache.py:92-212), the private
 * prefetch buffer (prefetcher.py:13-68), RpcQueue.submit/release
 * (rpc.py:82-113) and HostOs.pread (host_os.py:221).  Each entry point below
 * names the reference interface it replaces.  Plain pointers and sizes only:
 * no torch types cross this boundary (device buffers are raw CUDA pointers).
 *
 * Errors: every int-returning call returns 0 on success and a negative
 * GFS_E* code on failure; gfs_last_error() gives the thread's message.  The
 * Python layer maps them to GfsError (== the reference's SimError,
 * simcore.py:13).
 */
#ifndef GFS_H
#define GFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFS_ABI_VERSION 9  /* 9: k1_early; 8: k1_direct; 5: rpc_slots; 4: gfs_run_kernel (user kernels over gfs_device.cuh); 3: ondemand law */

enum { GFS_OK = 0, GFS_EINVAL = -1, GFS_ECUDA = -2, GFS_EIO = -3, GFS_ENOMEM = -4,
       GFS_ETIMEDOUT = -5, GFS_EDEVICE = -6, GFS_ESTATE = -7 };

/* gpufs.policy (gpu_cache.py:27-29) */
enum { GFS_POLICY_GLOBAL_LRU = 0, GFS_POLICY_PER_TB_LRA = 1 };
/* io.readahead: static = the reference span page+prefetch (prefetcher.py:13-25);
 * doubling = the span doubles on every sequential continuation up to ra_max_bytes;
 * ondemand ("adaptive" in the Python config) = the reference's Linux-style ondemand law
 *   (HostOs._decide, host_os.py:106-152) per TB stream: a cold sequential request of n pages
 *   opens max(n, min(4n, ra_max)) pages, the tail asynchronous with a marker; a request
 *   hitting the marker requests the next window (double, capped) asynchronously */
enum { GFS_RA_STATIC = 0, GFS_RA_DOUBLING = 1, GFS_RA_ONDEMAND = 2 };
/* ondemand windows end at the TB's segment end (its stride) or at EOF (the reference) */
enum { GFS_RA_CLAMP_SEGMENT = 0, GFS_RA_CLAMP_EOF = 1 };
/* io.transfer: zerocopy = SMs pull the span from per-CTA mapped pinned staging;
 * bounce = the daemon preads into a small (LLC-resident) per-worker pinned pool, the CTA
 *          pulls the whole span into its HBM landing slot at once and releases the buffer;
 * dma = daemon cudaMemcpyAsync's staging -> HBM landing, doorbell after it;
 * mapped_dma = memory-resident (tmpfs) files: the daemon DMAs each span straight from the
 *          pinned page-cache mapping into the HBM landing slot (no CPU copy);
 * mapped = memory-resident files: the daemon only answers the RPC, the CTA pulls the span
 *          from the pinned page-cache mapping into its HBM landing slot itself;
 * mapped_hybrid = mapped, but spans of >= 4 MiB go by copy engine (mapped_dma): SM pulls
 *          cap at ~51.5 GB/s on PCIe Gen5 x16, large copy-engine copies reach ~55, small
 *          copy-engine copies pay a fixed cost each;
 * pread_hybrid = the pread daemon for any file: O_DIRECT pread into a pinned pool, then spans
 *          of >= 4 MiB by cudaMemcpyAsync (dma), smaller ones pulled by the CTA (bounce) */
enum { GFS_XFER_ZEROCOPY = 0, GFS_XFER_DMA = 1, GFS_XFER_BOUNCE = 2, GFS_XFER_MAPPED = 3,
       GFS_XFER_MAPPED_ZC = 4, GFS_XFER_MAPPED_HYBRID = 5, GFS_XFER_PREAD_HYBRID = 6 };
/* gopen flags: read-only files are the only ones prefetched (prefetcher.py:22-24) */
enum { GFS_O_RDONLY = 0, GFS_O_RDWR = 2 };
/* log kinds (deterministic mode) */
enum { GFS_LOG_DELIVERIES = 0, GFS_LOG_RPCS = 1, GFS_LOG_VICTIMS = 2, GFS_LOG_WINDOWS = 3,
       GFS_LOG_TIMELINE = 4 };
/* timeline records (gfs_config.timeline): 4 int64 each —
 *   (kind << 56 | cta << 32 | tb, bytes, t_begin_ns, t_end_ns) on the GPU's global timer;
 *   kind: GFS_TL_RPC = request published .. its data ready (the PCIe transfer outstanding),
 *         GFS_TL_GREAD = one gread call, GFS_TL_CONSUME = the fused consumer over a request */
enum { GFS_TL_RPC = 0, GFS_TL_GREAD = 1, GFS_TL_CONSUME = 2 };

typedef struct gfs_config {
  int64_t page_size;       /* gpufs.page_size (multiple of 4096) */
  int64_t cache_bytes;     /* gpufs.cache_bytes: frame pool in HBM */
  int64_t prefetch_bytes;  /* gpufs.prefetch_bytes */
  int64_t staging_bytes;   /* rpc.staging_bytes: PCIe batch size (accounting, rpc.py:31-55) */
  int64_t ra_max_bytes;    /* io.ra_max_bytes: readahead window cap (doubling, ondemand) */
  int64_t ra_init_bytes;   /* io.ra_init_bytes: doubling first window (0 = page + prefetch) */
  int64_t max_request_bytes; /* largest gread request (raw mode sizes staging to it) */
  int32_t policy;          /* GFS_POLICY_* */
  int32_t resident_limit;  /* reference residency (gpu_exec.py:44-50): sets the LRA quota */
  int32_t readahead;       /* GFS_RA_* */
  int32_t transfer;        /* GFS_XFER_* */
  int32_t io_workers;      /* host daemon threads */
  int32_t io_direct;       /* O_DIRECT preads (aligned requests) */
  int32_t device;          /* CUDA ordinal */
  int32_t cta_threads;     /* threads per resident CTA (one CTA = one active TB) */
  int32_t max_ctas;        /* cap on resident CTAs (0 = min(resident_limit, occupancy)) */
  int32_t raw_mode;        /* mode.gpu_cache_disabled (gpu_exec.py:114-119) */
  int32_t pcie_disabled;   /* mode.pcie_disabled: accounting only */
  int32_t log;             /* record delivery / RPC / victim logs on the device */
  int32_t verify;          /* check every fetched word against the synthetic law */
  int32_t timeline;        /* record the GFS_LOG_TIMELINE log (mode.timeline) */
  int32_t k1_tma;          /* gpu.k1_copy: 1 = span -> frame/user copies by TMA bulk copies
                              through a shared-memory ring, 0 = 16-byte vector loads/stores */
  int32_t numa_pin;        /* io.numa_pin: daemon threads on the CPUs local to the GPU's PCIe root */
  int32_t lookahead;       /* gpu.lookahead: a page batch may run past a page-aligned request to
                              the TB's segment end (the next greads find their bytes delivered) */
  int32_t ra_clamp;        /* io.ra_clamp: GFS_RA_CLAMP_* (ondemand) */
  int32_t rpc_slots;       /* rpc.n_slots (0 = 128): the reference's slot partition tb % n_slots,
                              for the slot_collisions counter (rpc.py:25-28, 82-89) */
  int32_t k1_direct;       /* gpu.k1_direct: spans of the mapped transfers that the CTA would pull
                              are read by the span copy (K1) straight from the pinned file mapping
                              into frames + user buffer (one pass, no HBM landing copy) */
  int32_t k1_early;        /* gpu.k1_early: such a span is read before the daemon's answer comes
                              back (the answer is the span length, known from the file size); the
                              answer is collected before the CTA's next request and checked */
} gfs_config;

/* One gread program set (workloads.py:24-31 programs, flattened).
 * TB t reads segments segs[prog_off[t] .. prog_off[t+1]) in order, request_bytes
 * at a time (gpu_exec.py:95-105); its bytes land at dst + dst_off[t] + (position
 * within its program).  order[] is the activation order (gpu_exec.py:242-265). */
typedef struct gfs_program {
  int32_t n_tb;
  int32_t reserved;
  int64_t request_bytes;
  const int64_t* segs;     /* [n_segs][3]: file id, offset, length */
  const int64_t* prog_off; /* [n_tb + 1] */
  const int64_t* dst_off;  /* [n_tb] */
  const int32_t* order;    /* [n_tb] */
} gfs_program;

/* Counters: names follow gpuiosim.metrics.Metrics (metrics.py:12-46) + timing. */
#define GFS_STAT_FIELDS(X)                                                                    \
  X(greads) X(user_bytes) X(cache_hit_user_bytes) X(tag_mismatches) X(pc_lookups) X(pc_hits) \
  X(pc_hit_pending) X(pc_misses) X(pc_allocs) X(pc_evictions) X(pc_remaps) X(pb_hits)        \
  X(pb_misses) X(pb_filled_bytes) X(pb_consumed_bytes) X(pb_discarded_bytes) X(rpc_count)    \
  X(rpc_requested_bytes) X(slot_collisions) X(preads) X(pread_bytes) X(storage_bytes)       \
  X(pcie_bytes) X(pcie_transfers) X(victims) X(kernel_ns) X(wall_ns) X(ctas) X(word_mismatches) \
  X(wait_ns) X(meta_ns) X(copy_ns) X(lookup_ns) X(alloc_ns) X(install_ns) X(host_pread_ns) \
  X(host_idle_ns) X(host_xfer_ns) X(host_requests) X(io_workers) X(early_answers)

enum {
#define GFS_X(name) GFS_STAT_##name,
  GFS_STAT_FIELDS(GFS_X)
#undef GFS_X
  GFS_NSTATS
};

typedef struct gfs_stats {
  int64_t v[GFS_NSTATS];
} gfs_stats;

typedef struct gfs_ctx gfs_ctx;

/* ---- lifecycle: replaces Simulation.__init__ wiring (simulation.py:101-212) ---- */
int gfs_create(const gfs_config* cfg, gfs_ctx** out);
void gfs_destroy(gfs_ctx* ctx);

/* ---- files.  The reference has no gopen/gclose: "open" is WorkloadSpec.files /
 * read_only (workloads.py:24-31) and "close" is the TB-done drain + retire
 * (gpu_exec.py:281-291).  content_id >= 0 marks a synthetic file whose words
 * follow W(content_id, i) so the device can verify them (page_tag analogue,
 * gpu_exec.py:159-160); -1 = arbitrary content. ---- */
int gfs_gopen(gfs_ctx* ctx, const char* path, int flags, int64_t content_id, int* fid);
int gfs_gclose(gfs_ctx* ctx, int fid);
int gfs_file_size(gfs_ctx* ctx, int fid, int64_t* size);

/* ---- the hot path: every TB's gread loop (gpu_exec.py:95-239) on the GPU, fed by
 * the host daemon (rpc.py:144-229 + host_os.py:221).  dst: device buffer (NULL =
 * consume-only: pages are cached but not copied out).  Blocks until every TB is
 * done; cold page cache per run (as a fresh Simulation). ---- */
int gfs_run(gfs_ctx* ctx, const gfs_program* prog, void* dst, uint64_t dst_bytes, gfs_stats* out);

/* ---- streaming consumers fused into the gread loop.  After each gread
 * the TB runs the consumer over the bytes it just delivered (they are in L2), so compute
 * overlaps the other TBs' I/O — the real counterpart of workload.compute_ns_per_byte
 * (gpu_exec.py:127-129).  Elements decode from the file bytes: f32 = (u32 >> 8) * 2^-24. */
enum { GFS_CONSUME_NONE = 0, GFS_CONSUME_SUM64 = 1, GFS_CONSUME_GEMV_F32 = 2, GFS_CONSUME_NN_F32 = 3,
       GFS_CONSUME_GEMVT_F32 = 4, GFS_CONSUME_BICG_F32 = 5, GFS_CONSUME_KMEANS_F32 = 6 };
/* Shapes: the file is a row-major matrix A [rows, cols] of such f32 elements.
 *   GEMV   (gesummv, mvt 1st, atax 1st pass):  y  += A x          x [cols], y [rows]
 *   GEMVT  (mvt 2nd, atax 2nd pass):           y2 += A^T x2       x2 [rows], y2 [cols]
 *   BICG   (bicg q = A p, s = A^T r; mvt):     both in one pass
 *   KMEANS (Rodinia kmeans assignment step):   rows = points of `cols` features; each point
 *          goes to the nearest of k centroids x [k, cols] (squared distance summed over the
 *          features in order, IEEE fp32, lowest index on ties); y [k, cols] += the points'
 *          features per centroid, out [k] (u64) += points per centroid. */
#define GFS_KMEANS_MAX_K 16

typedef struct gfs_consumer {
  int32_t kind;             /* GFS_CONSUME_* */
  int32_t k;                /* KMEANS: number of centroids (1..GFS_KMEANS_MAX_K) */
  int64_t cols;             /* GEMV*, BICG, KMEANS: row length (elements, multiple of 4) */
  const float* x;           /* GEMV/BICG: device vector [cols]; KMEANS: centroids [k, cols] */
  float* y;                 /* GEMV/BICG: device vector [rows] (y += A x); KMEANS: sums [k, cols] */
  float qx, qy;             /* NN: query point (records are (lat, lng) pairs) */
  unsigned long long* out;  /* SUM64: device u64 += sum_i mix64(w_i ^ (i * golden)) over file words;
                               NN: device u64 atomicMin of (dist2 bits << 32 | record index);
                               KMEANS: device u64 [k] += points assigned per centroid */
  const float* x2;          /* GEMVT/BICG: device vector [rows] */
  float* y2;                /* GEMVT/BICG: device vector [cols] (y2 += A^T x2) */
} gfs_consumer;

/* gfs_run plus a consumer (cons may be NULL); requires a user buffer. */
int gfs_run_consume(gfs_ctx* ctx, const gfs_program* prog, void* dst, uint64_t dst_bytes,
                    const gfs_consumer* cons, gfs_stats* out);

/* ---- user kernels reading through the device-side gread (include/gfs_device.cuh;
 * SURVEY §8(b), reference ThreadBlock._gread gpu_exec.py:107-239).  gfs_run_kernel prepares a
 * run exactly as gfs_run does (cold page cache, fresh counters, daemon serving the RPC ring)
 * for n_tb threadblocks whose programs are the user's kernel, then calls launch() once, from
 * the calling thread, to launch that kernel on `stream`; it waits for the kernel and returns
 * the run's counters (and logs) like gfs_run.  order: activation order of the TB ids
 * (NULL = 0..n_tb-1).  Mapped transfers pin each open file whole.  The launch callback
 * returns 0, or nonzero to abort the run (GFS_EINVAL).  The built-in lookahead is off for
 * user kernels: a gread delivers only [offset, offset+size). ---- */
typedef struct gfs_launch {
  const void* dev;      /* device context (gfs_dev, gfs_device.cuh): pass *(const gfs_dev*)dev by value */
  int64_t dev_bytes;    /* sizeof(gfs_dev) the library was built with (launchers check it) */
  int32_t n_ctas;       /* grid: one CTA per resident TB slot */
  int32_t cta_threads;  /* block size: must equal the kernel's BS */
  int64_t smem_bytes;   /* dynamic shared memory the file layer needs */
  void* stream;         /* cudaStream_t to launch on */
  int32_t n_tb;
  int32_t reserved;
} gfs_launch;
typedef int (*gfs_launch_fn)(const gfs_launch* launch, void* user);
int gfs_run_kernel(gfs_ctx* ctx, int32_t n_tb, const int32_t* order, gfs_launch_fn launch, void* user,
                   gfs_stats* out);

/* ---- logs of the last run (metrics.deliveries, recorded trace, victim_log) ---- */
int gfs_log_len(gfs_ctx* ctx, int kind, int64_t* n);
int gfs_log_copy(gfs_ctx* ctx, int kind, int64_t* out, int64_t cap_records);

/* ---- device consumers ---- */
/* sum_i mix64(word_i ^ ((i + word_base) * golden)) over nbytes of a device buffer */
int gfs_checksum(gfs_ctx* ctx, const void* dev_buf, uint64_t nbytes, uint64_t word_base, uint64_t* out);
/* count words of dev_buf (laid out as prog's user buffer) that differ from W(content of file) */
int gfs_verify_dst(gfs_ctx* ctx, const gfs_program* prog, const void* dev_buf, uint64_t dst_bytes,
                   int64_t* mismatched_words);

/* ---- end-of-run invariant: GpuPageCache.check_unique_mapping (gpu_cache.py:217-224,
 * simulation.py:252-253) over the device page table the last run left.  Every mapped page
 * must name a settled frame (VALID, unpinned, not in flight) keyed by that (file, page), no
 * frame may be reachable from two pages, and no VALID frame of an open file may be
 * unreachable.  Fills *out and returns GFS_EDEVICE when any count but mapped_pages is
 * nonzero. ---- */
typedef struct gfs_mapping_check {
  int64_t mapped_pages;
  int64_t duplicate_frames;
  int64_t key_mismatches;
  int64_t unsettled;
  int64_t lost_frames;
} gfs_mapping_check;
int gfs_check_mapping(gfs_ctx* ctx, gfs_mapping_check* out);

/* ---- synthetic files (K6): write W(content_id, i) words, multi-threaded ---- */
int gfs_gen_file(const char* path, int64_t content_id, int64_t size, int threads);
/* the same words for [offset, offset+length) of a file of `size` bytes (created/extended
 * as needed): ranks of a sharded run write their own shards from GPU-local CPUs */
int gfs_gen_file_range(const char* path, int64_t content_id, int64_t size, int64_t offset,
                       int64_t length, int threads);

/* ---- comparison arms and roofline probes (bench.py; not on the gread path) ---- */
/* parallel sequential read of [offset, offset+size) of path; wall seconds */
int gfs_bench_storage(const char* path, int64_t offset, int64_t size, int threads, int64_t chunk,
                      int direct, double* seconds);
/* best-of-reps pinned host -> HBM cudaMemcpyAsync of `bytes`; seconds */
int gfs_bench_h2d(int device, int64_t bytes, int reps, double* best_seconds);
/* CPU I/O baseline: threads pread() into pinned buffers + cudaMemcpy into dst_dev
 * (sync = 1: blocking cudaMemcpy per chunk, the paper's CPU arm); wall seconds */
int gfs_bench_read_memcpy(const char* path, int64_t offset, int64_t size, void* dst_dev, int device,
                          int threads, int64_t chunk, int direct, int sync, double* seconds);

/* host-only replay of a recorded RPC trace (the reference's `gpuiosim replay`,
 * simulation.py:147-164): recs = [n_recs][4] (tb, file, offset, size);
 * record r is served by worker (tb % n_slots) / (n_slots / n_workers), each worker preads
 * its records back to back.  No GPU involved.  Errors: unknown file / read past EOF
 * (trace_workload, simulation.py:50-64) -> GFS_EINVAL. */
int gfs_replay(const char* const* paths, int n_files, const int64_t* recs, int64_t n_recs,
               int n_slots, int n_workers, int direct, int64_t* user_bytes, int64_t* preads,
               double* seconds);

/* ---- introspection ---- */
const char* gfs_last_error(void);
int gfs_abi_version(void);
int gfs_stat_count(void);
const char* gfs_stat_name(int i);
int gfs_resident_ctas(gfs_ctx* ctx);
/* the transfer this context uses: gfs_create probes whether copy-engine streams can make
 * progress while the persistent kernel runs (they cannot when CUDA_DEVICE_MAX_CONNECTIONS
 * was too small when CUDA started) and otherwise falls back to the SM-pull sibling
 * (mapped_dma / mapped_hybrid -> mapped, dma -> bounce); *downgraded_from = the requested
 * transfer then, else -1 */
int gfs_transfer(gfs_ctx* ctx, int* transfer, int* downgraded_from);

#ifdef __cplusplus
}
#endif
#endif /* GFS_H */
