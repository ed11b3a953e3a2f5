// gfs_host.cpp — host runtime of libgfs.so: context, files, pinned RPC ring, I/O daemon,
// run orchestration, synthetic-file generator.  C ABI declared in include/gfs.h.
//
// Daemon (replaces HostWorker, rpc.py:116-229, and HostOs.pread, host_os.py:221):
//   io_workers threads share one request ring in mapped pinned memory.  A worker claims
//   the next ring position (fetch_add), waits for the GPU to publish it, preads the span
//   (O_DIRECT when aligned) into the CTA slot's pinned staging buffer and completes it:
//     zerocopy: release-store of {nbytes, seq} into the slot's mapped response mailbox;
//               the CTA pulls the bytes over PCIe itself (K1);
//     dma:      cudaMemcpyAsync staging -> HBM landing on the worker's stream, then
//               cuStreamWriteValue64 of (nbytes << 32 | seq) into the slot's device
//               doorbell, ordered after the copy.
//   A shared ring (instead of the reference's tb % n_slots slot partitioning) keeps all
//   workers busy: the reference's worker-imbalance pathology (criterion 2) cannot occur.
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <immintrin.h>
#include <ctype.h>
#include <pthread.h>
#include <sched.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <string>
#include <thread>
#include <vector>

#include "gfs.h"
#include "gfs_shared.h"

namespace gfs {
cudaError_t launch_gread(const DevCtx& c, int cta_threads, cudaStream_t st);
cudaError_t occupancy_gread(int cta_threads, int* blocks_per_sm);
cudaError_t launch_queue_probe(const unsigned long long* flags, int n, uint64_t timeout_ns, int* ok,
                               cudaStream_t st);
int64_t gread_tma_offset(const gfs_consumer& k, int cta_threads);
int gread_tma_stages(const gfs_consumer& k, int cta_threads);
int64_t gread_launch_smem(const gfs_consumer& k, int cta_threads, int tma);
cudaError_t launch_check_mapping(const DevFile* files, int n_files, const unsigned long long* fkey,
                                 const uint32_t* fstate, uint32_t* owner, int64_t nframes,
                                 unsigned long long* out, int sms, cudaStream_t st);
cudaError_t launch_checksum(const void* buf, uint64_t nbytes, uint64_t word_base,
                            unsigned long long* out, int sms, cudaStream_t st);
cudaError_t launch_verify_dst(const void* buf, const int64_t* segs, const int64_t* seg_dst,
                              int64_t n_segs, const DevFile* files, unsigned long long* out,
                              int sms, cudaStream_t st);
}  // namespace gfs

using namespace gfs;

// ------------------------------------------------------------------- errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(GFS_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                               \
  } while (0)

static const char* const kStatNames[GFS_NSTATS] = {
#define GFS_X(name) #name,
    GFS_STAT_FIELDS(GFS_X)
#undef GFS_X
};

static int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

static uint64_t now_ns() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (uint64_t)t.tv_sec * 1000000000ull + (uint64_t)t.tv_nsec;
}

// ------------------------------------------------------------------- context

struct HostFile {
  std::string path;
  int fd_direct = -1;
  int fd_buffered = -1;
  int64_t size = 0;
  int64_t npages = 0;
  int read_only = 1;
  int64_t content_id = -1;
  uint32_t* d_pt = nullptr;
  uint8_t* map = nullptr;   // mapped modes: pinned mapping of [map_lo, map_lo + map_len)
  uint8_t* dmap = nullptr;  // and its device address
  int64_t map_lo = 0, map_len = 0;
  bool open = false;
};

static void unmap_file(HostFile& f) {
  if (f.map) {
    cudaHostUnregister(f.map);
    munmap(f.map, (size_t)f.map_len);
    f.map = f.dmap = nullptr;
    f.map_lo = f.map_len = 0;
  }
}

// Mapped transfers: pin the page-cache pages of [lo, hi) of a memory-resident file (tmpfs
// allows long-term pins of shmem pages; disk files do not) so spans can be pulled / DMA'd
// straight out of them.  Only the range a run reads is mapped (a rank maps its shard).
static int map_range(HostFile& f, int64_t lo, int64_t hi) {
  lo &= ~(int64_t)((2 << 20) - 1);
  hi = std::min(f.size, (hi + (2 << 20) - 1) & ~(int64_t)((2 << 20) - 1));
  if (f.map && f.map_lo <= lo && f.map_lo + f.map_len >= hi) return GFS_OK;
  unmap_file(f);
  const size_t len = (size_t)(hi - lo);
  void* m = MAP_FAILED;
  cudaError_t e = cudaErrorInvalidValue;
  // Pinning page-cache pages can fail transiently (the kernel migrating pages while memory
  // is tight); retry a few times before reporting.
  for (int attempt = 0; attempt < 4 && e != cudaSuccess; attempt++) {
    if (attempt) std::this_thread::sleep_for(std::chrono::milliseconds(250 * attempt));
    m = mmap(nullptr, len, PROT_READ, MAP_SHARED | MAP_POPULATE, f.fd_buffered, (off_t)lo);
    e = m == MAP_FAILED ? cudaErrorInvalidValue
                        : cudaHostRegister(m, len, cudaHostRegisterReadOnly | cudaHostRegisterPortable |
                                                       cudaHostRegisterMapped);
    if (m != MAP_FAILED && e != cudaSuccess) {
      // platforms without read-only registration: pin a shared read-write mapping of the
      // same pages (never written through; needs write permission on the file)
      cudaGetLastError();
      munmap(m, len);
      int rw = open(f.path.c_str(), O_RDWR);
      m = rw < 0 ? MAP_FAILED
                 : mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, rw, (off_t)lo);
      if (rw >= 0) close(rw);
      e = m == MAP_FAILED ? cudaErrorInvalidValue
                          : cudaHostRegister(m, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();  // do not leave a sticky error for the next launch check
      if (m != MAP_FAILED) munmap(m, len);
    }
  }
  if (m == MAP_FAILED || e != cudaSuccess) {
    return fail(GFS_EIO, "mapped transfers need a memory-resident file (tmpfs); pinning %s [%lld, %lld) failed: %s",
                f.path.c_str(), (long long)lo, (long long)hi,
                m == MAP_FAILED ? strerror(errno) : cudaGetErrorString(e));
  }
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, m, 0) != cudaSuccess) {
    cudaGetLastError();
    dp = m;  // UVA: the host address is the device address
  }
  f.map = (uint8_t*)m;
  f.dmap = (uint8_t*)dp;
  f.map_lo = lo;
  f.map_len = (int64_t)len;
  return GFS_OK;
}

template <typename T>
struct DevBuf {  // grow-only device buffer
  T* p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t count) {
    if (count <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct gfs_ctx {
  gfs_config cfg{};
  int sms = 0;
  int n_ctas = 0;
  int64_t nframes = 0, quota = 0, pb_cap = 0, slot_bytes = 0, gfifo_cap = 0;
  uint32_t ring_size = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // device memory
  uint8_t* d_frames = nullptr;
  unsigned long long* d_fkey = nullptr;
  uint32_t* d_fstate = nullptr;
  uint32_t* d_own_q = nullptr;
  uint32_t* d_retired = nullptr;
  unsigned long long* d_rpool = nullptr;  // retired FIFO heads/tails
  int ret_npools = 1;
  int landing_halves = 1;  // 2: asynchronous readahead fills one half while the CTA reads the other
  bool stream_pieces = false;  // copy-engine windows land piece by piece
  int64_t stream_piece = 0;
  unsigned long long* d_landed = nullptr;
  int64_t ret_pcap = 0;
  uint32_t* d_gfifo = nullptr;
  uint32_t* d_recycled = nullptr;
  DevGlobals* d_g = nullptr;
  uint8_t* d_landing = nullptr;
  unsigned long long* d_doorbell = nullptr;
  unsigned long long* d_done_pos = nullptr;
  long long* d_stats = nullptr;
  unsigned long long* d_scratch = nullptr;
  uint32_t* d_owner = nullptr;  // check_unique_mapping scratch (nframes), allocated on first use
  uint32_t* d_slot_busy = nullptr;  // [rpc_slots]: the reference slot partition's occupancy
  unsigned long long* h_served = nullptr;  // mapped: requests completed by the daemon
  DevBuf<int64_t> d_segs, d_prog_off, d_dst_off, d_seg_dst;
  DevBuf<int32_t> d_order;
  DevBuf<DevFile> d_files;
  DevBuf<long long> d_logs[5];
  unsigned long long log_cap[5] = {0, 0, 0, 0, 0};
  unsigned long long log_n[5] = {0, 0, 0, 0, 0};

  // mapped pinned host memory
  RpcReq* h_ring = nullptr;
  uint32_t* h_consumed = nullptr;  // [ring_size]: seq of the request the daemon last copied out of each entry
  RpcResp* h_resp = nullptr;
  uint8_t* h_staging = nullptr;

  std::vector<HostFile> files;

  // daemon
  std::vector<std::thread> workers;
  std::vector<int> local_cpus;  // daemon threads pinned here (empty = no pinning)
  std::vector<cudaStream_t> worker_streams;  // copy streams (shared by the workers)
  std::vector<cudaStream_t> bell_streams;    // doorbell streams
  std::vector<cudaEvent_t> bell_ev;          // per worker: "this copy is done"
  // DMA mode: per-worker pinned bounce buffers, few and small enough to stay resident in
  // the host LLC (pread writes them, the copy engine reads them right after)
  int nbounce = 0;
  uint8_t* h_bounce = nullptr;
  std::vector<cudaEvent_t> bounce_ev;  // [io_workers * nbounce]
  // bounce mode: the same pool, mapped; the GPU writes release words after pulling a span
  uint32_t* h_release = nullptr;       // [io_workers * nbounce] (mapped)
  std::vector<uint32_t> bounce_last;   // seq last stored in each buffer (0 = free)
  std::vector<char> bounce_ce;         // pread_hybrid: the buffer's last use was a copy-engine copy
  std::atomic<uint64_t> req_head{0};
  // daemon accounting for the current run (ns summed over workers)
  std::atomic<int64_t> t_pread{0}, t_idle{0}, t_xfer{0}, n_served{0};
  std::atomic<bool> stop{false};
  std::atomic<int> worker_error{0};
  // per-worker progress, for diagnosing a stalled request: last claimed ring position and
  // phase (0 waiting for the entry, 1 reading, 2 completing, 3 completed)
  std::atomic<uint64_t> w_pos[256];
  std::atomic<int> w_phase[256];
  bool has_run = false;
  // a run whose kernel never finished leaves the device and the daemon unusable: later
  // calls fail fast instead of timing out against workers parked on stale positions
  bool poisoned = false;
  int downgraded_from = -1;  // copy-engine transfer replaced by its SM-pull sibling (queue probe)
  int64_t ce_min = 4 << 20;  // mapped_hybrid: spans of at least this many bytes go by copy engine
  int probe_attempts = 0;    // copy-queue probe rounds gfs_create needed (1 = first streams fine)
  // driver entry point resolved through cudart (libgfs does not link libcuda, so it
  // loads on machines without a driver; CUDA calls then fail loudly)
  CUresult (*write_value64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
};

// ------------------------------------------------------------------- daemon

static int64_t do_pread(gfs_ctx* ctx, const HostFile& f, int64_t off, int64_t size, uint8_t* buf) {
  if (off >= f.size || size <= 0) return 0;
  int64_t n = std::min(size, f.size - off);
  bool direct = f.fd_direct >= 0 && (off & 4095) == 0 && (((uintptr_t)buf) & 4095) == 0;
  int fd = direct ? f.fd_direct : f.fd_buffered;
  int64_t want = direct ? round_up(n, 4096) : n;
  if (want > ctx->slot_bytes) want = n;  // never write past the staging slot
  int64_t got = 0;
  while (got < n) {
    ssize_t k = pread(fd, buf + got, (size_t)(want - got), (off_t)(off + got));
    if (k < 0) {
      if (errno == EINTR) continue;
      if (direct && errno == EINVAL) {  // filesystem refused O_DIRECT: buffered from here on
        direct = false;
        fd = f.fd_buffered;
        want = n;
        continue;
      }
      return -(int64_t)errno;
    }
    if (k == 0) break;
    got += k;
    if (direct && (got & 4095)) {  // short O_DIRECT read (EOF); finish buffered
      direct = false;
      fd = f.fd_buffered;
      want = n;
    }
  }
  return std::min(got, n);
}

// Host CPUs attached to the GPU's PCIe root (sysfs local_cpulist), limited to the CPUs this
// process may use; empty when unknown or when that is every usable CPU anyway.
static std::vector<int> gpu_local_cpus(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
    cudaGetLastError();
    return {};
  }
  std::string id(bus);
  for (auto& ch : id) ch = (char)tolower(ch);
  const size_t colon = id.find(':');
  if (colon != std::string::npos && colon > 4) id = id.substr(colon - 4);  // 8-digit domain
  FILE* fp = fopen(("/sys/bus/pci/devices/" + id + "/local_cpulist").c_str(), "r");
  if (!fp) return {};
  char line[4096] = {0};
  const bool ok = fgets(line, sizeof line, fp) != nullptr;
  fclose(fp);
  if (!ok) return {};
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  if (sched_getaffinity(0, sizeof allowed, &allowed) != 0) return {};
  std::vector<int> out;
  for (char* tok = strtok(line, ",\n"); tok; tok = strtok(nullptr, ",\n")) {
    int a = -1, b = -1;
    if (sscanf(tok, "%d-%d", &a, &b) == 2) {
    } else if (sscanf(tok, "%d", &a) == 1) {
      b = a;
    } else {
      continue;
    }
    for (int c = a; c <= b && c < CPU_SETSIZE; c++)
      if (c >= 0 && CPU_ISSET(c, &allowed)) out.push_back(c);
  }
  if ((int)out.size() >= CPU_COUNT(&allowed)) return {};  // no narrower than what we have
  return out;
}

static void worker_main(gfs_ctx* ctx, int wid) {
  if (!ctx->local_cpus.empty()) {  // NUMA-local to the GPU's PCIe root (north_star)
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : ctx->local_cpus) CPU_SET(c, &set);
    pthread_setaffinity_np(pthread_self(), sizeof set, &set);
  }
  const uint32_t mask = ctx->ring_size - 1;
  const bool dma = ctx->cfg.transfer == GFS_XFER_DMA;
  const bool bounce = ctx->cfg.transfer == GFS_XFER_BOUNCE;
  const bool hybrid = ctx->cfg.transfer == GFS_XFER_MAPPED_HYBRID;
  const bool phyb = ctx->cfg.transfer == GFS_XFER_PREAD_HYBRID;  // pread: large spans dma, small pulled
  const bool mapped_ce = ctx->cfg.transfer == GFS_XFER_MAPPED;     // copy engine from the mapping
  const bool mapped_zc = ctx->cfg.transfer == GFS_XFER_MAPPED_ZC;  // the CTA pulls it itself
  const bool from_map = mapped_ce || mapped_zc || hybrid;
  const int64_t ce_min = ctx->ce_min;  // hybrid: spans this large go by copy engine
  cudaStream_t st = (dma || mapped_ce || hybrid || phyb)
                        ? ctx->worker_streams[(size_t)wid % ctx->worker_streams.size()]
                        : nullptr;
  if (st) cudaSetDevice(ctx->cfg.device);
  uint64_t nreq = 0;
  while (!ctx->stop.load(std::memory_order_relaxed)) {
    uint64_t h = ctx->req_head.fetch_add(1, std::memory_order_relaxed);
    RpcReq* e = &ctx->h_ring[h & mask];
    const uint32_t seq = (uint32_t)(h + 1);
    uint64_t spins = 0;
    const uint64_t t_wait = now_ns();
    ctx->w_pos[wid].store(h, std::memory_order_relaxed);
    ctx->w_phase[wid].store(0, std::memory_order_relaxed);
    const uint64_t lap = ring_lap(h, mask + 1ull);
    uint64_t w0, w1, w2;
    for (;;) {  // the entry is complete when all three words carry this lap (see RpcReq)
      w0 = __atomic_load_n(&e->w[0], __ATOMIC_ACQUIRE);
      w1 = __atomic_load_n(&e->w[1], __ATOMIC_ACQUIRE);
      w2 = __atomic_load_n(&e->w[2], __ATOMIC_ACQUIRE);
      if ((w0 & 0xFFFF) == lap && (w1 & 0xFFFF) == lap && (w2 & 0xFFFF) == lap) break;
      if (ctx->stop.load(std::memory_order_relaxed)) return;
      if (++spins < 20000) {
        _mm_pause();
      } else {
        timespec ts{0, 20000};  // idle: back off to 20 us naps
        nanosleep(&ts, nullptr);
      }
    }
    const uint64_t t0 = now_ns();
    ctx->t_idle.fetch_add((int64_t)(t0 - t_wait), std::memory_order_relaxed);
    ctx->w_phase[wid].store(1, std::memory_order_relaxed);
    const int64_t off = (int64_t)(w0 >> 16), size = (int64_t)(w1 >> 32);
    const int fid = (int)((w1 >> 16) & 0xFFFF);
    const int slot = (int)((w2 >> 16) & 0x7FFF), half = (int)((w2 >> 31) & 1);
    // the entry's fields are copied out: the device may reuse it (ring wrap) from now on,
    // whether or not the CTA that asked has come back for its answer yet
    __atomic_store_n(&ctx->h_consumed[h & mask], seq, __ATOMIC_RELEASE);
    int64_t n;
    uint8_t* buf;
    int b = 0;
    if (dma) {  // next bounce buffer of this worker, once its previous copy has drained
      b = wid * ctx->nbounce + (int)(nreq % (uint64_t)ctx->nbounce);
      if (nreq >= (uint64_t)ctx->nbounce) cudaEventSynchronize(ctx->bounce_ev[b]);
      buf = ctx->h_bounce + (int64_t)b * ctx->slot_bytes;
    } else if (bounce || phyb) {  // next pool buffer, once the CTA that used it last pulled it out
      b = wid * ctx->nbounce + (int)(nreq % (uint64_t)ctx->nbounce);
      if (phyb && ctx->bounce_ce[b]) {  // (pread_hybrid) or its copy engine copy drained
        cudaEventSynchronize(ctx->bounce_ev[b]);
        ctx->bounce_ce[b] = 0;
      }
      const uint32_t last = ctx->bounce_last[b];
      uint64_t sp = 0;
      while (last && __atomic_load_n(&ctx->h_release[b], __ATOMIC_ACQUIRE) != last) {
        if (ctx->stop.load(std::memory_order_relaxed)) return;
        if (++sp > 200000) {
          timespec ts{0, 5000};
          nanosleep(&ts, nullptr);
        } else {
          _mm_pause();
        }
      }
      ctx->bounce_last[b] = seq;
      buf = ctx->h_bounce + (int64_t)b * ctx->slot_bytes;
    } else if (from_map) {
      buf = nullptr;
    } else {
      buf = ctx->h_staging + ((int64_t)slot * ctx->landing_halves + half) * ctx->slot_bytes;
    }
    nreq++;
    const bool bad = slot < 0 || slot >= ctx->n_ctas || fid < 0 || fid >= (int)ctx->files.size() ||
                     !ctx->files[fid].open || size > ctx->slot_bytes;
    if (bad) {
      n = -EINVAL;
    } else if (from_map) {  // no read at all: the span comes from the pinned mapping
      const HostFile& f = ctx->files[fid];
      n = off >= f.size ? 0 : std::min(size, f.size - off);
      buf = f.map + (off - f.map_lo);
    } else {
      n = do_pread(ctx, ctx->files[fid], off, size, buf);
    }
    const uint64_t t1 = now_ns();
    ctx->t_pread.fetch_add((int64_t)(t1 - t0), std::memory_order_relaxed);
    ctx->w_phase[wid].store(2, std::memory_order_relaxed);
    if (n < 0) ctx->worker_error.store((int)-n);
    // count it before completing: a launch that starts after this completion must see it
    __atomic_fetch_add(ctx->h_served, 1ull, __ATOMIC_SEQ_CST);
    if (dma || mapped_ce || hybrid || phyb) {
      const bool copy = !(hybrid || phyb) || n >= ce_min;  // hybrids: small spans are pulled by the CTA
      cudaError_t ce = cudaSuccess;
      cudaStream_t bs = ctx->bell_streams[(size_t)wid % ctx->bell_streams.size()];
      const int64_t li = (int64_t)slot * ctx->landing_halves + half;
      const int64_t piece = ctx->stream_piece;
      const bool streamed = copy && ctx->stream_pieces && n >= 2 * piece;
      if (n > 0 && copy && !streamed) {
        ce = cudaMemcpyAsync(ctx->d_landing + li * ctx->slot_bytes, buf, (size_t)n, cudaMemcpyHostToDevice, st);
        if (ce == cudaSuccess && (dma || phyb)) ce = cudaEventRecord(ctx->bounce_ev[b], st);
        if (phyb) {  // the copy engine frees the buffer: no CTA release to wait for
          ctx->bounce_ce[b] = 1;
          ctx->bounce_last[b] = 0;
        }
      }
      if (phyb && n <= 0) ctx->bounce_last[b] = 0;  // nothing to pull: the buffer stays free
      if (phyb && !copy && n > 0) {  // the CTA pulls it from pool buffer b: say which, before the doorbell
        RpcResp* r = &ctx->h_resp[li];
        r->buf = b;
        __atomic_thread_fence(__ATOMIC_RELEASE);
      }
      if (streamed) {
        // the window in pieces: after each, a landed marker; after the first, the doorbell —
        // the CTA starts on the first piece while the others copy
        for (int64_t o = 0; o < n && ce == cudaSuccess; o += piece) {
          const int64_t len = std::min(piece, n - o);
          ce = cudaMemcpyAsync(ctx->d_landing + li * ctx->slot_bytes + o, buf + o, (size_t)len,
                               cudaMemcpyHostToDevice, st);
          if (ce != cudaSuccess) break;
          cudaEventRecord(ctx->bell_ev[wid], st);
          cudaStreamWaitEvent(bs, ctx->bell_ev[wid], 0);
          const uint64_t pages = (uint64_t)((o + len + 4095) / 4096);
          CUresult cr = ctx->write_value64((CUstream)bs, (CUdeviceptr)(ctx->d_landed + li), (cuuint64_t)((pages << 32) | seq), 0);
          if (cr == CUDA_SUCCESS && o == 0)
            cr = ctx->write_value64((CUstream)bs, (CUdeviceptr)(ctx->d_doorbell + li),
                                    (cuuint64_t)(((uint64_t)n << 32) | seq), 0);
          if (cr != CUDA_SUCCESS) ce = cudaErrorUnknown;
        }
        if (ce == cudaSuccess && dma) ce = cudaEventRecord(ctx->bounce_ev[b], st);
      }
      if (ce != cudaSuccess) {
        ctx->worker_error.store(EIO);
        n = -EIO;
      }
      uint64_t v = ((uint64_t)(n < 0 ? 0xFFFFFFFFull : (uint64_t)n) << 32) | seq;
      if (!copy) v |= 1ull << 63;  // "not copied: pull it from the mapping"
      // The doorbell goes on a separate stream that waits for this copy: copy streams then
      // carry back-to-back copies only, so the engine never idles behind a memory op.
      if (!streamed || n < 0) {
        if (copy && n > 0) {
          cudaEventRecord(ctx->bell_ev[wid], st);
          cudaStreamWaitEvent(bs, ctx->bell_ev[wid], 0);
        }
        CUresult cr = ctx->write_value64((CUstream)bs, (CUdeviceptr)(ctx->d_doorbell + li), (cuuint64_t)v, 0);
        if (cr != CUDA_SUCCESS) ctx->worker_error.store(EIO);
      }
      // The driver may hold freshly enqueued work in its push buffer until the next call on
      // the stream; this worker may not make one for a while (it spins on the ring), and
      // the persistent kernel is waiting on exactly this doorbell.  Kick both streams.
      cudaStreamQuery(st);
      cudaStreamQuery(bs);
      ctx->t_xfer.fetch_add((int64_t)(now_ns() - t1), std::memory_order_relaxed);
    } else {
      RpcResp* r = &ctx->h_resp[(int64_t)slot * ctx->landing_halves + half];
      r->nbytes = n;
      r->buf = (mapped_zc || hybrid) ? -1 : b;
      if (bounce && n <= 0) ctx->bounce_last[b] = 0;  // nothing to pull: buffer stays free
      __atomic_store_n(&r->seq, seq, __ATOMIC_RELEASE);
    }
    ctx->n_served.fetch_add(1, std::memory_order_relaxed);
    ctx->w_phase[wid].store(3, std::memory_order_relaxed);
  }
}

static void stop_workers(gfs_ctx* ctx) {
  ctx->stop.store(true);
  for (auto& t : ctx->workers)
    if (t.joinable()) t.join();
  ctx->workers.clear();
}

// After a device error some ring positions were reserved but never written (rpc_submit
// gave up) and some bounce buffers were never released: workers stay parked on them and the
// next launch, whose ring base is the served count, would write positions nobody waits for.
// Restart the daemon from the served count with a clean ring and free buffers.
static void reset_daemon(gfs_ctx* ctx) {
  stop_workers(ctx);
  for (auto s : ctx->worker_streams)
    if (s) cudaStreamSynchronize(s);
  for (auto s : ctx->bell_streams)
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
  const uint64_t served = __atomic_load_n(ctx->h_served, __ATOMIC_ACQUIRE);
  memset(ctx->h_ring, 0, (size_t)ctx->ring_size * sizeof(RpcReq));
  memset(ctx->h_consumed, 0, (size_t)ctx->ring_size * 4);
  memset(ctx->h_resp, 0, (size_t)ctx->n_ctas * ctx->landing_halves * sizeof(RpcResp));
  if (ctx->h_release) memset(ctx->h_release, 0, ctx->bounce_last.size() * 4);
  std::fill(ctx->bounce_last.begin(), ctx->bounce_last.end(), 0u);
  std::fill(ctx->bounce_ce.begin(), ctx->bounce_ce.end(), (char)0);  // worker streams were synchronized
  if (ctx->d_doorbell) cudaMemset(ctx->d_doorbell, 0, (size_t)ctx->n_ctas * ctx->landing_halves * 8);
  if (ctx->d_landed) cudaMemset(ctx->d_landed, 0, (size_t)ctx->n_ctas * ctx->landing_halves * 8);
  ctx->req_head.store(served);
  ctx->stop.store(false);
  for (int w = 0; w < ctx->cfg.io_workers; w++) ctx->workers.emplace_back(worker_main, ctx, w);
}

// ------------------------------------------------------------------- lifecycle

static void free_all(gfs_ctx* ctx) {
  stop_workers(ctx);
  for (auto& f : ctx->files) {
    if (f.fd_direct >= 0) close(f.fd_direct);
    if (f.fd_buffered >= 0) close(f.fd_buffered);
    if (f.d_pt) cudaFree(f.d_pt);
    unmap_file(f);
  }
  ctx->files.clear();
  for (auto s : ctx->worker_streams)
    if (s) cudaStreamDestroy(s);
  for (auto s : ctx->bell_streams)
    if (s) cudaStreamDestroy(s);
  for (auto ev : ctx->bell_ev)
    if (ev) cudaEventDestroy(ev);
  void* dev[] = {ctx->d_frames, ctx->d_fkey, ctx->d_fstate, ctx->d_own_q, ctx->d_retired, ctx->d_rpool, ctx->d_landed,
                 ctx->d_gfifo, ctx->d_recycled, ctx->d_g, ctx->d_landing, ctx->d_doorbell,
                 ctx->d_done_pos, ctx->d_stats, ctx->d_scratch, ctx->d_owner, ctx->d_slot_busy};
  for (void* p : dev)
    if (p) cudaFree(p);
  ctx->d_segs.release();
  ctx->d_prog_off.release();
  ctx->d_dst_off.release();
  ctx->d_seg_dst.release();
  ctx->d_order.release();
  ctx->d_files.release();
  for (auto& l : ctx->d_logs) l.release();
  for (auto ev : ctx->bounce_ev)
    if (ev) cudaEventDestroy(ev);
  void* host[] = {ctx->h_ring, ctx->h_consumed, ctx->h_resp, ctx->h_staging, ctx->h_served, ctx->h_bounce,
                  ctx->h_release};
  for (void* p : host)
    if (p) cudaFreeHost(p);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
}

extern "C" int gfs_create(const gfs_config* cfg_in, gfs_ctx** out) {
  if (!cfg_in || !out) return fail(GFS_EINVAL, "gfs_create: null argument");
  *out = nullptr;
  gfs_config cfg = *cfg_in;
  if (cfg.page_size < 4096 || cfg.page_size % 4096)
    return fail(GFS_EINVAL, "page_size must be a positive multiple of 4096 (got %lld)",
                (long long)cfg.page_size);
  if (cfg.prefetch_bytes < 0 || cfg.prefetch_bytes % cfg.page_size)
    return fail(GFS_EINVAL, "prefetch_bytes must be a multiple of page_size");
  if (cfg.cache_bytes < cfg.page_size) return fail(GFS_EINVAL, "cache_bytes smaller than one page");
  if (cfg.resident_limit < 1) return fail(GFS_EINVAL, "resident_limit must be >= 1");
  if (cfg.staging_bytes < 1) return fail(GFS_EINVAL, "staging_bytes must be >= 1");
  if (cfg.policy != GFS_POLICY_GLOBAL_LRU && cfg.policy != GFS_POLICY_PER_TB_LRA)
    return fail(GFS_EINVAL, "unknown policy %d", cfg.policy);
  if (cfg.transfer < GFS_XFER_ZEROCOPY || cfg.transfer > GFS_XFER_PREAD_HYBRID)
    return fail(GFS_EINVAL, "unknown transfer %d", cfg.transfer);
  if (cfg.readahead < GFS_RA_STATIC || cfg.readahead > GFS_RA_ONDEMAND)
    return fail(GFS_EINVAL, "unknown readahead mode %d", cfg.readahead);
  if (cfg.readahead != GFS_RA_STATIC && (cfg.ra_max_bytes < cfg.page_size || cfg.ra_max_bytes % cfg.page_size))
    return fail(GFS_EINVAL, "ra_max_bytes must be a positive multiple of page_size");
  if (cfg.ra_init_bytes < 0 || cfg.ra_init_bytes % cfg.page_size)
    return fail(GFS_EINVAL, "ra_init_bytes must be 0 or a multiple of page_size");
  if (cfg.cta_threads != 128 && cfg.cta_threads != 256 && cfg.cta_threads != 512) cfg.cta_threads = 256;
  if (cfg.io_workers < 1) cfg.io_workers = 1;
  if (cfg.io_workers > 256) cfg.io_workers = 256;
  if (cfg.rpc_slots == 0) cfg.rpc_slots = 128;  // rpc.n_slots default (config.py)
  if (cfg.rpc_slots < 1) return fail(GFS_EINVAL, "rpc_slots must be >= 1");
  const int64_t nframes = cfg.cache_bytes / cfg.page_size;
  if (nframes >= (int64_t)PT_INFLIGHT) return fail(GFS_EINVAL, "too many frames (%lld)", (long long)nframes);
  const int64_t quota = nframes / cfg.resident_limit;  // gpu_cache.py:32-34
  if (cfg.policy == GFS_POLICY_PER_TB_LRA && quota < 1 && !cfg.raw_mode)
    return fail(GFS_EINVAL,
                "per-tb-lra needs cache_bytes/page_size >= resident TBs (%lld frames for %d TBs)",
                (long long)nframes, cfg.resident_limit);
  int64_t pb_cap = cfg.prefetch_bytes;
  if (cfg.readahead == GFS_RA_DOUBLING && cfg.ra_max_bytes - cfg.page_size > pb_cap)
    pb_cap = cfg.ra_max_bytes - cfg.page_size;
  // ondemand: a landing half holds a whole window or synchronous span, and an adopted window
  // is the private buffer in full (its first page included)
  if (cfg.readahead == GFS_RA_ONDEMAND)
    pb_cap = round_up(std::max(cfg.ra_max_bytes, cfg.page_size + cfg.prefetch_bytes), cfg.page_size);
  if (pb_cap / cfg.page_size >= MAX_PB_ENTRIES)
    return fail(GFS_EINVAL, "private buffer of %lld pages exceeds %d", (long long)(pb_cap / cfg.page_size),
                MAX_PB_ENTRIES - 1);

  gfs_ctx* ctx = new gfs_ctx();
  ctx->cfg = cfg;
  ctx->nframes = nframes;
  ctx->quota = quota;
  ctx->pb_cap = pb_cap;
  int64_t span_max = cfg.readahead == GFS_RA_ONDEMAND ? pb_cap : cfg.page_size + pb_cap;
  if (cfg.raw_mode) span_max = std::max<int64_t>(cfg.max_request_bytes, 4096);
  ctx->slot_bytes = round_up(span_max, 4096);
  // ondemand readahead: the next window lands in the other half while the CTA reads one
  ctx->landing_halves = (cfg.readahead == GFS_RA_ONDEMAND && !cfg.raw_mode) ? 2 : 1;
  auto bail = [&](int rc) {
    free_all(ctx);
    delete ctx;
    return rc;
  };
#define TRY(expr)                                                                            \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return bail(fail(GFS_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_)));          \
  } while (0)
  TRY(cudaSetDevice(cfg.device));
  TRY(cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, cfg.device));
  int per_sm = 0;
  TRY(occupancy_gread(cfg.cta_threads, &per_sm));
  int hw = std::max(1, per_sm) * ctx->sms;
  int want = cfg.max_ctas > 0 ? std::min(cfg.max_ctas, cfg.resident_limit) : cfg.resident_limit;
  ctx->n_ctas = std::max(1, std::min(want, hw));
  uint32_t q = 1;
  while (q < (uint32_t)(4 * ctx->n_ctas) || q < 1024) q <<= 1;
  ctx->ring_size = q;
  ctx->gfifo_cap = 2 * nframes + 65536;

  TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  TRY(cudaEventCreate(&ctx->ev0));
  TRY(cudaEventCreate(&ctx->ev1));
  if (cfg.transfer == GFS_XFER_DMA || cfg.transfer == GFS_XFER_MAPPED ||
      cfg.transfer == GFS_XFER_MAPPED_HYBRID || cfg.transfer == GFS_XFER_PREAD_HYBRID) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    TRY(cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &qr));
    if (!fn || qr != cudaDriverEntryPointSuccess)
      return bail(fail(GFS_ECUDA, "cuStreamWriteValue64 unavailable (stream memory operations)"));
    ctx->write_value64 = (CUresult(*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int))fn;
    // a few copy streams shared by the workers (streams are thread-safe): every extra
    // stream risks sharing a hardware queue with the persistent kernel's stream
    int nstreams = 2;
    if (const char* e = getenv("GFS_COPY_STREAMS")) nstreams = std::max(1, std::min(16, atoi(e)));  // experiments
    if (const char* e = getenv("GFS_CE_MIN_KIB")) ctx->ce_min = std::max(4, atoi(e)) * 1024ll;  // experiments
    // Copy-engine transfers complete while the persistent kernel runs: their streams must
    // not share a hardware queue with the kernel's stream (CUDA_DEVICE_MAX_CONNECTIONS too
    // small, or CUDA initialised before the package could raise it; with enough queues a
    // new stream can still land on the kernel stream's queue).  Probe it: a kernel on the
    // run stream waits (bounded) for one value written by each copy / doorbell stream.  If a
    // write queues behind the kernel, make new streams (up to 4 tries); if that never works,
    // fall back to the SM-pull transfer moving the same bytes (mapped_dma / mapped_hybrid ->
    // mapped, dma -> bounce).
    unsigned long long* d_flags = nullptr;
    TRY(cudaMalloc(&d_flags, (size_t)(4 * nstreams + 1) * 8));
    int ok = 0;
    std::vector<cudaStream_t> retired;  // kept alive while retrying so new streams move on
    for (int attempt = 0; attempt < 4 && !ok; attempt++) {
      for (auto s : ctx->worker_streams) retired.push_back(s);
      for (auto s : ctx->bell_streams) retired.push_back(s);
      ctx->worker_streams.assign((size_t)std::min(cfg.io_workers, nstreams), nullptr);
      ctx->bell_streams.assign((size_t)std::min(cfg.io_workers, nstreams), nullptr);
      for (auto& s : ctx->worker_streams) TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      for (auto& s : ctx->bell_streams) TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      std::vector<cudaStream_t> probe(ctx->worker_streams);
      probe.insert(probe.end(), ctx->bell_streams.begin(), ctx->bell_streams.end());
      int* d_ok = (int*)(d_flags + probe.size());
      TRY(cudaMemsetAsync(d_flags, 0, probe.size() * 8 + 8, ctx->stream));
      TRY(launch_queue_probe(d_flags, (int)probe.size(), 500ull * 1000000ull, d_ok, ctx->stream));
      for (size_t i = 0; i < probe.size(); i++) {
        if (ctx->write_value64((CUstream)probe[i], (CUdeviceptr)(d_flags + i), 1, 0) != CUDA_SUCCESS) {
          cudaFree(d_flags);
          return bail(fail(GFS_ECUDA, "cuStreamWriteValue64 failed on a copy stream"));
        }
        cudaStreamQuery(probe[i]);
      }
      TRY(cudaStreamSynchronize(ctx->stream));
      TRY(cudaMemcpy(&ok, d_ok, 4, cudaMemcpyDeviceToHost));
      TRY(cudaDeviceSynchronize());
      ctx->probe_attempts = attempt + 1;
    }
    for (auto s : retired) cudaStreamDestroy(s);
    cudaFree(d_flags);
    if (ok && ctx->probe_attempts > 1)
      fprintf(stderr, "libgfs: copy streams re-created %d time(s) to get hardware queues apart from the kernel's\n",
              ctx->probe_attempts - 1);
    if (!ok) {
      const int was = cfg.transfer;
      cfg.transfer = (was == GFS_XFER_DMA || was == GFS_XFER_PREAD_HYBRID) ? GFS_XFER_BOUNCE : GFS_XFER_MAPPED_ZC;
      ctx->cfg.transfer = cfg.transfer;
      ctx->downgraded_from = was;
      for (auto s : ctx->worker_streams) cudaStreamDestroy(s);
      for (auto s : ctx->bell_streams) cudaStreamDestroy(s);
      ctx->worker_streams.clear();
      ctx->bell_streams.clear();
      ctx->write_value64 = nullptr;
      const char* mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
      fprintf(stderr,
              "libgfs: copy streams share a hardware queue with the kernel stream "
              "(CUDA_DEVICE_MAX_CONNECTIONS=%s when CUDA started?): transfer %d -> %d (SM pull)\n",
              mc ? mc : "unset", was, cfg.transfer);
    }
  }
  if (!cfg.raw_mode) {
    TRY(cudaMalloc(&ctx->d_frames, (size_t)(nframes * cfg.page_size)));
    TRY(cudaMalloc(&ctx->d_fkey, (size_t)nframes * 8));
    TRY(cudaMalloc(&ctx->d_fstate, (size_t)nframes * 4));
    ctx->ret_npools = std::min(RET_POOLS, std::max(1, ctx->n_ctas));
    ctx->ret_pcap = nframes + 64;
    TRY(cudaMalloc(&ctx->d_retired, (size_t)ctx->ret_npools * (size_t)ctx->ret_pcap * 4));
    TRY(cudaMalloc(&ctx->d_rpool, (size_t)RET_POOLS * 16 * 8));
    TRY(cudaMalloc(&ctx->d_recycled, (size_t)nframes * 4));
    if (cfg.policy == GFS_POLICY_PER_TB_LRA)
      TRY(cudaMalloc(&ctx->d_own_q, (size_t)ctx->n_ctas * (size_t)std::max<int64_t>(quota, 1) * 4));
    else
      TRY(cudaMalloc(&ctx->d_gfifo, (size_t)ctx->gfifo_cap * 4));
  }
  TRY(cudaMalloc(&ctx->d_g, sizeof(DevGlobals)));
  TRY(cudaMalloc(&ctx->d_done_pos, (size_t)ctx->ring_size * 8));
  TRY(cudaMalloc(&ctx->d_stats, (size_t)ctx->n_ctas * GFS_NSTATS * 8));
  TRY(cudaMalloc(&ctx->d_scratch, 64));
  TRY(cudaMalloc(&ctx->d_slot_busy, (size_t)cfg.rpc_slots * 4));

  TRY(cudaHostAlloc(&ctx->h_ring, (size_t)ctx->ring_size * sizeof(RpcReq),
                    cudaHostAllocMapped | cudaHostAllocPortable));
  TRY(cudaHostAlloc(&ctx->h_consumed, (size_t)ctx->ring_size * 4, cudaHostAllocMapped | cudaHostAllocPortable));
  TRY(cudaHostAlloc(&ctx->h_resp, (size_t)ctx->n_ctas * ctx->landing_halves * sizeof(RpcResp),
                    cudaHostAllocMapped | cudaHostAllocPortable));
  if (cfg.transfer == GFS_XFER_ZEROCOPY)
    TRY(cudaHostAlloc(&ctx->h_staging, (size_t)(ctx->n_ctas * ctx->landing_halves * ctx->slot_bytes),
                      cudaHostAllocMapped | cudaHostAllocPortable));
  if (cfg.transfer == GFS_XFER_MAPPED_ZC)
    TRY(cudaMalloc(&ctx->d_landing, (size_t)(ctx->n_ctas * ctx->landing_halves * ctx->slot_bytes)));
  if (cfg.transfer == GFS_XFER_BOUNCE) {
    // ~24 MiB pool in total so it stays resident in the host LLC, 2..8 buffers per worker
    ctx->nbounce = (int)std::max<int64_t>(2, (24ll << 20) / (ctx->slot_bytes * cfg.io_workers));
    if (ctx->nbounce > 8) ctx->nbounce = 8;
    const int64_t nb = (int64_t)cfg.io_workers * ctx->nbounce;
    TRY(cudaHostAlloc(&ctx->h_bounce, (size_t)(ctx->slot_bytes * nb),
                      cudaHostAllocMapped | cudaHostAllocPortable));
    TRY(cudaHostAlloc(&ctx->h_release, (size_t)nb * 4, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(ctx->h_release, 0, (size_t)nb * 4);
    ctx->bounce_last.assign((size_t)nb, 0);
    TRY(cudaMalloc(&ctx->d_landing, (size_t)(ctx->n_ctas * ctx->landing_halves * ctx->slot_bytes)));
  }
  memset(ctx->h_ring, 0, (size_t)ctx->ring_size * sizeof(RpcReq));
  memset(ctx->h_consumed, 0, (size_t)ctx->ring_size * 4);
  memset(ctx->h_resp, 0, (size_t)ctx->n_ctas * ctx->landing_halves * sizeof(RpcResp));
  TRY(cudaHostAlloc(&ctx->h_served, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(ctx->h_served, 0, 64);
  if (cfg.transfer == GFS_XFER_DMA || cfg.transfer == GFS_XFER_MAPPED ||
      cfg.transfer == GFS_XFER_MAPPED_HYBRID || cfg.transfer == GFS_XFER_PREAD_HYBRID) {
    TRY(cudaMalloc(&ctx->d_landing, (size_t)(ctx->n_ctas * ctx->landing_halves * ctx->slot_bytes)));
    // experiments: GFS_STREAM_PIECE_MIB (0 = off, the default: whole-window copies measured
    // faster on the headline, 54.0 vs 51.9 GB/s with 4 MiB pieces)
    ctx->stream_piece = 0;
    if (const char* e = getenv("GFS_STREAM_PIECE_MIB")) ctx->stream_piece = (int64_t)atoi(e) << 20;
    ctx->stream_pieces = ctx->stream_piece > 0 && !cfg.raw_mode && cfg.transfer != GFS_XFER_MAPPED_HYBRID &&
                         cfg.transfer != GFS_XFER_PREAD_HYBRID &&
                         ctx->slot_bytes >= 2 * ctx->stream_piece;
    TRY(cudaMalloc(&ctx->d_landed, (size_t)ctx->n_ctas * ctx->landing_halves * 8));
    TRY(cudaMemset(ctx->d_landed, 0, (size_t)ctx->n_ctas * ctx->landing_halves * 8));
    TRY(cudaMalloc(&ctx->d_doorbell, (size_t)ctx->n_ctas * ctx->landing_halves * 8));
    TRY(cudaMemset(ctx->d_doorbell, 0, (size_t)ctx->n_ctas * ctx->landing_halves * 8));
    ctx->bell_ev.resize((size_t)cfg.io_workers, nullptr);
    for (auto& ev : ctx->bell_ev) TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  if (cfg.transfer == GFS_XFER_PREAD_HYBRID) {
    // a pool both the copy engine (large spans) and the CTAs (small spans, mapped) read
    ctx->nbounce = (int)std::max<int64_t>(2, (48ll << 20) / (ctx->slot_bytes * cfg.io_workers));
    if (ctx->nbounce > 8) ctx->nbounce = 8;
    const int64_t nb = (int64_t)cfg.io_workers * ctx->nbounce;
    TRY(cudaHostAlloc(&ctx->h_bounce, (size_t)(ctx->slot_bytes * nb), cudaHostAllocMapped | cudaHostAllocPortable));
    TRY(cudaHostAlloc(&ctx->h_release, (size_t)nb * 4, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(ctx->h_release, 0, (size_t)nb * 4);
    ctx->bounce_last.assign((size_t)nb, 0);
    ctx->bounce_ce.assign((size_t)nb, 0);
    ctx->bounce_ev.resize((size_t)nb, nullptr);
    for (auto& ev : ctx->bounce_ev) TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  if (cfg.transfer == GFS_XFER_DMA) {
    // ~48 MiB of bounce buffers in total (LLC-sized), at least 2 per worker
    ctx->nbounce = (int)std::max<int64_t>(2, (48ll << 20) / (ctx->slot_bytes * cfg.io_workers));
    if (ctx->nbounce > 8) ctx->nbounce = 8;
    TRY(cudaHostAlloc(&ctx->h_bounce, (size_t)(ctx->slot_bytes * cfg.io_workers * ctx->nbounce),
                      cudaHostAllocPortable));
    ctx->bounce_ev.resize((size_t)cfg.io_workers * ctx->nbounce, nullptr);
    for (auto& ev : ctx->bounce_ev) TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  TRY(cudaDeviceSynchronize());
#undef TRY
  if (cfg.numa_pin) ctx->local_cpus = gpu_local_cpus(cfg.device);
  for (int w = 0; w < cfg.io_workers; w++) ctx->workers.emplace_back(worker_main, ctx, w);
  *out = ctx;
  return GFS_OK;
}

extern "C" void gfs_destroy(gfs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
}

extern "C" int gfs_resident_ctas(gfs_ctx* ctx) { return ctx ? ctx->n_ctas : 0; }

extern "C" int gfs_transfer(gfs_ctx* ctx, int* transfer, int* downgraded_from) {
  if (!ctx || !transfer) return fail(GFS_EINVAL, "gfs_transfer: null argument");
  *transfer = ctx->cfg.transfer;
  if (downgraded_from) *downgraded_from = ctx->downgraded_from;

  return GFS_OK;
}

// ------------------------------------------------------------------- files

extern "C" int gfs_gopen(gfs_ctx* ctx, const char* path, int flags, int64_t content_id, int* fid) {
  if (!ctx || !path || !fid) return fail(GFS_EINVAL, "gfs_gopen: null argument");
  if (ctx->files.size() >= 65535) return fail(GFS_EINVAL, "gfs_gopen: at most 65535 files per context");
  HostFile f;
  f.path = path;
  f.read_only = (flags & GFS_O_RDWR) ? 0 : 1;
  f.content_id = content_id;
  f.fd_buffered = open(path, O_RDONLY);
  if (f.fd_buffered < 0) return fail(GFS_EIO, "open %s: %s", path, strerror(errno));
  if (ctx->cfg.io_direct) f.fd_direct = open(path, O_RDONLY | O_DIRECT);  // may be -1: buffered only
  struct stat sb;
  if (fstat(f.fd_buffered, &sb) != 0) {
    close(f.fd_buffered);
    if (f.fd_direct >= 0) close(f.fd_direct);
    return fail(GFS_EIO, "stat %s: %s", path, strerror(errno));
  }
  f.size = (int64_t)sb.st_size;
  if (f.size >= (1ll << 48)) {  // ring entries carry 48-bit offsets
    close(f.fd_buffered);
    if (f.fd_direct >= 0) close(f.fd_direct);
    return fail(GFS_EINVAL, "gfs_gopen: %s is larger than 256 TiB", path);
  }
  f.npages = (f.size + ctx->cfg.page_size - 1) / ctx->cfg.page_size + 1;
  cudaSetDevice(ctx->cfg.device);
  if (!ctx->cfg.raw_mode) {
    cudaError_t e = cudaMalloc(&f.d_pt, (size_t)f.npages * 4);
    if (e != cudaSuccess) {
      close(f.fd_buffered);
      if (f.fd_direct >= 0) close(f.fd_direct);
      return fail(GFS_ECUDA, "page table for %s: %s", path, cudaGetErrorString(e));
    }
  }
  f.open = true;
  ctx->files.push_back(f);
  *fid = (int)ctx->files.size() - 1;
  return GFS_OK;
}

extern "C" int gfs_gclose(gfs_ctx* ctx, int fid) {
  if (!ctx || fid < 0 || fid >= (int)ctx->files.size() || !ctx->files[fid].open)
    return fail(GFS_EINVAL, "gfs_gclose: bad file id %d", fid);
  HostFile& f = ctx->files[fid];
  cudaSetDevice(ctx->cfg.device);
  cudaStreamSynchronize(ctx->stream);
  if (f.fd_direct >= 0) close(f.fd_direct);
  if (f.fd_buffered >= 0) close(f.fd_buffered);
  if (f.d_pt) cudaFree(f.d_pt);
  unmap_file(f);
  f.fd_direct = f.fd_buffered = -1;
  f.d_pt = nullptr;
  f.open = false;
  return GFS_OK;
}

extern "C" int gfs_file_size(gfs_ctx* ctx, int fid, int64_t* size) {
  if (!ctx || !size || fid < 0 || fid >= (int)ctx->files.size() || !ctx->files[fid].open)
    return fail(GFS_EINVAL, "gfs_file_size: bad file id %d", fid);
  *size = ctx->files[fid].size;
  return GFS_OK;
}

// ------------------------------------------------------------------- run

static int upload_files(gfs_ctx* ctx) {
  std::vector<DevFile> df(ctx->files.size());
  for (size_t i = 0; i < ctx->files.size(); i++) {
    const HostFile& f = ctx->files[i];
    df[i].pt = f.d_pt;
    df[i].size = f.open ? f.size : 0;
    df[i].npages = f.npages;
    df[i].read_only = f.read_only;
    df[i].content_id = (int32_t)f.content_id;
    df[i].map = f.dmap ? f.dmap - f.map_lo : nullptr;  // map + file offset = device address
  }
  CUDA_TRY(ctx->d_files.reserve(std::max<size_t>(df.size(), 1)));
  if (!df.empty())
    CUDA_TRY(cudaMemcpyAsync(ctx->d_files.p, df.data(), df.size() * sizeof(DevFile),
                             cudaMemcpyHostToDevice, ctx->stream));
  return GFS_OK;
}

static int upload_program(gfs_ctx* ctx, const gfs_program* prog, int64_t* n_segs_out) {
  const int n_tb = prog->n_tb;
  const int64_t n_segs = prog->prog_off[n_tb];
  CUDA_TRY(ctx->d_segs.reserve((size_t)std::max<int64_t>(3 * n_segs, 3)));
  CUDA_TRY(ctx->d_prog_off.reserve((size_t)n_tb + 1));
  CUDA_TRY(ctx->d_dst_off.reserve((size_t)std::max(n_tb, 1)));
  CUDA_TRY(ctx->d_order.reserve((size_t)std::max(n_tb, 1)));
  if (n_segs)
    CUDA_TRY(cudaMemcpyAsync(ctx->d_segs.p, prog->segs, (size_t)(3 * n_segs) * 8,
                             cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(ctx->d_prog_off.p, prog->prog_off, (size_t)(n_tb + 1) * 8,
                           cudaMemcpyHostToDevice, ctx->stream));
  if (n_tb) {
    CUDA_TRY(cudaMemcpyAsync(ctx->d_dst_off.p, prog->dst_off, (size_t)n_tb * 8,
                             cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_order.p, prog->order, (size_t)n_tb * 4,
                             cudaMemcpyHostToDevice, ctx->stream));
  }
  *n_segs_out = n_segs;
  return GFS_OK;
}

static int validate_program(gfs_ctx* ctx, const gfs_program* prog, uint64_t dst_bytes, bool has_dst) {
  if (!prog || prog->n_tb < 0 || !prog->prog_off) return fail(GFS_EINVAL, "bad program");
  if (prog->request_bytes < 1) return fail(GFS_EINVAL, "request_bytes must be positive");
  if (ctx->cfg.raw_mode && prog->request_bytes > ctx->slot_bytes)
    return fail(GFS_EINVAL, "raw request of %lld bytes exceeds the staging slot (%lld)",
                (long long)prog->request_bytes, (long long)ctx->slot_bytes);
  std::vector<char> seen((size_t)prog->n_tb, 0);
  for (int k = 0; k < prog->n_tb; k++) {
    int t = prog->order[k];
    if (t < 0 || t >= prog->n_tb || seen[t]) return fail(GFS_EINVAL, "order is not a permutation");
    seen[t] = 1;
    if (prog->prog_off[k + 1] < prog->prog_off[k]) return fail(GFS_EINVAL, "prog_off not monotone");
  }
  for (int t = 0; t < prog->n_tb; t++) {
    int64_t pos = prog->dst_off[t];
    for (int64_t s = prog->prog_off[t]; s < prog->prog_off[t + 1]; s++) {
      int64_t fid = prog->segs[3 * s], off = prog->segs[3 * s + 1], len = prog->segs[3 * s + 2];
      if (fid < 0 || fid >= (int64_t)ctx->files.size() || !ctx->files[fid].open)
        return fail(GFS_EINVAL, "segment %lld names unopened file %lld", (long long)s, (long long)fid);
      if (off < 0 || len < 0) return fail(GFS_EINVAL, "negative segment offset/length");
      pos += len;
      if (has_dst && (uint64_t)pos > dst_bytes)
        return fail(GFS_EINVAL, "user buffer of %llu bytes too small for TB %d's program",
                    (unsigned long long)dst_bytes, t);
    }
  }
  return GFS_OK;
}

static int validate_consumer(const gfs_consumer* k, const gfs_program* prog, bool has_dst) {
  if (!k || k->kind == GFS_CONSUME_NONE) return GFS_OK;
  if (k->kind < GFS_CONSUME_NONE || k->kind > GFS_CONSUME_KMEANS_F32)
    return fail(GFS_EINVAL, "unknown consumer kind %d", k->kind);
  if (!has_dst) return fail(GFS_EINVAL, "consumers read the user buffer: dst is required");
  const bool matrix = k->kind == GFS_CONSUME_GEMV_F32 || k->kind == GFS_CONSUME_GEMVT_F32 ||
                      k->kind == GFS_CONSUME_BICG_F32 || k->kind == GFS_CONSUME_KMEANS_F32;
  if (matrix && (k->cols <= 0 || k->cols % 4))
    return fail(GFS_EINVAL, "matrix consumers need cols > 0, a multiple of 4");
  if ((k->kind == GFS_CONSUME_GEMV_F32 || k->kind == GFS_CONSUME_BICG_F32) && (!k->x || !k->y))
    return fail(GFS_EINVAL, "GEMV needs x [cols] and y [rows]");
  if ((k->kind == GFS_CONSUME_GEMVT_F32 || k->kind == GFS_CONSUME_BICG_F32) && (!k->x2 || !k->y2))
    return fail(GFS_EINVAL, "GEMVT needs x2 [rows] and y2 [cols]");
  if (k->kind == GFS_CONSUME_KMEANS_F32) {
    if (k->k < 1 || k->k > GFS_KMEANS_MAX_K)
      return fail(GFS_EINVAL, "kmeans needs 1 <= k <= %d centroids", GFS_KMEANS_MAX_K);
    if (!k->x || !k->y || !k->out) return fail(GFS_EINVAL, "kmeans needs x (centroids), y (sums), out (counts)");
    if (2 * (int64_t)k->k * k->cols * 4 + 4 * (int64_t)k->k > 32 * 1024)
      return fail(GFS_EINVAL, "kmeans state (2 k cols floats) must fit 32 KiB of shared memory");
  }
  if ((k->kind == GFS_CONSUME_SUM64 || k->kind == GFS_CONSUME_NN_F32) && !k->out)
    return fail(GFS_EINVAL, "consumer needs out");
  // every request starts on a record: 8 B words (sum64, nn), 16 B vectors (matrices),
  // whole points (kmeans)
  const int64_t align = k->kind == GFS_CONSUME_KMEANS_F32 ? k->cols * 4 : matrix ? 16 : 8;
  if (prog->request_bytes % align) return fail(GFS_EINVAL, "consumer needs %lld-byte aligned requests", (long long)align);
  const int64_t n_segs = prog->prog_off[prog->n_tb];
  for (int64_t s = 0; s < n_segs; s++)
    if (prog->segs[3 * s + 1] % align || prog->segs[3 * s + 2] % align)
      return fail(GFS_EINVAL, "consumer needs %lld-byte aligned segments", (long long)align);
  for (int t = 0; t < prog->n_tb; t++)
    if (prog->dst_off[t] % 16) return fail(GFS_EINVAL, "consumer needs 16-byte aligned user-buffer offsets");
  return GFS_OK;
}

static int run_prepared(gfs_ctx* ctx, const gfs_program* prog, void* dst, const gfs_consumer* cons,
                        gfs_launch_fn launch, void* user, gfs_stats* out, uint64_t w0);

extern "C" int gfs_run(gfs_ctx* ctx, const gfs_program* prog, void* dst, uint64_t dst_bytes,
                       gfs_stats* out) {
  return gfs_run_consume(ctx, prog, dst, dst_bytes, nullptr, out);
}

// A user kernel over the device gread (gfs_device.cuh): n_tb TBs with empty built-in
// programs; the kernel decides what each TB reads.
extern "C" int gfs_run_kernel(gfs_ctx* ctx, int32_t n_tb, const int32_t* order, gfs_launch_fn launch,
                              void* user, gfs_stats* out) {
  const uint64_t w0 = now_ns();
  if (!ctx || !launch || !out || n_tb < 0) return fail(GFS_EINVAL, "gfs_run_kernel: bad argument");
  if (ctx->poisoned)
    return fail(GFS_ESTATE, "context unusable: an earlier run's kernel never finished (destroy it)");
  if (ctx->cfg.raw_mode) return fail(GFS_EINVAL, "gfs_run_kernel: raw mode has no page cache to read through");
  std::vector<int64_t> prog_off((size_t)n_tb + 1, 0), dst_off((size_t)std::max(n_tb, 1), 0);
  std::vector<int32_t> ord((size_t)std::max(n_tb, 1));
  for (int i = 0; i < n_tb; i++) ord[i] = order ? order[i] : i;
  gfs_program prog{};
  prog.n_tb = n_tb;
  prog.request_bytes = ctx->cfg.page_size;
  prog.segs = nullptr;
  prog.prog_off = prog_off.data();
  prog.dst_off = dst_off.data();
  prog.order = ord.data();
  int rc = validate_program(ctx, &prog, 0, false);
  if (rc) return rc;
  const int xfer = ctx->cfg.transfer;
  if (xfer == GFS_XFER_MAPPED || xfer == GFS_XFER_MAPPED_ZC || xfer == GFS_XFER_MAPPED_HYBRID)
    for (auto& f : ctx->files)  // any byte of an open file may be read
      if (f.open && f.size > 0 && (rc = map_range(f, 0, f.size))) return rc;
  return run_prepared(ctx, &prog, nullptr, nullptr, launch, user, out, w0);
}

extern "C" int gfs_run_consume(gfs_ctx* ctx, const gfs_program* prog, void* dst, uint64_t dst_bytes,
                               const gfs_consumer* cons, gfs_stats* out) {
  const uint64_t w0 = now_ns();
  if (!ctx || !prog || !out) return fail(GFS_EINVAL, "gfs_run: null argument");
  if (ctx->poisoned)
    return fail(GFS_ESTATE, "context unusable: an earlier run's kernel never finished (destroy it)");
  int rc = validate_program(ctx, prog, dst_bytes, dst != nullptr);
  if (rc) return rc;
  if ((rc = validate_consumer(cons, prog, dst != nullptr))) return rc;
  const int xfer = ctx->cfg.transfer;
  if (xfer == GFS_XFER_MAPPED || xfer == GFS_XFER_MAPPED_ZC || xfer == GFS_XFER_MAPPED_HYBRID) {
    // pin what this run can touch: its segments plus one span of read-ahead past each end
    std::vector<int64_t> lo(ctx->files.size(), INT64_MAX), hi(ctx->files.size(), -1);
    for (int64_t s = 0; s < prog->prog_off[prog->n_tb]; s++) {
      const int64_t fid = prog->segs[3 * s], off = prog->segs[3 * s + 1], len = prog->segs[3 * s + 2];
      lo[fid] = std::min(lo[fid], off);
      hi[fid] = std::max(hi[fid], off + len + ctx->slot_bytes);
    }
    for (size_t f = 0; f < ctx->files.size(); f++)
      if (hi[f] > lo[f] && ctx->files[f].open && ctx->files[f].size > 0 && lo[f] < ctx->files[f].size)
        if ((rc = map_range(ctx->files[f], lo[f], hi[f]))) return rc;
  }
  return run_prepared(ctx, prog, dst, cons, nullptr, nullptr, out, w0);
}

// The run itself, shared by gfs_run_consume (the built-in strided driver) and
// gfs_run_kernel (a user kernel launched by `launch`).
static int run_prepared(gfs_ctx* ctx, const gfs_program* prog, void* dst, const gfs_consumer* cons,
                        gfs_launch_fn launch, void* user, gfs_stats* out, uint64_t w0) {
  int rc;
  CUDA_TRY(cudaSetDevice(ctx->cfg.device));
  const gfs_config& cfg = ctx->cfg;
  int64_t n_segs = 0;
  if ((rc = upload_files(ctx)) || (rc = upload_program(ctx, prog, &n_segs))) return rc;

  // log capacities: one delivery per page step, bounded by pages + 2 per request.  A user
  // kernel's reads are unknown: twice every open file's pages plus a margin per TB.
  int64_t pages = 0, requests = 0;
  for (int64_t s = 0; s < n_segs; s++) {
    int64_t len = prog->segs[3 * s + 2];
    pages += len / cfg.page_size + 2;
    requests += len / prog->request_bytes + 1;
  }
  if (launch) {
    for (auto& f : ctx->files)
      if (f.open) pages += 2 * f.npages;
    pages += 64 * (int64_t)prog->n_tb;
    requests = pages;
  }
  for (int k = 0; k < 5; k++) {
    ctx->log_cap[k] = 0;
    ctx->log_n[k] = 0;
  }
  if (cfg.timeline) {  // per request: one gread, at most one RPC, one consume
    const int64_t cap = 3 * requests + 2 * (int64_t)prog->n_tb + 16;
    CUDA_TRY(ctx->d_logs[GFS_LOG_TIMELINE].reserve((size_t)(cap * 4)));
    ctx->log_cap[GFS_LOG_TIMELINE] = (unsigned long long)cap;
  }
  if (cfg.log) {
    const int width[4] = {3, 4, 3, 2};
    const int64_t cap[4] = {pages + 2 * requests + 16, pages + 2 * requests + 16,
                            pages + 2 * requests + 16, pages + 2 * requests + 16};
    for (int k = 0; k < 4; k++) {
      CUDA_TRY(ctx->d_logs[k].reserve((size_t)(cap[k] * width[k])));
      ctx->log_cap[k] = (unsigned long long)cap[k];
    }
  }

  // cold cache + fresh run state (a new Simulation starts empty)
  for (auto& f : ctx->files)
    if (f.open && f.d_pt) CUDA_TRY(cudaMemsetAsync(f.d_pt, 0xFF, (size_t)f.npages * 4, ctx->stream));
  if (!cfg.raw_mode) {
    CUDA_TRY(cudaMemsetAsync(ctx->d_fstate, 0, (size_t)ctx->nframes * 4, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->d_retired, 0, (size_t)ctx->ret_npools * (size_t)ctx->ret_pcap * 4, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->d_rpool, 0, (size_t)RET_POOLS * 16 * 8, ctx->stream));
    if (ctx->d_gfifo) CUDA_TRY(cudaMemsetAsync(ctx->d_gfifo, 0, (size_t)ctx->gfifo_cap * 4, ctx->stream));
  }
  CUDA_TRY(cudaMemsetAsync(ctx->d_g, 0, sizeof(DevGlobals), ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->d_stats, 0, (size_t)ctx->n_ctas * GFS_NSTATS * 8, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->d_done_pos, 0, (size_t)ctx->ring_size * 8, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->d_slot_busy, 0, (size_t)cfg.rpc_slots * 4, ctx->stream));


  DevCtx c{};
  c.page_size = cfg.page_size;
  c.prefetch_bytes = cfg.prefetch_bytes;
  c.ra_max_bytes = cfg.ra_max_bytes;
  c.ra_init_bytes = std::min(cfg.ra_init_bytes, cfg.ra_max_bytes);
  c.pb_cap_bytes = ctx->pb_cap;
  c.slot_bytes = ctx->slot_bytes;
  c.staging_bytes = cfg.staging_bytes;
  c.request_bytes = prog->request_bytes;
  c.nframes = ctx->nframes;
  c.quota = ctx->quota;
  c.gfifo_cap = ctx->gfifo_cap;
  c.policy = cfg.policy;
  c.readahead = cfg.readahead;
  c.transfer = cfg.transfer;
  c.raw_mode = cfg.raw_mode;
  c.log = cfg.log;
  c.timeline = cfg.timeline;
  c.lookahead = launch ? 0 : cfg.lookahead;  // user greads deliver only their own range
  c.landing_halves = ctx->landing_halves;
  c.stream_pieces = ctx->stream_pieces ? 1 : 0;
  c.stream_piece = ctx->stream_piece;
  c.landed = ctx->d_landed;
  c.ra_clamp = cfg.ra_clamp;
  c.verify = cfg.verify;
  c.pcie_disabled = cfg.pcie_disabled;
  c.n_files = (int32_t)ctx->files.size();
  c.n_tb = prog->n_tb;
  c.n_ctas = ctx->n_ctas;
  c.n_sms = ctx->sms;
  c.spread = 1;
  if (const char* e = getenv("GFS_SPREAD")) c.spread = atoi(e);  // experiments
  c.ring_mask = ctx->ring_size - 1;
  c.timeout_ns = 60ull * 1000000000ull;
  c.segs = ctx->d_segs.p;
  c.prog_off = ctx->d_prog_off.p;
  c.dst_off = ctx->d_dst_off.p;
  c.order = ctx->d_order.p;
  c.dst = (uint8_t*)dst;
  c.files = ctx->d_files.p;
  c.frames = ctx->d_frames;
  c.fkey = ctx->d_fkey;
  c.fstate = ctx->d_fstate;
  c.own_q = ctx->d_own_q;
  c.retired = ctx->d_retired;
  c.rpool = ctx->d_rpool;
  c.ret_pcap = ctx->ret_pcap;
  c.ret_npools = ctx->ret_npools;
  c.gfifo = ctx->d_gfifo;
  c.recycled = ctx->d_recycled;
  c.g = ctx->d_g;
  c.ring = ctx->h_ring;
  c.ring_consumed = ctx->h_consumed;
  c.host_served = ctx->h_served;
  c.resp = ctx->h_resp;
  c.staging = ctx->h_staging;
  c.landing = ctx->d_landing;
  c.bounce = ctx->h_bounce;
  c.bounce_release = ctx->h_release;
  c.bounce_bytes = ctx->slot_bytes;
  c.doorbell = ctx->d_doorbell;
  c.done_pos = ctx->d_done_pos;
  c.slot_busy = ctx->d_slot_busy;
  c.ref_slots = cfg.rpc_slots;
  c.poll_first_ns = 2000;  // mailbox polls are PCIe reads queued behind the data: not too eager
  c.poll_ns = 4000;
  if (const char* e = getenv("GFS_POLL_NS")) c.poll_first_ns = c.poll_ns = (uint32_t)atoi(e);  // experiments
  c.k1_direct = cfg.k1_direct && (cfg.transfer == GFS_XFER_MAPPED_ZC || cfg.transfer == GFS_XFER_MAPPED_HYBRID);
  // K1 early: only where the daemon's answer is the span length (mapped transfers, K1 direct)
  // and the request is the static request_span / doubling RPC (not an ondemand window)
  c.k1_early = cfg.k1_early && c.k1_direct && cfg.readahead != GFS_RA_ONDEMAND;
  c.ce_min = ctx->ce_min;
  c.stats = ctx->d_stats;
  if (cons) c.cons = *cons;
  else c.cons.kind = GFS_CONSUME_NONE;
  c.tma = 0;
  c.tma_off = 0;
  if (cfg.k1_tma) {  // the stage ring needs room next to the consumer's shared state
    const int64_t off = gread_tma_offset(c.cons, cfg.cta_threads);
    if (off >= 0) {
      c.tma = 1;
      c.tma_off = (int32_t)off;
      c.tma_nst = gread_tma_stages(c.cons, cfg.cta_threads);
      if (const char* e = getenv("GFS_TMA_STAGES"))  // experiments: fewer stages than fit
        c.tma_nst = std::max(1, std::min(c.tma_nst, atoi(e)));
    }
  }
  for (int k = 0; k < 5; k++) {
    c.logs[k] = ctx->d_logs[k].p;
    c.log_cap[k] = ctx->log_cap[k];
  }
  ctx->worker_error.store(0);
  ctx->t_pread.store(0);
  ctx->t_idle.store(0);
  ctx->t_xfer.store(0);
  ctx->n_served.store(0);
  if (prog->n_tb > 0) {
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    cudaGetLastError();  // clear any stale non-sticky error before the launch check
    if (launch) {
      gfs_launch L{};
      L.dev = &c;
      L.dev_bytes = (int64_t)sizeof(DevCtx);
      L.n_ctas = ctx->n_ctas;
      L.cta_threads = cfg.cta_threads;
      L.smem_bytes = gread_launch_smem(c.cons, cfg.cta_threads, c.tma);
      L.stream = (void*)ctx->stream;
      L.n_tb = prog->n_tb;
      const int lr = launch(&L, user);
      cudaError_t le = cudaGetLastError();
      if (lr != 0 || le != cudaSuccess) {
        // nothing may be left running against the ring: wait for whatever did launch
        cudaStreamSynchronize(ctx->stream);
        reset_daemon(ctx);
        return fail(GFS_EINVAL, "gfs_run_kernel: launch callback failed (%d, %s)", lr, cudaGetErrorString(le));
      }
    } else {
      CUDA_TRY(launch_gread(c, cfg.cta_threads, ctx->stream));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
  }
  // wait (GIL is released by the ctypes caller); the kernel has its own device timeout
  const uint64_t deadline = now_ns() + 600ull * 1000000000ull;
  for (;;) {
    cudaError_t q = cudaStreamQuery(ctx->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      ctx->poisoned = true;  // sticky CUDA error: the context is gone
      return fail(GFS_ECUDA, "gread kernel failed: %s", cudaGetErrorString(q));
    }
    if (now_ns() > deadline) {
      ctx->poisoned = true;
      return fail(GFS_ETIMEDOUT, "gread kernel did not finish in 600 s");
    }
    // the daemon threads own the host cores while the kernel runs: poll lazily
    std::this_thread::sleep_for(std::chrono::microseconds(500));
  }
  float ms = 0.f;
  if (prog->n_tb > 0) CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));

  DevGlobals g{};
  CUDA_TRY(cudaMemcpy(&g, ctx->d_g, sizeof g, cudaMemcpyDeviceToHost));
  std::vector<long long> st((size_t)ctx->n_ctas * GFS_NSTATS);
  CUDA_TRY(cudaMemcpy(st.data(), ctx->d_stats, st.size() * 8, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  for (int b = 0; b < ctx->n_ctas; b++)
    for (int k = 0; k < GFS_NSTATS; k++) out->v[k] += st[(size_t)b * GFS_NSTATS + k];
  out->v[GFS_STAT_kernel_ns] = (int64_t)((double)ms * 1e6);
  out->v[GFS_STAT_ctas] = ctx->n_ctas;
  out->v[GFS_STAT_host_pread_ns] = ctx->t_pread.load();
  out->v[GFS_STAT_host_idle_ns] = ctx->t_idle.load();
  out->v[GFS_STAT_host_xfer_ns] = ctx->t_xfer.load();
  out->v[GFS_STAT_host_requests] = ctx->n_served.load();
  out->v[GFS_STAT_io_workers] = ctx->cfg.io_workers;
  for (int k = 0; k < 5; k++) ctx->log_n[k] = std::min(g.log_n[k], ctx->log_cap[k]);
  if (g.dbg[0] && getenv("GFS_DEBUG_MISMATCH"))
    fprintf(stderr, "gfs: first K1 word mismatch: tb %llu cta %llu fid %llu file offset %llu read %#llx "
            "landing half %llu span offset %llu batch pages %llu\n", g.dbg[1], g.dbg[7] >> 32, g.dbg[2], g.dbg[3],
            g.dbg[4], g.dbg[5], g.dbg[6], g.dbg[7] & 0xFFFFFFFFull);
  if (g.dbg[0] && getenv("GFS_DEBUG_MISMATCH"))
    fprintf(stderr, "gfs:   landing half last pulled file offset %llu (%llu bytes); pb_base %llu pb_off_adj %llu "
            "pb_count %llu j0 %llu; gread [%llu, %llu)\n", g.dbg[8], g.dbg[9], g.dbg[10], g.dbg[11], g.dbg[12],
            g.dbg[13], g.dbg[14], g.dbg[15]);
  ctx->has_run = true;
  out->v[GFS_STAT_wall_ns] = (int64_t)(now_ns() - w0);
  if (g.error) {
    static const char* names[] = {"none", "every frame is in flight (global-lru-dealloc)",
                                  "per-tb-lra: TB has no frames to recycle and none are free",
                                  "I/O error from the host daemon", "device wait timed out",
                                  "global FIFO overflow", "log overflow", "bad program",
                                  "private buffer overflow"};
    const char* what = g.error < 9 ? names[g.error] : "unknown";
    int werr = ctx->worker_error.load();
    std::string diag;
    if (g.error == ERR_TIMEOUT && g.error_info >= 21 && g.error_info <= 23) {
      // a request never completed: say where it is (ring entry, mailbox/doorbell, workers)
      const int mb = (int)(g.error_arg >> 32);  // mailbox / doorbell: slot * halves + half
      const int slot = mb / ctx->landing_halves;
      const uint32_t seq = (uint32_t)g.error_arg;
      char b[256];
      const RpcReq* e = &ctx->h_ring[(seq - 1) & (ctx->ring_size - 1)];
      snprintf(b, sizeof b, "; slot %d half %d seq %u: ring entry lap %u (want %u) slot %d, mailbox seq %u", slot,
               mb % ctx->landing_halves, seq, (unsigned)(e->w[2] & 0xFFFF),
               ring_lap(seq - 1, ctx->ring_size), (int)((e->w[2] >> 16) & 0x7FFF),
               slot < ctx->n_ctas ? ctx->h_resp[mb].seq : 0);
      diag += b;
      if (ctx->d_doorbell && slot < ctx->n_ctas) {
        unsigned long long bell = 0;
        cudaMemcpy(&bell, ctx->d_doorbell + mb, 8, cudaMemcpyDeviceToHost);
        snprintf(b, sizeof b, ", doorbell seq %u n %u", (uint32_t)bell, (uint32_t)(bell >> 32));
        diag += b;
      }
      snprintf(b, sizeof b, "; ring head %llu served %llu; workers",
               (unsigned long long)ctx->req_head.load(), (unsigned long long)*ctx->h_served);
      diag += b;
      for (int w = 0; w < ctx->cfg.io_workers && w < 256; w++) {
        snprintf(b, sizeof b, " %llu/%d", (unsigned long long)ctx->w_pos[w].load(), ctx->w_phase[w].load());
        diag += b;
      }
    }
    reset_daemon(ctx);  // the next run starts from a clean ring
    return fail(g.error == ERR_IO ? GFS_EIO : (g.error == ERR_TIMEOUT ? GFS_ETIMEDOUT : GFS_EDEVICE),
                "device error %d: %s (info %d, arg %llu)%s%s%s", g.error, what, g.error_info,
                (unsigned long long)g.error_arg, werr ? "; daemon errno: " : "",
                werr ? strerror(werr) : "", diag.c_str());
  }
  return GFS_OK;
}

// ------------------------------------------------------------------- logs

extern "C" int gfs_log_len(gfs_ctx* ctx, int kind, int64_t* n) {
  if (!ctx || !n || kind < 0 || kind > GFS_LOG_TIMELINE) return fail(GFS_EINVAL, "gfs_log_len: bad argument");
  *n = (int64_t)ctx->log_n[kind];
  return GFS_OK;
}

extern "C" int gfs_log_copy(gfs_ctx* ctx, int kind, int64_t* out, int64_t cap_records) {
  if (!ctx || !out || kind < 0 || kind > GFS_LOG_TIMELINE) return fail(GFS_EINVAL, "gfs_log_copy: bad argument");
  const int width[5] = {3, 4, 3, 2, 4};
  int64_t n = std::min<int64_t>((int64_t)ctx->log_n[kind], cap_records);
  if (n > 0)
    CUDA_TRY(cudaMemcpy(out, ctx->d_logs[kind].p, (size_t)(n * width[kind]) * 8, cudaMemcpyDeviceToHost));
  return GFS_OK;
}

// ------------------------------------------------------------------- consumers

extern "C" int gfs_checksum(gfs_ctx* ctx, const void* dev_buf, uint64_t nbytes, uint64_t word_base,
                            uint64_t* out) {
  if (!ctx || !out || (!dev_buf && nbytes)) return fail(GFS_EINVAL, "gfs_checksum: bad argument");
  CUDA_TRY(cudaSetDevice(ctx->cfg.device));
  CUDA_TRY(cudaMemsetAsync(ctx->d_scratch, 0, 8, ctx->stream));
  if (nbytes) CUDA_TRY(launch_checksum(dev_buf, nbytes, word_base, ctx->d_scratch, ctx->sms, ctx->stream));
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, ctx->d_scratch, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *out = v;
  return GFS_OK;
}

// check_unique_mapping (gpu_cache.py:217-224) over the page table the last run left.
extern "C" int gfs_check_mapping(gfs_ctx* ctx, gfs_mapping_check* out) {
  if (!ctx || !out) return fail(GFS_EINVAL, "gfs_check_mapping: null argument");
  if (ctx->poisoned) return fail(GFS_ESTATE, "context unusable");
  memset(out, 0, sizeof *out);
  if (ctx->cfg.raw_mode || !ctx->has_run) return GFS_OK;  // no page cache / nothing cached yet
  CUDA_TRY(cudaSetDevice(ctx->cfg.device));
  if (!ctx->d_owner) CUDA_TRY(cudaMalloc(&ctx->d_owner, (size_t)ctx->nframes * 4));
  int rc = upload_files(ctx);
  if (rc) return rc;
  CUDA_TRY(cudaMemsetAsync(ctx->d_owner, 0xFF, (size_t)ctx->nframes * 4, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->d_scratch, 0, 64, ctx->stream));
  CUDA_TRY(launch_check_mapping(ctx->d_files.p, (int)ctx->files.size(), ctx->d_fkey, ctx->d_fstate, ctx->d_owner,
                                ctx->nframes, ctx->d_scratch, ctx->sms, ctx->stream));
  unsigned long long v[5] = {0, 0, 0, 0, 0};
  CUDA_TRY(cudaMemcpyAsync(v, ctx->d_scratch, sizeof v, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  out->mapped_pages = (int64_t)v[0];
  out->duplicate_frames = (int64_t)v[1];
  out->key_mismatches = (int64_t)v[2];
  out->unsettled = (int64_t)v[3];
  out->lost_frames = (int64_t)v[4];
  if (v[1] || v[2] || v[3] || v[4])
    return fail(GFS_EDEVICE,
                "check_unique_mapping: %llu frames reached from two pages, %llu key mismatches, "
                "%llu unsettled entries, %llu valid frames unreachable (of %llu mapped pages)",
                v[1], v[2], v[3], v[4], v[0]);
  return GFS_OK;
}

extern "C" int gfs_verify_dst(gfs_ctx* ctx, const gfs_program* prog, const void* dev_buf,
                              uint64_t dst_bytes, int64_t* mismatched_words) {
  if (!ctx || !prog || !dev_buf || !mismatched_words) return fail(GFS_EINVAL, "gfs_verify_dst: null argument");
  int rc = validate_program(ctx, prog, dst_bytes, true);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(ctx->cfg.device));
  int64_t n_segs = 0;
  if ((rc = upload_files(ctx)) || (rc = upload_program(ctx, prog, &n_segs))) return rc;
  std::vector<int64_t> seg_dst((size_t)std::max<int64_t>(n_segs, 1));
  for (int t = 0; t < prog->n_tb; t++) {
    int64_t pos = prog->dst_off[t];
    for (int64_t s = prog->prog_off[t]; s < prog->prog_off[t + 1]; s++) {
      seg_dst[s] = pos;
      pos += prog->segs[3 * s + 2];
    }
  }
  CUDA_TRY(ctx->d_seg_dst.reserve(seg_dst.size()));
  CUDA_TRY(cudaMemcpyAsync(ctx->d_seg_dst.p, seg_dst.data(), seg_dst.size() * 8, cudaMemcpyHostToDevice,
                           ctx->stream));
  CUDA_TRY(cudaMemsetAsync(ctx->d_scratch, 0, 8, ctx->stream));
  if (n_segs)
    CUDA_TRY(launch_verify_dst(dev_buf, ctx->d_segs.p, ctx->d_seg_dst.p, n_segs, ctx->d_files.p,
                               ctx->d_scratch, ctx->sms, ctx->stream));
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpyAsync(&v, ctx->d_scratch, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *mismatched_words = (int64_t)v;
  return GFS_OK;
}

// ------------------------------------------------------------------- synthetic files (K6)

static inline uint64_t h_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

extern "C" int gfs_gen_file(const char* path, int64_t content_id, int64_t size, int threads) {
  if (!path || size < 0 || content_id < 0) return fail(GFS_EINVAL, "gfs_gen_file: bad argument");
  int fd = open(path, O_CREAT | O_WRONLY | O_TRUNC, 0644);
  if (fd < 0) return fail(GFS_EIO, "create %s: %s", path, strerror(errno));
  close(fd);
  return gfs_gen_file_range(path, content_id, size, 0, size, threads);
}

extern "C" int gfs_gen_file_range(const char* path, int64_t content_id, int64_t size, int64_t offset,
                                  int64_t length, int threads) {
  if (!path || size < 0 || content_id < 0 || offset < 0 || length < 0 || offset + length > size ||
      offset % 8)
    return fail(GFS_EINVAL, "gfs_gen_file_range: bad argument");
  int fd = open(path, O_CREAT | O_WRONLY, 0644);
  if (fd < 0) return fail(GFS_EIO, "create %s: %s", path, strerror(errno));
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (sb.st_size != size && ftruncate(fd, (off_t)size) != 0)) {
    close(fd);
    return fail(GFS_EIO, "truncate %s: %s", path, strerror(errno));
  }
  if (threads < 1) threads = 1;
  const int64_t chunk = 8 << 20;
  const int64_t nchunks = (length + chunk - 1) / chunk;
  std::atomic<int64_t> next{0};
  std::atomic<int> err{0};
  auto body = [&]() {
    std::vector<uint64_t> buf((size_t)(chunk / 8) + 1);
    for (;;) {
      int64_t k = next.fetch_add(1);
      if (k >= nchunks || err.load()) return;
      const int64_t off = offset + k * chunk, n = std::min(chunk, offset + length - off);
      const int64_t w0 = off >> 3, nw = (n + 7) >> 3;
      for (int64_t i = 0; i < nw; i++) {
        int64_t wi = w0 + i;
        uint64_t tag = h_mix64(((uint64_t)content_id << 40) ^ (uint64_t)(wi >> 9) ^ 0xA5A5A5A5A5A5A5A5ull);
        buf[(size_t)i] = h_mix64(tag ^ (uint64_t)wi);
      }
      const uint8_t* p = (const uint8_t*)buf.data();
      int64_t done = 0;
      while (done < n) {
        ssize_t w = pwrite(fd, p + done, (size_t)(n - done), (off_t)(off + done));
        if (w < 0) {
          if (errno == EINTR) continue;
          err.store(errno);
          return;
        }
        done += w;
      }
    }
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; t++) ts.emplace_back(body);
  for (auto& t : ts) t.join();
  if (!err.load() && fsync(fd) != 0) err.store(errno);
  close(fd);
  if (err.load()) return fail(GFS_EIO, "write %s: %s", path, strerror(err.load()));
  return GFS_OK;
}

// ------------------------------------------------------------------- introspection

extern "C" const char* gfs_last_error(void) { return g_err.c_str(); }
extern "C" int gfs_abi_version(void) { return GFS_ABI_VERSION; }
extern "C" int gfs_stat_count(void) { return GFS_NSTATS; }
extern "C" const char* gfs_stat_name(int i) { return (i >= 0 && i < GFS_NSTATS) ? kStatNames[i] : nullptr; }

// lets the baseline translation unit report through the same thread-local error slot
extern "C" int gfs_internal_fail(int code, const char* msg) { return fail(code, "%s", msg); }
