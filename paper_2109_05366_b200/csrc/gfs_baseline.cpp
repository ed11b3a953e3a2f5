// gfs_baseline.cpp — the comparison arms and roofline probes the north_star asks for,
// measured natively on the same box as the gread path:
//   * storage roofline: parallel sequential O_DIRECT read of a file;
//   * PCIe roofline: pinned host -> HBM cudaMemcpyAsync bandwidth;
//   * the traditional CPU I/O baseline (paper §3): host
//     threads pread() the file into pinned buffers and cudaMemcpy it into HBM.
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "gfs.h"

extern "C" int gfs_internal_fail(int code, const char* msg);

static double now_s() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static int failf(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return gfs_internal_fail(code, buf);
}

static int64_t read_fully(int fd, uint8_t* buf, int64_t want, int64_t off) {
  int64_t got = 0;
  while (got < want) {
    ssize_t k = pread(fd, buf + got, (size_t)(want - got), (off_t)(off + got));
    if (k < 0) {
      if (errno == EINTR) continue;
      return -(int64_t)errno;
    }
    if (k == 0) break;
    got += k;
  }
  return got;
}

extern "C" int gfs_bench_storage(const char* path, int64_t offset, int64_t size, int threads,
                                 int64_t chunk, int direct, double* seconds) {
  if (!path || !seconds || threads < 1 || chunk < 4096 || (direct && (chunk % 4096 || offset % 4096)))
    return failf(GFS_EINVAL, "gfs_bench_storage: bad argument");
  std::atomic<int64_t> next{0};
  std::atomic<int> err{0};
  const int64_t nchunks = (size + chunk - 1) / chunk;
  auto body = [&]() {
    int fd = open(path, O_RDONLY | (direct ? O_DIRECT : 0));
    if (fd < 0) {
      err.store(errno);
      return;
    }
    void* buf = nullptr;
    if (posix_memalign(&buf, 4096, (size_t)chunk)) {
      err.store(ENOMEM);
      close(fd);
      return;
    }
    for (;;) {
      int64_t k = next.fetch_add(1);
      if (k >= nchunks || err.load()) break;
      int64_t off = offset + k * chunk, n = std::min(chunk, offset + size - off);
      int64_t r = read_fully(fd, (uint8_t*)buf, direct ? (n + 4095) / 4096 * 4096 : n, off);
      if (r < 0) {
        err.store((int)-r);
        break;
      }
    }
    free(buf);
    close(fd);
  };
  double t0 = now_s();
  std::vector<std::thread> ts;
  for (int i = 0; i < threads; i++) ts.emplace_back(body);
  for (auto& t : ts) t.join();
  *seconds = now_s() - t0;
  if (err.load()) return failf(GFS_EIO, "storage probe on %s: %s", path, strerror(err.load()));
  return GFS_OK;
}

extern "C" int gfs_bench_h2d(int device, int64_t bytes, int reps, double* best_seconds) {
  if (!best_seconds || bytes < 1 || reps < 1) return failf(GFS_EINVAL, "gfs_bench_h2d: bad argument");
  cudaError_t e;
  void *h = nullptr, *d = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  float best = 1e30f;
  if ((e = cudaSetDevice(device)) || (e = cudaHostAlloc(&h, (size_t)bytes, cudaHostAllocDefault)) ||
      (e = cudaMalloc(&d, (size_t)bytes)) || (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) ||
      (e = cudaEventCreate(&a)) || (e = cudaEventCreate(&b)))
    goto out;
  memset(h, 1, (size_t)bytes);
  for (int r = 0; r < reps + 1; r++) {
    cudaEventRecord(a, st);
    cudaMemcpyAsync(d, h, (size_t)bytes, cudaMemcpyHostToDevice, st);
    cudaEventRecord(b, st);
    if ((e = cudaEventSynchronize(b))) goto out;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0) best = std::min(best, ms);  // first is a warm-up
  }
  *best_seconds = best / 1e3;
out:
  if (a) cudaEventDestroy(a);
  if (b) cudaEventDestroy(b);
  if (st) cudaStreamDestroy(st);
  if (d) cudaFree(d);
  if (h) cudaFreeHost(h);
  if (e) return failf(GFS_ECUDA, "h2d probe: %s", cudaGetErrorString(e));
  return GFS_OK;
}

// CPU I/O baseline: `threads` host threads each own a contiguous share of
// [offset, offset+size); each preads `chunk`-sized pieces into two pinned buffers
// (double buffering) and copies them to dst + (piece - offset) with cudaMemcpyAsync on
// its own stream.  threads == 1 with sync == 1 is the paper's "CPU I/O" arm: one
// thread, read() then a blocking cudaMemcpy per chunk.
extern "C" int gfs_bench_read_memcpy(const char* path, int64_t offset, int64_t size, void* dst_dev,
                                     int device, int threads, int64_t chunk, int direct, int sync,
                                     double* seconds) {
  if (!path || !dst_dev || !seconds || threads < 1 || chunk < 4096 || chunk % 4096)
    return failf(GFS_EINVAL, "gfs_bench_read_memcpy: bad argument");
  if (direct && offset % 4096) direct = 0;
  cudaError_t ce = cudaSetDevice(device);
  if (ce) return failf(GFS_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(ce));
  std::atomic<int> err{0};
  std::atomic<int> cerr{0};
  const int64_t per = (size + threads - 1) / threads / chunk * chunk + chunk;
  std::vector<uint8_t*> bufs((size_t)threads * 2, nullptr);
  std::vector<cudaStream_t> streams((size_t)threads, nullptr);
  std::vector<cudaEvent_t> evs((size_t)threads * 2, nullptr);
  for (int t = 0; t < threads && !ce; t++) {
    for (int k = 0; k < 2 && !ce; k++) {
      ce = cudaHostAlloc((void**)&bufs[2 * t + k], (size_t)chunk, cudaHostAllocDefault);
      if (!ce) ce = cudaEventCreateWithFlags(&evs[2 * t + k], cudaEventDisableTiming);
    }
    if (!ce) ce = cudaStreamCreateWithFlags(&streams[t], cudaStreamNonBlocking);
  }
  double el = 0;
  if (!ce) {
    auto body = [&](int t) {
      cudaSetDevice(device);
      int fd = open(path, O_RDONLY | (direct ? O_DIRECT : 0));
      if (fd < 0) {
        err.store(errno);
        return;
      }
      const int64_t lo = offset + (int64_t)t * per, hi = std::min(offset + size, lo + per);
      int k = 0;
      for (int64_t pos = lo; pos < hi; pos += chunk, k ^= 1) {
        const int64_t n = std::min(chunk, hi - pos);
        uint8_t* b = bufs[2 * t + k];
        if (!sync) cudaEventSynchronize(evs[2 * t + k]);  // the copy that used b is done
        int64_t r = read_fully(fd, b, direct ? (n + 4095) / 4096 * 4096 : n, pos);
        if (r < n) {
          err.store(r < 0 ? (int)-r : EIO);
          break;
        }
        uint8_t* d = (uint8_t*)dst_dev + (pos - offset);
        cudaError_t e = sync ? cudaMemcpy(d, b, (size_t)n, cudaMemcpyHostToDevice)
                             : cudaMemcpyAsync(d, b, (size_t)n, cudaMemcpyHostToDevice, streams[t]);
        if (!e && !sync) e = cudaEventRecord(evs[2 * t + k], streams[t]);
        if (e) {
          cerr.store((int)e);
          break;
        }
      }
      if (!sync) cudaStreamSynchronize(streams[t]);
      close(fd);
    };
    double t0 = now_s();
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; t++) ts.emplace_back(body, t);
    for (auto& th : ts) th.join();
    el = now_s() - t0;
  }
  for (auto b : bufs)
    if (b) cudaFreeHost(b);
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto s : streams)
    if (s) cudaStreamDestroy(s);
  if (ce) return failf(GFS_ECUDA, "read+memcpy setup: %s", cudaGetErrorString(ce));
  if (cerr.load()) return failf(GFS_ECUDA, "read+memcpy copy: %s", cudaGetErrorString((cudaError_t)cerr.load()));
  if (err.load()) return failf(GFS_EIO, "read+memcpy read: %s", strerror(err.load()));
  *seconds = el;
  return GFS_OK;
}

// ---------------------------------------------------------------- host-only trace replay
//
// The paper's §3.3 methodology and the reference's `gpuiosim replay`
// (simulation.py:147-164, HostStream :67-95): the RPC trace a GPU run recorded is replayed
// by host threads alone — no GPU, no PCIe — to separate the host I/O cost of the GPU's
// access pattern from the GPU side.  Record r goes to worker
// slot_for_threadblock(tb, n_slots) / (n_slots / n_workers) (rpc.py:27-28); each worker
// issues its records back to back (HostStream._next), each a pread of
// min(size, file_size - offset) bytes (host_os.py:221-230) into a private buffer.
extern "C" int gfs_replay(const char* const* paths, int n_files, const int64_t* recs, int64_t n_recs,
                          int n_slots, int n_workers, int direct, int64_t* user_bytes,
                          int64_t* preads, double* seconds) {
  if (!paths || n_files < 1 || !recs || n_recs < 1 || n_slots < 1 || n_workers < 1 ||
      n_slots % n_workers || !user_bytes || !preads || !seconds)
    return failf(GFS_EINVAL, "gfs_replay: bad argument (n_slots must be a multiple of n_workers)");
  const int per_worker = n_slots / n_workers;
  std::vector<int> fd_d(n_files, -1), fd_b(n_files, -1);
  std::vector<int64_t> fsize(n_files, 0);
  auto close_all = [&]() {
    for (int f = 0; f < n_files; f++) {
      if (fd_d[f] >= 0) close(fd_d[f]);
      if (fd_b[f] >= 0) close(fd_b[f]);
    }
  };
  for (int f = 0; f < n_files; f++) {
    fd_b[f] = open(paths[f], O_RDONLY);
    if (fd_b[f] < 0) {
      int e = errno;
      close_all();
      return failf(GFS_EIO, "gfs_replay: open %s: %s", paths[f], strerror(e));
    }
    fsize[f] = lseek(fd_b[f], 0, SEEK_END);
    if (direct) fd_d[f] = open(paths[f], O_RDONLY | O_DIRECT);  // -1: buffered only
  }
  // group per worker, keeping trace order within a worker; validate like trace_workload
  std::vector<std::vector<int64_t>> groups(n_workers);
  int64_t max_size = 0;
  for (int64_t i = 0; i < n_recs; i++) {
    const int64_t tb = recs[4 * i], fid = recs[4 * i + 1], off = recs[4 * i + 2], size = recs[4 * i + 3];
    if (tb < 0 || fid < 0 || fid >= n_files || off < 0 || size <= 0) {
      close_all();
      return failf(GFS_EINVAL, "trace record %lld: unknown file or bad field", (long long)i);
    }
    if (off + size > fsize[fid]) {
      close_all();
      return failf(GFS_EINVAL, "trace record %lld: read past EOF", (long long)i);
    }
    groups[(tb % n_slots) / per_worker].push_back(i);
    max_size = std::max(max_size, size);
  }
  const int64_t buf_bytes = (max_size + 8191) / 4096 * 4096;
  std::atomic<int64_t> bytes{0}, count{0};
  std::atomic<int> err{0};
  auto body = [&](int w) {
    void* buf = nullptr;
    if (posix_memalign(&buf, 4096, (size_t)buf_bytes)) {
      err.store(ENOMEM);
      return;
    }
    int64_t b = 0, c = 0;
    for (int64_t i : groups[w]) {
      if (err.load(std::memory_order_relaxed)) break;
      const int64_t fid = recs[4 * i + 1], off = recs[4 * i + 2];
      const int64_t n = std::min(recs[4 * i + 3], fsize[fid] - off);
      const bool dio = fd_d[fid] >= 0 && (off & 4095) == 0;
      int64_t r = read_fully(dio ? fd_d[fid] : fd_b[fid], (uint8_t*)buf, dio ? (n + 4095) / 4096 * 4096 : n, off);
      if (r < 0 && dio && r == -EINVAL) r = read_fully(fd_b[fid], (uint8_t*)buf, n, off);
      if (r < 0) {
        err.store((int)-r);
        break;
      }
      b += std::min(r, n);
      c++;
    }
    bytes.fetch_add(b);
    count.fetch_add(c);
    free(buf);
  };
  const double t0 = now_s();
  std::vector<std::thread> th;
  for (int w = 0; w < n_workers; w++)
    if (!groups[w].empty()) th.emplace_back(body, w);
  for (auto& t : th) t.join();
  *seconds = now_s() - t0;
  close_all();
  if (err.load()) return failf(GFS_EIO, "gfs_replay: pread failed: %s", strerror(err.load()));
  *user_bytes = bytes.load();
  *preads = count.load();
  return GFS_OK;
}
