// Host-side daemon probe: how fast can T threads move a tmpfs/disk file into HBM?
//   mode zc   : pread spans into a pinned pool (no GPU copy)            -> host pread rate
//   mode dma  : pread into a pinned bounce pool, cudaMemcpyAsync to HBM -> end-to-end rate
// Pool size decides whether staging stays LLC-resident.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
  if (argc < 7) {
    printf("usage: %s file size_mb threads span_kb pool_mb mode(zc|dma) [direct]\n", argv[0]);
    return 1;
  }
  const char* path = argv[1];
  const int64_t size = (int64_t)atoll(argv[2]) << 20;
  const int T = atoi(argv[3]);
  const int64_t span = (int64_t)atoll(argv[4]) << 10;
  const int64_t pool = (int64_t)atoll(argv[5]) << 20;
  const bool dma = !strcmp(argv[6], "dma");
  const bool direct = argc > 7 ? atoi(argv[7]) : 1;
  uint8_t* h;
  cudaHostAlloc((void**)&h, pool, cudaHostAllocMapped | cudaHostAllocPortable);
  memset(h, 0, pool);
  uint8_t* d = nullptr;
  if (dma) cudaMalloc(&d, size);
  const int64_t nbuf = pool / span;
  const int64_t per_thread = nbuf / T;
  std::atomic<int64_t> next{0};
  const int64_t nspans = size / span;
  auto body = [&](int t) {
    int fd = open(path, O_RDONLY | (direct ? O_DIRECT : 0));
    cudaStream_t st;
    std::vector<cudaEvent_t> ev(per_thread);
    if (dma) {
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    int64_t k, i = 0;
    while ((k = next.fetch_add(1)) < nspans) {
      int64_t b = t * per_thread + (i % per_thread);
      if (dma && i >= per_thread) cudaEventSynchronize(ev[i % per_thread]);
      uint8_t* buf = h + b * span;
      int64_t got = 0;
      while (got < span) {
        ssize_t r = pread(fd, buf + got, span - got, k * span + got);
        if (r <= 0) break;
        got += r;
      }
      if (dma) {
        cudaMemcpyAsync(d + k * span, buf, span, cudaMemcpyHostToDevice, st);
        cudaEventRecord(ev[i % per_thread], st);
      }
      i++;
    }
    if (dma) cudaStreamSynchronize(st);
    close(fd);
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++) th.emplace_back(body, t);
  for (auto& x : th) x.join();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("%s T=%d span=%lldK pool=%lldM direct=%d: %.2f GB/s\n", dma ? "dma" : "zc", T,
         (long long)(span >> 10), (long long)(pool >> 20), direct, size / s / 1e9);
  return 0;
}
