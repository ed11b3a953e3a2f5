// Copy-engine H2D from a cudaHostRegister'ed tmpfs mapping vs cudaHostAlloc memory,
// chunk sizes and stream counts: is the mapped_dma path limited by the source pages?
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <chrono>
#include <cstdio>
#include <cstring>

static double run(const char* name, uint8_t* src, uint8_t* dst, size_t bytes, size_t chunk, int ns,
                  cudaStream_t* st) {
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  size_t n = bytes / chunk;
  for (size_t i = 0; i < n; i++)
    cudaMemcpyAsync(dst + i * chunk, src + i * chunk, chunk, cudaMemcpyHostToDevice, st[i % ns]);
  cudaDeviceSynchronize();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("%s chunk=%zuK streams=%d: %.2f GB/s\n", name, chunk >> 10, ns, bytes / s / 1e9);
  return bytes / s / 1e9;
}

int main() {
  const size_t bytes = 2ull << 30;
  const char* path = "/dev/shm/gfs_probe_ce.bin";
  int fd = open(path, O_CREAT | O_RDWR | O_TRUNC, 0644);
  if (ftruncate(fd, bytes)) return 1;
  uint8_t* m = (uint8_t*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, 0);
  memset(m, 3, bytes);
  cudaError_t e = cudaHostRegister(m, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  printf("register tmpfs: %s\n", cudaGetErrorString(e));
  uint8_t* h;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  memset(h, 3, bytes);
  uint8_t* d;
  cudaMalloc(&d, bytes);
  cudaStream_t st[8];
  for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (size_t chunk : {(size_t)1 << 20, (size_t)4 << 20, (size_t)16 << 20}) {
    for (int ns : {1, 4}) {
      run("hostalloc", h, d, bytes, chunk, ns, st);
      run("tmpfs-map", m, d, bytes, chunk, ns, st);
    }
  }
  cudaHostUnregister(m);
  munmap(m, bytes);
  close(fd);
  unlink(path);
  return 0;
}
