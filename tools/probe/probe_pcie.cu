// PCIe probe: H2D cudaMemcpyAsync bandwidth vs size/streams, zero-copy kernel read BW,
// GPU<->host mapped-memory ping-pong latency.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <thread>
#include <atomic>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x);if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e));exit(1);}}while(0)

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) dst[i] = src[i];
}
__global__ void pingpong(volatile uint32_t* req, volatile uint32_t* resp, int iters, unsigned long long* out) {
  unsigned long long t0 = clock64();
  for (int i = 1; i <= iters; i++) {
    *req = i; __threadfence_system();
    while (*resp != (uint32_t)i) {}
  }
  *out = clock64() - t0;
}
int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("gpu %s sms %d pcie bus %d asyncEngines %d\n", p.name, p.multiProcessorCount, p.pciBusID, p.asyncEngineCount);
  size_t MAX = 1ull << 30;
  void *h, *d; CK(cudaHostAlloc(&h, MAX, cudaHostAllocMapped)); CK(cudaMalloc(&d, MAX));
  memset(h, 1, MAX);
  cudaStream_t st[8]; for (int i = 0; i < 8; i++) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t sz = 4096; sz <= MAX; sz *= 4) {
    for (int ns : {1, 4}) {
      size_t total = std::max(sz, (size_t)256 << 20); int n = total / sz;
      // warm
      for (int i = 0; i < std::min(n,64); i++) CK(cudaMemcpyAsync((char*)d + (i * sz) % MAX, (char*)h + (i * sz) % MAX, sz, cudaMemcpyHostToDevice, st[i % ns]));
      CK(cudaDeviceSynchronize());
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < n; i++) CK(cudaMemcpyAsync((char*)d + (i * sz) % MAX, (char*)h + (i * sz) % MAX, sz, cudaMemcpyHostToDevice, st[i % ns]));
      CK(cudaDeviceSynchronize());
      double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      printf("H2D memcpy sz=%zuK streams=%d n=%d: %.2f GB/s (%.2f us/copy)\n", sz >> 10, ns, n, total / dt / 1e9, dt / n * 1e6);
    }
  }
  // D2H too
  { cudaEventRecord(e0, st[0]); CK(cudaMemcpyAsync(h, d, MAX, cudaMemcpyDeviceToHost, st[0])); cudaEventRecord(e1, st[0]); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("D2H 1G: %.2f GB/s\n", MAX / ms / 1e6); }
  // zero-copy kernel reads
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  for (int blocks : {148, 296, 592, 1184}) for (int thr : {256, 512, 1024}) {
    size_t n = MAX / 16;
    zc_read<<<blocks, thr>>>((const uint4*)hd, (uint4*)d, n); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); zc_read<<<blocks, thr>>>((const uint4*)hd, (uint4*)d, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("zero-copy read blocks=%d thr=%d: %.2f GB/s\n", blocks, thr, MAX / ms / 1e6);
  }
  // ping-pong latency: GPU writes req in mapped host mem, host thread echoes into resp (mapped host mem)
  uint32_t *hreq, *hresp; CK(cudaHostAlloc(&hreq, 4096, cudaHostAllocMapped)); CK(cudaHostAlloc(&hresp, 4096, cudaHostAllocMapped));
  *hreq = 0; *hresp = 0; uint32_t *dreq, *dresp; cudaHostGetDevicePointer((void**)&dreq, hreq, 0); cudaHostGetDevicePointer((void**)&dresp, hresp, 0);
  unsigned long long* dout; cudaMalloc(&dout, 8);
  int iters = 20000; std::atomic<bool> stop{false};
  std::thread echo([&] { volatile uint32_t* r = hreq; volatile uint32_t* s = hresp; uint32_t last = 0;
    while (!stop.load(std::memory_order_relaxed)) { uint32_t v = *r; if (v != last) { last = v; *s = v; } } });
  auto t0 = std::chrono::steady_clock::now();
  pingpong<<<1, 1>>>(dreq, dresp, iters, dout); CK(cudaDeviceSynchronize());
  double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  stop = true; echo.join();
  printf("mapped ping-pong round trip: %.2f us\n", dt / iters * 1e6);
  // host-written flag in device memory via cuStreamWriteValue32 after a memcpy: latency of memcpy(64K)+write
  return 0;
}
