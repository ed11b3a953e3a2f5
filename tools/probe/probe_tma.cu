// Probe: host(pinned, mapped) -> HBM pull bandwidth by SMs, LDG.128 vs TMA bulk copies.
// Question: do cp.async.bulk reads of system memory use the PCIe link more efficiently
// (larger read requests) than 16-byte vector loads (51.4 GB/s measured)?
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("ERR %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e));         \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void ldg_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * s < n; i += 4 * s) {
    uint4 a = __ldcv(src + i), b = __ldcv(src + i + s), c = __ldcv(src + i + 2 * s), d = __ldcv(src + i + 3 * s);
    dst[i] = a; dst[i + s] = b; dst[i + 2 * s] = c; dst[i + 3 * s] = d;
  }
  for (; i < n; i += s) dst[i] = __ldcv(src + i);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// One elected thread per CTA streams `chunk`-byte pieces host -> smem (TMA bulk, mbarrier
// completion) -> HBM (TMA bulk store), STAGES deep.
template <int STAGES>
__global__ void tma_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t bytes,
                         uint32_t chunk) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; s++)
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nchunks = bytes / chunk;
  uint32_t phase[STAGES] = {0};
  size_t k0 = blockIdx.x;
  // prologue
  int issued = 0;
  for (int s = 0; s < STAGES; s++) {
    size_t k = k0 + (size_t)s * gridDim.x;
    if (k >= nchunks) break;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sbuf + (size_t)s * chunk)),
        "l"(src + k * chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
        : "memory");
    issued++;
  }
  for (size_t it = 0;; it++) {
    int s = (int)(it % STAGES);
    size_t k = k0 + it * gridDim.x;
    if (k >= nchunks) break;
    // wait for stage s
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bar[s])), "r"(phase[s]));
    }
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + k * chunk),
                 "r"(smem_u32(sbuf + (size_t)s * chunk)), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stage reusable
    size_t kn = k0 + (it + STAGES) * gridDim.x;
    if (kn < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(chunk));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sbuf + (size_t)s * chunk)),
          "l"(src + kn * chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
          : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 2ull << 30;
  uint8_t *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  memset(h, 7, bytes);
  CK(cudaMalloc(&d, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int blocks : {148, 296, 592}) {
    ldg_copy<<<blocks, 256>>>((const uint4*)h, (uint4*)d, bytes / 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    ldg_copy<<<blocks, 256>>>((const uint4*)h, (uint4*)d, bytes / 16);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 blocks=%d: %.2f GB/s\n", blocks, bytes / ms / 1e6);
  }
  for (uint32_t chunk : {4096u, 16384u, 32768u, 65536u}) {
    for (int blocks : {148, 296}) {
      const int STAGES = 4;
      size_t smem = (size_t)STAGES * chunk;
      if (smem > 200 * 1024) continue;
      CK(cudaFuncSetAttribute(tma_copy<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tma_copy<STAGES><<<blocks, 32, smem>>>(h, d, bytes, chunk);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      tma_copy<STAGES><<<blocks, 32, smem>>>(h, d, bytes, chunk);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      cudaEventElapsedTime(&ms, a, b);
      printf("TMA bulk chunk=%uK stages=%d blocks=%d: %.2f GB/s\n", chunk >> 10, STAGES, blocks,
             bytes / ms / 1e6);
    }
  }
  // correctness spot check
  uint8_t x = 0;
  CK(cudaMemcpy(&x, d + bytes - 1, 1, cudaMemcpyDeviceToHost));
  printf("check %d\n", x);
  cudaEventRecord(a);
  CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice));
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  printf("cudaMemcpy 2 GiB: %.2f GB/s\n", bytes / ms / 1e6);
  // SM pulls and a copy-engine copy sharing the link: does the mix beat either alone?
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (double frac : {0.25, 0.5, 0.75}) {
    size_t ce = (size_t)(bytes * frac) & ~(size_t)0xFFFF, sm = bytes - ce;
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, ce, cudaMemcpyHostToDevice, s2);
    ldg_copy<<<296, 256, 0, s1>>>((const uint4*)(h + ce), (uint4*)(d + ce), sm / 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    printf("mixed CE %.0f%% + SM: %.2f GB/s\n", frac * 100, bytes / ms / 1e6);
  }
  return 0;
}
