// user_gemv.cu — a user kernel written against the public device API (include/gfs_device.cuh):
// y = A x over a row-major f32 matrix file, every TB reading its stride of rows through
// gfs::gread (the reference's TB program, gpu_exec.py:95-129, with the consumer as the TB's
// compute).  It is what an application outside this package writes: it includes only
// gfs_device.cuh / gfs.h, links libgfs.so, and drives the run with gfs_run_kernel.
//
// Access pattern = gen_sequential_strided (workloads.py:66-81) over one file: TB t reads
// [t * stride, (t + 1) * stride) in request-sized greads, so its counters equal the built-in driver's for that program.
// Elements decode from the file bytes as the built-in consumers do: f32 = (u32 >> 8) * 2^-24.
#include <cuda_runtime.h>

#include "gfs.h"
#include "gfs_device.cuh"

namespace {

struct GemvArgs {
  int fid;
  int64_t stride, request, cols;
  const float* x;
  float* y;
  uint8_t* dst;     // the matrix as delivered
  int stream_hint;  // bound readahead to the TB's stride (io.ra_clamp=segment)
};

__device__ __forceinline__ float dec(uint32_t u) { return (float)(u >> 8) * (1.0f / 16777216.0f); }

template <int BS>
__global__ void __launch_bounds__(BS) user_gemv_kernel(gfs_dev dev, GemvArgs a) {
  gfs::run_threadblocks<BS>(dev, [&](gfs::Tb& tb) {
    const int64_t lo = (int64_t)tb.id * a.stride, hi = lo + a.stride;
    const int64_t row_bytes = a.cols * 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (a.stream_hint) gfs::stream(tb, lo, hi);  // the TB's readahead stream is its stride
    for (int64_t off = lo; off < hi; off += a.request) {
      const int64_t want = a.request < hi - off ? a.request : hi - off;
      const int64_t n = gfs::gread<BS>(tb, a.fid, off, want, a.dst + off);
      if (n < 0) return;
      __syncthreads();  // every thread's part of the delivery is in dst
      // rows of this request: one warp per row, 16-byte vectors along the row
      const int64_t r0 = off / row_bytes, nr = n / row_bytes;
      for (int64_t r = warp; r < nr; r += BS / 32) {
        const uint4* row = (const uint4*)(a.dst + (r0 + r) * row_bytes);
        float acc = 0.f;
        for (int64_t v = lane; v < a.cols / 4; v += 32) {
          const uint4 q = __ldcg(row + v);
          const float4 xv = *(const float4*)(a.x + 4 * v);
          acc += dec(q.x) * xv.x + dec(q.y) * xv.y + dec(q.z) * xv.z + dec(q.w) * xv.w;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.y[r0 + r] = acc;
      }
      if (n < want) return;  // EOF
    }
  });
}

int launch(const gfs_launch* l, void* user) {
  if (l->dev_bytes != (int64_t)sizeof(gfs_dev)) return -1;  // built against another libgfs
  const GemvArgs& a = *(const GemvArgs*)user;
  const gfs_dev& d = *(const gfs_dev*)l->dev;
  cudaStream_t st = (cudaStream_t)l->stream;
  const size_t smem = (size_t)l->smem_bytes;
  switch (l->cta_threads) {
    case 128:
      if (cudaFuncSetAttribute(user_gemv_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -1;
      user_gemv_kernel<128><<<l->n_ctas, 128, smem, st>>>(d, a);
      break;
    case 256:
      if (cudaFuncSetAttribute(user_gemv_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -1;
      user_gemv_kernel<256><<<l->n_ctas, 256, smem, st>>>(d, a);
      break;
    case 512:
      if (cudaFuncSetAttribute(user_gemv_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) return -1;
      user_gemv_kernel<512><<<l->n_ctas, 512, smem, st>>>(d, a);
      break;
    default:
      return -1;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace

// y[rows] = A x for the matrix file fid of file_bytes bytes (rows = file_bytes / (4 cols)),
// n_tb TBs of file_bytes / n_tb bytes each (whole rows), request-sized greads into dst.
extern "C" int gfs_example_gemv(gfs_ctx* ctx, int fid, int64_t file_bytes, int32_t n_tb, int64_t request_bytes,
                                int64_t cols, const float* x, float* y, void* dst, int stream_hint,
                                const int32_t* order, gfs_stats* out) {
  if (n_tb < 1 || cols < 4 || cols % 4 || file_bytes % n_tb || request_bytes < 1 || !x || !y || !dst)
    return GFS_EINVAL;
  GemvArgs a;
  a.fid = fid;
  a.stride = file_bytes / n_tb;
  a.request = request_bytes;
  a.cols = cols;
  a.x = x;
  a.y = y;
  a.dst = (uint8_t*)dst;
  a.stream_hint = stream_hint;
  if (a.stride % (cols * 4) || request_bytes % (cols * 4)) return GFS_EINVAL;  // whole rows per gread
  return gfs_run_kernel(ctx, n_tb, order, launch, &a, out);
}
