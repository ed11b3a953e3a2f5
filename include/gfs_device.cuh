/* gfs_device.cuh — the device-side gread for user kernels (header-only).
 *
 * Replaces the reference's per-threadblock file calls: ThreadBlock._gread / _page_step /
 * _finish_gread (pkg/src/gpuiosim/gpu_exec.py:107-239), driven by the TB program loop and
 * the dispatcher (gpu_exec.py:95-105, 242-291).  A user kernel reads files through the same
 * HBM page cache, private prefetch buffer, readahead law and host RPC ring as the built-in
 * strided driver (gfs_run); the host side is gfs_run_kernel (gfs.h).
 *
 *   #include "gfs_device.cuh"          // nvcc -I<repo>/include -gencode arch=compute_100a,code=sm_100a
 *
 *   template <int BS>
 *   __global__ void __launch_bounds__(BS) my_kernel(gfs_dev dev, ...) {
 *     gfs::run_threadblocks<BS>(dev, [&](gfs::Tb& tb) {      // once per TB id, TB-collective
 *       for (...) {
 *         int64_t n = gfs::gread<BS>(tb, fid, off, size, dst);  // every thread calls it
 *         if (n < 0) return;                                  // run failed (see gfs_last_error)
 *         ... use dst[0, n) ...                               // n < size: EOF (short read)
 *       }
 *     });
 *   }
 *
 *   static int launch(const gfs_launch* l, void* arg) {       // gfs_run_kernel calls this
 *     my_kernel<256><<<l->n_ctas, l->cta_threads, l->smem_bytes, (cudaStream_t)l->stream>>>(
 *         *(const gfs_dev*)l->dev, ...);
 *     return cudaGetLastError() == cudaSuccess ? 0 : -1;
 *   }
 *
 * Rules (they are what make the cache lock-free):
 *  - launch exactly l->n_ctas CTAs of l->cta_threads threads with l->smem_bytes of dynamic
 *    shared memory; the dynamic shared memory belongs to the file layer (K1 stage ring).
 *    Each CTA is one resident TB slot: its RPC mailbox, landing buffer and own-frame queue.
 *  - gread is TB-collective: all BS threads call it with the same arguments, at most one
 *    outstanding RPC per TB.  dst is a device pointer (or nullptr:
 *    pages are cached, nothing is copied out).
 *  - the body runs once per TB id 0..n_tb-1 in the run's dispatch order; when it returns
 *    the TB is closed: private buffer drained, own frames retired (≙ gclose,
 *    gpu_exec.py:281-291).
 */
#pragma once
#include "../paper_2109_05366_b200/csrc/gfs_device_impl.cuh"

/* The device context gfs_run_kernel hands to the launch callback (gfs_launch.dev). */
typedef gfs::DevCtx gfs_dev;

namespace gfs {

/* One threadblock of the run: which TB id it is, and its readahead stream bounds. */
struct Tb {
  const DevCtx* c;
  Smem* s;
  int id;             /* the reference's tb (0 .. n_tb-1) */
  int bad_words;      /* synthetic files: delivered words that broke W(f, i) */
  int64_t stream_lo;  /* readahead windows stay inside [stream_lo, stream_hi) of the file */
  int64_t stream_hi;
};

/* Optional: bound this TB's readahead stream to [lo, hi) of the file (io.ra_clamp=segment:
 * a strided TB's stream is its stride).  Default: the whole file (windows end at EOF, the
 * reference's host_os._decide).  Collective; call between greads. */
__device__ inline void stream(Tb& t, int64_t lo, int64_t hi) {
  t.stream_lo = lo;
  t.stream_hi = hi;
}

/* gread(fid, offset, size) into dst (gpu_exec.py:107-239): returns the bytes delivered
 * (< size at EOF), or -1 when the run failed (bad arguments, I/O error, timeout). */
template <int BS>
__device__ int64_t gread(Tb& t, int fid, int64_t offset, int64_t size, void* dst) {
  const DevCtx& c = *t.c;
  Smem& s = *t.s;
  if (fid < 0 || fid >= c.n_files || offset < 0 || size < 0) {
    if (threadIdx.x == 0) set_error(c, ERR_BAD_PROGRAM, t.id, (unsigned long long)fid);
    __syncthreads();
    return -1;
  }
  if (threadIdx.x == 0) {
    s.seg_lo = t.stream_lo;
    s.seg_hi = t.stream_hi;
    s.seg_ord = 0;
  }
  // (no barrier needed: gread's first decisions are thread 0's; it barriers before any
  // other thread reads the TB state)
  return gread<BS>(c, s, fid, offset, size, t.stream_hi, (uint8_t*)dst, t.bad_words);
}

/* Persistent TB loop: this CTA runs TB ids from the dispatcher until none are left;
 * body(Tb&) is called collectively once per TB. */
template <int BS, class Body>
__device__ void run_threadblocks(const DevCtx& c, Body&& body) {
  __shared__ Smem s;
  if (blockIdx.x >= (unsigned)c.n_ctas) return;  // more CTAs than slots: the extras idle
  if (blockDim.x != BS) {
    if (threadIdx.x == 0) set_error(c, ERR_BAD_PROGRAM, -2, blockDim.x);
    return;
  }
  cta_begin<BS>(c, s);
  Tb t;
  t.c = &c;
  t.s = &s;
  t.bad_words = 0;
  for (;;) {
    const int tb = next_tb(c, s);
    if (tb < 0) break;
    tb_begin(c, s, tb);
    t.id = tb;
    t.stream_lo = 0;
    t.stream_hi = INT64_MAX / 4;
    body(t);
    if (__syncthreads_or(has_error(c))) break;  // one decision for the whole CTA
    tb_end<BS>(c, s);
  }
  cta_end(c, s, t.bad_words);
}

}  // namespace gfs
