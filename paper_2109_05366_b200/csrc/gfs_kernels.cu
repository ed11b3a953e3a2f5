// gfs_kernels.cu — sm_100a device side of the GPUfs-style sequential-read layer.
//
// K3  gread_driver : persistent grid, one CTA per resident TB slot.  Each CTA pulls TB
//                    ids from the dispatcher ticket and runs that TB's gread loop
//                    (reference gpu_exec.py:95-239) against the HBM page cache:
//                    lookup+claim in a direct-mapped page table, per-TB LRA or global
//                    LRU-dealloc allocation (gpu_cache.py:104-179), private prefetch
//                    buffer (prefetcher.py:38-68), RPC to the host daemon through a
//                    mapped pinned ring (rpc.py:82-113), completion polling.
// K1  span copy    : staging (mapped pinned, zero-copy) or HBM landing (DMA) -> frame
//                    and user buffer in one pass, 16-byte vectors, word-law verify.
// K2  hit copy     : frame -> user buffer (16 B vectors, congruence-aware).
// K4  checksum / verify_dst consumers over a device buffer.
//
// Metadata decisions of a TB are made by thread 0 (they are inherently sequential in the
// reference: page p's RPC fills the private buffer that serves page p+1); every data
// movement is done by the whole CTA.
#include "gfs_device_impl.cuh"

namespace gfs {

// ------------------------------------------------------------ fused consumers (K4)

struct ConsAcc {
  unsigned long long sum = 0;     // SUM64 partial
  unsigned long long nn = ~0ull;  // NN partial minimum
};

__device__ __forceinline__ float decode_f32(uint32_t u) { return (float)(u >> 8) * (1.0f / 16777216.0f); }

constexpr int GEMV_ROWS = 1024;          // rows of one request accumulated in shared memory
constexpr int GEMVT_SMEM_COLS = 8192;    // A^T x2 accumulated per CTA in shared memory up to this

constexpr int64_t CONS_SMEM_MAX = 48 * 1024;  // dynamic shared memory cap: 4 CTAs/SM still fit

// Kmeans keeps one private [k, cols] accumulator (and counts) per warp when it fits: lanes
// then update distinct words with plain shared stores, no atomics.  Needs cols >= 32.
__host__ __device__ inline bool kmeans_warp_acc(const gfs_consumer& k, int bs) {
  const int64_t w = bs / 32, kd = (int64_t)k.k * k.cols;
  return k.cols >= 32 && (1 + w) * kd * 4 + w * k.k * 4 <= CONS_SMEM_MAX;
}

// Dynamic shared memory a consumer needs (the launch passes it; 0 for the plain gread path).
__host__ __device__ inline int64_t consumer_smem_bytes(const gfs_consumer& k, int bs) {
  if ((k.kind == GFS_CONSUME_GEMVT_F32 || k.kind == GFS_CONSUME_BICG_F32) && k.cols <= GEMVT_SMEM_COLS)
    return k.cols * 4;
  if (k.kind == GFS_CONSUME_KMEANS_F32) {  // + the centroids transposed, [cols][k rounded to 4]
    const int64_t w = bs / 32, kd = (int64_t)k.k * k.cols;
    const int64_t base = kmeans_warp_acc(k, bs) ? (1 + w) * kd * 4 + w * k.k * 4 : 2 * kd * 4 + k.k * 4;
    return (base + 15) / 16 * 16 + (int64_t)k.cols * ((k.k + 3) / 4 * 4) * 4;
  }
  return 0;
}

// Float offset of the transposed centroid copy in the kmeans consumer's shared memory.
__host__ __device__ inline int64_t kmeans_ct_off(const gfs_consumer& k, int bs) {
  const int64_t kp4 = (int64_t)k.cols * ((k.k + 3) / 4 * 4) * 4;
  return (consumer_smem_bytes(k, bs) - kp4) / 4;
}

// Where the K1 stage ring starts in dynamic shared memory, and the launch's total.
__host__ __device__ inline int64_t tma_ring_offset(const gfs_consumer& k, int bs) {
  return (consumer_smem_bytes(k, bs) + 127) / 128 * 128;
}
// Stages of the ring: five when they fit beside the consumer's state, else four.  Five
// stages (40 KiB) + the static control block still let 4 CTAs (592 TBs) share an SM.
inline int tma_ring_stages(const gfs_consumer& k, int bs) {
  return tma_ring_offset(k, bs) + TMA_NST_MAX * TMA_CH <= CONS_SMEM_MAX ? TMA_NST_MAX : TMA_NST;
}
inline int64_t gread_smem_bytes(const gfs_consumer& k, int bs, int tma) {
  return tma ? tma_ring_offset(k, bs) + tma_ring_stages(k, bs) * TMA_CH : consumer_smem_bytes(k, bs);
}

// y += A x over the request's rows (cols % 4 == 0: one row per 16-byte vector).
template <int BS>
__device__ void gemv_part(const gfs_consumer& k, const uint4* v4, int64_t ne, int64_t e0) {
  __shared__ float rows[GEMV_ROWS];
  const int tid = threadIdx.x;
  const int64_t M = k.cols;
  const int64_t row_lo = e0 / M, row_hi = (e0 + ne - 1) / M;
  const bool local = row_hi - row_lo < GEMV_ROWS;
  // element e0 + l sits at (row_lo + (r0 + l) / M, (r0 + l) % M): 32-bit division
  const uint32_t r0 = (uint32_t)(e0 - row_lo * M), M32 = (uint32_t)M;
  if (local)
    for (int i = tid; i <= (int)(row_hi - row_lo); i += BS) rows[i] = 0.f;
  __syncthreads();
  for (int64_t i = tid; i < (ne >> 2); i += BS) {
    const uint4 u = __ldcg(v4 + i);
    const uint32_t l = r0 + 4 * (uint32_t)i;
    const uint32_t q = l / M32;
    const int64_t row = row_lo + q, col = l - q * M32;
    const float4 xv = *(const float4*)(k.x + col);
    float p = decode_f32(u.x) * xv.x + decode_f32(u.y) * xv.y + decode_f32(u.z) * xv.z +
              decode_f32(u.w) * xv.w;
    // a warp's 32 consecutive vectors usually share one row: reduce them first
    const unsigned active = __activemask();
    const int64_t row0 = __shfl_sync(active, row, __ffs(active) - 1);
    if (active == 0xffffffffu && __all_sync(active, row == row0)) {
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      if ((threadIdx.x & 31) == 0) {
        if (local) atomicAdd(&rows[row - row_lo], p);
        else atomicAdd(&k.y[row], p);
      }
    } else if (local) {
      atomicAdd(&rows[row - row_lo], p);
    } else {
      atomicAdd(&k.y[row], p);
    }
  }
  __syncthreads();
  if (local)
    for (int i = tid; i <= (int)(row_hi - row_lo); i += BS) atomicAdd(&k.y[row_lo + i], rows[i]);
  __syncthreads();
}

// y2 += A^T x2: a warp's vectors cover consecutive columns, so the per-CTA shared
// accumulator (held across every TB the CTA runs, flushed once) sees no same-address
// conflicts; wider matrices accumulate straight into y2.
__device__ void gemvt_part(const gfs_consumer& k, float* acc, const uint4* v4, int64_t ne, int64_t e0,
                           int tid, int bs) {
  const int64_t M = k.cols;
  const bool sm = M <= GEMVT_SMEM_COLS;
  const int64_t row_lo = e0 / M;
  const uint32_t r0 = (uint32_t)(e0 - row_lo * M), M32 = (uint32_t)M;
  if (sm && M % (4 * bs) == 0 && M / (4 * bs) <= 4) {
    // Each thread meets the same <= 4 column quads in every row of the request (the
    // vector stride 4 bs divides the row): sum them in registers, then add them to the
    // CTA accumulator once — threads own disjoint columns, so plain shared adds.
    const int nq = (int)(M / (4 * bs));
    float a[4][4] = {};
    const int64_t nv = ne >> 2;
    for (int64_t i0 = tid; i0 < nv; i0 += (int64_t)bs * nq) {
#pragma unroll
      for (int m = 0; m < 4; m++) {  // static indices: a[][] stays in registers
        const int64_t i = i0 + (int64_t)m * bs;
        if (m < nq && i < nv) {
          const uint4 u = __ldcg(v4 + i);
          const uint32_t l = r0 + 4 * (uint32_t)i;
          const float xr = k.x2[row_lo + l / M32];
          a[m][0] += decode_f32(u.x) * xr;
          a[m][1] += decode_f32(u.y) * xr;
          a[m][2] += decode_f32(u.z) * xr;
          a[m][3] += decode_f32(u.w) * xr;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 4; m++) {
      if (m < nq) {
        const uint32_t col = (r0 + 4 * (uint32_t)(tid + m * bs)) % M32;
        acc[col + 0] += a[m][0];
        acc[col + 1] += a[m][1];
        acc[col + 2] += a[m][2];
        acc[col + 3] += a[m][3];
      }
    }
    return;
  }
  for (int64_t i = tid; i < (ne >> 2); i += bs) {
    const uint4 u = __ldcg(v4 + i);
    const uint32_t l = r0 + 4 * (uint32_t)i;
    const uint32_t q = l / M32;
    const int64_t row = row_lo + q, col = l - q * M32;
    const float xr = k.x2[row];
    float* dst = sm ? acc + col : k.y2 + col;
    atomicAdd(dst + 0, decode_f32(u.x) * xr);
    atomicAdd(dst + 1, decode_f32(u.y) * xr);
    atomicAdd(dst + 2, decode_f32(u.z) * xr);
    atomicAdd(dst + 3, decode_f32(u.w) * xr);
  }
}

// Kmeans assignment + accumulation, one thread per point.  Distances are summed over the
// features in order with IEEE round-to-nearest steps and no contraction (the bits a
// float32 reference gets).  Warp-uniform loop: a warp takes 32 consecutive points per
// step.  The point bytes were just delivered into the user buffer (never read by this SM
// before), so L1-cached loads are coherent here: the distance pass brings the lines into
// L1 and the accumulation pass re-reads them from there instead of from L2.
template <int BS>
__device__ void kmeans_part(const gfs_consumer& k, float* smem, const uint8_t* data, int64_t np) {
  const int K = k.k;
  const int D = (int)k.cols;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int W = BS / 32;
  const bool wacc = kmeans_warp_acc(k, BS);
  const float* cent = smem;
  float* acc = smem + K * D + (wacc ? warp * K * D : 0);
  unsigned* cnt = (unsigned*)(smem + K * D + (wacc ? W : 1) * K * D) + (wacc ? warp * K : 0);
  for (int64_t pb = (int64_t)warp * 32; pb < np; pb += BS) {
    const int64_t p = pb + lane;
    const bool valid = p < np;
    const uint4* pv = (const uint4*)(data + (valid ? p : 0) * (int64_t)D * 4);
    int best = 0;
    if (valid) {
      float d[GFS_KMEANS_MAX_K];
#pragma unroll
      for (int c = 0; c < GFS_KMEANS_MAX_K; c++) d[c] = 0.f;
      // 16 features per round: the point's four 16-byte loads are issued together (one L2
      // round trip instead of four), then summed in feature order
      for (int j0 = 0; j0 < D; j0 += 16) {
        uint4 uu[4];
#pragma unroll
        for (int r = 0; r < 4; r++)
          uu[r] = j0 + 4 * r < D ? __ldca(pv + (j0 >> 2) + r) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int j = j0 + 4 * r;
          if (j >= D) break;
          const uint4 u = uu[r];
          const float v[4] = {decode_f32(u.x), decode_f32(u.y), decode_f32(u.z), decode_f32(u.w)};
#pragma unroll
          for (int c = 0; c < GFS_KMEANS_MAX_K; c++) {
            if (c < K) {  // one 16-byte broadcast load of the centroid's 4 features (D % 4 == 0)
              const float4 cv = *(const float4*)(cent + c * D + j);
              const float cq[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const float df = __fsub_rn(v[q], cq[q]);
                d[c] = __fadd_rn(d[c], __fmul_rn(df, df));
              }
            }
          }
        }
      }
      float bd = d[0];
#pragma unroll
      for (int c = 1; c < GFS_KMEANS_MAX_K; c++)
        if (c < K && d[c] < bd) { bd = d[c]; best = c; }
    }
    const uint32_t* pw = (const uint32_t*)pv;
    float* row = acc + best * D;
    if (wacc) {
      for (int c = 0; c < K; c++) {  // per-warp counts: one ballot per centroid
        const unsigned m = __ballot_sync(0xffffffffu, valid && best == c);
        if (lane == 0) cnt[c] += __popc(m);
      }
      // lanes start at different features (cols >= 32), so in every step the 32 lanes
      // touch 32 distinct words of this warp's accumulator: plain read-modify-write
      // (the point's words are re-read 8 at a time so one memory latency covers 8 steps)
      int t = 0;
      for (; t + 8 <= D; t += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          int j = lane + t + u;
          if (j >= D) j -= D;
          v[u] = valid ? decode_f32(__ldca(pw + j)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          int j = lane + t + u;
          if (j >= D) j -= D;
          if (valid) row[j] += v[u];
          __syncwarp();
        }
      }
      for (; t < D; t++) {
        int j = lane + t;
        if (j >= D) j -= D;
        if (valid) row[j] += decode_f32(__ldca(pw + j));
        __syncwarp();
      }
    } else if (valid) {
      atomicAdd(&cnt[best], 1u);
      int t = 0;
      for (; t + 4 <= D; t += 4) {  // 4 loads in flight per latency
        float v[4];
        int jj[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          int j = lane + t + u;
          while (j >= D) j -= D;
          jj[u] = j;
          v[u] = decode_f32(__ldca(pw + j));
        }
#pragma unroll
        for (int u = 0; u < 4; u++) atomicAdd(&row[jj[u]], v[u]);
      }
      for (; t < D; t++) {
        int j = lane + t;
        while (j >= D) j -= D;
        atomicAdd(&row[j], decode_f32(__ldca(pw + j)));
      }
    }
  }
}

// Kmeans through a per-warp shared-memory stage (the K1 TMA ring, idle between greads): a
// warp loads its 32 points with coalesced 16-byte loads, all in flight at once, decodes them
// into rows rotated by the point index (feature f of point p at column (f + p) mod D, so
// the 32 lanes reading "their" feature j hit distinct banks), then runs the distance and
// accumulation passes out of shared memory.  One memory round trip per 32 points instead of
// one per feature group; the arithmetic and its order are those of kmeans_part.
__host__ __device__ inline bool kmeans_staged_fits(const gfs_consumer& k, int bs) {
  return (int64_t)(bs / 32) * 32 * k.cols * 4 <= TMA_NST * TMA_CH;
}

template <int BS>
__device__ void kmeans_part_staged(const gfs_consumer& k, float* smem, const uint8_t* data, int64_t np,
                                   float* ring) {
  const int K = k.k;
  const int D = (int)k.cols;
  const int q4 = D >> 2;  // 16-byte vectors per point
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int W = BS / 32;
  const bool wacc = kmeans_warp_acc(k, BS);
  const float* cent = smem;
  float* acc = smem + K * D + (wacc ? warp * K * D : 0);
  unsigned* cnt = (unsigned*)(smem + K * D + (wacc ? W : 1) * K * D) + (wacc ? warp * K : 0);
  float* stg = ring + (int64_t)warp * 32 * D;
  const float* prow = stg + lane * D;
  const int kp = (K + 3) / 4 * 4;
  const float* ct = smem + kmeans_ct_off(k, BS);
  const int rot = lane % D;
  for (int64_t pb = (int64_t)warp * 32; pb < np; pb += BS) {
    const int64_t p = pb + lane;
    const bool valid = p < np;
    const int nq = (int)min((int64_t)32, np - pb) * q4;
    const uint4* src = (const uint4*)(data + pb * (int64_t)D * 4);
    __syncwarp();  // the previous step's reads of the stage are done
    for (int q0 = 0; q0 < nq; q0 += 32 * 8) {
      uint4 u[8];
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int q = q0 + lane + 32 * i;
        if (q < nq) u[i] = __ldcg(src + q);
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int q = q0 + lane + 32 * i;
        if (q < nq) {
          const int pp = q / q4, f0 = (q - pp * q4) * 4;
          float* row = stg + pp * D;
          int col = f0 + pp % D;
          if (col >= D) col -= D;
          const float v4[4] = {decode_f32(u[i].x), decode_f32(u[i].y), decode_f32(u[i].z), decode_f32(u[i].w)};
#pragma unroll
          for (int r = 0; r < 4; r++) {
            row[col] = v4[r];
            if (++col == D) col = 0;
          }
        }
      }
    }
    __syncwarp();
    int best = 0;
    if (valid) {
      // four centroids per sweep over the features (one broadcast 16-byte load of their
      // feature j from the transposed copy, four independent chains), features in order
      float bd = 0.f;
      for (int c0 = 0; c0 < K; c0 += 4) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        int col = rot;
#pragma unroll 4
        for (int j = 0; j < D; j++) {
          const float v = prow[col];
          if (++col == D) col = 0;
          const float4 cv = *(const float4*)(ct + j * kp + c0);
          float df;
          df = __fsub_rn(v, cv.x);
          a0 = __fadd_rn(a0, __fmul_rn(df, df));
          df = __fsub_rn(v, cv.y);
          a1 = __fadd_rn(a1, __fmul_rn(df, df));
          df = __fsub_rn(v, cv.z);
          a2 = __fadd_rn(a2, __fmul_rn(df, df));
          df = __fsub_rn(v, cv.w);
          a3 = __fadd_rn(a3, __fmul_rn(df, df));
        }
        const float a[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int i = 0; i < 4; i++)  // first minimum wins, as in kmeans_part
          if (c0 + i < K && (c0 + i == 0 || a[i] < bd)) {
            bd = a[i];
            best = c0 + i;
          }
      }
    }
    float* row = acc + best * D;
    if (wacc) {
      for (int c = 0; c < K; c++) {
        const unsigned m = __ballot_sync(0xffffffffu, valid && best == c);
        if (lane == 0) cnt[c] += __popc(m);
      }
      // lane L adds feature (L + t) mod D in step t: 32 distinct accumulator words per step;
      // that feature sits at stage column (L + t + L) mod D of the lane's row
      int j = lane % D, sc = (2 * lane) % D;
      for (int t = 0; t < D; t++) {
        if (valid) row[j] += prow[sc];
        __syncwarp();
        if (++j == D) j = 0;
        if (++sc == D) sc = 0;
      }
    } else if (valid) {
      atomicAdd(&cnt[best], 1u);
      int j = lane % D, sc = (2 * lane) % D;
      for (int t = 0; t < D; t++) {
        atomicAdd(&row[j], prow[sc]);
        if (++j == D) j = 0;
        if (++sc == D) sc = 0;
      }
    }
  }
}

// All threads, once per launch before the first TB: zero / load the consumer's shared state.
__device__ void consume_init(const DevCtx& c, float* smem) {
  const gfs_consumer& k = c.cons;
  const int64_t n = consumer_smem_bytes(k, blockDim.x) / 4;
  if (n == 0) return;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) smem[i] = 0.f;
  if (k.kind == GFS_CONSUME_KMEANS_F32) {
    __syncthreads();  // the zeroing above used another thread -> index mapping
    for (int64_t i = threadIdx.x; i < (int64_t)k.k * k.cols; i += blockDim.x) smem[i] = k.x[i];
    const int kp = (k.k + 3) / 4 * 4;  // transposed copy, zero-padded centroids
    float* ct = smem + kmeans_ct_off(k, blockDim.x);
    for (int64_t i = threadIdx.x; i < (int64_t)k.cols * kp; i += blockDim.x) {
      const int64_t j = i / kp, c = i - j * kp;
      ct[i] = c < k.k ? k.x[c * k.cols + j] : 0.f;
    }
  }
  __syncthreads();
}

// Consume the n bytes the TB just delivered (`data`, in the user buffer) that came from
// file offset `file_off`.  All threads.
template <int BS>
__device__ void consume(const DevCtx& c, float* smem, const uint8_t* data, int64_t n, int64_t file_off,
                        ConsAcc& acc) {
  const int tid = threadIdx.x;
  const gfs_consumer& k = c.cons;
  if (n <= 0) return;
  if (k.kind == GFS_CONSUME_SUM64) {  // words of the file, position-weighted
    const int64_t nw = n >> 3, w0 = file_off >> 3;
    const uint64_t* w = (const uint64_t*)data;
    for (int64_t i = tid; i < nw; i += BS)
      acc.sum += mix64(__ldcg(w + i) ^ ((uint64_t)(w0 + i) * 0x9E3779B97F4A7C15ull));
  } else if (k.kind == GFS_CONSUME_NN_F32) {  // records (lat, lng): nearest to (qx, qy)
    const int64_t nr = n >> 3, r0 = file_off >> 3;
    const uint2* rec = (const uint2*)data;
    for (int64_t i = tid; i < nr; i += BS) {
      const uint2 u = __ldcg(rec + i);
      // IEEE single-precision steps without contraction: the same bits numpy float32 gets
      const float lat = __fsub_rn(__fmul_rn(decode_f32(u.x), 180.0f), 90.0f);
      const float lng = __fsub_rn(__fmul_rn(decode_f32(u.y), 360.0f), 180.0f);
      const float dx = __fsub_rn(lat, k.qx), dy = __fsub_rn(lng, k.qy);
      const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      const unsigned long long key =
          ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned long long)(uint32_t)(r0 + i);
      acc.nn = key < acc.nn ? key : acc.nn;
    }
  } else if (k.kind == GFS_CONSUME_GEMV_F32) {
    gemv_part<BS>(k, (const uint4*)data, n >> 2, file_off >> 2);
  } else if (k.kind == GFS_CONSUME_GEMVT_F32) {
    gemvt_part(k, smem, (const uint4*)data, n >> 2, file_off >> 2, tid, BS);
  } else if (k.kind == GFS_CONSUME_BICG_F32) {
    gemvt_part(k, smem, (const uint4*)data, n >> 2, file_off >> 2, tid, BS);
    gemv_part<BS>(k, (const uint4*)data, n >> 2, file_off >> 2);
  } else if (k.kind == GFS_CONSUME_KMEANS_F32) {
    if (c.tma && kmeans_staged_fits(k, BS))  // the K1 ring is free between greads
      kmeans_part_staged<BS>(k, smem, data, n / (k.cols * 4), (float*)((uint8_t*)smem + c.tma_off));
    else
      kmeans_part<BS>(k, smem, data, n / (k.cols * 4));
  }
}

template <int BS>
__device__ void consume_flush(const DevCtx& c, float* smem, ConsAcc& acc) {
  const int kind = c.cons.kind;
  const gfs_consumer& k = c.cons;
  if (kind == GFS_CONSUME_GEMVT_F32 || kind == GFS_CONSUME_BICG_F32 || kind == GFS_CONSUME_KMEANS_F32) {
    __syncthreads();
    if (kind == GFS_CONSUME_KMEANS_F32) {
      const int64_t kd = (int64_t)k.k * k.cols;
      const int nacc = kmeans_warp_acc(k, BS) ? BS / 32 : 1;  // accumulator copies
      for (int64_t i = threadIdx.x; i < kd; i += BS) {
        float v = 0.f;
        for (int w = 0; w < nacc; w++) v += smem[kd + w * kd + i];
        if (v != 0.f) atomicAdd(&k.y[i], v);
      }
      const unsigned* cnt = (const unsigned*)(smem + (1 + nacc) * kd);
      for (int i = threadIdx.x; i < k.k; i += BS) {
        unsigned long long v = 0;
        for (int w = 0; w < nacc; w++) v += cnt[w * k.k + i];
        if (v) atomicAdd(&k.out[i], v);
      }
    } else if (k.cols <= GEMVT_SMEM_COLS) {
      for (int64_t i = threadIdx.x; i < k.cols; i += BS)
        if (smem[i] != 0.f) atomicAdd(&k.y2[i], smem[i]);
    }
    return;
  }
  if (kind != GFS_CONSUME_SUM64 && kind != GFS_CONSUME_NN_F32) return;
  unsigned long long v = kind == GFS_CONSUME_SUM64 ? acc.sum : acc.nn;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = kind == GFS_CONSUME_SUM64 ? v + w : (w < v ? w : v);
  }
  if ((threadIdx.x & 31) == 0) {
    if (kind == GFS_CONSUME_SUM64) atomicAdd(c.cons.out, v);
    else atomicMin(c.cons.out, v);
  }
}

// TB program (gpu_exec.py:95-105) and TB done (drain + retire, gpu_exec.py:281-291).
template <int BS>
__device__ bool run_tb(const DevCtx& c, Smem& s, float* cons_smem, int tb, int& bad_words, ConsAcc& acc) {
  const int tid = threadIdx.x;
  tb_begin(c, s, tb);
  int64_t pos = c.dst_off[tb];
  const int64_t s0 = c.prog_off[tb], s1 = c.prog_off[tb + 1];
  for (int64_t sg = s0; sg < s1; sg++) {
    const int64_t fid = c.segs[3 * sg], base = c.segs[3 * sg + 1], len = c.segs[3 * sg + 2];
    if (fid < 0 || fid >= c.n_files) {
      if (tid == 0) set_error(c, ERR_BAD_PROGRAM, tb, (unsigned long long)sg);
      return false;
    }
    if (c.lookahead && sg > s0) {  // bytes delivered ahead belong to the segment that fetched them
      // a gread answered from the lookahead range returns without a block barrier: every
      // thread must have read la_* there before it is cleared
      __syncthreads();
      if (tid == 0) s.la_fid = -1;
      __syncthreads();
    }
    if (tid == 0) {  // the requests of this segment start at base + k * request_bytes
      s.seg_lo = base;
      s.seg_hi = base + len;
      s.seg_ord = sg - s0;
    }
    int64_t seg_off = 0;
    while (seg_off < len) {
      int64_t size = c.request_bytes < len - seg_off ? c.request_bytes : len - seg_off;
      uint8_t* d = c.dst ? c.dst + pos + seg_off : nullptr;
      const uint64_t tg = c.timeline ? globaltimer() : 0;
      int64_t got = gread<BS>(c, s, fid, base + seg_off, size, base + len, d, bad_words);
      if (got < 0) return false;
      if (c.timeline && tid == 0) tl_rec(c, GFS_TL_GREAD, tb, got, tg, globaltimer());
      if (c.cons.kind != GFS_CONSUME_NONE && d) {
        const uint64_t tc = c.timeline ? globaltimer() : 0;
        consume<BS>(c, cons_smem, d, got, base + seg_off, acc);
        if (c.timeline) {
          __syncthreads();
          if (tid == 0) tl_rec(c, GFS_TL_CONSUME, tb, got, tc, globaltimer());
        }
      }
      seg_off += got;
      if (got < size) break;  // short read: rest of the segment is skipped
    }
    pos += len;
  }
  tb_end<BS>(c, s);
  return true;
}

template <int BS>
__global__ void __launch_bounds__(BS, 4) gread_driver(DevCtx c) {
  __shared__ Smem s;
  cta_begin<BS>(c, s);
  extern __shared__ __align__(128) float cons_smem[];  // consumer state, then the K1 stage ring
  consume_init(c, cons_smem);
  int bad_words = 0;
  ConsAcc acc;
  for (;;) {
    const int tb = next_tb(c, s);
    if (tb < 0) break;
    if (!run_tb<BS>(c, s, cons_smem, tb, bad_words, acc)) break;
  }
  consume_flush<BS>(c, cons_smem, acc);
  cta_end(c, s, bad_words);
}

// ------------------------------------------------------------------ K4 consumers

__global__ void checksum_kernel(const uint8_t* buf, uint64_t nbytes, uint64_t word_base,
                                unsigned long long* out) {
  const uint64_t nw = nbytes >> 3;
  const uint64_t* w = (const uint64_t*)buf;
  uint64_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 2;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < nw; i += stride) {
    if (i + 1 < nw) {
      uint4 q = __ldcs((const uint4*)(w + i));
      uint64_t lo = ((uint64_t)q.y << 32) | q.x, hi = ((uint64_t)q.w << 32) | q.z;
      acc += mix64(lo ^ ((i + word_base) * 0x9E3779B97F4A7C15ull));
      acc += mix64(hi ^ ((i + 1 + word_base) * 0x9E3779B97F4A7C15ull));
    } else {
      acc += mix64(w[i] ^ ((i + word_base) * 0x9E3779B97F4A7C15ull));
    }
  }
  if ((nbytes & 7) && blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t last = 0;
    for (uint64_t b = 0; b < (nbytes & 7); b++) last |= (uint64_t)buf[(nw << 3) + b] << (8 * b);
    acc += mix64(last ^ ((nw + word_base) * 0x9E3779B97F4A7C15ull));
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ uint64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += part[i];
    atomicAdd(out, (unsigned long long)t);
  }
}

// Compare the user buffer with the synthetic law, segment by segment.
__global__ void verify_dst_kernel(const uint8_t* buf, const int64_t* segs, const int64_t* seg_dst,
                                  int64_t n_segs, const DevFile* files,
                                  unsigned long long* mismatches) {
  unsigned long long bad = 0;
  for (int64_t sg = blockIdx.x; sg < n_segs; sg += gridDim.x) {
    const int64_t fid = segs[3 * sg], off = segs[3 * sg + 1];
    int64_t len = segs[3 * sg + 2];
    const DevFile& F = files[fid];
    if (F.content_id < 0) continue;
    if (off + len > F.size) len = F.size > off ? F.size - off : 0;
    const uint8_t* d = buf + seg_dst[sg];
    if ((((uintptr_t)d - (uintptr_t)off) & 7) == 0) {
      int64_t head = (8 - (off & 7)) & 7;
      if (head > len) head = len;
      for (int64_t i = threadIdx.x; i < head; i += blockDim.x) {
        int64_t fo = off + i;
        bad += d[i] != (uint8_t)(word_law(F.content_id, fo >> 3) >> (8 * (fo & 7)));
      }
      const uint64_t* dw = (const uint64_t*)(d + head);
      const int64_t w0 = (off + head) >> 3, nw = (len - head) >> 3;
      for (int64_t i = threadIdx.x; i < nw; i += blockDim.x)
        bad += __ldcs(dw + i) != word_law(F.content_id, w0 + i);
      for (int64_t i = head + (nw << 3) + threadIdx.x; i < len; i += blockDim.x) {
        int64_t fo = off + i;
        bad += d[i] != (uint8_t)(word_law(F.content_id, fo >> 3) >> (8 * (fo & 7)));
      }
    } else {
      for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
        int64_t fo = off + i;
        bad += d[i] != (uint8_t)(word_law(F.content_id, fo >> 3) >> (8 * (fo & 7)));
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatches, bad);
}

// ------------------------------------------------------------------ end-of-run invariants

// GpuPageCache.check_unique_mapping (gpu_cache.py:217-224, called from
// simulation.py:252-253), over the lock-free table: every PTE that names a frame must name a
// settled (VALID, unpinned, not in flight) frame whose key is that (file, page), and no frame
// may be reachable from two PTEs.  owner[] (nframes, 0xFF-filled) records the first PTE
// that reached each frame.  out: [0] mapped pages, [1] frames reached twice, [2] key
// mismatches, [3] unsettled entries (claimed / in flight / not valid / pinned).
__global__ void check_mapping_pt_kernel(const DevFile* files, int n_files, const unsigned long long* fkey,
                                        const uint32_t* fstate, uint32_t* owner, int64_t nframes,
                                        unsigned long long* out) {
  unsigned long long n[4] = {0, 0, 0, 0};
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int f = 0; f < n_files; f++) {
    const DevFile& F = files[f];
    if (!F.pt) continue;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < F.npages; p += step) {
      const uint32_t e = F.pt[p];
      if (e == PT_EMPTY) continue;
      n[0]++;
      if (e == PT_CLAIMED || (e & PT_INFLIGHT) || (int64_t)e >= nframes) {
        n[3]++;
        continue;
      }
      if (atomicCAS(&owner[e], 0xFFFFFFFFu, (uint32_t)p) != 0xFFFFFFFFu) n[1]++;
      if (fkey[e] != page_key(f, p)) n[2]++;
      if (fstate[e] != FR_VALID) n[3]++;  // VALID with a zero refcount
    }
  }
  for (int k = 0; k < 4; k++) {
    unsigned long long v = n[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[k], v);
  }
}

// out[4]: VALID frames of an open file that no PTE reaches (a cached page the table lost).
__global__ void check_mapping_frames_kernel(const DevFile* files, int n_files, const unsigned long long* fkey,
                                            const uint32_t* fstate, const uint32_t* owner, int64_t nframes,
                                            unsigned long long* out) {
  unsigned long long v = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nframes; i += (int64_t)gridDim.x * blockDim.x) {
    if (!(fstate[i] & FR_VALID) || owner[i] != 0xFFFFFFFFu) continue;
    const int64_t fid = (int64_t)(fkey[i] >> 40);
    v += fid < n_files && files[fid].pt != nullptr;  // frames of closed files have no table
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&out[4], v);
}

// ------------------------------------------------------------------ host-side launchers

cudaError_t launch_gread(const DevCtx& c, int cta_threads, cudaStream_t st) {
  const size_t smem = (size_t)gread_smem_bytes(c.cons, cta_threads, c.tma);
  if (smem > 0) {  // beyond the default dynamic limit (48 KiB minus the static Smem) needs opt-in
    cudaError_t e = cudaSuccess;
    switch (cta_threads) {
      case 128: e = cudaFuncSetAttribute(gread_driver<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
      case 512: e = cudaFuncSetAttribute(gread_driver<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
      default: e = cudaFuncSetAttribute(gread_driver<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); break;
    }
    if (e != cudaSuccess) return e;
  }
  switch (cta_threads) {
    case 128: gread_driver<128><<<c.n_ctas, 128, smem, st>>>(c); break;
    case 512: gread_driver<512><<<c.n_ctas, 512, smem, st>>>(c); break;
    default: gread_driver<256><<<c.n_ctas, 256, smem, st>>>(c); break;
  }
  return cudaGetLastError();
}

// K1 stage ring placement for this launch: offset (bytes), or -1 when the consumer state
// and the ring together would not fit the dynamic shared memory available without opt-in.
// Dynamic shared memory a launch of the gread path needs (gfs_run_kernel passes it on).
int64_t gread_launch_smem(const gfs_consumer& k, int cta_threads, int tma) {
  return gread_smem_bytes(k, cta_threads, tma);
}

int gread_tma_stages(const gfs_consumer& k, int cta_threads) { return tma_ring_stages(k, cta_threads); }

int64_t gread_tma_offset(const gfs_consumer& k, int cta_threads) {
  const int64_t off = tma_ring_offset(k, cta_threads);
  return off + TMA_NST * TMA_CH <= CONS_SMEM_MAX ? off : -1;
}

// Copy-queue probe (gfs_create): waits, bounded, until each of n flags was written by its
// copy / doorbell stream while this kernel occupies the run stream.
__global__ void queue_probe_kernel(const unsigned long long* flags, int n, uint64_t timeout_ns, int* ok) {
  const uint64_t t0 = globaltimer();
  for (int i = 0; i < n; i++)
    while (ld_acquire_sys64(flags + i) != 1ull) {
      if (globaltimer() - t0 > timeout_ns) {
        *ok = 0;
        return;
      }
      __nanosleep(1000);
    }
  *ok = 1;
}

cudaError_t launch_queue_probe(const unsigned long long* flags, int n, uint64_t timeout_ns, int* ok,
                               cudaStream_t st) {
  queue_probe_kernel<<<1, 1, 0, st>>>(flags, n, timeout_ns, ok);
  return cudaGetLastError();
}

cudaError_t occupancy_gread(int cta_threads, int* blocks_per_sm) {
  switch (cta_threads) {
    case 128: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, gread_driver<128>, 128, 0);
    case 512: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, gread_driver<512>, 512, 0);
    default: return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, gread_driver<256>, 256, 0);
  }
}

cudaError_t launch_check_mapping(const DevFile* files, int n_files, const unsigned long long* fkey,
                                 const uint32_t* fstate, uint32_t* owner, int64_t nframes,
                                 unsigned long long* out, int sms, cudaStream_t st) {
  check_mapping_pt_kernel<<<sms * 4, 512, 0, st>>>(files, n_files, fkey, fstate, owner, nframes, out);
  check_mapping_frames_kernel<<<sms * 4, 512, 0, st>>>(files, n_files, fkey, fstate, owner, nframes, out);
  return cudaGetLastError();
}

cudaError_t launch_checksum(const void* buf, uint64_t nbytes, uint64_t word_base,
                            unsigned long long* out, int sms, cudaStream_t st) {
  int grid = sms * 4;
  checksum_kernel<<<grid, 512, 0, st>>>((const uint8_t*)buf, nbytes, word_base, out);
  return cudaGetLastError();
}

cudaError_t launch_verify_dst(const void* buf, const int64_t* segs, const int64_t* seg_dst,
                              int64_t n_segs, const DevFile* files, unsigned long long* out,
                              int sms, cudaStream_t st) {
  int grid = (int)(n_segs < (int64_t)sms * 8 ? n_segs : (int64_t)sms * 8);
  if (grid < 1) grid = 1;
  verify_dst_kernel<<<grid, 512, 0, st>>>((const uint8_t*)buf, segs, seg_dst, n_segs, files, out);
  return cudaGetLastError();
}

}  // namespace gfs
