// gfs_device_impl.cuh — the device file layer shared by the persistent gread driver
// (gfs_kernels.cu) and user kernels (include/gfs_device.cuh): page cache, private
// buffer, readahead, RPC ring, K1/K2 copies and the TB-collective gread
// (reference gpu_exec.py:95-239, gpu_cache.py:92-224, prefetcher.py:13-68, rpc.py:82-113).
//
// Header-only: every translation unit that includes it compiles its own copy of the
// device code (no relocatable device code needed).  All state is reached through the
// DevCtx the host fills (gfs_host.cpp) and the per-CTA Smem block.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gfs_shared.h"

namespace gfs {

// ------------------------------------------------------------------ primitives

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// W(f, i) = mix64(page_tag(f, i >> 9) ^ i): the synthetic content law.
__device__ __forceinline__ uint64_t block_tag(int64_t cid, int64_t i) {
  return mix64(((uint64_t)cid << 40) ^ (uint64_t)(i >> 9) ^ 0xA5A5A5A5A5A5A5A5ull);
}
__device__ __forceinline__ uint64_t word_law(int64_t cid, int64_t i) {
  return mix64(block_tag(cid, i) ^ (uint64_t)i);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// refcount pin with acquire semantics: the frame key read after it cannot be satisfied from
// a line cached before the pin (the key is then read from L2 with __ldcg)
__device__ __forceinline__ uint32_t atomic_add_acquire_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acquire.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Hand a host pool buffer back to the daemon.  Only *loads* from the buffer precede it, and
// they have all returned (the caller passed a barrier after using the values), so a relaxed
// system-scope store is enough: no membar.sys, which would wait behind the link's reads.
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// device-memory counters shared by CTAs: relaxed loads at GPU scope (no system-scope
// strong load needed: the host never writes them while the kernel runs)
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ TMA bulk copies

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}

// global -> shared bulk copy completing `bytes` of transaction count on `bar` (one thread)
__device__ __forceinline__ void tma_load(void* sdst, const void* gsrc, uint32_t bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// shared -> global bulk copy in the current bulk group (one thread)
__device__ __forceinline__ void tma_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes -> generic readers
}

// source kinds for K1/K2 loads
enum { SRC_HBM = 0, SRC_SYS = 1 };

template <int SRC>
__device__ __forceinline__ uint4 ld16(const uint4* p) {
  if (SRC == SRC_SYS) return __ldcv(p);  // mapped pinned host memory: always refetch
  return __ldcg(p);                      // HBM written by other SMs / copy engine: bypass L1
}
template <int SRC>
__device__ __forceinline__ uint8_t ld1(const uint8_t* p) {
  if (SRC == SRC_SYS) return *(volatile const uint8_t*)p;
  return __ldcg((const unsigned char*)p);
}

// ----------------------------------------------------------------- CTA state

constexpr int TMA_NST = 4;        // K1 stage ring: stages (at least)
constexpr int TMA_NST_MAX = 5;    // ... and at most, when the consumer's shared state leaves room
// stage and mbarrier phase of chunk g in an n-stage ring (n = 4 or 5: constant divisors)
__device__ __forceinline__ int stage_of(unsigned long long g, int n) { return n == 5 ? (int)(g % 5) : (int)(g & 3); }
__device__ __forceinline__ uint32_t phase_of(unsigned long long g, int n) {
  return n == 5 ? (uint32_t)((g / 5) & 1) : (uint32_t)((g >> 2) & 1);
}
constexpr int OD_MARKS = 4;       // readahead markers remembered per TB stream
constexpr int64_t TMA_CH = 8192;  // bytes per stage (one bulk load, 1-2 bulk stores per page)

struct Smem {
  unsigned long long tma_bar[TMA_NST_MAX];    // stage "full" mbarriers (tx-count)
  unsigned long long tma_empty[TMA_NST_MAX];  // stage "checked" mbarriers (one arrival per checker warp)
  unsigned long long tma_seq;             // chunks staged since launch (stage / parity)
  uint32_t tma_epend;                     // bit st: stage st awaits its checkers before reuse
  uint32_t tma_epar;                      // bit st: parity of that pending phase
  // broadcast from thread 0
  int act;
  int abort;
  uint32_t frame;
  int64_t n;        // RPC result bytes
  int64_t nb;       // bytes installed into the frame
  int64_t src_off;  // offset of the page inside the span buffer
  int64_t k;        // dispatcher ticket
  int any_bad;
  uint64_t t_copy0;
  // bounce mode: span waiting in a host pool buffer to be pulled into the HBM landing slot
  int64_t pull_n;
  int32_t pull_buf;  // bounce buffer to release afterwards, -1 = none (mapped file)
  uint32_t pull_seq;
  const uint8_t* pull_src;
  // TB state (thread 0)
  int tb;
  int64_t own_head, own_len;
  long long last_gfifo_pos;
  int64_t pb_fid, pb_base, pb_count, pb_filled;
  int64_t ra_win, ra_next_fid, ra_next_page;
  int pending_seen;
  long long st[GFS_NSTATS];
  // batched page walk (gread_batch): one entry per page of the batch
  struct {
    int n_empty, k, status, nvict, nret, ret_lane0, own_lane0, j0, ret_pool, src_half;
    int early, fb_h, fb_od;         // page 0's RPC submitted before the frame work (fetch_begin)
    int64_t fb_span;
    uint32_t fb_seq;
    unsigned long long fb_pos;
    unsigned tail_mask, part_mask;  // pages with a sub-16 B EOF tail / a partial delivery
    int64_t total;                  // bytes this batch delivers
    int64_t rpc_n;
    int64_t sync_m;                 // ondemand: pages of the synchronous span (od_plan_sync)
    unsigned long long ret_pos;
    int64_t own_head0, own_tail0;
    uint32_t frame[32];
    int32_t nb[32];
    int64_t src_off[32];
    int32_t vict[32];  // 1 = frame must be evicted before reuse
  } b;
  int64_t pb_last_nb;        // bytes of the last private-buffer entry
  int fresh_done;            // this CTA saw the never-used frames run out (they never return)
  // lookahead: file bytes [la_lo, la_hi) of la_fid were delivered ahead of their gread
  int64_t la_fid, la_lo, la_hi;
  // landing halves: span_half holds the private buffer's bytes; fetch_half received the last
  // synchronous span (its page 0 is read from there; it becomes span_half only when the span
  // refills the private buffer, i.e. brings more than one page); pull_half is where a pending
  // CTA pull (bounce / mapped transfers) lands
  int span_half, fetch_half, pull_half, src_half;
  // streamed windows, per landing half: the last request into it and how much has landed
  uint32_t st_seq[2];
  int64_t st_n[2], st_landed[2];
  int64_t page_size_cached;  // c.page_size, for the smem-only pb_take
  int64_t pb_off_adj;        // span offset of entry i = i * page - pb_off_adj (pg for adopted windows)
  // ondemand readahead (io.readahead=adaptive, host_os.py:106-152), one stream per TB
  struct {
    int64_t fid, ws, wsize, async, prev_end;          // ReadaheadState, in pages
    int64_t mark[OD_MARKS];                            // marker pages (-1 = none)
    long long dec_key;                                 // gread instance decided last
    int64_t run_page, run_n;                           // async run decided, not yet submitted
    int64_t cap;                                       // next marker past the walk position
  } od;
  // the current gread and segment (ondemand: which request a page belongs to)
  int64_t g_lo, g_hi, seg_lo, seg_hi;
  long long seg_ord;
  int g_la;
  // landing halves holding a pending (requested, not adopted) readahead window
  struct {
    int pending, deferred;
    int64_t fid, page, span;
    uint32_t seq, age;
    unsigned long long pos;
  } hp[2];
  uint32_t hp_age;
  uint32_t rpc_out;  // this TB's requests outstanding (submitted, not yet waited for)
  int direct[2];       // half h's span is read straight from the pinned file mapping (K1 direct)
  int sm_rank;         // this CTA's start order among the CTAs on its SM
  int first_ticket;    // next_tb has not handed this CTA a TB yet
  // K1 early: a static request whose span K1 read before the daemon's answer (collected and
  // checked by early_collect before the CTA's next request / at TB end)
  struct {
    int on, half, polled;
    uint32_t seq;
    unsigned long long pos;
    int64_t fid, off, n;
    uint64_t t_sub;
  } early;
  // the answer's mailbox line, fetched by an asynchronous bulk copy while K1 runs
  unsigned long long poll_bar;
  uint32_t poll_par;
  uint4 poll_buf;
  int64_t pull_off;            // file offset of the span waiting to be pulled
  int64_t dbg_land_off[2], dbg_land_n[2];  // what each landing half last received (diagnostics)
  uint32_t pb_absent[MAX_PB_ENTRIES / 32];  // private-buffer entries consumed / dropped
};

enum { A_HIT = 1, A_PBHIT = 2, A_RPC = 3, A_ABORT = 4 };

#define ST(name) s.st[GFS_STAT_##name]

__device__ void set_error(const DevCtx& c, int code, int info, unsigned long long arg) {
  if (atomicCAS(&c.g->error, 0, code) == 0) {
    c.g->error_info = info;
    c.g->error_arg = arg;
  }
}

__device__ __forceinline__ bool has_error(const DevCtx& c) {
  int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&c.g->error) : "memory");
  return v != 0;
}

// spin helper: true while waiting may continue (no error, no timeout)
__device__ __forceinline__ bool keep_waiting(const DevCtx& c, uint64_t t0, int info) {
  if (has_error(c)) return false;
  if (globaltimer() - t0 > c.timeout_ns) {
    set_error(c, ERR_TIMEOUT, info, 0);
    return false;
  }
  return true;
}

// mbarrier wait with the device timeout: false (error set) instead of spinning forever.
__device__ bool mbar_wait_t(const DevCtx& c, unsigned long long* bar, uint32_t parity, int info,
                            unsigned long long arg) {
  const uint64_t t0 = globaltimer();
  for (;;) {
    uint32_t done = 0;
    for (int k = 0; k < 64 && !done; k++)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(smem_u32(bar)), "r"(parity)
                   : "memory");
    if (done) return true;
    if (has_error(c)) return false;
    if (globaltimer() - t0 > c.timeout_ns) {  // arg: chunk sequence << 16 | stage << 8 | chunk
      set_error(c, ERR_TIMEOUT, info, arg);
      return false;
    }
  }
}

__device__ void log_rec(const DevCtx& c, int kind, long long a, long long b, long long d, long long e) {
  if (!c.log) return;
  unsigned long long i = atomicAdd(&c.g->log_n[kind], 1ull);
  if (i >= c.log_cap[kind]) {
    set_error(c, ERR_LOG_OVERFLOW, kind, i);
    return;
  }
  const int width = kind == GFS_LOG_RPCS ? 4 : (kind == GFS_LOG_WINDOWS ? 2 : 3);
  long long* r = c.logs[kind] + i * width;
  r[0] = a;
  r[1] = b;
  if (width > 2) r[2] = d;
  if (width > 3) r[3] = e;
}

// Timeline record (thread 0; gfs_config.timeline): what a CTA was doing, and when.
// First K1 word mismatch of the run (diagnostics only; rare by construction).
__device__ void note_mismatch(const DevCtx& c, const Smem& s, int64_t fid, int64_t file_off, uint64_t got,
                              int64_t span_off, int pages) {
  if (atomicCAS(&c.g->dbg[0], 0ull, 1ull) != 0ull) return;
  c.g->dbg[1] = (unsigned long long)s.tb;
  c.g->dbg[2] = (unsigned long long)fid;
  c.g->dbg[3] = (unsigned long long)file_off;
  c.g->dbg[4] = got;
  c.g->dbg[5] = (unsigned long long)s.b.src_half;
  c.g->dbg[6] = (unsigned long long)span_off;
  c.g->dbg[7] = (unsigned long long)pages | ((unsigned long long)blockIdx.x << 32);
  c.g->dbg[8] = (unsigned long long)s.dbg_land_off[s.b.src_half];
  c.g->dbg[9] = (unsigned long long)s.dbg_land_n[s.b.src_half];
  c.g->dbg[10] = (unsigned long long)s.pb_base;
  c.g->dbg[11] = (unsigned long long)s.pb_off_adj;
  c.g->dbg[12] = (unsigned long long)s.pb_count;
  c.g->dbg[13] = (unsigned long long)(s.b.j0);
  c.g->dbg[14] = (unsigned long long)s.g_lo;
  c.g->dbg[15] = (unsigned long long)s.g_hi;
}

__device__ void tl_rec(const DevCtx& c, int kind, int tb, long long bytes, uint64_t t0, uint64_t t1) {
  if (!c.timeline) return;
  unsigned long long i = atomicAdd(&c.g->log_n[GFS_LOG_TIMELINE], 1ull);
  if (i >= c.log_cap[GFS_LOG_TIMELINE]) return;  // full: later records are dropped
  long long* r = c.logs[GFS_LOG_TIMELINE] + i * 4;
  r[0] = ((long long)kind << 56) | ((long long)blockIdx.x << 32) | (long long)(uint32_t)tb;
  r[1] = bytes;
  r[2] = (long long)t0;
  r[3] = (long long)t1;
}

// ------------------------------------------------------------ frame ownership

__device__ __forceinline__ unsigned long long page_key(int64_t fid, int64_t page) {
  return ((unsigned long long)fid << 40) | (unsigned long long)page;
}

// Unmap a VALID, unreferenced frame (gpu_cache.py:139-147, 165-178).  Fails if a
// reader holds a reference or the frame is not valid.
__device__ bool try_evict(const DevCtx& c, Smem& s, uint32_t v) {
  if (atomicCAS(&c.fstate[v], FR_VALID, 0u) != FR_VALID) return false;
  unsigned long long key = c.fkey[v];
  int64_t vfid = (int64_t)(key >> 40), vpage = (int64_t)(key & ((1ull << 40) - 1));
  atomicCAS(&c.files[vfid].pt[vpage], v, PT_EMPTY);
  log_rec(c, GFS_LOG_VICTIMS, s.tb, vfid, vpage, 0);
  ST(victims)++;
  return true;
}

// Lane-safe variant (no smem counters, no log): returns the victim's key, or ~0 if the
// frame is referenced / not valid right now.
__device__ unsigned long long try_unmap(const DevCtx& c, uint32_t v) {
  if (atomicCAS(&c.fstate[v], FR_VALID, 0u) != FR_VALID) return ~0ull;
  unsigned long long key = c.fkey[v];
  atomicCAS(&c.files[key >> 40].pt[key & ((1ull << 40) - 1)], v, PT_EMPTY);
  return key;
}

__device__ bool evict_spin(const DevCtx& c, Smem& s, uint32_t v) {
  uint64_t t0 = globaltimer();
  while (!try_evict(c, s, v)) {
    if (!keep_waiting(c, t0, 10)) return false;
    __nanosleep(100);
  }
  return true;
}

__device__ uint32_t take_recycled(const DevCtx& c) {
  if (ld_volatile_u64(&c.g->recycled_n) == 0) return PT_EMPTY;
  while (atomicCAS(&c.g->recycled_lock, 0, 1) != 0) __nanosleep(32);
  __threadfence();
  uint32_t f = PT_EMPTY;
  if (c.g->recycled_n > 0) f = c.recycled[--c.g->recycled_n];
  __threadfence();
  atomicExch(&c.g->recycled_lock, 0);
  return f;
}

// A free frame (never used, or released at EOF), or PT_EMPTY when none is left.
__device__ uint32_t take_free(const DevCtx& c) {
  if (ld_volatile_u64(&c.g->fresh_next) < (unsigned long long)c.nframes) {
    unsigned long long k = atomicAdd(&c.g->fresh_next, 1ull);
    if (k < (unsigned long long)c.nframes) return (uint32_t)k;
  }
  return take_recycled(c);
}

// Retired frames (gpu_cache.py:158-167, 208-212) live in ret_npools FIFOs: a finished TB
// retires into its CTA's FIFO, and a TB reclaims from its CTA's FIFO first, then from the
// others in order.  Which retired frame a TB gets is schedule-dependent in the reference
// too whenever several TBs are resident (SURVEY.md §8c rule 4); the counts are not (every
// reclaim is one remap of a valid frame), and with one resident CTA there is one FIFO —
// exactly the reference's global oldest-first order.  Spreading the FIFOs keeps hundreds of
// CTAs from serialising on one head counter.
__device__ __forceinline__ unsigned long long* rp_head(const DevCtx& c, int p) { return c.rpool + 16 * p; }
__device__ __forceinline__ unsigned long long* rp_tail(const DevCtx& c, int p) { return c.rpool + 16 * p + 1; }
__device__ __forceinline__ uint32_t* rp_entry(const DevCtx& c, int p, unsigned long long pos) {
  return c.retired + (int64_t)p * c.ret_pcap + (int64_t)(pos % (unsigned long long)c.ret_pcap);
}

// Reserve up to `want` consecutive entries of one FIFO (home first); returns how many, with
// the FIFO and first position in *pool / *pos.  One round trip per CAS attempt.
__device__ int retired_reserve(const DevCtx& c, int want, int* pool, unsigned long long* pos) {
  const int home = (int)(blockIdx.x % (unsigned)c.ret_npools);
  for (int q = 0; q < c.ret_npools; q++) {
    const int p = home + q < c.ret_npools ? home + q : home + q - c.ret_npools;
    unsigned long long h = ld_volatile_u64(rp_head(c, p)), t = ld_volatile_u64(rp_tail(c, p));
    for (;;) {
      if (h >= t) {
        t = ld_volatile_u64(rp_tail(c, p));
        if (h >= t) break;
      }
      const unsigned long long take = t - h < (unsigned long long)want ? t - h : (unsigned long long)want;
      const unsigned long long prev = atomicCAS(rp_head(c, p), h, h + take);
      if (prev == h) {
        *pool = p;
        *pos = h;
        return (int)take;
      }
      h = prev;
    }
  }
  return 0;
}

// Take the value of a reserved entry once its pusher has written it.
__device__ uint32_t retired_take(const DevCtx& c, int pool, unsigned long long pos, bool* ok) {
  uint32_t* e = rp_entry(c, pool, pos);
  const uint64_t t0 = globaltimer();
  uint32_t v;
  while ((v = ld_acquire_gpu(e)) == 0) {
    if (!keep_waiting(c, t0, 11)) break;
  }
  *e = 0;
  *ok = v != 0;
  return v - 1;
}

__device__ uint32_t retired_pop(const DevCtx& c) {
  int pool;
  unsigned long long pos;
  if (retired_reserve(c, 1, &pool, &pos) == 0) return PT_EMPTY;
  bool ok;
  const uint32_t f = retired_take(c, pool, pos, &ok);
  return ok ? f : PT_EMPTY;
}

__device__ __forceinline__ void own_push(const DevCtx& c, Smem& s, uint32_t f) {
  c.own_q[(int64_t)blockIdx.x * c.quota + (s.own_head + s.own_len) % c.quota] = f;
  s.own_len++;
}

// per-tb-lra allocation (gpu_cache.py:149-179)
__device__ uint32_t alloc_per_tb(const DevCtx& c, Smem& s) {
  if (s.own_len < c.quota) {
    uint32_t f = take_free(c);
    if (f != PT_EMPTY) {
      own_push(c, s, f);
      ST(pc_allocs)++;
      return f;
    }
    uint32_t v = retired_pop(c);
    if (v != PT_EMPTY) {
      if (!evict_spin(c, s, v)) return PT_EMPTY;
      ST(pc_remaps)++;
      own_push(c, s, v);
      return v;
    }
    if (has_error(c)) return PT_EMPTY;
  }
  if (s.own_len == 0) {
    set_error(c, ERR_NO_FRAME, s.tb, 0);
    return PT_EMPTY;
  }
  int64_t qi = (int64_t)blockIdx.x * c.quota + s.own_head % c.quota;
  uint32_t v = c.own_q[qi];
  s.own_head++;
  s.own_len--;
  if (!evict_spin(c, s, v)) return PT_EMPTY;
  ST(pc_remaps)++;
  own_push(c, s, v);  // remapped in place, now the most recently allocated
  return v;
}

__device__ void gfifo_append(const DevCtx& c, Smem& s, uint32_t f) {
  unsigned long long pos = atomicAdd(&c.g->g_tail, 1ull);
  if (pos - ld_volatile_u64(&c.g->g_head) >= (unsigned long long)c.gfifo_cap) {
    set_error(c, ERR_FIFO_OVERFLOW, 0, pos);
    return;
  }
  st_release_gpu(&c.gfifo[pos % c.gfifo_cap], f + 1);
  s.last_gfifo_pos = (long long)pos;
}

// global-lru-dealloc allocation (gpu_cache.py:126-147).  Fresh frames are handed out
// lock-free (their FIFO position is their ticket order); eviction scans the global
// allocation-order FIFO for the first valid, unreferenced frame under the global lock.
__device__ uint32_t alloc_global(const DevCtx& c, Smem& s) {
  uint32_t f = take_free(c);
  if (f != PT_EMPTY) {
    gfifo_append(c, s, f);
    ST(pc_allocs)++;
    return f;
  }
  uint64_t t0 = globaltimer();
  for (;;) {
    while (atomicCAS(&c.g->lock, 0, 1) != 0) {
      if (!keep_waiting(c, t0, 12)) return PT_EMPTY;
      __nanosleep(64);
    }
    __threadfence();
    uint32_t victim = PT_EMPTY;
    unsigned long long head = c.g->g_head;
    unsigned long long tail = ld_volatile_u64(&c.g->g_tail);
    for (unsigned long long p = head; p < tail; p++) {
      uint32_t* e = &c.gfifo[p % c.gfifo_cap];
      uint32_t val;
      while ((val = ld_acquire_gpu(e)) == 0) {  // reserved, not yet written
        if (!keep_waiting(c, t0, 13)) break;
      }
      if (val == 0) break;
      if (val == RING_TOMB) continue;
      if (try_evict(c, s, val - 1)) {
        victim = val - 1;
        *e = RING_TOMB;
        break;
      }
    }
    // drop leading tombstones
    while (head < tail && *(volatile uint32_t*)&c.gfifo[head % c.gfifo_cap] == RING_TOMB) {
      c.gfifo[head % c.gfifo_cap] = 0;
      head++;
    }
    c.g->g_head = head;
    __threadfence();
    atomicExch(&c.g->lock, 0);
    if (victim != PT_EMPTY) {
      gfifo_append(c, s, victim);
      ST(pc_evictions)++;
      ST(pc_allocs)++;
      return victim;
    }
    // every frame in flight or referenced: the reference fails here; a real GPU
    // may see transient references, so retry until the timeout.
    if (!keep_waiting(c, t0, 14)) {
      if (c.g->error == ERR_TIMEOUT) c.g->error = ERR_ALL_INFLIGHT;
      return PT_EMPTY;
    }
    __nanosleep(200);
  }
}

// zero-byte RPC result: unbind the in-flight frame (gpu_cache.py:191-206)
__device__ void release_frame(const DevCtx& c, Smem& s, uint32_t f, uint32_t* pte) {
  if (c.policy == GFS_POLICY_GLOBAL_LRU) {
    if (s.last_gfifo_pos >= 0) c.gfifo[s.last_gfifo_pos % c.gfifo_cap] = RING_TOMB;
  } else {
    s.own_len--;  // it is the newest own frame
  }
  atomicAnd(&c.fstate[f], ~FR_VALID);  // keep transient readers' pins (refcount bits)
  st_release_gpu(pte, PT_EMPTY);
  while (atomicCAS(&c.g->recycled_lock, 0, 1) != 0) __nanosleep(32);
  __threadfence();
  c.recycled[c.g->recycled_n++] = f;
  __threadfence();
  atomicExch(&c.g->recycled_lock, 0);
}

// ---------------------------------------------------------- private buffer

__device__ int64_t page_bytes(const DevFile& F, int64_t pg, int64_t page) {
  int64_t b = F.size - page * pg;
  return b < pg ? b : pg;
}

// prefetcher.py:38-50.  The fill's pages are base+1 .. base+m-1 of one RPC span; their
// bytes stay in the slot's span buffer at (page - base) * pg.
__device__ void pb_fill(const DevCtx& c, Smem& s, int64_t fid, int64_t base, int64_t m,
                        int64_t rest_bytes) {
  // Entries 1..cnt-1 are whole pages and entry cnt holds the rest (short only at EOF), so
  // the buffer is (count, last entry's bytes, an absent-bitmap) instead of a byte count per
  // entry.  Fill order semantics of the reference: entries are offered in page order and
  // one that does not fit the capacity is dropped (counted as discarded).
  ST(pb_discarded_bytes) += s.pb_filled;  // every unconsumed entry is stale
  s.pb_fid = fid;
  s.pb_base = base;
  s.pb_off_adj = 0;
  const int64_t pg = c.page_size;
  int64_t cnt = m - 1;
  if (cnt >= MAX_PB_ENTRIES) {
    set_error(c, ERR_PB, (int)cnt, 0);
    cnt = MAX_PB_ENTRIES - 1;
  }
  const int64_t last = rest_bytes - (cnt - 1) * pg;
  const int64_t kept_full = min(cnt - 1, c.pb_cap_bytes / pg);
  int64_t filled = kept_full * pg;
  const bool last_fits = filled + last <= c.pb_cap_bytes;
  ST(pb_discarded_bytes) += (cnt - 1 - kept_full) * pg + (last_fits ? 0 : last);  // no room
  if (last_fits) filled += last;
  ST(pb_filled_bytes) += filled;
  s.pb_filled = filled;
  s.pb_count = cnt;
  s.pb_last_nb = last;
  for (int64_t w = 0; w <= (cnt >> 5); w++) {  // bit set = entry absent
    const int64_t lo = w << 5;
    uint32_t present = 0;
    const int64_t a = lo > 1 ? lo : 1, b = kept_full < lo + 31 ? kept_full : lo + 31;
    if (a <= b) present = (b - a + 1 == 32 ? 0xFFFFFFFFu : ((1u << (b - a + 1)) - 1u)) << (a - lo);
    if (last_fits && cnt >= lo && cnt <= lo + 31) present |= 1u << (cnt - lo);
    s.pb_absent[w] = ~present;
  }
}

__device__ __forceinline__ bool pb_present(const Smem& s, int64_t i) {
  return !((s.pb_absent[i >> 5] >> (i & 31)) & 1u);
}

__device__ __forceinline__ bool pb_has(const Smem& s, int64_t fid, int64_t page) {
  const int64_t i = page - s.pb_base;
  return s.pb_count > 0 && fid == s.pb_fid && i >= 1 && i <= s.pb_count && pb_present(s, i);
}

// prefetcher.py:52-61
__device__ int64_t pb_take(Smem& s, int64_t fid, int64_t page) {
  int64_t i = page - s.pb_base;
  if (s.pb_count > 0 && fid == s.pb_fid && i >= 1 && i <= s.pb_count && pb_present(s, i)) {
    const int64_t nb = i == s.pb_count ? s.pb_last_nb : s.page_size_cached;
    s.pb_absent[i >> 5] |= 1u << (i & 31);
    s.pb_filled -= nb;
    ST(pb_hits)++;
    ST(pb_consumed_bytes) += nb;
    return nb;
  }
  ST(pb_misses)++;
  return 0;
}

// Consecutive private-buffer entries present from `page` on (at most maxn), by bitmap
// words: the run pb_has() would walk page by page.
__device__ int pb_run(const Smem& s, int64_t fid, int64_t page, int maxn) {
  if (s.pb_count <= 0 || fid != s.pb_fid) return 0;
  const int64_t i = page - s.pb_base;
  if (i < 1 || i > s.pb_count) return 0;
  const int64_t lim = min((int64_t)maxn, s.pb_count - i + 1);
  int64_t n = 0;
  while (n < lim) {
    const int64_t k = i + n;
    const uint32_t w = s.pb_absent[k >> 5] >> (k & 31);  // bit set = absent
    if (w) {
      n += __ffs(w) - 1;
      break;
    }
    n += 32 - (k & 31);
  }
  return (int)min(n, lim);
}

// pb_take (prefetcher.py:52-61) of n consecutive present entries from `page`, at once:
// the same counters as n single takes.  Returns their bytes.
__device__ int64_t pb_take_run(Smem& s, int64_t page, int n) {
  const int64_t i = page - s.pb_base;
  for (int64_t k = i; k < i + n;) {
    const int b = (int)(k & 31);
    const int m = (int)min((int64_t)(32 - b), i + n - k);
    s.pb_absent[k >> 5] |= (m == 32 ? 0xFFFFFFFFu : ((1u << m) - 1u)) << b;
    k += m;
  }
  int64_t bytes = (int64_t)n * s.page_size_cached;
  if (i + n - 1 == s.pb_count) bytes += s.pb_last_nb - s.page_size_cached;
  s.pb_filled -= bytes;
  ST(pb_hits) += n;
  ST(pb_consumed_bytes) += bytes;
  return bytes;
}

// request_span (prefetcher.py:13-25) + the doubling window (io.readahead=doubling)
// Pure part of request_span: the span an RPC at `page` would have, and the doubling
// window it implies (no state change).
__device__ int64_t span_peek(const DevCtx& c, const Smem& s, int64_t fid, int64_t page,
                             int64_t seg_end, int64_t* new_win) {
  const DevFile& F = c.files[fid];
  const int64_t pg = c.page_size;
  const int64_t off = page * pg;
  *new_win = s.ra_win;
  if (off >= F.size) return 0;
  const bool ro = F.read_only != 0;
  int64_t want = (ro && c.prefetch_bytes > 0) ? pg + c.prefetch_bytes : pg;
  if (c.readahead == GFS_RA_DOUBLING && ro) {
    const int64_t base = c.ra_init_bytes > pg + c.prefetch_bytes ? c.ra_init_bytes : pg + c.prefetch_bytes;
    int64_t win = base;
    if (s.ra_win > 0 && fid == s.ra_next_fid && page == s.ra_next_page)
      win = 2 * s.ra_win < c.ra_max_bytes ? 2 * s.ra_win : c.ra_max_bytes;
    *new_win = win;
    want = win;
    const int64_t seg_lim = (seg_end + pg - 1) / pg * pg - off;  // stay inside this TB's segment
    if (want > seg_lim) want = seg_lim;
    if (want < pg) want = pg;
  }
  return want < F.size - off ? want : F.size - off;
}

__device__ int64_t rpc_span(const DevCtx& c, Smem& s, int64_t fid, int64_t page, int64_t seg_end) {
  int64_t win;
  const int64_t span = span_peek(c, s, fid, page, seg_end, &win);
  if (span > 0 && c.readahead == GFS_RA_DOUBLING && c.files[fid].read_only) {
    s.ra_win = win;
    s.ra_next_fid = fid;
    s.ra_next_page = page + (span + c.page_size - 1) / c.page_size;
    log_rec(c, GFS_LOG_WINDOWS, s.tb, span, 0, 0);
  }
  return span;
}

// ----------------------------------------------------------------------- RPC

__device__ __forceinline__ void account_transfer(const DevCtx& c, Smem& s, int64_t n) {
  ST(preads)++;
  ST(pread_bytes) += n;
  ST(storage_bytes) += n;
  if (!c.pcie_disabled && n > 0) {
    ST(pcie_bytes) += n;
    ST(pcie_transfers) += (n + c.staging_bytes - 1) / c.staging_bytes;  // rpc.py:31-55
  }
}

// Submit one request for this CTA's slot into landing half `half` (thread 0): rpc.py:82-102.
// Returns false on abort; *seq_out / *pos_out identify it for rpc_wait.
__device__ bool rpc_submit(const DevCtx& c, Smem& s, int64_t fid, int64_t off, int64_t size, int half,
                           uint32_t* seq_out, unsigned long long* pos_out) {
  const unsigned slot = blockIdx.x;
  const unsigned long long Q = (unsigned long long)c.ring_mask + 1;
  const unsigned long long local = atomicAdd(&c.g->req_local, 1ull);
  const unsigned long long pos = c.g->req_base + local;
  uint64_t t0 = globaltimer();
  if (local >= Q) {
    // ring position pos - Q (same entry) must have been copied out by the daemon: its
    // answer came back (done_pos, device memory, the cheap check) or the daemon marked the
    // entry consumed (mapped host memory).  The second check matters: a pending readahead
    // window may stay unanswered-for (not waited on) for any number of requests, and its
    // own CTA may be the one waiting here.
    const unsigned long long need = pos - Q + 1;
    while (ld_volatile_u64(&c.done_pos[pos & c.ring_mask]) < need &&
           ld_acquire_sys(&c.ring_consumed[pos & c.ring_mask]) != (uint32_t)need) {
      if (!keep_waiting(c, t0, 20)) return false;
      __nanosleep(200);
    }
  }
  RpcReq* e = &c.ring[pos & c.ring_mask];
  const uint32_t seq = (uint32_t)(pos + 1);
  const unsigned long long lap = ring_lap(pos, Q);  // every word carries it (see RpcReq)
  const unsigned long long w0 = ((unsigned long long)off << 16) | lap;
  const unsigned long long w1 = ((unsigned long long)(uint32_t)size << 32) | ((unsigned long long)(fid & 0xFFFF) << 16) | lap;
  const unsigned long long w2 = ((unsigned long long)(uint32_t)s.tb << 32) |
                                ((unsigned long long)((slot | ((unsigned)half << 15)) & 0xFFFF) << 16) | lap;
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&e->w[0]), "l"(w0) : "memory");
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&e->w[1]), "l"(w1) : "memory");
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(&e->w[2]), "l"(w2) : "memory");
  *seq_out = seq;
  *pos_out = pos;
  // the reference's slot partition (rpc.py:25-28, 82-89): TB tb owns slot tb % n_slots and
  // a request finding that slot occupied is a collision.  Counted on the real timing; the
  // device does not serialise on it (every resident CTA has its own mailbox).
  // (this TB's own outstanding readahead windows are not collisions: the reference's OS
  // readahead runs inside the host's pread, not through the slot)
  if (atomicAdd(&c.slot_busy[s.tb % c.ref_slots], 1u) > s.rpc_out) ST(slot_collisions)++;
  s.rpc_out++;
  return true;
}

// A request's answer has been seen (thread 0): its ring entry and slot are free again.
__device__ __forceinline__ void rpc_retire(const DevCtx& c, Smem& s, unsigned long long pos) {
  atomicMax(&c.done_pos[pos & c.ring_mask], pos + 1);
  atomicSub(&c.slot_busy[s.tb % c.ref_slots], 1u);  // slot released when the data is ready (rpc.py:104-113)
  s.rpc_out--;
}

// Wait for the completion of request (seq, pos) of file `fid` at `off` (thread 0):
// rpc.py:192-229.  Returns bytes read, or -1 on abort.
__device__ int64_t rpc_wait(const DevCtx& c, Smem& s, int64_t fid, int64_t off, uint32_t seq,
                            unsigned long long pos, int half, bool first_nap = true) {
  const unsigned slot = blockIdx.x;
  const uint64_t t0 = globaltimer();
  const uint64_t tw = globaltimer();
  int64_t n;
  s.direct[half] = 0;  // what lands in this half now: the answer says
  if (c.transfer == GFS_XFER_DMA || c.transfer == GFS_XFER_MAPPED) {
    const unsigned long long* bell = &c.doorbell[(int64_t)slot * c.landing_halves + half];
    for (;;) {
      uint64_t v = ld_acquire_sys64(bell);
      if ((uint32_t)v == seq) {
        n = (int64_t)(v >> 32);
        if (n == 0xFFFFFFFFll) n = -1;
        break;
      }
      if (!keep_waiting(c, t0, 21)) {
        c.g->error_arg = ((unsigned long long)(slot * c.landing_halves + half) << 32) | seq;
        return -1;
      }
      __nanosleep(256);
    }
  } else if (c.transfer == GFS_XFER_MAPPED_HYBRID || c.transfer == GFS_XFER_PREAD_HYBRID) {
    // the daemon answers either by copy engine (doorbell in HBM, data already in the landing
    // slot) or by mailbox (the CTA pulls the span from the pinned page-cache mapping)
    // (both answers arrive through the HBM doorbell, so nothing polls host memory: bit 63
    // set = "not copied, pull it yourself")
    const unsigned long long* bell = &c.doorbell[(int64_t)slot * c.landing_halves + half];
    for (;;) {
      const uint64_t v = ld_acquire_sys64(bell);
      if ((uint32_t)v == seq) {
        n = (int64_t)((v >> 32) & 0x7FFFFFFFull);
        if (n == 0x7FFFFFFFll) n = -1;
        if ((v >> 63) && n > 0) {
          if (c.transfer == GFS_XFER_PREAD_HYBRID) {  // in pool buffer r->buf (written before the doorbell)
            const RpcResp* r = &c.resp[(int64_t)slot * c.landing_halves + half];
            s.pull_n = n;
            s.pull_buf = (int32_t)ld_acquire_sys((const uint32_t*)&r->buf);
            s.pull_src = c.bounce + (int64_t)s.pull_buf * c.bounce_bytes;
            s.pull_seq = seq;
            s.pull_off = off;
            s.pull_half = half;
          } else if (c.k1_direct) {
            s.direct[half] = 1;  // K1 reads it from the mapping: no pull, no landing copy
          } else {
            s.pull_n = n;
            s.pull_buf = -1;
            s.pull_src = c.files[fid].map + off;
            s.pull_off = off;
            s.pull_half = half;
          }
        }
        break;
      }
      if (!keep_waiting(c, t0, 23)) {
        c.g->error_arg = ((unsigned long long)(slot * c.landing_halves + half) << 32) | seq;
        return -1;
      }
      __nanosleep(256);
    }
  } else {
    const RpcResp* r = &c.resp[(int64_t)slot * c.landing_halves + half];
    if (first_nap) __nanosleep(c.poll_first_ns);
    for (;;) {
      if (ld_acquire_sys(&r->seq) == seq) {
        n = *(volatile const int64_t*)&r->nbytes;
        if (c.transfer == GFS_XFER_BOUNCE && n > 0) {  // pulled by the whole CTA (pull_span)
          s.pull_n = n;
          s.pull_buf = *(volatile const int32_t*)&r->buf;
          s.pull_src = c.bounce + (int64_t)s.pull_buf * c.bounce_bytes;
          s.pull_off = off;
          s.pull_half = half;
          s.pull_seq = seq;
        } else if (c.transfer == GFS_XFER_MAPPED_ZC && n > 0 && c.k1_direct) {
          s.direct[half] = 1;  // K1 reads it from the mapping: no pull, no landing copy
        } else if (c.transfer == GFS_XFER_MAPPED_ZC && n > 0) {  // straight from the page cache
          s.pull_n = n;
          s.pull_buf = -1;
          s.pull_src = c.files[fid].map + off;
          s.pull_off = off;
          s.pull_half = half;
          s.pull_off = off;
        }
        break;
      }
      if (!keep_waiting(c, t0, 22)) {
        c.g->error_arg = ((unsigned long long)(slot * c.landing_halves + half) << 32) | seq;
        return -1;
      }
      __nanosleep(c.poll_ns);
    }
  }
  rpc_retire(c, s, pos);
  if (c.stream_pieces && n > 0) {  // the doorbell comes after the first piece
    s.st_seq[half] = seq;
    s.st_n[half] = n;
    s.st_landed[half] = n >= 2 * c.stream_piece ? c.stream_piece : n;
  }
  const uint64_t tr = globaltimer();
  ST(wait_ns) += (long long)(tr - tw);
  tl_rec(c, GFS_TL_RPC, s.tb, n, tw, tr);
  if (n < 0) {
    set_error(c, ERR_IO, (int)fid, (unsigned long long)off);
    return -1;
  }
  return n;
}

// Streamed windows (thread 0): wait until the first `need` bytes of the last request into
// landing half `h` have landed.  False on abort.
__device__ bool wait_landed(const DevCtx& c, Smem& s, int h, int64_t need) {
  if (!c.stream_pieces || need <= s.st_landed[h]) return true;
  if (need > s.st_n[h]) need = s.st_n[h];
  const unsigned long long* p = &c.landed[(int64_t)blockIdx.x * c.landing_halves + h];
  const uint64_t t0 = globaltimer();
  while (need > s.st_landed[h]) {
    const uint64_t v = ld_acquire_sys64(p);
    if ((uint32_t)v == s.st_seq[h]) {
      const int64_t got = (int64_t)(v >> 32) * 4096;
      s.st_landed[h] = got < s.st_n[h] ? got : s.st_n[h];
      if (need <= s.st_landed[h]) break;
    }
    if (!keep_waiting(c, t0, 24)) return false;
    __nanosleep(128);
  }
  return true;
}

// Where the current span (page 0 + private-buffer pages) lives.
__device__ __forceinline__ const uint8_t* half_base(const DevCtx& c, int h) {
  if (c.transfer == GFS_XFER_ZEROCOPY)
    return c.staging + ((int64_t)blockIdx.x * c.landing_halves + h) * c.slot_bytes;
  return c.landing + ((int64_t)blockIdx.x * c.landing_halves + h) * c.slot_bytes;
}
__device__ __forceinline__ const uint8_t* span_base(const DevCtx& c, const Smem& s) {
  return half_base(c, s.span_half);
}

// K1 early (gpu.k1_early, thread 0).  For the mapped transfers with K1 direct the daemon's
// answer to a static request carries nothing but the span length, min(size, file size - off)
// (gfs_host.cpp io_worker, `from_map`), and "read it from the mapping" — for mapped_hybrid
// when that length is below the copy-engine size.  The device knows both, so K1 starts on the
// span at once instead of after a mailbox round trip over the loaded link; the request is the
// same (same ring entry, counters and trace), only its wait moves: early_collect waits for the
// answer before the CTA's next request and at TB end, and a length other than the one K1
// used (the file changed under the mapping) fails the run with ERR_IO.
__device__ bool early_eligible(const DevCtx& c, int64_t n) {
  return c.k1_early && n > 0 &&
         (c.transfer == GFS_XFER_MAPPED_ZC || (c.transfer == GFS_XFER_MAPPED_HYBRID && n < c.ce_min));
}

//
// Reading the answer is itself a PCIe read, and with the link loaded by K1's reads such a read
// returns only after the bytes queued ahead of it (~10-20 us).  So K1's producer fetches the
// mailbox line asynchronously (early_poll: a 16-byte bulk copy into shared memory, issued once
// the span's first chunk is in — by then the daemon has answered) and early_collect finds the
// answer already on chip; when the copy caught the mailbox before the answer (or anything
// does not match) it falls back to polling.
__device__ __forceinline__ void early_poll(const DevCtx& c, Smem& s) {
  // (mapped_hybrid answers through the HBM doorbell: nothing to fetch over the link)
  if (!s.early.on || s.early.polled || c.transfer != GFS_XFER_MAPPED_ZC) return;
  s.early.polled = 1;
  const RpcResp* r = &c.resp[(int64_t)blockIdx.x * c.landing_halves + s.early.half];
  tma_load(&s.poll_buf, r, 16, &s.poll_bar);
}

__device__ bool early_collect(const DevCtx& c, Smem& s) {
  if (!s.early.on) return true;
  s.early.on = 0;
  if (s.early.polled) {
    s.early.polled = 0;
    const uint32_t par = s.poll_par;
    s.poll_par ^= 1u;
    if (!mbar_wait_t(c, &s.poll_bar, par, 43, s.early.pos)) return false;
    const int64_t n = (int64_t)(((unsigned long long)s.poll_buf.y << 32) | s.poll_buf.x);
    if (s.poll_buf.z == s.early.seq && n == s.early.n) {  // answered: no poll on the link
      rpc_retire(c, s, s.early.pos);
      ST(early_answers)++;
      tl_rec(c, GFS_TL_RPC, s.tb, n, s.early.t_sub, globaltimer());
      return true;
    }
  }
  const int64_t n = rpc_wait(c, s, s.early.fid, s.early.off, s.early.seq, s.early.pos, s.early.half, false);
  if (n < 0) return false;
  if (n != s.early.n || !s.direct[s.early.half]) {
    set_error(c, ERR_IO, (int)s.early.fid, (unsigned long long)s.early.off);
    return false;
  }
  return true;
}

// Submit and wait (the reference's synchronous RPC).
__device__ int64_t rpc_call(const DevCtx& c, Smem& s, int64_t fid, int64_t off, int64_t size, int half = 0) {
  uint32_t seq;
  unsigned long long pos;
  if (!early_collect(c, s)) return -1;
  if (!wait_landed(c, s, half, s.st_n[half])) return -1;  // the half's previous window is in
  if (!rpc_submit(c, s, fid, off, size, half, &seq, &pos)) return -1;
  return rpc_wait(c, s, fid, off, seq, pos, half);
}

// ------------------------------------------------------------- ondemand readahead
//
// io.readahead=adaptive is the reference's Linux-style ondemand law (HostOs._decide,
// host_os.py:106-152) run per TB stream on the device.  A "read" is one gread request
// (the reference's pread).  Its decision is taken the first time the walk meets one of its
// pages that is missing (not cached, not in the private buffer, not in a pending window) or
// a readahead marker — the reference decides at pread entry on "any page missing or any
// marker" (host_os.py:255-265); the inputs are the same, the walk only takes it lazily.
//   cold sequential read of n pages: window max(n, min(4n, ra_max)); the requested pages
//     are fetched synchronously, the rest asynchronously, marker on the first async page;
//   a read hitting the marker: the next window (double, capped at ra_max) asynchronously,
//     marker on its first page (a marker that does not match the window state rebuilds it
//     from the resident run around it, the reference's context recovery);
//   a non-sequential read: exactly its missing pages, window state reset.
// Asynchronous windows land in the CTA's other landing half while it consumes the current
// one and are adopted as the private buffer when the walk reaches them.  Windows are clamped
// at EOF (io.ra_clamp=eof, the reference) or at the TB's segment end (segment, the default:
// a TB's stream is its stride, and the law sees only that segment's pages).

__device__ __forceinline__ int64_t od_pages(const DevCtx& c, int64_t bytes) {
  return (bytes + c.page_size - 1) / c.page_size;
}

__device__ bool od_in_pending(const DevCtx& c, const Smem& s, int64_t fid, int64_t p, int* h_out) {
  for (int h = 0; h < 2; h++)
    if (s.hp[h].pending && s.hp[h].fid == fid && p >= s.hp[h].page &&
        p < s.hp[h].page + od_pages(c, s.hp[h].span)) {
      if (h_out) *h_out = h;
      return true;
    }
  return false;
}

// Resident for the law (the sequentiality test and the resident run): cached or being
// fetched by anyone, in the private buffer, or in a pending window — except this TB's own
// claims [ex_lo, ex_hi) for the request being decided, which nothing has fetched yet.  With
// the segment clamp the stream sees only its own segment (what other TBs cached next to it
// would make the decision depend on their progress).
__device__ bool od_resident(const DevCtx& c, const Smem& s, int64_t fid, int64_t p, int64_t ex_lo,
                            int64_t ex_hi) {
  const DevFile& F = c.files[fid];
  if (p < 0 || p >= od_pages(c, F.size)) return false;
  if (c.ra_clamp == GFS_RA_CLAMP_SEGMENT && (p < s.seg_lo / c.page_size || p >= od_pages(c, s.seg_hi)))
    return false;
  if (pb_has(s, fid, p) || od_in_pending(c, s, fid, p, nullptr)) return true;
  if (p >= ex_lo && p < ex_hi) return false;
  return ld_acquire_gpu(&F.pt[p]) != PT_EMPTY;
}

// Page limit of the stream: EOF, or the end of the TB's segment.
__device__ int64_t od_limit(const DevCtx& c, const Smem& s, int64_t fid) {
  int64_t lim = od_pages(c, c.files[fid].size);
  if (c.ra_clamp == GFS_RA_CLAMP_SEGMENT) {
    const int64_t se = od_pages(c, s.seg_hi);
    if (se < lim) lim = se;
  }
  return lim;
}

// The request page p belongs to, as pages [*gs, *ge), and its instance key.  With lookahead
// a batch walks the TB's next requests too; they start at seg_lo + k * request_bytes.
__device__ long long od_request_of(const DevCtx& c, const Smem& s, int64_t fid, int64_t p, int64_t* gs,
                                   int64_t* ge) {
  const int64_t pg = c.page_size, fs = c.files[fid].size;
  int64_t lo = s.g_lo, hi = s.g_hi;
  if (s.g_la) {
    lo = s.seg_lo + (p * pg - s.seg_lo) / c.request_bytes * c.request_bytes;
    hi = lo + c.request_bytes < s.seg_hi ? lo + c.request_bytes : s.seg_hi;
  }
  if (hi > fs) hi = fs;
  *gs = lo / pg;
  *ge = od_pages(c, hi);
  return (s.seg_ord << 32) | (long long)((lo - s.seg_lo) / c.request_bytes);
}

// HostOs._resident_run (host_os.py:88-103): the resident run [*rs, *re) around page m,
// each scan capped at ra_max pages.
__device__ void od_resident_run(const DevCtx& c, const Smem& s, int64_t fid, int64_t m, int64_t ex_lo,
                                int64_t ex_hi, int64_t* rs, int64_t* re) {
  const int64_t ra_max = c.ra_max_bytes / c.page_size, np = od_pages(c, c.files[fid].size);
  int64_t a = m;
  while (m - a < ra_max && a > 0 && od_resident(c, s, fid, a - 1, ex_lo, ex_hi)) a--;
  int64_t e = m + 1;
  while (e - m <= ra_max && e < np && od_resident(c, s, fid, e, ex_lo, ex_hi)) e++;
  *rs = a;
  *re = e;
}

__device__ void od_add_mark(Smem& s, int64_t page) {
  for (int i = 0; i < OD_MARKS; i++)
    if (s.od.mark[i] < 0) {
      s.od.mark[i] = page;
      return;
    }
  for (int i = 0; i + 1 < OD_MARKS; i++) s.od.mark[i] = s.od.mark[i + 1];  // drop the oldest
  s.od.mark[OD_MARKS - 1] = page;
}

__device__ void od_reset(Smem& s, int64_t fid) {
  s.od.fid = fid;
  s.od.ws = s.od.wsize = s.od.async = 0;
  s.od.prev_end = -1;
  for (int i = 0; i < OD_MARKS; i++) s.od.mark[i] = -1;
  s.od.dec_key = -1;
  s.od.run_n = 0;
}

// HostOs._decide (host_os.py:106-152) for the request [gs, ge) (thread 0).  Updates the
// window state and markers; the asynchronous run to request goes to s.od.run_page/run_n
// (run_n = 0: none).  Returns the window bytes window_history records (0 = none).
__device__ int64_t od_decide(const DevCtx& c, Smem& s, int64_t fid, int64_t gs, int64_t ge, int64_t ex_lo,
                             int64_t ex_hi) {
  const int64_t pg = c.page_size, ra_max = c.ra_max_bytes / pg;
  const int64_t lim = od_limit(c, s, fid);
  const int64_t npages = ge - gs, req_end = ge;
  s.od.run_n = 0;
  int64_t marker = -1;
  for (int i = 0; i < OD_MARKS; i++) {  // each marker triggers at most once
    const int64_t m = s.od.mark[i];
    if (m >= gs && m < ge) {
      s.od.mark[i] = -1;
      if (marker < 0 || m < marker) marker = m;
    }
  }
  if (marker >= 0) {
    int64_t ns, nz;
    if (s.od.wsize > 0 && marker == s.od.ws + s.od.wsize - s.od.async) {
      ns = max(s.od.ws + s.od.wsize, req_end);
      nz = min(2 * s.od.wsize, ra_max);
    } else {  // context recovery
      int64_t rs, re;
      od_resident_run(c, s, fid, marker, ex_lo, ex_hi, &rs, &re);
      ns = max(re, req_end);
      nz = min(2 * max(re - rs, (int64_t)1), ra_max);
    }
    nz = min(nz, max(lim - ns, (int64_t)0));
    s.od.prev_end = req_end;
    if (nz == 0) {
      s.od.ws = gs;
      s.od.wsize = s.od.async = 0;
      return 0;
    }
    s.od.ws = ns;
    s.od.wsize = s.od.async = nz;
    s.od.run_page = ns;
    s.od.run_n = nz;
    od_add_mark(s, ns);
    return nz * pg;
  }
  const bool seq = gs == 0 || gs == s.od.prev_end ||
                   (gs > 0 && od_resident(c, s, fid, gs - 1, ex_lo, ex_hi));
  s.od.prev_end = req_end;
  if (!seq) {
    s.od.ws = gs;
    s.od.wsize = s.od.async = 0;
    return 0;
  }
  int64_t w = max(npages, min(4 * npages, ra_max));
  w = min(w, max(lim - gs, npages));
  s.od.ws = gs;
  s.od.wsize = w;
  s.od.async = w - npages;
  if (s.od.async <= 0) return w * pg;
  s.od.run_page = req_end;
  s.od.run_n = s.od.async;
  od_add_mark(s, req_end);
  return w * pg;
}

// Request `span` bytes at `page` into landing half h (thread 0), with its RPC record and
// counters.  A pending window under bounce transfers is requested only when adopted: a CTA
// must not hold a host pool buffer while it waits for another request.
__device__ bool od_submit(const DevCtx& c, Smem& s, int64_t fid, int64_t page, int64_t span, int h,
                          bool pending) {
  log_rec(c, GFS_LOG_RPCS, s.tb, fid, page * c.page_size, span);
  ST(rpc_count)++;
  ST(rpc_requested_bytes) += span;
  s.hp[h].fid = fid;
  s.hp[h].page = page;
  s.hp[h].span = span;
  s.hp[h].age = ++s.hp_age;
  s.hp[h].pending = pending;
  // a window pulled out of a host pool buffer would hold that buffer until adopted
  const int64_t nexp = span < c.files[fid].size - page * c.page_size ? span : c.files[fid].size - page * c.page_size;
  s.hp[h].deferred = pending && (c.transfer == GFS_XFER_BOUNCE ||
                                 (c.transfer == GFS_XFER_PREAD_HYBRID && nexp < c.ce_min));
  if (s.hp[h].deferred) return true;
  if (!wait_landed(c, s, h, s.st_n[h])) return false;
  return rpc_submit(c, s, fid, page * c.page_size, span, h, &s.hp[h].seq, &s.hp[h].pos);
}

// Wait for half h's request (submitting a deferred one first); counts its transfer.
__device__ int64_t od_wait(const DevCtx& c, Smem& s, int h) {
  const int64_t off = s.hp[h].page * c.page_size;
  if (s.hp[h].deferred) {
    s.hp[h].deferred = 0;
    if (!wait_landed(c, s, h, s.st_n[h])) return -1;
    if (!rpc_submit(c, s, s.hp[h].fid, off, s.hp[h].span, h, &s.hp[h].seq, &s.hp[h].pos)) return -1;
  }
  s.hp[h].pending = 0;
  const int64_t n = rpc_wait(c, s, s.hp[h].fid, off, s.hp[h].seq, s.hp[h].pos, h);
  if (n >= 0) account_transfer(c, s, n);
  return n;
}

// A pending window the TB will not consume: wait for it and drop it (its bytes moved:
// they show up as prefetch waste).
__device__ int od_drain(const DevCtx& c, Smem& s, int h) {
  const int64_t n = od_wait(c, s, h);
  if (n < 0 || !wait_landed(c, s, h, n)) return -1;
  if (s.pull_n > 0) {  // never pulled: hand a bounce buffer straight back
    if (s.pull_buf >= 0) {
      st_relaxed_sys(&c.bounce_release[s.pull_buf], s.pull_seq);
    }
    s.pull_n = 0;
  }
  return 0;
}

// Landing half for a new span (thread 0): one without a pending window — the half not
// holding the private buffer first; taking the private buffer's half discards its
// unconsumed entries — else the older pending window is drained.  `avoid`: a half taken
// by the span requested alongside.  -1 on abort.
__device__ int od_pick_half(const DevCtx& c, Smem& s, int avoid) {
  const int a = s.span_half ^ 1, b = s.span_half;
  int h = -1;
  if (a != avoid && !s.hp[a].pending) h = a;
  else if (b != avoid && !s.hp[b].pending) h = b;
  if (h < 0) {
    for (int k = 0; k < 2; k++)
      if (k != avoid && (h < 0 || s.hp[k].age < s.hp[h].age)) h = k;
    if (od_drain(c, s, h) < 0) return -1;
  }
  if (h == s.span_half && s.pb_count > 0) {
    ST(pb_discarded_bytes) += s.pb_filled;
    s.pb_filled = 0;
    s.pb_count = 0;
  }
  return h;
}

__device__ bool od_submit_run(const DevCtx& c, Smem& s, int64_t fid, int avoid) {
  if (s.od.run_n <= 0) return true;
  const int64_t pg = c.page_size, fs = c.files[fid].size;
  int64_t span = s.od.run_n * pg;
  if (span > fs - s.od.run_page * pg) span = fs - s.od.run_page * pg;
  s.od.run_n = 0;
  if (span <= 0) return true;
  const int h = od_pick_half(c, s, avoid);
  return h >= 0 && od_submit(c, s, fid, s.od.run_page, span, h, true);
}

// Take the request decision for page p's request if it has not been taken (thread 0).
__device__ void od_decide_once(const DevCtx& c, Smem& s, int64_t fid, int64_t p, int64_t ex_lo, int64_t ex_hi,
                               int64_t* ge_out) {
  int64_t gs, ge;
  const long long key = od_request_of(c, s, fid, p, &gs, &ge);
  *ge_out = ge;
  if (key == s.od.dec_key) return;
  s.od.dec_key = key;
  const int64_t w = od_decide(c, s, fid, gs, ge, ex_lo, ex_hi);
  if (w > 0) log_rec(c, GFS_LOG_WINDOWS, s.tb, w, 0, 0);
}

// Walk position p0, before a batch (thread 0): a marker there fires its request's
// decision (the next window is requested); a pending window holding p0 is adopted as the
// private buffer (all its pages are entries: pb_off_adj).  Sets od.cap, the next marker or
// pending window past p0: batches and hit runs stop before it.  False on abort.
__device__ bool od_top(const DevCtx& c, Smem& s, int64_t fid, int64_t p0) {
  s.od.cap = INT64_MAX;
  if (!c.files[fid].read_only) return true;
  for (int i = 0; i < OD_MARKS; i++)
    if (s.od.mark[i] == p0) {
      int64_t ge;
      od_decide_once(c, s, fid, p0, 0, 0, &ge);
      if (!od_submit_run(c, s, fid, -1)) return false;
      break;
    }
  int h;
  if (od_in_pending(c, s, fid, p0, &h)) {
    const int64_t head = s.hp[h].page;
    const int64_t n = od_wait(c, s, h);
    if (n < 0) return false;
    s.span_half = h;
    if (n > 0) {
      pb_fill(c, s, fid, head - 1, od_pages(c, n) + 1, n);
      s.pb_off_adj = c.page_size;
    } else {
      ST(pb_discarded_bytes) += s.pb_filled;
      s.pb_filled = 0;
      s.pb_count = 0;
    }
  }
  for (int i = 0; i < OD_MARKS; i++)
    if (s.od.mark[i] > p0 && s.od.mark[i] < s.od.cap) s.od.cap = s.od.mark[i];
  for (int k = 0; k < 2; k++)  // a pending window is adopted at its first page the walk reaches
    if (s.hp[k].pending && s.hp[k].fid == fid && s.hp[k].page > p0 && s.hp[k].page < s.od.cap)
      s.od.cap = s.hp[k].page;
  return true;
}

// A synchronous miss at p0 with this TB's claims [ex_lo, ex_hi) (thread 0): the request's
// decision, then the synchronous span — the missing pages from p0 to the request's end or
// the first resident page, at most one landing half.  Returns its pages.
__device__ int64_t od_plan_sync(const DevCtx& c, Smem& s, int64_t fid, int64_t p0, int64_t ex_lo, int64_t ex_hi) {
  int64_t ge;
  od_decide_once(c, s, fid, p0, ex_lo, ex_hi, &ge);
  int64_t lim = p0 + c.slot_bytes / c.page_size;
  if (ge < lim) lim = ge;
  const int64_t np = od_pages(c, c.files[fid].size);
  if (np < lim) lim = np;
  int64_t q = p0 + 1;
  while (q < lim && !od_resident(c, s, fid, q, ex_lo, ex_hi)) q++;
  return q - p0;
}

// TB done: drop windows it did not reach.
__device__ int od_drain_all(const DevCtx& c, Smem& s) {
  for (int h = 0; h < 2; h++)
    if (s.hp[h].pending && od_drain(c, s, h) < 0) return -1;
  return 0;
}

// The span starting at `page` (thread 0): request_span + RPC (prefetcher.py:13-25,
// rpc.py:82-229); under ondemand readahead the synchronous span of the request's missing
// pages (sync_pages from od_plan_sync; < 0 = plan it here, claims [page, page + 1)).  In two
// halves so that a batch overlaps the RPC round trip with its frame allocation and eviction
// (the request is the same; only its wait moves): fetch_begin submits, fetch_end waits and
// accounts.  False / -1 on abort.
__device__ bool fetch_begin(const DevCtx& c, Smem& s, int64_t fid, int64_t page, int64_t seg_end,
                            int64_t sync_pages) {
  const int64_t pg = c.page_size;
  if (!early_collect(c, s)) return false;  // the previous request's answer, before the next one
  if (c.readahead == GFS_RA_ONDEMAND && c.files[fid].read_only) {
    if (sync_pages < 0) sync_pages = od_plan_sync(c, s, fid, page, page, page + 1);
    const int64_t fs = c.files[fid].size;
    int64_t span = sync_pages * pg;
    if (span > fs - page * pg) span = fs - page * pg;
    s.b.fb_od = 1;
    s.b.fb_span = span;
    s.b.fb_h = -1;
    if (span <= 0) {
      s.od.run_n = 0;
      return true;
    }
    const int hs = od_pick_half(c, s, -1);
    if (hs < 0 || !od_submit(c, s, fid, page, span, hs, false)) return false;
    if (!od_submit_run(c, s, fid, hs)) return false;
    s.b.fb_h = hs;
    return true;
  }
  int h = 0;
  if (c.readahead == GFS_RA_ONDEMAND && (h = od_pick_half(c, s, -1)) < 0) return false;  // non-RO file
  const int64_t span = rpc_span(c, s, fid, page, seg_end);
  s.b.fb_od = 0;
  s.b.fb_h = h;
  s.b.fb_span = span;
  if (span > 0) {
    if (!wait_landed(c, s, h, s.st_n[h])) return false;  // the half's previous window is in
    if (!rpc_submit(c, s, fid, page * pg, span, h, &s.b.fb_seq, &s.b.fb_pos)) return false;
  }
  return true;
}

__device__ int64_t fetch_end(const DevCtx& c, Smem& s, int64_t fid, int64_t page, int64_t* span_out,
                             bool early = false) {
  const int64_t span = s.b.fb_span;
  *span_out = span;
  if (s.b.fb_od) {
    if (span <= 0) return 0;
    const int64_t n = od_wait(c, s, s.b.fb_h);
    s.fetch_half = s.b.fb_h;
    return n;
  }
  const int h = s.b.fb_h;
  const int64_t pg = c.page_size;
  const int64_t fs = c.files[fid].size;
  const int64_t en = span > 0 && page * pg < fs ? min(span, fs - page * pg) : 0;  // the answer's length
  int64_t n;
  if (early && early_eligible(c, en)) {  // K1 early: read it now, collect the answer later
    s.early.on = 1;
    s.early.half = h;
    s.early.seq = s.b.fb_seq;
    s.early.pos = s.b.fb_pos;
    s.early.fid = fid;
    s.early.off = page * pg;
    s.early.n = en;
    s.early.polled = 0;
    s.early.t_sub = globaltimer();
    s.direct[h] = 1;
    n = en;
  } else {
    n = span > 0 ? rpc_wait(c, s, fid, page * pg, s.b.fb_seq, s.b.fb_pos, h) : 0;
  }
  if (n >= 0) {
    log_rec(c, GFS_LOG_RPCS, s.tb, fid, page * pg, span);
    ST(rpc_count)++;
    ST(rpc_requested_bytes) += span;
    account_transfer(c, s, n);
  }
  s.fetch_half = h;
  return n;
}

__device__ int64_t fetch_span(const DevCtx& c, Smem& s, int64_t fid, int64_t page, int64_t seg_end,
                              int64_t* span_out, int64_t sync_pages = -1) {
  if (!fetch_begin(c, s, fid, page, seg_end, sync_pages)) return -1;
  return fetch_end(c, s, fid, page, span_out);
}

// ------------------------------------------------------------------ copies (all threads)

// Generic congruence-aware copy of n bytes (K2 and partial deliveries).
template <int BS, int SRC>
__device__ void copy_bytes(uint8_t* dst, const uint8_t* src, int64_t n) {
  const int tid = threadIdx.x;
  if (n <= 0) return;
  uintptr_t d = (uintptr_t)dst, sp = (uintptr_t)src;
  if (((d ^ sp) & 15) == 0) {
    int64_t head = (int64_t)((16 - (d & 15)) & 15);
    if (head > n) head = n;
    if (tid < head) dst[tid] = ld1<SRC>(src + tid);
    int64_t body = (n - head) >> 4;
    const uint4* s4 = (const uint4*)(src + head);
    uint4* d4 = (uint4*)(dst + head);
    int64_t v = tid;
    for (; v + 3 * BS < body; v += 4 * BS) {
      uint4 a = ld16<SRC>(s4 + v), b = ld16<SRC>(s4 + v + BS);
      uint4 x = ld16<SRC>(s4 + v + 2 * BS), y = ld16<SRC>(s4 + v + 3 * BS);
      d4[v] = a;
      d4[v + BS] = b;
      d4[v + 2 * BS] = x;
      d4[v + 3 * BS] = y;
    }
    for (; v < body; v += BS) d4[v] = ld16<SRC>(s4 + v);
    int64_t t0 = head + (body << 4);
    for (int64_t i = t0 + tid; i < n; i += BS) dst[i] = ld1<SRC>(src + i);
  } else {
    for (int64_t i = tid; i < n; i += BS) dst[i] = ld1<SRC>(src + i);
  }
}

// Bounce mode (all threads): pull the span the daemon left in a host pool buffer into this
// CTA's HBM landing slot in one bulk pass, then hand the buffer back to its worker.
template <int BS>
__device__ void pull_span(const DevCtx& c, Smem& s) {
  if (s.pull_n <= 0) return;
  copy_bytes<BS, SRC_SYS>((uint8_t*)half_base(c, s.pull_half), s.pull_src, s.pull_n);
  if (threadIdx.x == 0) {
    s.dbg_land_off[s.pull_half] = s.pull_off;
    s.dbg_land_n[s.pull_half] = s.pull_n;
  }
  // the landing slot is read next by cp.async.bulk (async proxy): order these generic-proxy
  // stores before it (each writing thread fences, the barrier below publishes)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();  // every load has returned: the buffer may be reused
  if (threadIdx.x == 0) {
    if (s.pull_buf >= 0) {
      st_relaxed_sys(&c.bounce_release[s.pull_buf], s.pull_seq);
    }
    s.pull_n = 0;
  }
  __syncthreads();
}

// K1: copy a page's nb bytes from the span buffer into its frame (and, when the page is
// delivered whole to a 16 B-aligned destination, into the user buffer in the same pass),
// checking every word against W(cid, .).  Returns this thread's mismatching-word count.
template <int BS, int SRC>
__device__ int copy_page_in(uint8_t* frame, uint8_t* dst_whole, const uint8_t* src, int64_t nb,
                            int64_t file_off, int64_t cid) {
  const int tid = threadIdx.x;
  int bad = 0;
  const bool chk = cid >= 0;
  const int64_t nv = nb >> 4;
  const uint4* s4 = (const uint4*)src;
  uint4* f4 = (uint4*)frame;
  uint4* d4 = (uint4*)dst_whole;
  const int64_t w0 = file_off >> 3;
  int64_t v = tid;
  for (; v + 3 * BS < nv; v += 4 * BS) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) q[u] = ld16<SRC>(s4 + v + u * BS);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      f4[v + u * BS] = q[u];
      if (d4) d4[v + u * BS] = q[u];
      if (chk) {
        int64_t wi = w0 + 2 * (v + u * BS);
        uint64_t lo = ((uint64_t)q[u].y << 32) | q[u].x, hi = ((uint64_t)q[u].w << 32) | q[u].z;
        bad += (lo != word_law(cid, wi)) + (hi != word_law(cid, wi + 1));
      }
    }
  }
  for (; v < nv; v += BS) {
    uint4 q = ld16<SRC>(s4 + v);
    f4[v] = q;
    if (d4) d4[v] = q;
    if (chk) {
      int64_t wi = w0 + 2 * v;
      uint64_t lo = ((uint64_t)q.y << 32) | q.x, hi = ((uint64_t)q.w << 32) | q.z;
      bad += (lo != word_law(cid, wi)) + (hi != word_law(cid, wi + 1));
    }
  }
  for (int64_t i = (nv << 4) + tid; i < nb; i += BS) {  // sub-16 B tail (EOF pages)
    uint8_t b = ld1<SRC>(src + i);
    frame[i] = b;
    if (dst_whole) dst_whole[i] = b;
    if (chk) {
      int64_t fo = file_off + i;
      uint64_t w = word_law(cid, fo >> 3);
      bad += b != (uint8_t)(w >> (8 * (fo & 7)));
    }
  }
  return bad;
}

// ------------------------------------------------------------ batched page walk
//
// The cold sequential case — a run of pages none of which is cached — is walked as one
// batch instead of page by page: warp 0 looks up and claims up to 32 pages at once, thread
// 0 plans the frame allocations for all of them in page order (the reference's sequence
// of allocation decisions, gpu_cache.py:104-179), warp 0 evicts the victims in parallel,
// the whole CTA copies every page span buffer -> frame (+ user buffer) in one pass, and
// warp 0 installs them.  Every counter, log record and victim is the same as the
// per-page walk would produce for the same TB; only pages that are hits, in flight or
// raced by another TB take the per-page path.


// Reserve n consecutive log records (one atomic); ~0 when logging is off / full.
__device__ unsigned long long log_reserve(const DevCtx& c, int kind, int n) {
  if (!c.log || n <= 0) return ~0ull;
  unsigned long long b = atomicAdd(&c.g->log_n[kind], (unsigned long long)n);
  if (b + n > c.log_cap[kind]) {
    set_error(c, ERR_LOG_OVERFLOW, kind, b);
    return ~0ull;
  }
  return b;
}

__device__ __forceinline__ void log_put3(const DevCtx& c, int kind, unsigned long long i, long long a,
                                         long long b, long long d) {
  long long* r = c.logs[kind] + i * 3;
  r[0] = a;
  r[1] = b;
  r[2] = d;
}

// per-tb-lra plan for k pages (thread 0); returns how many pages get a frame now.  Fresh
// frames first, then retired frames of finished TBs, then the TB's own oldest frames —
// the latter only while they predate this batch (so a batch never recycles itself).
__device__ int plan_per_tb(const DevCtx& c, Smem& s, int k) {
  const int64_t len0 = s.own_len;
  const int a = (int)min((int64_t)k, max((int64_t)0, c.quota - len0));
  int g = 0;
  if (a > 0 && !s.fresh_done) {
    unsigned long long old = atomicAdd(&c.g->fresh_next, (unsigned long long)a);
    if (old + a >= (unsigned long long)c.nframes) s.fresh_done = 1;
    if (old < (unsigned long long)c.nframes)
      g = (int)min((unsigned long long)a, (unsigned long long)c.nframes - old);
    for (int j = 0; j < g; j++) s.b.frame[j] = (uint32_t)(old + j);
  }
  while (g < a) {  // frames released at EOF (rare)
    uint32_t f = take_recycled(c);
    if (f == PT_EMPTY) break;
    s.b.frame[g++] = f;
  }
  for (int j = 0; j < g; j++) s.b.vict[j] = 0;
  int r = 0;
  if (g < a) {  // retired frames, oldest first: one contiguous range of one FIFO
    int pool = 0;
    unsigned long long pos = 0;
    r = retired_reserve(c, a - g, &pool, &pos);
    s.b.ret_pos = pos;
    s.b.ret_pool = pool;
  }
  int hd = k - g - r;  // own-head remaps
  if (hd > len0) hd = (int)len0;
  const int kk = g + r + hd;
  for (int j = g; j < kk; j++) s.b.vict[j] = 1;
  s.b.nret = r;
  s.b.ret_lane0 = g;
  s.b.own_lane0 = g + r;
  s.b.own_head0 = s.own_head;
  s.b.own_tail0 = s.own_head + len0;
  s.b.nvict = r + hd;
  s.own_head += hd;
  s.own_len = len0 + g + r;
  ST(pc_allocs) += g;
  ST(pc_remaps) += r + hd;
  return kk;
}

// global-lru-dealloc plan for k pages (thread 0).  Fresh frames lock-free; victims are the
// first valid, unreferenced frames of the global allocation-order FIFO, taken under the
// global lock (gpu_cache.py:126-147).  Victims are unmapped here (vict = 0 afterwards).
__device__ int plan_global(const DevCtx& c, Smem& s, int k) {
  int g = 0;
  if (!s.fresh_done) {
    unsigned long long old = atomicAdd(&c.g->fresh_next, (unsigned long long)k);
    if (old + k >= (unsigned long long)c.nframes) s.fresh_done = 1;
    if (old < (unsigned long long)c.nframes)
      g = (int)min((unsigned long long)k, (unsigned long long)c.nframes - old);
    for (int j = 0; j < g; j++) s.b.frame[j] = (uint32_t)(old + j);
  }
  while (g < k) {
    uint32_t f = take_recycled(c);
    if (f == PT_EMPTY) break;
    s.b.frame[g++] = f;
  }
  if (g > 0) {
    unsigned long long pos = atomicAdd(&c.g->g_tail, (unsigned long long)g);
    if (pos + g - ld_volatile_u64(&c.g->g_head) >= (unsigned long long)c.gfifo_cap) {
      set_error(c, ERR_FIFO_OVERFLOW, 0, pos);
      return 0;
    }
    for (int j = 0; j < g; j++) st_release_gpu(&c.gfifo[(pos + j) % c.gfifo_cap], s.b.frame[j] + 1);
    s.last_gfifo_pos = (long long)(pos + g - 1);
  }
  ST(pc_allocs) += g;
  int found = 0;
  if (g < k) {
    uint64_t t0 = globaltimer();
    while (atomicCAS(&c.g->lock, 0, 1) != 0) {
      if (!keep_waiting(c, t0, 15)) return 0;
      __nanosleep(64);
    }
    __threadfence();
    unsigned long long head = c.g->g_head;
    const unsigned long long tail = ld_volatile_u64(&c.g->g_tail);
    for (unsigned long long p = head; p < tail && g + found < k; p++) {
      uint32_t* e = &c.gfifo[p % c.gfifo_cap];
      uint32_t val;
      while ((val = ld_acquire_gpu(e)) == 0) {  // reserved, not yet written
        if (!keep_waiting(c, t0, 16)) break;
      }
      if (val == 0) break;
      if (val == RING_TOMB) continue;
      unsigned long long key = try_unmap(c, val - 1);
      if (key == ~0ull) continue;  // in flight or referenced: skipped (gpu_cache.py:133-137)
      *e = RING_TOMB;
      s.b.frame[g + found] = val - 1;
      log_rec(c, GFS_LOG_VICTIMS, s.tb, (long long)(key >> 40), (long long)(key & ((1ull << 40) - 1)), 0);
      found++;
    }
    while (head < tail && *(volatile uint32_t*)&c.gfifo[head % c.gfifo_cap] == RING_TOMB) {
      c.gfifo[head % c.gfifo_cap] = 0;
      head++;
    }
    c.g->g_head = head;
    __threadfence();
    atomicExch(&c.g->lock, 0);
    if (found > 0) {
      unsigned long long pos = atomicAdd(&c.g->g_tail, (unsigned long long)found);
      for (int j = 0; j < found; j++)
        st_release_gpu(&c.gfifo[(pos + j) % c.gfifo_cap], s.b.frame[g + j] + 1);
      s.last_gfifo_pos = (long long)(pos + found - 1);
    }
    ST(pc_evictions) += found;
    ST(pc_allocs) += found;
    ST(victims) += found;
  }
  for (int j = 0; j < g + found; j++) s.b.vict[j] = 0;
  s.b.nvict = 0;
  return g + found;
}

// One batch of cold pages starting at g_pos (all threads).  Returns delivered bytes,
// 0 = not applicable (the caller takes the per-page path), -1 = abort.
template <int BS>
__device__ int64_t gread_batch(const DevCtx& c, Smem& s, int64_t fid, int64_t g_pos, int64_t g_end,
                               int64_t seg_end, uint8_t* d0, int& bad_words, const uint8_t* span_buf) {
  const int tid = threadIdx.x, lane = tid & 31;
  const bool w0 = tid < 32;
  const DevFile& F = c.files[fid];
  const int64_t pg = c.page_size, fs = F.size;
  const int64_t p0 = g_pos / pg;
  const int64_t lim = g_end < fs ? g_end : fs;
  int nmax = (int)min((int64_t)32, (lim + pg - 1) / pg - p0);
  if (c.policy == GFS_POLICY_GLOBAL_LRU) nmax = (int)min((int64_t)nmax, max((int64_t)1, c.nframes / 4));
  uint32_t* pt = F.pt;
  uint64_t t_start = 0;
  long long wait0 = 0;
  if (tid == 0) {
    t_start = globaltimer();
    wait0 = ST(wait_ns);
  }
  if (c.readahead == GFS_RA_ONDEMAND) {  // markers and pending windows at the walk position
    if (tid == 0) {
      if (!od_top(c, s, fid, p0)) set_error(c, ERR_IO, (int)fid, (unsigned long long)p0);
      s.abort = has_error(c);
    }
    __syncthreads();
    if (s.abort) return -1;  // block-uniform
    pull_span<BS>(c, s);     // an adopted window pulled by the CTA (bounce / mapped)
    span_buf = span_base(c, s);
    if (s.od.cap - p0 < nmax) nmax = (int)(s.od.cap - p0);
  }

  // (A) warp 0: look up and claim the leading run of uncached pages
  if (w0) {
    // claim straight away (one round trip): the batch is the leading run of claimed pages
    bool ok = lane < nmax && atomicCAS(&pt[p0 + lane], PT_EMPTY, PT_CLAIMED) == PT_EMPTY;
    unsigned got = __ballot_sync(0xffffffffu, ok);
    int kc = (~got == 0u) ? 32 : __ffs(~got) - 1;
    if (ok && lane >= kc) st_release_gpu(&pt[p0 + lane], PT_EMPTY);  // beyond a raced page
    if (lane == 0) s.b.n_empty = kc;
  }
  __syncthreads();
  const int kc = s.b.n_empty;
  if (kc < 1) return 0;

  // (B) thread 0: how many of them this batch can serve, and their frames
  if (tid == 0) {
    const uint64_t tb0 = globaltimer();
    ST(lookup_ns) += (long long)(tb0 - t_start);  // batch phase A: claims (incl. ondemand top)
    s.t_copy0 = tb0;
    int kp = 1;
    s.b.sync_m = -1;
    if (pb_has(s, fid, p0)) {
      kp = max(1, pb_run(s, fid, p0, kc));
    } else if (c.readahead == GFS_RA_ONDEMAND && F.read_only) {
      s.b.sync_m = od_plan_sync(c, s, fid, p0, p0, p0 + kc);  // the request's decision first
      kp = (int)min((int64_t)kc, max((int64_t)1, s.b.sync_m));
    } else {
      int64_t win;
      const int64_t span = span_peek(c, s, fid, p0, seg_end, &win);
      int64_t m = (span + pg - 1) / pg;                        // pages the RPC brings
      if (m - 1 > c.pb_cap_bytes / pg) m = 1 + c.pb_cap_bytes / pg;  // private-buffer room
      kp = (int)min((int64_t)kc, max((int64_t)1, m));
    }
    int kk = c.policy == GFS_POLICY_GLOBAL_LRU ? plan_global(c, s, kp) : plan_per_tb(c, s, kp);
    if (has_error(c)) kk = 0;
    // page 0's RPC goes out now: its round trip overlaps the evictions of (C)
    s.b.early = 0;
    if (kk >= 1 && !pb_has(s, fid, p0)) {
      if (fetch_begin(c, s, fid, p0, seg_end, s.b.sync_m)) {
        s.b.early = 1;
      } else {
        if (!has_error(c)) set_error(c, ERR_IO, (int)fid, (unsigned long long)p0);
        kk = 0;
      }
    }
    s.b.k = kk;
  }
  __syncthreads();
  const int kk = s.b.k;
  if (w0 && lane < kc && lane >= kk) st_release_gpu(&pt[p0 + lane], PT_EMPTY);  // not this batch
  if (kk < 1) {
    __syncthreads();
    return has_error(c) ? -1 : 0;
  }

  // (C) warp 0: victims (own-head / retired frames) and the own-queue update
  if (w0 && c.policy == GFS_POLICY_PER_TB_LRA) {
    uint32_t f = PT_EMPTY;
    bool abort = false;
    if (lane < kk && s.b.vict[lane]) {
      if (lane < s.b.own_lane0) {  // retired range
        bool ok;
        f = retired_take(c, s.b.ret_pool, s.b.ret_pos + (lane - s.b.ret_lane0), &ok);
        abort = !ok;
      } else {  // own oldest frames
        f = c.own_q[(int64_t)blockIdx.x * c.quota + (s.b.own_head0 + (lane - s.b.own_lane0)) % c.quota];
      }
    }
    __syncwarp();
    if (lane < kk && s.b.vict[lane]) {
      if (!abort) s.b.frame[lane] = f;
      unsigned long long key = ~0ull;
      uint64_t t0 = globaltimer();
      while (!abort && (key = try_unmap(c, f)) == ~0ull) {  // wait out transient readers
        if (!keep_waiting(c, t0, 10)) {
          abort = true;
          break;
        }
        __nanosleep(100);
      }
      s.b.src_off[lane] = (long long)key;  // scratch: victim key for the log below
    }
    __syncwarp();
    const int nv = s.b.nvict;
    unsigned long long base = 0;
    if (lane == 0) base = log_reserve(c, GFS_LOG_VICTIMS, nv);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base != ~0ull && lane < kk && s.b.vict[lane]) {
      const unsigned long long key = (unsigned long long)s.b.src_off[lane];
      log_put3(c, GFS_LOG_VICTIMS, base + (lane - s.b.ret_lane0), s.tb, (long long)(key >> 40),
               (long long)(key & ((1ull << 40) - 1)));
    }
    if (lane == 0) ST(victims) += nv;
    if (lane < kk)  // pushes at the tail, in page order
      c.own_q[(int64_t)blockIdx.x * c.quota + (s.b.own_tail0 + lane) % c.quota] = s.b.frame[lane];
  }
  __syncthreads();
  if (has_error(c)) return -1;

  // (D) thread 0: lookups/misses, the private-buffer walk and the RPC (prefetcher.py)
  // Page 0 of the batch is a private-buffer hit or the RPC's own page; every later page
  // is a private-buffer hit (planned in (B)), taken as one run.
  if (tid == 0) {
    ST(alloc_ns) += (long long)(globaltimer() - s.t_copy0);  // batch phases B + C: plan, RPC out, evictions
    int status = 0, j0 = 0;
    ST(pc_lookups) += kk;
    ST(pc_misses) += kk;
    if (!pb_has(s, fid, p0)) {
      const int64_t page = p0;
      ST(pb_misses)++;
      j0 = 1;
      int64_t span;
      const int64_t n = s.b.early ? fetch_end(c, s, fid, page, &span, true)
                                  : fetch_span(c, s, fid, page, seg_end, &span, s.b.sync_m);
      if (n < 0) {
        status = 2;
      } else if (n == 0) {
        set_error(c, ERR_IO, (int)fid, (unsigned long long)page);
        status = 2;
      }
      if (status == 0) {
        const int64_t nb0 = n < pg ? n : pg;
        s.b.nb[0] = (int32_t)nb0;
        s.b.src_off[0] = 0;
        const int64_t m = (n + pg - 1) / pg;
        if (m > 1) {  // the span refills the private buffer, in the half it landed in
          pb_fill(c, s, fid, page, m, n - nb0);
          s.span_half = s.fetch_half;
        }
      }
    }
    // every page of a batch comes from one half: the fetched span's (page 0, and the
    // private-buffer pages it brought), or the private buffer's
    s.b.src_half = j0 ? s.fetch_half : s.span_half;
    if (status == 0 && j0 < kk) {
      if (pb_run(s, fid, p0 + j0, kk - j0) < kk - j0) {  // planned but absent: file shrank
        set_error(c, ERR_IO, (int)fid, (unsigned long long)(p0 + j0));
        status = 2;
      } else {
        pb_take_run(s, p0 + j0, kk - j0);
      }
    }
    s.b.status = status;
    s.b.j0 = j0;
  }
  __syncthreads();
  if (s.b.status != 0) return -1;
  const bool direct = s.direct[s.b.src_half];
  // an RPC may have switched landing halves; a direct span is read at its file offsets
  span_buf = direct ? F.map : half_base(c, s.b.src_half);
  if (w0) {  // private-buffer pages' bytes and span offsets; bind frames to their pages
    if (lane >= s.b.j0 && lane < kk) {
      const int64_t i = p0 + lane - s.pb_base;
      s.b.nb[lane] = (int32_t)(i == s.pb_count ? s.pb_last_nb : pg);
      s.b.src_off[lane] = i * pg - s.pb_off_adj;
    }
    if (direct && lane < kk) s.b.src_off[lane] = (p0 + lane) * pg;
    if (lane < kk) c.fkey[s.b.frame[lane]] = page_key(fid, p0 + lane);
    __syncwarp();
    // which pages need the byte-wise tail copy or a partial delivery, and the batch's bytes
    const int64_t in0b = g_pos - p0 * pg;
    const bool dok = d0 != nullptr && ((((uintptr_t)d0 - (uintptr_t)in0b)) & 15) == 0;
    long long want = 0;
    bool tail = false, part = false;
    if (lane < kk) {
      const int64_t ps = (p0 + lane) * pg, nbj = s.b.nb[lane];
      const int64_t lo = ps > g_pos ? ps : g_pos;
      const int64_t hi = ps + nbj < g_end ? ps + nbj : g_end;
      want = hi - lo;
      tail = (nbj & 15) != 0;
      part = d0 != nullptr && !(dok && ps >= g_pos && ps + nbj <= g_end && !tail);
    }
    const unsigned tm = __ballot_sync(0xffffffffu, tail), pm = __ballot_sync(0xffffffffu, part);
    for (int o = 16; o > 0; o >>= 1) want += __shfl_xor_sync(0xffffffffu, want, o);
    if (lane == 0) {
      // streamed window: the batch's span bytes must have landed
      int64_t need = 0;
      for (int j = 0; j < kk; j++) need = max(need, (int64_t)s.b.src_off[j] + s.b.nb[j]);
      if (!wait_landed(c, s, s.b.src_half, need)) set_error(c, ERR_TIMEOUT, 24, 0);
      s.b.tail_mask = tm;
      s.b.part_mask = pm;
      s.b.total = want;
      const uint64_t t1 = globaltimer();
      ST(meta_ns) += (long long)(t1 - t_start) - (ST(wait_ns) - wait0);  // RPC waits counted apart
      s.t_copy0 = t1;
    }
  }
  __syncthreads();
  pull_span<BS>(c, s);

  // (E) all threads: K1 over the whole batch — span buffer -> frames (+ user buffer)
  const int64_t vpp = pg >> 4;  // 16-byte vectors per page
  const int64_t nvec = (int64_t)kk * vpp;
  const int64_t in0 = g_pos - p0 * pg;
  const bool dst_ok = d0 != nullptr && ((((uintptr_t)d0 - (uintptr_t)in0)) & 15) == 0;
  const bool chk = c.verify && F.content_id >= 0;
  const int64_t cid = F.content_id;
  int bad = 0;
  const uint4* src4 = (const uint4*)(span_buf + s.b.src_off[0]);  // pages are consecutive
  const bool contiguous = s.b.src_off[kk - 1] == s.b.src_off[0] + (int64_t)(kk - 1) * pg;
  bool full_pages = true;
  for (int j = 0; j < kk; j++) full_pages &= s.b.nb[j] == pg;
  const bool sys_src = c.transfer == GFS_XFER_ZEROCOPY || direct;  // pinned host memory
  const bool use_tma = c.tma && c.transfer != GFS_XFER_ZEROCOPY && contiguous && full_pages &&
                       (((uintptr_t)src4) & 15) == 0;
  if (use_tma) {
    // K1 by TMA: thread 0 streams the batch HBM -> shared-memory stage ring -> frames (and
    // whole pages -> user buffer) with bulk copies, TMA_NST stages in flight.  With the
    // word check on, warps 1.. check each stage while it sits in shared memory and arrive on
    // its "checked" mbarrier; thread 0 waits for that only before refilling the stage —
    // producer and checkers never meet at a block barrier inside the batch.
    extern __shared__ __align__(128) float cons_smem[];
    uint8_t* ring = (uint8_t*)cons_smem + c.tma_off;
    const int64_t total_b = (int64_t)kk * pg;
    const int nch = (int)((total_b + TMA_CH - 1) / TMA_CH);
    const int NST = c.tma_nst;  // stages in flight (4, or 5 when the shared state leaves room)
    const unsigned long long G0 = s.tma_seq;
    const uint8_t* srcb = (const uint8_t*)src4;
    const int warp = tid >> 5;
    auto load = [&](int i) {  // thread 0
      const int st = stage_of(G0 + i, NST);
      if (s.tma_epend & (1u << st)) {  // the stage's last chunk must be checked before reuse
        mbar_wait_t(c, &s.tma_empty[st], (s.tma_epar >> st) & 1u, 42,
                    ((G0 + i) << 16) | ((unsigned long long)st << 8) | (unsigned)(i & 0xff));
        s.tma_epend &= ~(1u << st);
        s.tma_epar ^= 1u << st;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int64_t cb = min(TMA_CH, total_b - (int64_t)i * TMA_CH);
      tma_load(ring + st * TMA_CH, srcb + (int64_t)i * TMA_CH, (uint32_t)cb, &s.tma_bar[st]);
    };
    if (tid == 0) {
      // landing bytes written by the copy engine / generic proxy, read by the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for (int i = 0; i < nch && i < NST; i++) load(i);
    }
    for (int i = 0; i < nch; i++) {
      const unsigned long long G = G0 + i;
      const int st = stage_of(G, NST);
      const uint32_t par = phase_of(G, NST);
      const int64_t b0 = (int64_t)i * TMA_CH;
      const int64_t cb = min(TMA_CH, total_b - b0);
      const uint8_t* sbuf = ring + st * TMA_CH;
      if (chk && warp > 0) {  // checkers
        mbar_wait_t(c, &s.tma_bar[st], par, 41, (G << 16) | ((unsigned long long)st << 8) | (unsigned)(i & 0xff));
        const uint4* sv = (const uint4*)sbuf;
        const int64_t wbase = (p0 * pg + b0) >> 3;
        for (int64_t v = tid - 32; v < (cb >> 4); v += BS - 32) {
          const uint4 q = sv[v];
          const int64_t wi = wbase + 2 * v;
          const uint64_t tag = block_tag(cid, wi);
          const uint64_t lo = ((uint64_t)q.y << 32) | q.x, hi = ((uint64_t)q.w << 32) | q.z;
          const int nb2 = (lo != mix64(tag ^ (uint64_t)wi)) + (hi != mix64(tag ^ (uint64_t)(wi + 1)));
          if (nb2) note_mismatch(c, s, fid, wi * 8, lo, s.b.src_off[0] + b0 + 16 * v, kk);
          bad += nb2;
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&s.tma_empty[st]);
      }
      if (tid == 0) {  // producer
        mbar_wait_t(c, &s.tma_bar[st], par, 40, (G << 16) | ((unsigned long long)st << 8) | (unsigned)(i & 0xff));
        if (i == 0) early_poll(c, s);  // the span's answer, fetched while the rest streams
        // the chunk's pieces: page j gets [max(b0, j pg), min(b0 + cb, (j+1) pg))
        for (int64_t b = b0; b < b0 + cb;) {
          const int j = (int)(b / pg);
          const int64_t e = min(b0 + cb, (int64_t)(j + 1) * pg);
          const int64_t po = b - (int64_t)j * pg;
          tma_store(c.frames + (int64_t)s.b.frame[j] * pg + po, sbuf + (b - b0), (uint32_t)(e - b));
          const int64_t ps = (p0 + j) * pg;
          if (dst_ok && ps >= g_pos && ps + pg <= g_end)
            tma_store(d0 + (ps - g_pos) + po, sbuf + (b - b0), (uint32_t)(e - b));
          b = e;
        }
        tma_commit();
        if (chk) s.tma_epend |= 1u << st;
        if (i >= 1 && i - 1 + NST < nch) {  // refill the stage chunk i - 1 used
          tma_wait_read<1>();               // its stores have read it (chunk i's may not)
          load(i - 1 + NST);
        }
      }
    }
    if (tid == 0) tma_wait_all();
    __syncthreads();  // every thread has read G0 and is done with the ring
    if (tid == 0) s.tma_seq = G0 + nch;  // read again only after later block barriers
  } else {
  // vector v of the batch is vector w of page j: shifts when the page size is a power of 2
  const int vsh = (pg & (pg - 1)) == 0 ? __ffsll(pg) - 1 - 4 : -1;
  for (int64_t v0 = tid; v0 < nvec; v0 += 4 * BS) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = v0 + u * BS;
      if (v < nvec) {
        const int j = (int)(vsh >= 0 ? v >> vsh : v / vpp);
        const int64_t w = v - (int64_t)j * vpp;
        const uint4* sp = contiguous ? src4 + v : (const uint4*)(span_buf + s.b.src_off[j]) + w;
        q[u] = (w << 4) < s.b.nb[j] ? (!sys_src ? ld16<SRC_HBM>(sp) : ld16<SRC_SYS>(sp))
                                    : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t v = v0 + u * BS;
      if (v >= nvec) break;
      const int j = (int)(vsh >= 0 ? v >> vsh : v / vpp);
      const int64_t w = v - (int64_t)j * vpp;
      const int64_t nbj = s.b.nb[j];
      if ((w << 4) + 16 > nbj) continue;  // sub-16 B EOF tail: byte loop below
      ((uint4*)(c.frames + (int64_t)s.b.frame[j] * pg))[w] = q[u];
      // whole-page deliveries go straight to the user buffer in the same pass
      const int64_t ps = (p0 + j) * pg;
      if (dst_ok && ps >= g_pos && ps + nbj <= g_end)
        ((uint4*)(d0 + (ps - g_pos)))[w] = q[u];
      if (chk) {  // both words of a vector share one 4 KiB block tag
        const int64_t wi = (ps >> 3) + 2 * w;
        const uint64_t tag = block_tag(cid, wi);
        const uint64_t lo = ((uint64_t)q[u].y << 32) | q[u].x, hi = ((uint64_t)q[u].w << 32) | q[u].z;
        const int nb2 = (lo != mix64(tag ^ (uint64_t)wi)) + (hi != mix64(tag ^ (uint64_t)(wi + 1)));
        if (nb2) note_mismatch(c, s, fid, wi * 8, lo, s.b.src_off[j] + 16 * w, kk);
        bad += nb2;
      }
    }
  }
  }  // LDG path
  for (unsigned m = s.b.tail_mask; m; m &= m - 1) {  // EOF page tails not a multiple of 16 B
    const int j = __ffs(m) - 1;
    const int64_t nbj = s.b.nb[j];
    const uint8_t* sp = span_buf + s.b.src_off[j];
    uint8_t* fp = c.frames + (int64_t)s.b.frame[j] * pg;
    for (int64_t i = (nbj & ~(int64_t)15) + tid; i < nbj; i += BS) {
      const uint8_t b = !sys_src ? ld1<SRC_HBM>(sp + i) : ld1<SRC_SYS>(sp + i);
      fp[i] = b;
      if (chk) {
        const int64_t fo = (p0 + j) * pg + i;
        bad += b != (uint8_t)(word_law(cid, fo >> 3) >> (8 * (fo & 7)));
      }
    }
  }
  bad_words += bad;
  const int any_bad = __syncthreads_or(bad);
  // partial deliveries (first page entered mid-page, last page cut by the request, EOF
  // tails, misaligned user buffers) from the frames just written
  const int64_t total = s.b.total;
  for (unsigned m = s.b.part_mask; m; m &= m - 1) {
    const int j = __ffs(m) - 1;
    const int64_t ps = (p0 + j) * pg, nbj = s.b.nb[j];
    const int64_t lo = ps > g_pos ? ps : g_pos;
    const int64_t hi = ps + nbj < g_end ? ps + nbj : g_end;
    copy_bytes<BS, SRC_HBM>(d0 + (lo - g_pos), c.frames + (int64_t)s.b.frame[j] * pg + (lo - ps), hi - lo);
  }
  if (s.b.part_mask) __syncthreads();

  // (F) warp 0: install (data, then VALID, then the page-table entry) and deliveries
  if (w0) {
    if (lane == 0) {
      const uint64_t t_in = globaltimer();
      ST(copy_ns) += (long long)(t_in - s.t_copy0);
      s.t_copy0 = t_in;
    }
    __threadfence();  // frame data before VALID and the PTE (this fence makes the store a release)
    if (lane < kk) {
      atomicOr(&c.fstate[s.b.frame[lane]], FR_VALID);
      *(volatile uint32_t*)&pt[p0 + lane] = s.b.frame[lane];
    }
    unsigned long long base = 0;
    if (lane == 0) base = log_reserve(c, GFS_LOG_DELIVERIES, kk);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base != ~0ull && lane < kk) log_put3(c, GFS_LOG_DELIVERIES, base + lane, s.tb, fid, p0 + lane);
    if (lane == 0) {
      ST(user_bytes) += total;
      if (any_bad) ST(tag_mismatches)++;
      ST(install_ns) += (long long)(globaltimer() - s.t_copy0);
    }
  }
  __syncthreads();
  return total;
}

// One batch of cached pages starting at g_pos (all threads): gpu_exec.py:156-166 for a run
// of up to 32 pages at once — warp 0 looks up and pins the leading run of valid frames,
// every thread copies frame -> user buffer, warp 0 unpins and delivers.  Same lookups,
// hits, bytes and delivery log as the page-by-page walk.  Returns delivered bytes, 0 when
// page p0 is not a valid cached page (the caller takes the per-page path: pending pages,
// races, misses).
template <int BS>
__device__ int64_t gread_hits(const DevCtx& c, Smem& s, int64_t fid, int64_t g_pos, int64_t g_end,
                              uint8_t* d0) {
  const int tid = threadIdx.x, lane = tid & 31;
  const bool w0 = tid < 32;
  const DevFile& F = c.files[fid];
  const int64_t pg = c.page_size, fs = F.size;
  const int64_t p0 = g_pos / pg;
  const int64_t lim = g_end < fs ? g_end : fs;
  int nmax = (int)min((int64_t)32, (lim + pg - 1) / pg - p0);
  if (c.readahead == GFS_RA_ONDEMAND && s.od.cap - p0 < nmax) nmax = (int)(s.od.cap - p0);  // markers
  if (w0) {
    bool ok = false;
    uint32_t f = 0;
    if (lane < nmax) {
      const uint32_t e = ld_acquire_gpu(&F.pt[p0 + lane]);
      if (e != PT_EMPTY && e != PT_CLAIMED && !(e & PT_INFLIGHT)) {
        const uint32_t old = atomic_add_acquire_gpu(&c.fstate[e], FR_REF);  // pin against eviction
        if ((old & FR_VALID) && __ldcg(&c.fkey[e]) == page_key(fid, p0 + lane)) {
          ok = true;
          f = e;
        } else {
          atomicSub(&c.fstate[e], FR_REF);
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    const int run = (~m == 0u) ? 32 : __ffs(~m) - 1;
    if (ok && lane >= run) atomicSub(&c.fstate[f], FR_REF);  // beyond the run
    if (lane < run) s.b.frame[lane] = f;
    if (lane == 0) s.b.k = run;
  }
  __syncthreads();
  const int kh = s.b.k;
  if (kh == 0) return 0;
  // copy frames -> user buffer: one flattened vector loop when every page is delivered
  // whole to a 16 B-aligned destination, else page by page
  const int64_t end_b = min(lim, (p0 + kh) * pg);
  const bool whole = d0 != nullptr && g_pos == p0 * pg && end_b == (p0 + kh) * pg && (((uintptr_t)d0) & 15) == 0;
  if (whole) {
    const int64_t vpp = pg >> 4, nvec = (int64_t)kh * vpp;
    const int vsh = (pg & (pg - 1)) == 0 ? __ffsll(pg) - 1 - 4 : -1;
    for (int64_t v0 = tid; v0 < nvec; v0 += 4 * BS) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t v = v0 + u * BS;
        if (v < nvec) {
          const int j = (int)(vsh >= 0 ? v >> vsh : v / vpp);
          q[u] = __ldcg((const uint4*)(c.frames + (int64_t)s.b.frame[j] * pg) + (v - (int64_t)j * vpp));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t v = v0 + u * BS;
        if (v < nvec) ((uint4*)d0)[v] = q[u];
      }
    }
  } else if (d0) {
    for (int j = 0; j < kh; j++) {
      const int64_t ps = (p0 + j) * pg;
      const int64_t lo = ps > g_pos ? ps : g_pos;
      const int64_t pe = ps + pg < fs ? ps + pg : fs;
      const int64_t hi = pe < g_end ? pe : g_end;
      copy_bytes<BS, SRC_HBM>(d0 + (lo - g_pos), c.frames + (int64_t)s.b.frame[j] * pg + (lo - ps), hi - lo);
    }
  }
  __syncthreads();
  if (w0) {
    long long want = 0;
    if (lane < kh) {
      atomicSub(&c.fstate[s.b.frame[lane]], FR_REF);
      const int64_t ps = (p0 + lane) * pg;
      const int64_t lo = ps > g_pos ? ps : g_pos;
      const int64_t pe = ps + pg < fs ? ps + pg : fs;
      want = (pe < g_end ? pe : g_end) - lo;
    }
    for (int o = 16; o > 0; o >>= 1) want += __shfl_xor_sync(0xffffffffu, want, o);
    unsigned long long base = 0;
    if (lane == 0) base = log_reserve(c, GFS_LOG_DELIVERIES, kh);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base != ~0ull && lane < kh) log_put3(c, GFS_LOG_DELIVERIES, base + lane, s.tb, fid, p0 + lane);
    if (lane == 0) {
      ST(pc_lookups) += kh;
      ST(pc_hits) += kh;
      ST(user_bytes) += want;
      ST(cache_hit_user_bytes) += want;
      s.b.total = want;
    }
  }
  __syncthreads();
  return s.b.total;
}

// ----------------------------------------------------------------- gread (all threads)

// One gread of `size` bytes at `offset` of `fid` (gpu_exec.py:107-239).  `dst` is the
// user-buffer address of byte `offset` (nullptr = consume-only).  Returns delivered bytes,
// or -1 when the run aborts.
template <int BS>
__device__ int64_t gread(const DevCtx& c, Smem& s, int64_t fid, int64_t offset, int64_t size,
                         int64_t seg_end, uint8_t* dst, int& bad_words) {
  const int tid = threadIdx.x;
  const int64_t pg = c.page_size;
  const DevFile& F = c.files[fid];
  const int64_t fs = F.size;
  const uint8_t* span_buf = half_base(c, 0);  // raw mode: one span in half 0
  if (tid == 0) {
    ST(greads)++;
    s.g_lo = offset;
    s.g_hi = offset + size;
    s.g_la = c.lookahead && (offset % pg) == 0 && (c.request_bytes % pg) == 0;
    if (c.readahead == GFS_RA_ONDEMAND && fid != s.od.fid) od_reset(s, fid);  // a new stream
  }

  if (c.raw_mode) {  // gpu_exec.py:114-119, 131-138: whole request, no page cache
    if (tid == 0) {
      int64_t n = rpc_call(c, s, fid, offset, size);
      s.n = n;
      if (n >= 0) {
        log_rec(c, GFS_LOG_RPCS, s.tb, fid, offset, size);
        ST(rpc_count)++;
        ST(rpc_requested_bytes) += size;
        account_transfer(c, s, n);
        ST(user_bytes) += n;
      }
    }
    __syncthreads();
    pull_span<BS>(c, s);
    int64_t n = s.n;
    if (n < 0) return -1;
    if (dst) {
      if (s.direct[0]) copy_bytes<BS, SRC_SYS>(dst, F.map + offset, n);  // straight from the mapping
      else if (c.transfer != GFS_XFER_ZEROCOPY) copy_bytes<BS, SRC_HBM>(dst, span_buf, n);
      else copy_bytes<BS, SRC_SYS>(dst, span_buf, n);
    }
    __syncthreads();
    return n;
  }

  int64_t g_pos = offset;
  const int64_t g_end = offset + size;
  uint32_t* pt = F.pt;
  // Lookahead (gpu.lookahead): with page-aligned requests a batch may run past this request
  // to the end of the TB's segment — the pages the TB's next greads would walk, in the same
  // order, with the same lookups, allocations, private-buffer takes, installs and
  // deliveries (straight into their user-buffer positions).  Those greads then find their
  // bytes delivered.  Every counter and log is what the request-by-request walk produces.
  const bool la = c.lookahead && (offset % pg) == 0 && (c.request_bytes % pg) == 0;
  const int64_t d_end = la ? (seg_end < fs ? seg_end : fs) : g_end;
  if (fid == s.la_fid && offset >= s.la_lo && offset < s.la_hi) {
    const int64_t covered = (s.la_hi < g_end ? s.la_hi : g_end) - offset;
    if (covered >= size) return size;
    g_pos = offset + covered;
  }
  for (;;) {
    if (g_pos >= g_end || g_pos >= fs) return (g_pos < g_end ? g_pos : g_end) - offset;
    const int64_t page = g_pos / pg;
    const int64_t page_end = (page + 1) * pg < fs ? (page + 1) * pg : fs;
    int64_t want = (g_end < page_end ? g_end : page_end) - g_pos;
    const int64_t in_page = g_pos - page * pg;
    const unsigned long long key = page_key(fid, page);

    {  // cold run of pages: batched walk
      const int64_t got = gread_batch<BS>(c, s, fid, g_pos, d_end, seg_end,
                                          dst ? dst + (g_pos - offset) : nullptr, bad_words, span_buf);
      if (got < 0) return -1;
      const int64_t hits = got > 0 ? 0 : gread_hits<BS>(c, s, fid, g_pos, d_end,
                                                      dst ? dst + (g_pos - offset) : nullptr);
      if (got > 0 || hits > 0) {
        g_pos += got + hits;
        if (g_pos > g_end) {  // delivered ahead: remember for the next greads of this TB
          if (tid == 0) {
            s.la_fid = fid;
            s.la_lo = g_end;
            s.la_hi = g_pos;
          }
          __syncthreads();
        }
        continue;
      }
    }

    if (tid == 0) {  // ---- decide (gpu_exec.py:142-199) ----
      int act = A_ABORT;
      ST(pc_lookups)++;
      bool pending = false;
      uint64_t t0 = globaltimer();
      const long long wait0 = ST(wait_ns);
      uint32_t f = PT_EMPTY;
      bool miss = false;
      for (;;) {
        if (has_error(c)) break;
        uint32_t e = ld_acquire_gpu(&pt[page]);
        if (e == PT_CLAIMED || (e != PT_EMPTY && (e & PT_INFLIGHT))) {
          if (!pending) {  // another TB is fetching it: single flight, wait (:167-172)
            ST(pc_hit_pending)++;
            pending = true;
          }
          if (!keep_waiting(c, t0, 30)) break;
          __nanosleep(128);
          continue;
        }
        if (pending) {  // woken: the reference re-runs _page_step, one more lookup
          ST(pc_lookups)++;
          pending = false;
        }
        if (e == PT_EMPTY) {
          if (atomicCAS(&pt[page], PT_EMPTY, PT_CLAIMED) == PT_EMPTY) {
            miss = true;
            break;
          }
          continue;
        }
        uint32_t old = atomic_add_acquire_gpu(&c.fstate[e], FR_REF);
        if ((old & FR_VALID) && __ldcg(&c.fkey[e]) == key) {
          f = e;
          act = A_HIT;
          ST(pc_hits)++;
          break;
        }
        atomicSub(&c.fstate[e], FR_REF);  // remapped under us: look again
      }
      if (miss) {
        ST(pc_misses)++;
        // ondemand: decision + synchronous span before the frame allocation may evict pages
        int64_t sync_m = -1;
        if (c.readahead == GFS_RA_ONDEMAND && F.read_only && !pb_has(s, fid, page))
          sync_m = od_plan_sync(c, s, fid, page, page, page + 1);
        const uint64_t ta = globaltimer();
        ST(lookup_ns) += (long long)(ta - t0);
        f = c.policy == GFS_POLICY_GLOBAL_LRU ? alloc_global(c, s) : alloc_per_tb(c, s);
        ST(alloc_ns) += (long long)(globaltimer() - ta);
        if (f != PT_EMPTY) {
          c.fkey[f] = key;
          st_release_gpu(&pt[page], f | PT_INFLIGHT);
          int64_t nb = pb_take(s, fid, page);
          if (nb > 0) {
            act = A_PBHIT;
            s.nb = nb;
            s.src_off = (page - s.pb_base) * pg - s.pb_off_adj;
            s.src_half = s.span_half;
          } else {
            int64_t span;
            int64_t n = fetch_span(c, s, fid, page, seg_end, &span, sync_m);
            if (n >= 0) {
              act = A_RPC;
              s.n = n;
              s.nb = n < pg ? n : pg;
              s.src_off = 0;
              s.src_half = s.fetch_half;
            }
          }
        }
      }
      if ((act == A_PBHIT || act == A_RPC) && !wait_landed(c, s, s.src_half, s.src_off + s.nb))
        act = A_ABORT;
      if (has_error(c)) act = A_ABORT;
      s.act = act;
      s.frame = f;
      const uint64_t t1 = globaltimer();
      ST(meta_ns) += (long long)(t1 - t0) - (ST(wait_ns) - wait0);
      s.t_copy0 = t1;
    }
    __syncthreads();
    pull_span<BS>(c, s);
    const int act = s.act;
    const uint32_t f = s.frame;
    if (act == A_ABORT) return -1;
    uint8_t* fmem = c.frames + (int64_t)f * pg;
    uint8_t* d = dst ? dst + (g_pos - offset) : nullptr;

    if (act == A_HIT) {  // K2: frame -> user buffer
      if (d) copy_bytes<BS, SRC_HBM>(d, fmem + in_page, want);
      __syncthreads();
      if (tid == 0) {
        atomicSub(&c.fstate[f], FR_REF);
        ST(user_bytes) += want;
        ST(cache_hit_user_bytes) += want;
        log_rec(c, GFS_LOG_DELIVERIES, s.tb, fid, page, 0);
      }
      g_pos += want;
      continue;
    }

    if (act == A_RPC && s.n == 0) {  // zero bytes: page at/after EOF (gpu_exec.py:207-211)
      if (tid == 0) release_frame(c, s, f, &pt[page]);
      __syncthreads();
      return g_pos - offset;
    }

    // K1: span buffer -> frame (+ user buffer)
    const int64_t nb = s.nb;
    if (act == A_RPC) {  // the page may be cut short by the returned byte count
      const int64_t pend = page * pg + nb < fs ? page * pg + nb : fs;
      want = (g_end < pend ? g_end : pend) - g_pos;
    }
    const bool whole = d && in_page == 0 && want == nb && (((uintptr_t)d & 15) == 0);
    const bool direct = s.direct[s.src_half];  // straight from the pinned mapping (K1 direct)
    const uint8_t* src = direct ? F.map + page * pg : half_base(c, s.src_half) + s.src_off;
    int bad = c.transfer != GFS_XFER_ZEROCOPY && !direct
                  ? copy_page_in<BS, SRC_HBM>(fmem, whole ? d : nullptr, src, nb, page * pg,
                                              c.verify ? F.content_id : -1)
                  : copy_page_in<BS, SRC_SYS>(fmem, whole ? d : nullptr, src, nb, page * pg,
                                              c.verify ? F.content_id : -1);
    bad_words += bad;
    int page_bad = __syncthreads_or(bad);
    if (d && !whole) {
      copy_bytes<BS, SRC_HBM>(d, fmem + in_page, want);
      __syncthreads();
    }
    if (tid == 0) {  // install (gpu_cache.py:181-189): data first, then VALID, then the PTE
      const uint64_t t_in = globaltimer();
      ST(copy_ns) += (long long)(t_in - s.t_copy0);
      __threadfence();
      atomicOr(&c.fstate[f], FR_VALID);
      st_release_gpu(&pt[page], f);
      if (page_bad) ST(tag_mismatches)++;
      if (act == A_RPC) {
        int64_t m = (s.n + pg - 1) / pg;
        if (m > 1) {
          pb_fill(c, s, fid, page, m, s.n - nb);
          s.span_half = s.fetch_half;
        }
      }
      ST(user_bytes) += want;
      log_rec(c, GFS_LOG_DELIVERIES, s.tb, fid, page, 0);
      ST(install_ns) += (long long)(globaltimer() - t_in);
    }
    g_pos += want;
    __syncthreads();
  }
}

// ------------------------------------------------------------ TB lifecycle
// Shared by the persistent driver (gread_driver) and user kernels (gfs_device.cuh).

// CTA start: counters, the K1 stage-ring barriers and this launch's RPC ring base.
template <int BS>
__device__ void cta_begin(const DevCtx& c, Smem& s) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < GFS_NSTATS; i++) s.st[i] = 0;
    s.pull_n = 0;
    s.span_half = s.fetch_half = s.pull_half = s.src_half = 0;
    s.hp[0].pending = s.hp[1].pending = 0;
    s.hp_age = 0;
    s.dbg_land_off[0] = s.dbg_land_off[1] = -1;
    s.direct[0] = s.direct[1] = 0;
    s.dbg_land_n[0] = s.dbg_land_n[1] = 0;
    s.st_seq[0] = s.st_seq[1] = 0;
    s.st_n[0] = s.st_n[1] = 0;
    s.st_landed[0] = s.st_landed[1] = 0;
    s.tma_seq = 0;
    s.fresh_done = 0;
    s.tma_epend = 0;
    s.tma_epar = 0;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s.sm_rank = smid < (uint32_t)GFS_MAX_SMS ? (int)atomicAdd(&c.g->sm_ctas[smid], 1u) : 0;
    s.first_ticket = 1;
    if (c.tma) {
      for (int i = 0; i < TMA_NST_MAX; i++) {
        mbar_init(&s.tma_bar[i], 1);
        mbar_init(&s.tma_empty[i], BS / 32 - 1);  // the checker warps
      }
      mbar_init(&s.poll_bar, 1);
      s.poll_par = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ring base for this launch: the daemon's completed-request count
    if (atomicCAS(&c.g->base_state, 0, 1) == 0) {
      c.g->req_base = ld_acquire_sys64(c.host_served);
      __threadfence();
      atomicExch(&c.g->base_state, 2);
    } else {
      while (*(volatile int*)&c.g->base_state != 2) __nanosleep(64);
      __threadfence();
    }
  }
  __syncthreads();
}

// Dispatcher (gpu_exec.py:242-265): the next TB id in activation order, or -1 when every
// TB has been handed out (or the run failed).
//
// Which CTA takes which ticket is free (per-TB observables are schedule-invariant), and it
// matters when there are fewer TBs than resident CTAs: 64 TBs taken by whichever CTAs come
// first put two or three of them on one SM, where they share its load/TMA issue and run
// ~30 % slower than the rest, and the pass waits for them (C3 64 TBs x 4 KiB: most TBs done
// at 45 ms, the SM-sharing ones at 56-62 ms).  So a CTA that is the r-th to start on its
// SM takes its first ticket only once r x (SMs in use) tickets are gone — the first wave is
// one TB per SM, then two, ... — or after 50 us, whichever comes first.
__device__ int next_tb(const DevCtx& c, Smem& s) {
  if (threadIdx.x == 0 && s.first_ticket) {
    s.first_ticket = 0;
    if (c.spread && s.sm_rank > 0) {
      const int used = c.n_sms < c.n_ctas ? c.n_sms : c.n_ctas;
      const unsigned long long want = (unsigned long long)s.sm_rank * (unsigned long long)used;
      const uint64_t t0 = globaltimer();
      for (;;) {
        const unsigned long long k = ld_volatile_u64(&c.g->next_tb);
        if (k >= want || k >= (unsigned long long)c.n_tb || has_error(c) || globaltimer() - t0 > 50000) break;
        __nanosleep(256);
      }
    }
  }
  if (threadIdx.x == 0) s.k = has_error(c) ? (int64_t)c.n_tb : (int64_t)atomicAdd(&c.g->next_tb, 1ull);
  __syncthreads();
  const int64_t k = s.k;
  __syncthreads();
  return k < c.n_tb ? c.order[k] : -1;
}

// TB start: an empty private buffer, own-frame queue and readahead stream.
__device__ void tb_begin(const DevCtx& c, Smem& s, int tb) {
  if (threadIdx.x == 0) {
    s.tb = tb;
    s.own_head = 0;
    s.own_len = 0;
    s.pb_count = 0;
    s.pb_filled = 0;
    s.pb_fid = -1;
    s.pb_last_nb = 0;
    s.page_size_cached = c.page_size;
    s.pb_base = 0;
    s.ra_win = 0;
    s.ra_next_fid = -1;
    s.ra_next_page = -1;
    s.pb_off_adj = 0;
    od_reset(s, -1);
    s.last_gfifo_pos = -1;
    s.la_fid = -1;
    s.la_lo = s.la_hi = 0;
    s.seg_lo = 0;
    s.seg_hi = 0;
    s.seg_ord = 0;
    s.rpc_out = 0;
    s.early.on = 0;
    s.early.polled = 0;
  }
  __syncthreads();
}

// TB done (on_tb_done ≙ gclose, gpu_exec.py:281-291): drain the private buffer, retire
// the own frames into a reclaim pool (their pages stay hittable).
template <int BS>
__device__ void tb_end(const DevCtx& c, Smem& s) {
  const int tid = threadIdx.x;
  __shared__ unsigned long long ret_pos;
  if (tid == 0) {
    if (!early_collect(c, s)) set_error(c, ERR_IO, -1, 0);
    if (od_drain_all(c, s) < 0) set_error(c, ERR_IO, -1, 0);
    ST(pb_discarded_bytes) += s.pb_filled;
    s.pb_filled = 0;
    s.pb_count = 0;
    if (c.policy == GFS_POLICY_PER_TB_LRA && s.own_len > 0)
      ret_pos = atomicAdd(rp_tail(c, (int)(blockIdx.x % (unsigned)c.ret_npools)), (unsigned long long)s.own_len);
  }
  __syncthreads();
  if (c.policy == GFS_POLICY_PER_TB_LRA && s.own_len > 0) {
    const int pool = (int)(blockIdx.x % (unsigned)c.ret_npools);
    for (int64_t i = tid; i < s.own_len; i += BS) {
      uint32_t f = c.own_q[(int64_t)blockIdx.x * c.quota + (s.own_head + i) % c.quota];
      st_release_gpu(rp_entry(c, pool, ret_pos + i), f + 1);
    }
  }
  __syncthreads();
}

// CTA end: word mismatches seen by the K1 checks, counters out.
__device__ void cta_end(const DevCtx& c, Smem& s, int bad_words) {
  const int tid = threadIdx.x;
  __shared__ int mism;
  if (tid == 0) mism = 0;
  __syncthreads();
  if (bad_words) atomicAdd(&mism, bad_words);
  __syncthreads();
  if (tid == 0) {
    s.st[GFS_STAT_word_mismatches] += mism;
    long long* out = c.stats + (int64_t)blockIdx.x * GFS_NSTATS;
    for (int i = 0; i < GFS_NSTATS; i++) out[i] = s.st[i];
    atomicAdd(&c.g->done_ctas, 1ull);
  }
}

}  // namespace gfs
