/*
 * gfs_oracle.c — CPU restatement of the reference's sequential gread path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (libgfs.so) never
 * links or calls it.
 *
 * What it restates (reference = /root/reference/pkg/src/gpuiosim):
 *   - content oracle mix64/page_tag ............ simcore.py:68-73, 116-122
 *   - TB request loop (_next_request) .......... gpu_exec.py:95-105
 *   - gread entry + raw mode ................... gpu_exec.py:107-120, 131-138
 *   - short-read rule (_finish_gread) .......... gpu_exec.py:122-129
 *   - per-page walk (_page_step) ............... gpu_exec.py:142-199
 *   - RPC completion (_on_slot_ready) .......... gpu_exec.py:201-231
 *   - deliveries (_deliver) .................... gpu_exec.py:233-239
 *   - TB done: drain + retire (on_tb_done) ..... gpu_exec.py:281-291
 *   - page cache policies ...................... gpu_cache.py:32-212
 *   - request_span / PrivateBuffer ............. prefetcher.py:13-68
 *   - RPC accounting, page split, PCIe batches . rpc.py:31-55, 91-102, 201-220
 *   - pread EOF contract ....................... host_os.py:221-233
 *
 * Schedule: TBs run one at a time to completion in the given dispatch order
 * (the reference's behaviour at resident_limit == 1, tests/test_acceptance.py
 * tiny_oracle).  For sequential strided workloads with page-aligned strides
 * every per-TB observable (deliveries, RPC records, private-buffer counters,
 * misses, alloc/evict/remap COUNTS) is schedule-invariant, so this canonical
 * schedule is also the oracle for resident_limit > 1; victim identities are
 * compared only where the reference itself is order-invariant.
 *
 * Data: when a source is attached (real file paths, or the synthetic word
 * generator) the oracle also moves real bytes: staging -> frame / private
 * buffer -> user buffer, exactly like the device path, so user buffers and
 * checksums can be compared byte-for-byte.
 *
 * Readahead modes:
 *   0 static   — request_span, prefetcher.py:13-25 (the reference GPU prefetcher);
 *   1 doubling — the RPC span doubles on every sequential continuation up to
 *                ra_max_bytes, clamped to EOF and to the TB's segment end;
 *   2 ondemand — io.readahead=adaptive: HostOs._decide's Linux ondemand law
 *                (host_os.py:106-152, _resident_run :88-103) applied per TB stream to
 *                the gread requests, with the device's two landing halves: the
 *                synchronous span of a request's missing pages, asynchronous windows
 *                pending in the other half, adopted as the private buffer when the walk
 *                reaches them.  Pinned against the reference's own window_history
 *                (tests/golden/window_*.json, made by tests/golden/make_windows.py).
 */
#define _GNU_SOURCE
#include <errno.h>
#include <fcntl.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <unistd.h>

#include "gfs_oracle.h"

/* ------------------------------------------------------------------ content */

static inline uint64_t mix64(uint64_t x) { /* simcore.py:68-73 */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_mix64(uint64_t x) { return mix64(x); }

uint64_t orc_page_tag(int64_t fid, int64_t page) { /* simcore.py:116-122 */
  return mix64(((uint64_t)fid << 40) ^ (uint64_t)page ^ 0xA5A5A5A5A5A5A5A5ull);
}

/* Word i (8-byte index) of synthetic file fid: W(f,i) = mix64(page_tag(f, i>>9) ^ i). */
uint64_t orc_word(int64_t fid, int64_t i) {
  return mix64(orc_page_tag(fid, i >> 9) ^ (uint64_t)i);
}

/* Fill buf with bytes [off, off+n) of synthetic file fid (any alignment). */
void orc_gen_bytes(int64_t fid, int64_t off, int64_t n, uint8_t* buf) {
  int64_t pos = off, end = off + n;
  while (pos < end) {
    int64_t wi = pos >> 3;
    uint64_t w = orc_word(fid, wi);
    int64_t lo = pos - (wi << 3);
    int64_t take = 8 - lo;
    if (take > end - pos) take = end - pos;
    memcpy(buf + (pos - off), ((uint8_t*)&w) + lo, (size_t)take);
    pos += take;
  }
}

/* Write the synthetic words of [offset, offset+length) of a file of `size` bytes (created
 * or extended as needed): the reference arm's input, made without the product library. */
int orc_gen_file_range(const char* path, int64_t content_id, int64_t size, int64_t offset, int64_t length) {
  if (!path || size < 0 || offset < 0 || length < 0 || offset + length > size || (offset & 7)) return -1;
  int fd = open(path, O_CREAT | O_WRONLY, 0644);
  if (fd < 0) return -1;
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (sb.st_size != size && ftruncate(fd, (off_t)size) != 0)) {
    close(fd);
    return -1;
  }
  const int64_t chunk = 8 << 20;
  uint8_t* buf = (uint8_t*)malloc((size_t)chunk);
  int rc = buf ? 0 : -1;
  for (int64_t o = offset; rc == 0 && o < offset + length; o += chunk) {
    int64_t n = offset + length - o < chunk ? offset + length - o : chunk;
    orc_gen_bytes(content_id, o, n, buf);
    for (int64_t done = 0; done < n;) {
      ssize_t w = pwrite(fd, buf + done, (size_t)(n - done), (off_t)(o + done));
      if (w < 0 && errno == EINTR) continue;
      if (w <= 0) {
        rc = -1;
        break;
      }
      done += w;
    }
  }
  free(buf);
  if (close(fd) != 0) rc = -1;
  return rc;
}

/* Position-sensitive checksum of a byte buffer viewed as little-endian u64
 * words (zero padded): sum_i mix64(word_i ^ (i * golden)) mod 2^64. */
uint64_t orc_checksum(const uint8_t* buf, int64_t n, int64_t word_base) {
  uint64_t s = 0;
  int64_t nw = n >> 3;
  const uint64_t* w = (const uint64_t*)buf;
  for (int64_t i = 0; i < nw; i++)
    s += mix64(w[i] ^ ((uint64_t)(i + word_base) * 0x9E3779B97F4A7C15ull));
  if (n & 7) {
    uint64_t last = 0;
    memcpy(&last, buf + (nw << 3), (size_t)(n & 7));
    s += mix64(last ^ ((uint64_t)(nw + word_base) * 0x9E3779B97F4A7C15ull));
  }
  return s;
}

/* -------------------------------------------------------------- utilities */

static const char* const STAT_NAMES[ORC_NSTATS] = {
#define X(name) #name,
    ORC_STAT_FIELDS(X)
#undef X
};

const char* orc_stat_name(int i) { return (i >= 0 && i < ORC_NSTATS) ? STAT_NAMES[i] : NULL; }
int orc_nstats(void) { return ORC_NSTATS; }

typedef struct {
  int64_t* v;
  int64_t n, cap; /* in int64 elements */
} vec_t;

static int vec_push(vec_t* a, const int64_t* rec, int width) {
  if (a->n + width > a->cap) {
    int64_t ncap = a->cap ? a->cap * 2 : 1024;
    while (ncap < a->n + width) ncap *= 2;
    int64_t* nv = (int64_t*)realloc(a->v, (size_t)ncap * sizeof(int64_t));
    if (!nv) return -1;
    a->v = nv;
    a->cap = ncap;
  }
  memcpy(a->v + a->n, rec, (size_t)width * sizeof(int64_t));
  a->n += width;
  return 0;
}

/* frame states */
enum { F_FREE = 0, F_INFLIGHT = 1, F_VALID = 2 };
enum { OD_MARKS = 4 }; /* readahead markers remembered per TB stream (the device's bound) */

typedef struct {
  int64_t fid, page;
  int32_t state;
  int32_t nbytes;
  int64_t alloc_seq;
  int32_t owner;
} frame_t;

struct orc_run_s {
  orc_cfg cfg;
  char err[256];
  int64_t stats[ORC_NSTATS];
  vec_t deliveries; /* (tb, fid, page) */
  vec_t rpcs;       /* (tb, fid, offset, size) */
  vec_t victims;    /* (tb, fid, page) */
  vec_t windows;    /* (tb, span) per RPC in doubling mode; (tb, window bytes) per ondemand decision */
  uint64_t checksum;

  /* page cache */
  int64_t nframes, quota, next_fresh, alloc_seq;
  frame_t* frames;
  int32_t** pt; /* per file: page -> frame index or -1 */
  int64_t* free_stack;
  int64_t free_top, free_frames;
  /* global FIFO (allocation order), ring of frame indices; -1 = tombstone */
  int64_t* gfifo;
  int64_t g_head, g_tail, g_cap;
  /* per-tb-lra: own queue of the running TB, retired FIFO */
  int64_t* own;
  int64_t own_head, own_len;
  int64_t* retired;
  int64_t r_head, r_len;
  /* private buffer */
  int64_t pb_fid, pb_first, pb_count, pb_filled;
  int32_t* pb_nbytes; /* per entry, 0 = consumed/absent */
  int64_t pb_cap_bytes;
  /* doubling readahead state */
  int64_t ra_win, ra_next_fid, ra_next_page;
  /* ondemand readahead: the TB's stream (host_os.py ReadaheadState + markers) */
  int64_t od_fid, od_ws, od_wsize, od_async, od_prev_end;
  int64_t od_mark[OD_MARKS];
  long long od_dec_key;
  int64_t od_run_page, od_run_n;
  /* the current gread and segment */
  int64_t g_lo, g_hi, seg_lo, seg_hi;
  long long seg_ord;
  /* the two landing halves: a pending window (requested, not adopted) and its bytes */
  struct {
    int pending;
    int64_t fid, page, span, n;
    uint32_t age;
  } hp[2];
  uint32_t hp_age;
  int span_half;
  uint8_t* half_mem[2];
  int64_t staging_pages; /* a landing half / span buffer, in pages (ondemand sync span cap) */

  /* data plane */
  uint8_t* frame_mem;
  uint8_t* pb_mem;
  uint8_t* staging;
  int64_t staging_cap;
  int* fds;
};

static int fail(orc_run* r, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(r->err, sizeof r->err, fmt, ap);
  va_end(ap);
  return -1;
}

#define S(name) r->stats[ORC_STAT_##name]

static int materialized(const orc_run* r) { return r->cfg.source != ORC_SRC_NONE; }

/* ---------------------------------------------------------- source reads */

/* pread the span into staging; returns bytes (EOF-clamped, host_os.py:221-233). */
static int64_t source_read(orc_run* r, int64_t fid, int64_t off, int64_t size) {
  int64_t fsize = r->cfg.file_sizes[fid];
  if (off >= fsize || size <= 0) return 0;
  int64_t n = size < fsize - off ? size : fsize - off;
  if (!materialized(r)) return n;
  if (r->cfg.source == ORC_SRC_SYNTH) {
    orc_gen_bytes(fid, off, n, r->staging);
    return n;
  }
  /* real file: O_DIRECT needs 4 KiB aligned length; EOF clamps the count */
  int64_t want = r->cfg.io_direct ? ((n + 4095) & ~(int64_t)4095) : n;
  int64_t got = 0;
  while (got < n) {
    ssize_t k = pread(r->fds[fid], r->staging + got, (size_t)(want - got), (off_t)(off + got));
    if (k < 0) {
      if (errno == EINTR) continue;
      return -1;
    }
    if (k == 0) break;
    got += k;
  }
  return got < n ? got : n;
}

/* ------------------------------------------------------------ page cache */

static void pt_set(orc_run* r, int64_t fid, int64_t page, int64_t frame) {
  r->pt[fid][page] = (int32_t)frame;
}

static void unmap_victim(orc_run* r, int tb, int64_t v) {
  frame_t* f = &r->frames[v];
  pt_set(r, f->fid, f->page, -1);
  int64_t rec[3] = {tb, f->fid, f->page};
  vec_push(&r->victims, rec, 3);
  f->state = F_FREE;
}

static int64_t take_free(orc_run* r) {
  r->free_frames--;
  if (r->free_top > 0) return r->free_stack[--r->free_top];
  return r->next_fresh++;
}

/* gpu_cache.py:126-147 */
static int64_t alloc_global(orc_run* r, int tb) {
  if (r->free_frames > 0) {
    S(pc_allocs)++;
    return take_free(r);
  }
  /* first valid frame in allocation order; in-flight frames are skipped */
  int64_t victim = -1, vpos = -1;
  for (int64_t p = r->g_head; p < r->g_tail; p++) {
    int64_t fi = r->gfifo[p % r->g_cap];
    if (fi >= 0 && r->frames[fi].state == F_VALID) {
      victim = fi;
      vpos = p;
      break;
    }
  }
  if (victim < 0) return fail(r, "global-lru-dealloc: every frame is in flight"), -1;
  r->gfifo[vpos % r->g_cap] = -1;
  while (r->g_head < r->g_tail && r->gfifo[r->g_head % r->g_cap] < 0) r->g_head++;
  unmap_victim(r, tb, victim);
  S(pc_evictions)++;
  S(pc_allocs)++;
  return victim;
}

/* gpu_cache.py:149-179 */
static int64_t alloc_per_tb(orc_run* r, int tb) {
  if (r->own_len < r->quota) {
    if (r->free_frames > 0) {
      int64_t fi = take_free(r);
      r->own[(r->own_head + r->own_len++) % r->quota] = fi;
      S(pc_allocs)++;
      return fi;
    }
    if (r->r_len > 0) {
      int64_t v = r->retired[r->r_head % r->nframes];
      r->r_head++;
      r->r_len--;
      if (r->frames[v].state != F_VALID) return fail(r, "retired frame in flight"), -1;
      unmap_victim(r, tb, v);
      S(pc_remaps)++;
      r->own[(r->own_head + r->own_len++) % r->quota] = v;
      return v;
    }
  }
  if (r->own_len == 0)
    return fail(r, "per-tb-lra: tb %d has no frames to recycle and none are free", tb), -1;
  int64_t v = r->own[r->own_head % r->quota];
  r->own_head++;
  if (r->frames[v].state != F_VALID) return fail(r, "per-tb victim in flight"), -1;
  unmap_victim(r, tb, v);
  S(pc_remaps)++;
  r->own[(r->own_head + r->own_len - 1) % r->quota] = v; /* re-append at tail */
  return v;
}

/* gpu_cache.py:104-124 */
static int64_t cache_allocate(orc_run* r, int tb, int64_t fid, int64_t page) {
  int64_t fi = r->cfg.policy == ORC_POLICY_GLOBAL ? alloc_global(r, tb) : alloc_per_tb(r, tb);
  if (fi < 0) return -1;
  frame_t* f = &r->frames[fi];
  f->fid = fid;
  f->page = page;
  f->state = F_INFLIGHT;
  f->owner = tb;
  f->alloc_seq = r->alloc_seq++;
  pt_set(r, fid, page, fi);
  if (r->cfg.policy == ORC_POLICY_GLOBAL) r->gfifo[(r->g_tail++) % r->g_cap] = fi;
  return fi;
}

/* gpu_cache.py:191-206 (zero-byte RPC result past EOF) */
static void cache_release(orc_run* r, int64_t fi) {
  frame_t* f = &r->frames[fi];
  pt_set(r, f->fid, f->page, -1);
  if (r->cfg.policy == ORC_POLICY_GLOBAL) {
    for (int64_t p = r->g_tail - 1; p >= r->g_head; p--)
      if (r->gfifo[p % r->g_cap] == fi) {
        r->gfifo[p % r->g_cap] = -1;
        break;
      }
    while (r->g_tail > r->g_head && r->gfifo[(r->g_tail - 1) % r->g_cap] < 0) r->g_tail--;
  } else {
    r->own_len--; /* released frame is the newest own frame */
  }
  r->free_stack[r->free_top++] = fi;
  r->free_frames++;
  f->state = F_FREE;
}

/* gpu_cache.py:208-212 */
static void retire_tb(orc_run* r) {
  for (int64_t i = 0; i < r->own_len; i++) {
    r->retired[(r->r_head + r->r_len) % r->nframes] = r->own[(r->own_head + i) % r->quota];
    r->r_len++;
  }
  r->own_head = 0;
  r->own_len = 0;
}

/* -------------------------------------------------------- private buffer */

static int64_t page_bytes(const orc_run* r, int64_t fid, int64_t page) {
  int64_t pg = r->cfg.page_size, fs = r->cfg.file_sizes[fid];
  int64_t b = fs - page * pg;
  return b < pg ? b : pg;
}

static void pb_discard_all(orc_run* r) { /* prefetcher.py:40-43, 63-68 */
  for (int64_t i = 0; i < r->pb_count; i++) S(pb_discarded_bytes) += r->pb_nbytes[i];
  r->pb_count = 0;
  r->pb_filled = 0;
}

/* prefetcher.py:38-50: pages are [first, first+n) of fid, staged after page 0.
 * Entries that do not fit the capacity are dropped (counted as discarded). */
static void pb_fill(orc_run* r, int64_t fid, int64_t first, int64_t n, int64_t nbytes_total) {
  pb_discard_all(r);
  r->pb_fid = fid;
  r->pb_first = first;
  int64_t remaining = nbytes_total;
  for (int64_t i = 0; i < n; i++) {
    int64_t nb = page_bytes(r, fid, first + i);
    if (nb > remaining) nb = remaining;
    remaining -= nb;
    r->pb_nbytes[i] = 0;
    if (r->pb_filled + nb > r->pb_cap_bytes) {
      S(pb_discarded_bytes) += nb; /* no room, never served */
      continue;
    }
    r->pb_nbytes[i] = (int32_t)nb;
    r->pb_filled += nb;
    S(pb_filled_bytes) += nb;
  }
  r->pb_count = n;
}

/* prefetcher.py:52-61; returns nbytes or 0 on miss */
static int64_t pb_take(orc_run* r, int64_t fid, int64_t page) {
  int64_t i = page - r->pb_first;
  if (r->pb_count > 0 && fid == r->pb_fid && i >= 0 && i < r->pb_count && r->pb_nbytes[i] > 0) {
    int64_t nb = r->pb_nbytes[i];
    r->pb_nbytes[i] = 0;
    r->pb_filled -= nb;
    S(pb_hits)++;
    S(pb_consumed_bytes) += nb;
    return nb;
  }
  S(pb_misses)++;
  return 0;
}

/* -------------------------------------------------------------- RPC path */

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* rpc.py:201-220: pcie batches of <= staging_bytes (greedy packing with
 * splitting makes the batch count ceil(nbytes / staging_bytes)). */
static void account_transfer(orc_run* r, int64_t nbytes) {
  S(preads)++;
  S(pread_bytes) += nbytes;
  S(storage_bytes) += nbytes;
  if (!r->cfg.pcie_disabled && nbytes > 0) {
    S(pcie_bytes) += nbytes;
    S(pcie_transfers) += ceil_div(nbytes, r->cfg.staging_bytes);
  }
}

static void log_rpc(orc_run* r, int tb, int64_t fid, int64_t off, int64_t size) {
  int64_t rec[4] = {tb, fid, off, size};
  vec_push(&r->rpcs, rec, 4);
  S(rpc_count)++;
  S(rpc_requested_bytes) += size;
}

/* prefetcher.py:13-25 (+ doubling extension) */
static int64_t rpc_span(orc_run* r, int tb, int64_t fid, int64_t page, int64_t seg_end) {
  int64_t pg = r->cfg.page_size, fs = r->cfg.file_sizes[fid];
  int64_t off = page * pg;
  if (off >= fs) return 0;
  int ro = r->cfg.read_only[fid];
  int64_t pf = r->cfg.prefetch_bytes;
  int64_t want = (ro && pf > 0) ? pg + pf : pg;
  if (r->cfg.readahead == ORC_RA_DOUBLING && ro) {
    int64_t base = pg + pf;
    int64_t init = r->cfg.ra_init_bytes < r->cfg.ra_max_bytes ? r->cfg.ra_init_bytes : r->cfg.ra_max_bytes;
    if (init > base) base = init; /* io.ra_init_bytes: a larger first window */
    if (r->ra_win > 0 && fid == r->ra_next_fid && page == r->ra_next_page) {
      r->ra_win = 2 * r->ra_win;
      if (r->ra_win > r->cfg.ra_max_bytes) r->ra_win = r->cfg.ra_max_bytes;
    } else {
      r->ra_win = base;
    }
    want = r->ra_win;
    int64_t seg_lim = ceil_div(seg_end, pg) * pg - off; /* stay inside the TB's segment */
    if (want > seg_lim) want = seg_lim;
    if (want < pg) want = pg;
  }
  int64_t span = want < fs - off ? want : fs - off;
  if (r->cfg.readahead == ORC_RA_DOUBLING && ro) {
    r->ra_next_fid = fid;
    r->ra_next_page = page + ceil_div(span, pg);
    int64_t rec[2] = {tb, span};
    vec_push(&r->windows, rec, 2);
  }
  (void)tb;
  return span;
}

/* ------------------------------------------------------- ondemand readahead */

static int64_t od_pages(const orc_run* r, int64_t bytes) { return ceil_div(bytes, r->cfg.page_size); }

static int od_pb_has(const orc_run* r, int64_t fid, int64_t page) {
  int64_t i = page - r->pb_first;
  return r->pb_count > 0 && fid == r->pb_fid && i >= 0 && i < r->pb_count && r->pb_nbytes[i] > 0;
}

static int od_in_pending(const orc_run* r, int64_t fid, int64_t p) {
  for (int h = 0; h < 2; h++)
    if (r->hp[h].pending && r->hp[h].fid == fid && p >= r->hp[h].page &&
        p < r->hp[h].page + od_pages(r, r->hp[h].span))
      return h;
  return -1;
}

/* host_os.py:91-92 + in-flight pages: cached, in the private buffer or in a pending
 * window; page `ex` (the miss being decided, just allocated) is not fetched yet. */
static int od_resident(const orc_run* r, int64_t fid, int64_t p, int64_t ex) {
  if (p < 0 || p >= od_pages(r, r->cfg.file_sizes[fid])) return 0;
  /* segment clamp: the stream sees only its own segment */
  if (r->cfg.ra_clamp == ORC_CLAMP_SEGMENT && (p < r->seg_lo / r->cfg.page_size || p >= od_pages(r, r->seg_hi)))
    return 0;
  if (od_pb_has(r, fid, p) || od_in_pending(r, fid, p) >= 0) return 1;
  if (p == ex) return 0;
  return r->pt[fid][p] >= 0;
}

static int64_t od_limit(const orc_run* r, int64_t fid) {
  int64_t lim = od_pages(r, r->cfg.file_sizes[fid]);
  if (r->cfg.ra_clamp == ORC_CLAMP_SEGMENT && od_pages(r, r->seg_hi) < lim) lim = od_pages(r, r->seg_hi);
  return lim;
}

/* The current gread as pages [*gs, *ge) and its instance key (segment ordinal, index). */
static long long od_request(const orc_run* r, int64_t fid, int64_t* gs, int64_t* ge) {
  int64_t hi = r->g_hi < r->cfg.file_sizes[fid] ? r->g_hi : r->cfg.file_sizes[fid];
  *gs = r->g_lo / r->cfg.page_size;
  *ge = od_pages(r, hi);
  return (r->seg_ord << 32) | (long long)((r->g_lo - r->seg_lo) / r->cfg.request_bytes);
}

static void od_add_mark(orc_run* r, int64_t page) {
  for (int i = 0; i < OD_MARKS; i++)
    if (r->od_mark[i] < 0) {
      r->od_mark[i] = page;
      return;
    }
  for (int i = 0; i + 1 < OD_MARKS; i++) r->od_mark[i] = r->od_mark[i + 1]; /* drop the oldest */
  r->od_mark[OD_MARKS - 1] = page;
}

static void od_reset(orc_run* r, int64_t fid) {
  r->od_fid = fid;
  r->od_ws = r->od_wsize = r->od_async = 0;
  r->od_prev_end = -1;
  for (int i = 0; i < OD_MARKS; i++) r->od_mark[i] = -1;
  r->od_dec_key = -1;
  r->od_run_n = 0;
}

static int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }

/* host_os.py:106-152 (HostOs._decide) for the request [gs, ge); _resident_run :88-103.
 * Returns the window bytes window_history records (0 = none); the asynchronous run goes
 * to od_run_page / od_run_n. */
static int64_t od_decide(orc_run* r, int64_t fid, int64_t gs, int64_t ge, int64_t ex) {
  const int64_t pg = r->cfg.page_size, ra_max = r->cfg.ra_max_bytes / pg;
  const int64_t lim = od_limit(r, fid), npages = ge - gs, req_end = ge;
  r->od_run_n = 0;
  int64_t marker = -1;
  for (int i = 0; i < OD_MARKS; i++) {
    int64_t m = r->od_mark[i];
    if (m >= gs && m < ge) {
      r->od_mark[i] = -1; /* each marker triggers at most once */
      if (marker < 0 || m < marker) marker = m;
    }
  }
  if (marker >= 0) {
    int64_t ns, nz;
    if (r->od_wsize > 0 && marker == r->od_ws + r->od_wsize - r->od_async) {
      ns = i64max(r->od_ws + r->od_wsize, req_end);
      nz = i64min(2 * r->od_wsize, ra_max);
    } else { /* context recovery: the resident run around the marker */
      int64_t a = marker, e = marker + 1, np = od_pages(r, r->cfg.file_sizes[fid]);
      while (marker - a < ra_max && a > 0 && od_resident(r, fid, a - 1, ex)) a--;
      while (e - marker <= ra_max && e < np && od_resident(r, fid, e, ex)) e++;
      ns = i64max(e, req_end);
      nz = i64min(2 * i64max(e - a, 1), ra_max);
    }
    nz = i64min(nz, i64max(lim - ns, 0));
    r->od_prev_end = req_end;
    if (nz == 0) {
      r->od_ws = gs;
      r->od_wsize = r->od_async = 0;
      return 0;
    }
    r->od_ws = ns;
    r->od_wsize = r->od_async = nz;
    r->od_run_page = ns;
    r->od_run_n = nz;
    od_add_mark(r, ns);
    return nz * pg;
  }
  int seq = gs == 0 || gs == r->od_prev_end || (gs > 0 && od_resident(r, fid, gs - 1, ex));
  r->od_prev_end = req_end;
  if (!seq) {
    r->od_ws = gs;
    r->od_wsize = r->od_async = 0;
    return 0;
  }
  int64_t w = i64max(npages, i64min(4 * npages, ra_max));
  w = i64min(w, i64max(lim - gs, npages));
  r->od_ws = gs;
  r->od_wsize = w;
  r->od_async = w - npages;
  if (r->od_async <= 0) return w * pg;
  r->od_run_page = req_end;
  r->od_run_n = r->od_async;
  od_add_mark(r, req_end);
  return w * pg;
}

static void od_decide_once(orc_run* r, int tb, int64_t fid, int64_t ex, int64_t* ge_out) {
  int64_t gs, ge;
  long long key = od_request(r, fid, &gs, &ge);
  *ge_out = ge;
  if (key == r->od_dec_key) return;
  r->od_dec_key = key;
  int64_t w = od_decide(r, fid, gs, ge, ex);
  if (w > 0) {
    int64_t rec[2] = {tb, w};
    vec_push(&r->windows, rec, 2);
  }
}

/* A window the TB will not consume: dropped (its transfer was counted at request). */
static void od_drain(orc_run* r, int h) { r->hp[h].pending = 0; }

/* Landing half for a new span: one without a pending window, the half not holding the
 * private buffer first (taking the private buffer's half discards its entries), else the
 * older pending window is dropped.  `avoid`: the half of the span requested alongside. */
static int od_pick_half(orc_run* r, int avoid) {
  int a = r->span_half ^ 1, b = r->span_half, h = -1;
  if (a != avoid && !r->hp[a].pending) h = a;
  else if (b != avoid && !r->hp[b].pending) h = b;
  if (h < 0) {
    for (int k = 0; k < 2; k++)
      if (k != avoid && (h < 0 || r->hp[k].age < r->hp[h].age)) h = k;
    od_drain(r, h);
  }
  if (h == r->span_half && r->pb_count > 0) pb_discard_all(r);
  return h;
}

/* Request `span` bytes at `page` (rpc.py:82-102): the RPC record, the read, the transfer. */
static int64_t od_request_span(orc_run* r, int tb, int64_t fid, int64_t page, int64_t span, uint8_t* buf) {
  log_rpc(r, tb, fid, page * r->cfg.page_size, span);
  int64_t n = source_read(r, fid, page * r->cfg.page_size, span);
  if (n < 0) return fail(r, "pread failed: %s", strerror(errno)), -1;
  if (buf && materialized(r)) memcpy(buf, r->staging, (size_t)n);
  account_transfer(r, n);
  return n;
}

static int od_submit_run(orc_run* r, int tb, int64_t fid, int avoid) {
  if (r->od_run_n <= 0) return 0;
  const int64_t pg = r->cfg.page_size, fs = r->cfg.file_sizes[fid];
  int64_t span = r->od_run_n * pg;
  if (span > fs - r->od_run_page * pg) span = fs - r->od_run_page * pg;
  r->od_run_n = 0;
  if (span <= 0) return 0;
  int h = od_pick_half(r, avoid);
  int64_t n = od_request_span(r, tb, fid, r->od_run_page, span, r->half_mem[h]);
  if (n < 0) return -1;
  r->hp[h].pending = 1;
  r->hp[h].fid = fid;
  r->hp[h].page = r->od_run_page;
  r->hp[h].span = span;
  r->hp[h].n = n;
  r->hp[h].age = ++r->hp_age;
  return 0;
}

/* Walk position `page` (before its lookup): a marker there fires its request's decision; a
 * pending window holding the page becomes the private buffer (all its pages). */
static int od_top(orc_run* r, int tb, int64_t fid, int64_t page) {
  for (int i = 0; i < OD_MARKS; i++)
    if (r->od_mark[i] == page) {
      int64_t ge;
      od_decide_once(r, tb, fid, -1, &ge);
      if (od_submit_run(r, tb, fid, -1) < 0) return -1;
      break;
    }
  int h = od_in_pending(r, fid, page);
  if (h >= 0) {
    r->hp[h].pending = 0;
    r->span_half = h;
    int64_t n = r->hp[h].n;
    if (n > 0) {
      pb_fill(r, fid, r->hp[h].page, od_pages(r, n), n);
      if (r->pb_mem) memcpy(r->pb_mem, r->half_mem[h], (size_t)(n < r->pb_cap_bytes ? n : r->pb_cap_bytes));
    } else {
      pb_discard_all(r);
    }
  }
  return 0;
}

static void deliver(orc_run* r, int tb, int64_t fid, int64_t g_pos, int64_t want, int hit,
                    const uint8_t* src, uint8_t* dst) {
  S(user_bytes) += want;
  if (hit) S(cache_hit_user_bytes) += want;
  if (r->cfg.log) {
    int64_t rec[3] = {tb, fid, g_pos / r->cfg.page_size};
    vec_push(&r->deliveries, rec, 3);
  }
  if (dst && src) memcpy(dst, src, (size_t)want);
}

/* gpu_exec.py:107-239.  Returns delivered bytes or -1 on error.
 * dst points at the user-buffer position of byte `offset` (or NULL). */
static int64_t gread(orc_run* r, int tb, int64_t fid, int64_t offset, int64_t size, int64_t seg_end,
                     uint8_t* dst) {
  S(greads)++;
  int64_t pg = r->cfg.page_size;
  int64_t fs = r->cfg.file_sizes[fid];
  if (r->cfg.raw_mode) { /* gpu_exec.py:114-119, 131-138 */
    log_rpc(r, tb, fid, offset, size);
    int64_t n = 0, done = 0;
    /* raw request may exceed the staging buffer: read in staging-sized pieces */
    while (done < size) {
      int64_t piece = size - done;
      if (materialized(r) && piece > r->staging_cap) piece = r->staging_cap;
      int64_t k = source_read(r, fid, offset + done, piece);
      if (k < 0) return fail(r, "pread failed: %s", strerror(errno)), -1;
      if (dst && materialized(r)) memcpy(dst + done, r->staging, (size_t)k);
      n += k;
      done += piece;
      if (k < piece) break;
    }
    S(preads)++;
    S(pread_bytes) += n;
    S(storage_bytes) += n;
    if (!r->cfg.pcie_disabled && n > 0) {
      S(pcie_bytes) += n;
      S(pcie_transfers) += ceil_div(n, r->cfg.staging_bytes);
    }
    S(user_bytes) += n;
    return n;
  }
  int64_t g_pos = offset, g_end = offset + size;
  const int od = r->cfg.readahead == ORC_RA_ONDEMAND && r->cfg.read_only[fid];
  if (r->cfg.readahead == ORC_RA_ONDEMAND) {
    r->g_lo = offset;
    r->g_hi = offset + size;
    if (fid != r->od_fid) od_reset(r, fid); /* a new stream */
  }
  for (;;) {
    if (g_pos >= g_end || g_pos >= fs) return g_pos - offset;
    int64_t page = g_pos / pg;
    int64_t page_end = (page + 1) * pg < fs ? (page + 1) * pg : fs;
    int64_t want = (g_end < page_end ? g_end : page_end) - g_pos;
    int64_t in_page = g_pos - page * pg;
    uint8_t* d = dst ? dst + (g_pos - offset) : NULL;
    if (od && od_top(r, tb, fid, page) < 0) return -1;

    S(pc_lookups)++;
    int64_t fi = r->pt[fid][page];
    if (fi >= 0) {
      frame_t* f = &r->frames[fi];
      if (f->state != F_VALID) return fail(r, "in-flight frame under the sequential schedule"), -1;
      S(pc_hits)++;
      deliver(r, tb, fid, g_pos, want, 1, r->frame_mem ? r->frame_mem + fi * pg + in_page : NULL, d);
      g_pos += want;
      continue;
    }
    S(pc_misses)++;
    /* ondemand: the request's decision and its synchronous span are taken on the miss,
     * before the page's frame is allocated (allocation may evict pages the scan sees) */
    int64_t od_span = 0;
    if (od && !od_pb_has(r, fid, page)) {
      int64_t ge;
      od_decide_once(r, tb, fid, -1, &ge);
      int64_t lim = i64min(i64min(ge, page + r->staging_pages), od_pages(r, fs));
      int64_t q = page + 1;
      while (q < lim && !od_resident(r, fid, q, -1)) q++;
      od_span = i64min((q - page) * pg, fs - page * pg);
    }
    fi = cache_allocate(r, tb, fid, page);
    if (fi < 0) return -1;
    frame_t* f = &r->frames[fi];
    uint8_t* fmem = r->frame_mem ? r->frame_mem + fi * pg : NULL;
    int64_t nb = pb_take(r, fid, page);
    if (nb > 0) { /* gpu_exec.py:174-189 */
      if (fmem) memcpy(fmem, r->pb_mem + (page - r->pb_first) * pg, (size_t)nb);
      f->state = F_VALID;
      f->nbytes = (int32_t)nb;
      deliver(r, tb, fid, g_pos, want, 0, fmem ? fmem + in_page : NULL, d);
      g_pos += want;
      continue;
    }
    int64_t span, n;
    if (od) { /* the synchronous span planned above, then the decided async run */
      span = od_span;
      int hs = od_pick_half(r, -1);
      log_rpc(r, tb, fid, page * pg, span);
      if (od_submit_run(r, tb, fid, hs) < 0) return -1;
      r->span_half = hs;
    } else {
      int ph = 0;
      if (r->cfg.readahead == ORC_RA_ONDEMAND) r->span_half = ph = od_pick_half(r, -1); /* non-RO file */
      (void)ph;
      span = rpc_span(r, tb, fid, page, seg_end);
      log_rpc(r, tb, fid, page * pg, span);
    }
    n = source_read(r, fid, page * pg, span);
    if (n < 0) return fail(r, "pread failed: %s", strerror(errno)), -1;
    account_transfer(r, n);
    if (n == 0) { /* gpu_exec.py:207-211 */
      cache_release(r, fi);
      return g_pos - offset;
    }
    int64_t nb0 = n < pg ? n : pg;
    if (fmem) memcpy(fmem, r->staging, (size_t)nb0);
    f->state = F_VALID;
    f->nbytes = (int32_t)nb0;
    int64_t rest_pages = ceil_div(n, pg) - 1;
    if (rest_pages > 0) {
      pb_fill(r, fid, page + 1, rest_pages, n - nb0);
      if (r->pb_mem) {
        int64_t cp = n - nb0 < r->pb_cap_bytes ? n - nb0 : r->pb_cap_bytes;
        memcpy(r->pb_mem, r->staging + pg, (size_t)cp);
      }
    }
    int64_t pend = page * pg + nb0 < fs ? page * pg + nb0 : fs;
    want = (g_end < pend ? g_end : pend) - g_pos;
    deliver(r, tb, fid, g_pos, want, 0, fmem ? fmem + in_page : NULL, d);
    g_pos += want;
  }
}

/* ------------------------------------------------------------------- run */

static int setup(orc_run* r) {
  const orc_cfg* c = &r->cfg;
  if (c->page_size < 1 || c->request_bytes < 1 || c->staging_bytes < 1)
    return fail(r, "page_size, request_bytes and staging_bytes must be positive");
  if (c->prefetch_bytes % c->page_size) return fail(r, "prefetch_bytes must be a multiple of page_size");
  if (c->cache_bytes < c->page_size) return fail(r, "cache_bytes smaller than one page");
  if (c->resident_limit < 1) return fail(r, "resident_limit must be >= 1");
  r->nframes = c->cache_bytes / c->page_size;
  r->quota = r->nframes / c->resident_limit; /* gpu_cache.py:32-34 */
  if (c->policy == ORC_POLICY_PER_TB && r->quota < 1 && !c->raw_mode)
    return fail(r, "per-tb-lra needs cache_bytes/page_size >= resident TBs (%lld frames for %d TBs)",
                (long long)r->nframes, c->resident_limit);
  r->free_frames = r->nframes;
  if (!c->raw_mode) {
    r->frames = (frame_t*)calloc((size_t)r->nframes, sizeof(frame_t));
    r->free_stack = (int64_t*)malloc((size_t)r->nframes * sizeof(int64_t));
    r->g_cap = r->nframes + 1;
    r->gfifo = (int64_t*)malloc((size_t)r->g_cap * sizeof(int64_t));
    r->own = (int64_t*)malloc((size_t)(r->quota > 0 ? r->quota : 1) * sizeof(int64_t));
    r->retired = (int64_t*)malloc((size_t)r->nframes * sizeof(int64_t));
    r->pt = (int32_t**)calloc((size_t)c->n_files, sizeof(int32_t*));
    if (!r->frames || !r->free_stack || !r->gfifo || !r->own || !r->retired || !r->pt)
      return fail(r, "out of host memory");
    for (int f = 0; f < c->n_files; f++) {
      int64_t np = ceil_div(c->file_sizes[f], c->page_size) + 1;
      r->pt[f] = (int32_t*)malloc((size_t)np * sizeof(int32_t));
      if (!r->pt[f]) return fail(r, "out of host memory");
      memset(r->pt[f], 0xff, (size_t)np * sizeof(int32_t));
    }
  }
  int64_t pb_cap = c->prefetch_bytes;
  if (c->readahead == ORC_RA_DOUBLING && c->ra_max_bytes - c->page_size > pb_cap)
    pb_cap = c->ra_max_bytes - c->page_size;
  if (c->readahead == ORC_RA_ONDEMAND) { /* a landing half holds a whole window */
    if (c->ra_max_bytes < c->page_size || c->ra_max_bytes % c->page_size)
      return fail(r, "ra_max_bytes must be a positive multiple of page_size");
    pb_cap = i64max(c->ra_max_bytes, c->page_size + c->prefetch_bytes);
  }
  r->pb_cap_bytes = pb_cap;
  int64_t max_span = c->readahead == ORC_RA_ONDEMAND ? pb_cap : c->page_size + pb_cap;
  r->staging_pages = max_span / c->page_size;
  r->pb_nbytes = (int32_t*)calloc((size_t)(max_span / c->page_size + 2), sizeof(int32_t));
  if (!r->pb_nbytes) return fail(r, "out of host memory");
  if (materialized(r)) {
    r->staging_cap = max_span;
    if (c->raw_mode) r->staging_cap = c->request_bytes < (64 << 20) ? c->request_bytes : (64 << 20);
    r->staging_cap = (r->staging_cap + 4095) & ~(int64_t)4095;
    if (posix_memalign((void**)&r->staging, 4096, (size_t)r->staging_cap + 4096))
      return fail(r, "out of host memory");
    if (!c->raw_mode) {
      if (c->readahead == ORC_RA_ONDEMAND)
        for (int h = 0; h < 2; h++)
          if (!(r->half_mem[h] = (uint8_t*)malloc((size_t)max_span))) return fail(r, "out of host memory");
      r->frame_mem = (uint8_t*)malloc((size_t)(r->nframes * c->page_size));
      r->pb_mem = (uint8_t*)malloc((size_t)(pb_cap > 0 ? pb_cap : 1));
      if (!r->frame_mem || !r->pb_mem) return fail(r, "out of host memory for the frame pool");
    }
  }
  if (c->source == ORC_SRC_FILES) {
    r->fds = (int*)malloc((size_t)c->n_files * sizeof(int));
    for (int f = 0; f < c->n_files; f++) {
      r->fds[f] = open(c->paths[f], O_RDONLY | (c->io_direct ? O_DIRECT : 0));
      if (r->fds[f] < 0) return fail(r, "open %s: %s", c->paths[f], strerror(errno));
    }
  }
  return 0;
}

static int execute(orc_run* r) {
  const orc_cfg* c = &r->cfg;
  for (int k = 0; k < c->n_tb; k++) {
    int tb = c->order ? c->order[k] : k;
    if (tb < 0 || tb >= c->n_tb) return fail(r, "bad dispatch order entry %d", tb);
    /* TB start: fresh private buffer and readahead state */
    r->pb_count = 0;
    r->pb_filled = 0;
    r->ra_win = 0;
    r->ra_next_fid = -1;
    r->ra_next_page = -1;
    od_reset(r, -1);
    r->hp[0].pending = r->hp[1].pending = 0;
    r->span_half = 0;
    int64_t pos = c->dst_off ? c->dst_off[tb] : 0;
    for (int64_t s = c->prog_off[tb]; s < c->prog_off[tb + 1]; s++) { /* gpu_exec.py:95-105 */
      int64_t fid = c->segs[3 * s], base = c->segs[3 * s + 1], len = c->segs[3 * s + 2];
      if (fid < 0 || fid >= c->n_files) return fail(r, "segment names unknown file %lld", (long long)fid);
      r->seg_lo = base; /* requests of this segment start at base + k * request_bytes */
      r->seg_hi = base + len;
      r->seg_ord = s - c->prog_off[tb];
      int64_t seg_off = 0;
      while (seg_off < len) {
        int64_t size = c->request_bytes < len - seg_off ? c->request_bytes : len - seg_off;
        uint8_t* d = c->dst ? c->dst + pos + seg_off : NULL;
        int64_t got = gread(r, tb, fid, base + seg_off, size, base + len, d);
        if (got < 0) return -1;
        seg_off += got;
        if (got < size) break; /* short read: rest of the segment skipped (gpu_exec.py:124-126) */
      }
      pos += len;
    }
    /* on_tb_done: drain + retire (gpu_exec.py:281-286); windows never reached are dropped */
    od_drain(r, 0);
    od_drain(r, 1);
    pb_discard_all(r);
    if (!c->raw_mode && c->policy == ORC_POLICY_PER_TB) retire_tb(r);
  }
  if (c->dst && c->checksum_bytes > 0) r->checksum = orc_checksum(c->dst, c->checksum_bytes, 0);
  return 0;
}

orc_run* orc_create(const orc_cfg* cfg) {
  orc_run* r = (orc_run*)calloc(1, sizeof(orc_run));
  if (!r) return NULL;
  r->cfg = *cfg;
  return r;
}

int orc_execute(orc_run* r) {
  if (setup(r) != 0) return -1;
  return execute(r);
}

const char* orc_error(const orc_run* r) { return r->err; }
uint64_t orc_result_checksum(const orc_run* r) { return r->checksum; }

void orc_stats_copy(const orc_run* r, int64_t* out) {
  memcpy(out, r->stats, sizeof r->stats);
  out[ORC_STAT_victims] = r->victims.n / 3;
}

int64_t orc_log_len(const orc_run* r, int kind) {
  switch (kind) {
    case ORC_LOG_DELIVERIES: return r->deliveries.n / 3;
    case ORC_LOG_RPCS: return r->rpcs.n / 4;
    case ORC_LOG_VICTIMS: return r->victims.n / 3;
    case ORC_LOG_WINDOWS: return r->windows.n / 2;
  }
  return -1;
}

void orc_log_copy(const orc_run* r, int kind, int64_t* out) {
  const vec_t* v = kind == ORC_LOG_DELIVERIES ? &r->deliveries
                   : kind == ORC_LOG_RPCS     ? &r->rpcs
                   : kind == ORC_LOG_VICTIMS  ? &r->victims
                                              : &r->windows;
  memcpy(out, v->v, (size_t)v->n * sizeof(int64_t));
}

void orc_destroy(orc_run* r) {
  if (!r) return;
  free(r->deliveries.v);
  free(r->rpcs.v);
  free(r->victims.v);
  free(r->windows.v);
  free(r->frames);
  free(r->free_stack);
  free(r->gfifo);
  free(r->own);
  free(r->retired);
  if (r->pt) {
    for (int f = 0; f < r->cfg.n_files; f++) free(r->pt[f]);
    free(r->pt);
  }
  free(r->pb_nbytes);
  free(r->frame_mem);
  free(r->pb_mem);
  free(r->half_mem[0]);
  free(r->half_mem[1]);
  free(r->staging);
  if (r->fds) {
    for (int f = 0; f < r->cfg.n_files; f++)
      if (r->fds[f] >= 0) close(r->fds[f]);
    free(r->fds);
  }
  free(r);
}
