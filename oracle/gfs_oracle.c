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
 * Extension beyond the reference (documented in DESIGN.md): readahead mode 1
 * ("adaptive") doubles the RPC span on every sequential continuation up to
 * ra_max_bytes (the ondemand doubling law of host_os.py:124-128), clamped to
 * EOF and to the end of the TB's current segment.
 */
#define _GNU_SOURCE
#include <errno.h>
#include <fcntl.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
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
  vec_t windows;    /* (tb, span) per RPC in adaptive mode */
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
  /* adaptive readahead state */
  int64_t ra_win, ra_next_fid, ra_next_page;

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

/* prefetcher.py:13-25 (+ adaptive extension) */
static int64_t rpc_span(orc_run* r, int tb, int64_t fid, int64_t page, int64_t seg_end) {
  int64_t pg = r->cfg.page_size, fs = r->cfg.file_sizes[fid];
  int64_t off = page * pg;
  if (off >= fs) return 0;
  int ro = r->cfg.read_only[fid];
  int64_t pf = r->cfg.prefetch_bytes;
  int64_t want = (ro && pf > 0) ? pg + pf : pg;
  if (r->cfg.readahead == ORC_RA_ADAPTIVE && ro) {
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
  if (r->cfg.readahead == ORC_RA_ADAPTIVE && ro) {
    r->ra_next_fid = fid;
    r->ra_next_page = page + ceil_div(span, pg);
    int64_t rec[2] = {tb, span};
    vec_push(&r->windows, rec, 2);
  }
  (void)tb;
  return span;
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
  for (;;) {
    if (g_pos >= g_end || g_pos >= fs) return g_pos - offset;
    int64_t page = g_pos / pg;
    int64_t page_end = (page + 1) * pg < fs ? (page + 1) * pg : fs;
    int64_t want = (g_end < page_end ? g_end : page_end) - g_pos;
    int64_t in_page = g_pos - page * pg;
    uint8_t* d = dst ? dst + (g_pos - offset) : NULL;

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
    int64_t span = rpc_span(r, tb, fid, page, seg_end);
    log_rpc(r, tb, fid, page * pg, span);
    int64_t n = source_read(r, fid, page * pg, span);
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
  if (c->readahead == ORC_RA_ADAPTIVE && c->ra_max_bytes - c->page_size > pb_cap)
    pb_cap = c->ra_max_bytes - c->page_size;
  r->pb_cap_bytes = pb_cap;
  int64_t max_span = c->page_size + pb_cap;
  r->pb_nbytes = (int32_t*)calloc((size_t)(max_span / c->page_size + 2), sizeof(int32_t));
  if (!r->pb_nbytes) return fail(r, "out of host memory");
  if (materialized(r)) {
    r->staging_cap = max_span;
    if (c->raw_mode) r->staging_cap = c->request_bytes < (64 << 20) ? c->request_bytes : (64 << 20);
    r->staging_cap = (r->staging_cap + 4095) & ~(int64_t)4095;
    if (posix_memalign((void**)&r->staging, 4096, (size_t)r->staging_cap + 4096))
      return fail(r, "out of host memory");
    if (!c->raw_mode) {
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
    int64_t pos = c->dst_off ? c->dst_off[tb] : 0;
    for (int64_t s = c->prog_off[tb]; s < c->prog_off[tb + 1]; s++) { /* gpu_exec.py:95-105 */
      int64_t fid = c->segs[3 * s], base = c->segs[3 * s + 1], len = c->segs[3 * s + 2];
      if (fid < 0 || fid >= c->n_files) return fail(r, "segment names unknown file %lld", (long long)fid);
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
    /* on_tb_done: drain + retire (gpu_exec.py:281-286) */
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
  free(r->staging);
  if (r->fds) {
    for (int f = 0; f < r->cfg.n_files; f++)
      if (r->fds[f] >= 0) close(r->fds[f]);
    free(r->fds);
  }
  free(r);
}
