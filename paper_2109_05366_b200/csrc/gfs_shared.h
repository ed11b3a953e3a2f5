// gfs_shared.h — layouts shared by the host runtime (gfs_host.cpp) and the
// device kernels (gfs_kernels.cu).  Plain PODs; every pointer is either device
// memory or mapped pinned host memory (UVA), as noted.
#pragma once
#include <stdint.h>

#include "gfs.h"

namespace gfs {

constexpr uint32_t PT_EMPTY = 0xFFFFFFFFu;    // page-table entry: not cached
constexpr uint32_t PT_CLAIMED = 0xFFFFFFFEu;  // claimed by a TB, frame not bound yet
constexpr uint32_t PT_INFLIGHT = 0x80000000u; // frame bound, data not installed
constexpr uint32_t FR_VALID = 1u;             // frame state bit 0; refcount in bits 1..
constexpr uint32_t FR_REF = 2u;
constexpr uint32_t RING_TOMB = 0xFFFFFFFFu;   // global FIFO tombstone
constexpr int MAX_PB_ENTRIES = 16384;         // private-buffer entries per TB (smem bitmap)
constexpr int RET_POOLS = 32;                 // retired-frame FIFOs (per-tb-lra reclaim)
// Copy-engine windows of at least 2 pieces can land piece by piece, each piece followed
// by a "landed" marker: the CTA starts on the first piece while the rest copy.

// Request record in the mapped request ring (device writes, host daemon reads): three
// 64-bit words, each tagged in its low 16 bits with the entry's lap (ring position / ring
// size, mod 65535, + 1).  A 64-bit store from the GPU reaches host memory as one piece and
// an aligned 64-bit load on the host is atomic, so the daemon takes the entry once all three
// words show the lap it expects — the device needs no system-scope fence to publish a
// request (a membar.sys waits behind the link's read traffic: ~30 us per request under
// load; 16-byte stores are not seen whole by the host).
//   w0 = offset << 16 | lap                        (offsets < 2^48)
//   w1 = size << 32 | fid << 16 | lap              (size < 2^32, fid < 2^16)
//   w2 = tb << 32 | (slot | half << 15) << 16 | lap  (slot < 2^15)
struct alignas(32) RpcReq {
  unsigned long long w[4];  // w[3] unused
};
__host__ __device__ inline uint32_t ring_lap(unsigned long long pos, unsigned long long q) {
  return (uint32_t)((pos / q) % 65535ull) + 1u;
}

// Response mailbox per CTA slot (host writes, device polls).  One cache line
// each so concurrent workers never share a line.
struct alignas(64) RpcResp {
  int64_t nbytes;   // bytes read (EOF-clamped), < 0 = -errno
  uint32_t seq;     // request seq this answers (written last, release)
  int32_t buf;      // bounce mode: pool buffer holding the data
  uint32_t pad[12];
};

struct DevFile {
  uint32_t* pt;       // page table: npages entries (device)
  int64_t size;
  int64_t npages;
  int32_t read_only;
  int32_t content_id; // >= 0: synthetic law W(content_id, i); -1 = unverified
  const uint8_t* map; // mapped transfers: device pointer of the pinned file mapping
};

constexpr int GFS_MAX_SMS = 256;

// Global run state in device memory (zeroed per run).
struct DevGlobals {
  unsigned long long next_tb;      // dispatcher ticket
  unsigned long long fresh_next;   // never-used frames handed out in order
  unsigned long long ret_head, ret_tail;  // retired FIFO (per-tb-lra)
  unsigned long long g_head, g_tail;      // global FIFO (global-lru-dealloc)
  unsigned long long req_local;    // requests produced by this launch
  unsigned long long req_base;     // ring position of this launch's first request
  int base_state;                  // 0 = unset, 1 = being set, 2 = ready
  int pad0;
  unsigned long long log_n[5];     // log record counts
  unsigned long long recycled_n;   // released (EOF) frames stack depth
  int lock;                        // global policy structural lock
  int recycled_lock;
  int error;                       // first error code (GFS_E*), 0 = ok
  int error_info;
  unsigned long long error_arg;
  unsigned long long done_ctas;
  uint32_t sm_ctas[GFS_MAX_SMS];   // CTAs of this launch started on each SM (cta_begin)
  // first K1 word mismatch seen (diagnostics, GFS_DEBUG_MISMATCH): set, tb, fid, file
  // offset of the word, the word read, landing half, span offset, batch pages | cta << 32,
  // then the landing half's last pull (file offset, bytes), pb_base, pb_off_adj, pb_count,
  // batch first page, j0
  unsigned long long dbg[16];
};

enum { ERR_NONE = 0, ERR_ALL_INFLIGHT = 1, ERR_NO_FRAME = 2, ERR_IO = 3, ERR_TIMEOUT = 4,
       ERR_FIFO_OVERFLOW = 5, ERR_LOG_OVERFLOW = 6, ERR_BAD_PROGRAM = 7, ERR_PB = 8 };

struct DevCtx {
  // configuration
  int64_t page_size;
  int64_t prefetch_bytes;
  int64_t ra_max_bytes;
  int64_t ra_init_bytes;     // doubling first window (>= page + prefetch, <= ra_max)
  int64_t pb_cap_bytes;      // private-buffer capacity (bytes)
  int64_t slot_bytes;        // span buffer bytes per CTA slot
  int64_t staging_bytes;     // PCIe batch accounting unit
  int64_t request_bytes;
  int64_t nframes;
  int64_t quota;             // per-TB LRA queue cap
  int64_t gfifo_cap;
  int32_t policy, readahead, transfer, raw_mode, log, verify, pcie_disabled, timeline;
  int32_t tma;               // K1 by TMA bulk copies through the shared-memory stage ring
  int32_t lookahead;         // batches may run past a page-aligned request (gpu.lookahead)
  int32_t ra_clamp;          // ondemand windows end at EOF or at the TB's segment end
  int32_t landing_halves;    // landing slots per CTA (2 with ondemand readahead)
  int32_t stream_pieces;     // copy-engine windows land piece by piece (landed markers)
  int64_t stream_piece;      // piece bytes (windows of >= 2 pieces are streamed)
  unsigned long long* landed;  // [n_ctas * landing_halves]: (4 KiB pages landed << 32) | seq
  int32_t tma_off;           // byte offset of the stage ring in dynamic shared memory
  int32_t tma_nst;           // stages in the ring
  int32_t n_files, n_tb, n_ctas;
  int32_t n_sms;      // SMs of the device: first TBs go one per SM (next_tb)
  int32_t spread;     // 0 = plain ticket order (GFS_SPREAD=0, experiments)
  uint32_t ring_mask;
  uint64_t timeout_ns;
  // program (device)
  const int64_t* segs;
  const int64_t* prog_off;
  const int64_t* dst_off;
  const int32_t* order;
  uint8_t* dst;              // user buffer or nullptr
  // files (device)
  const DevFile* files;
  // page cache (device)
  uint8_t* frames;
  unsigned long long* fkey;  // (fid << 40) | page
  uint32_t* fstate;
  uint32_t* own_q;           // [n_ctas][quota]
  uint32_t* retired;         // [ret_npools][ret_pcap], value + 1, 0 = empty
  unsigned long long* rpool; // [RET_POOLS][16]: head at [16 p], tail at [16 p + 1] (own 128 B line)
  int64_t ret_pcap;          // entries per retired FIFO (>= frames: a frame is in at most one)
  int32_t ret_npools;        // min(RET_POOLS, n_ctas): CTA b retires into FIFO b % ret_npools
  uint32_t* gfifo;           // [gfifo_cap], value + 1, 0 = reserved-unwritten
  uint32_t* recycled;        // [nframes]
  DevGlobals* g;
  // RPC (mapped pinned host memory, device-usable pointers)
  RpcReq* ring;
  const uint32_t* ring_consumed;  // [ring_mask + 1]: seq the daemon last copied out of each entry
  // Requests completed by the daemon so far (mapped host memory).  Read once per launch
  // as the ring base: every earlier request is complete when a launch starts, so the
  // daemon's next expected position equals it — also under profiler kernel replay,
  // which restores device memory but not the daemon's progress.
  const unsigned long long* host_served;
  RpcResp* resp;
  uint8_t* staging;          // [n_ctas][landing_halves][slot_bytes] (zerocopy span buffers)
  // DMA mode (device)
  uint8_t* landing;          // [n_ctas][slot_bytes]
  unsigned long long* doorbell; // [n_ctas] (nbytes << 32 | seq), written by cuStreamWriteValue64
  // bounce mode (mapped pinned host memory): worker pool and per-buffer release words
  uint8_t* bounce;
  uint32_t* bounce_release;  // [n_bounce]: seq of the request whose data was pulled out
  int64_t bounce_bytes;
  // ring reuse guard (device)
  unsigned long long* done_pos;  // [ring_mask + 1]: last completed ring position + 1 per entry
  // the reference's RPC slot partition (rpc.n_slots): requests outstanding per slot tb % n
  uint32_t* slot_busy;
  int32_t ref_slots;
  uint32_t poll_first_ns, poll_ns;  // host-memory mailbox polling: first wait, then period
  int32_t k1_direct;         // pulled spans (mapped, small mapped_hybrid) are read by K1 straight
                             // from the pinned file mapping: no landing copy
  int32_t k1_early;          // static spans K1 reads from the mapping start before the answer (checked later)
  int64_t ce_min;            // mapped_hybrid / pread_hybrid: spans of at least this size go by copy engine
  // fused consumer (gfs_run_consume)
  gfs_consumer cons;
  // counters (device): [n_ctas][GFS_NSTATS]
  long long* stats;
  // logs (device): [cap][width]
  long long* logs[5];
  unsigned long long log_cap[5];
};

}  // namespace gfs
