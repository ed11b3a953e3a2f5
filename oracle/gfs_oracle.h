/* gfs_oracle.h — CPU restatement of the reference gread path (TEST INFRASTRUCTURE ONLY).
 * See gfs_oracle.c for the reference file:line map.  Never linked by libgfs. */
#ifndef GFS_ORACLE_H
#define GFS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Counter names follow gpuiosim.metrics.Metrics (metrics.py:12-46) plus
 * storage_bytes (bytes pread from storage) and victims (victim log length). */
#define ORC_STAT_FIELDS(X)                                                                    \
  X(greads) X(user_bytes) X(cache_hit_user_bytes) X(tag_mismatches) X(pc_lookups) X(pc_hits) \
  X(pc_hit_pending) X(pc_misses) X(pc_allocs) X(pc_evictions) X(pc_remaps) X(pb_hits)        \
  X(pb_misses) X(pb_filled_bytes) X(pb_consumed_bytes) X(pb_discarded_bytes) X(rpc_count)    \
  X(rpc_requested_bytes) X(slot_collisions) X(preads) X(pread_bytes) X(storage_bytes)       \
  X(pcie_bytes) X(pcie_transfers) X(victims)

enum {
#define X(name) ORC_STAT_##name,
  ORC_STAT_FIELDS(X)
#undef X
  ORC_NSTATS
};

enum { ORC_POLICY_GLOBAL = 0, ORC_POLICY_PER_TB = 1 };
enum { ORC_RA_STATIC = 0, ORC_RA_DOUBLING = 1, ORC_RA_ONDEMAND = 2 };
enum { ORC_CLAMP_SEGMENT = 0, ORC_CLAMP_EOF = 1 };
enum { ORC_SRC_NONE = 0, ORC_SRC_SYNTH = 1, ORC_SRC_FILES = 2 };
enum { ORC_LOG_DELIVERIES = 0, ORC_LOG_RPCS = 1, ORC_LOG_VICTIMS = 2, ORC_LOG_WINDOWS = 3 };

typedef struct {
  int64_t page_size, cache_bytes, prefetch_bytes, request_bytes, staging_bytes, ra_max_bytes;
  int64_t ra_init_bytes; /* doubling first window (0 = page + prefetch) */
  int32_t policy, resident_limit, raw_mode, readahead, pcie_disabled, log;
  int32_t n_files, n_tb;
  int32_t ra_clamp, reserved; /* ondemand windows end at the TB's segment or at EOF */
  const int64_t* file_sizes;   /* n_files */
  const uint8_t* read_only;    /* n_files */
  const int64_t* prog_off;     /* n_tb + 1, index into segs (in segments) */
  const int64_t* segs;         /* 3 * n_segs: fid, offset, length */
  const int32_t* order;        /* dispatch order (n_tb) or NULL = round-robin */
  const int64_t* dst_off;      /* n_tb: user-buffer offset of each TB's program, or NULL */
  uint8_t* dst;                /* host user buffer or NULL */
  int64_t checksum_bytes;      /* bytes of dst to checksum after the run (0 = none) */
  int32_t source;              /* ORC_SRC_* */
  int32_t io_direct;           /* open files with O_DIRECT */
  const char* const* paths;    /* n_files, for ORC_SRC_FILES */
} orc_cfg;

typedef struct orc_run_s orc_run;

orc_run* orc_create(const orc_cfg* cfg);
int orc_execute(orc_run* r); /* 0 ok, -1 error (orc_error) */
const char* orc_error(const orc_run* r);
void orc_stats_copy(const orc_run* r, int64_t* out); /* ORC_NSTATS values */
int64_t orc_log_len(const orc_run* r, int kind);
void orc_log_copy(const orc_run* r, int kind, int64_t* out);
uint64_t orc_result_checksum(const orc_run* r);
void orc_destroy(orc_run* r);

int orc_nstats(void);
const char* orc_stat_name(int i);
uint64_t orc_mix64(uint64_t x);
uint64_t orc_page_tag(int64_t fid, int64_t page);
uint64_t orc_word(int64_t fid, int64_t i);
void orc_gen_bytes(int64_t fid, int64_t off, int64_t n, uint8_t* buf);
uint64_t orc_checksum(const uint8_t* buf, int64_t n, int64_t word_base);
int orc_gen_file_range(const char* path, int64_t content_id, int64_t size, int64_t offset, int64_t length);

#ifdef __cplusplus
}
#endif
#endif
