/*
 * tgs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the TideGS working-set
 * step (arXiv 2605.20150): Level-1 block culling (Eq.
 * Kt_def), Tide residency selection and differential streaming (PAPER.md:
 * 268-322, Alg. 1), eviction/write-back with dirty tracking (PAPER.md:238-251,
 * 290-293), optimizer-state placement and the masked Adam
 * update (Eq. masked_update).  Silent points follow the
 * readings listed in DESIGN.md §3 ("R1".."R22").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the
 * CUDA path (paper_2605_20150_b200/) and neither side includes the other.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions whose result is fixed
 * only by an invented reading say "parity unpinned" in DESIGN.md §4.
 */
#ifndef TGS_ORACLE_H
#define TGS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_EINVAL = 1, OR_ESTATE = 2, OR_ENONFINITE = 6 };
enum { OR_PERSIST = 0, OR_COLD_RESTART = 1 };

typedef struct {
  uint64_t n_gaussians;
  uint32_t dim;          /* 59 */
  uint32_t block_size;   /* B */
  uint32_t capacity;     /* C (per shard) */
  uint32_t pool_slots;   /* P >= C; 0 -> 2C */
  uint32_t max_cameras;
  uint32_t max_age;      /* A_max */
  uint32_t quota_num, quota_den; /* beta */
  double lambda, gamma;
  int32_t moments;       /* OR_PERSIST / OR_COLD_RESTART */
  int32_t tide;          /* 1 = differential, 0 = restage-all ablation */
  int32_t world_size, rank;
  int32_t refresh_bounds; /* NEXT f2 (R25): grow r_k after each update; needs track_all */
} or_config;

typedef struct {
  uint64_t iter, n_visible, n_resident, n_active_blocks, n_stage_in, n_evict, n_evict_dirty,
      n_active_rows, h2d_bytes, d2h_bytes, flush_bytes, n_flush_blocks, readmissions,
      cold_restart_updates, total_updates, resident_streak_sum, streak_count,
      k_inter_sum, k_union_sum;  /* sum over activates of |K_t n K_{t+1}|, |K_t u K_{t+1}| */
} or_stats;

typedef void (*or_fill_fn)(void* user, uint64_t k_global, float* out /* B*59 */);
typedef void (*or_grad_fn)(void* user, uint64_t k_global, uint64_t t, float* out /* B*59 */);
typedef void (*or_mask_fn)(void* user, uint64_t k_global, uint64_t t, uint32_t* words);

typedef struct or_ctx or_ctx;

/* bounds_global: K x 4 floats for ALL global blocks; the shard keeps k%G==rank */
int or_create(const or_config* cfg, const float* bounds_global, or_fill_fn fill, void* fill_user,
              int track_all, or_ctx** out);
void or_destroy(or_ctx* c);
/* data (theta, m, v, Adam values) are kept only for tracked blocks */
int or_track_block(or_ctx* c, uint64_t k_global);

int or_activate(or_ctx* c, const float* planes /* J x 6 x 4 */, uint32_t J);
int or_step_adam(or_ctx* c, const float* lr /* 59 */, float beta1, float beta2, float eps,
                 or_grad_fn grad, void* grad_user, or_mask_fn mask, void* mask_user);
int or_flush(or_ctx* c);

/* lists of the last activate, ascending global ids:
 * 0 K_{t+1}, 1 R_{t+1}, 2 S+, 3 S-, 4 Omega, 5 A = R n K; slots where defined */
uint32_t or_get_list(or_ctx* c, int which, uint32_t* blocks, int32_t* slots, uint32_t cap);
uint32_t or_get_percam(or_ctx* c, uint32_t j, uint32_t* blocks, uint32_t cap);
/* S- entries that were dirty (written back) in the last activate */
uint32_t or_get_evicted_dirty(or_ctx* c, uint32_t* blocks, uint32_t cap);
void or_get_slot_map(or_ctx* c, int64_t* slot_to_block /* P, global ids, -1 free */);
void or_get_stats(or_ctx* c, or_stats* s);
/* lowest (gid*59+attr) of a non-finite gradient in an active row, or UINT64_MAX */
uint64_t or_nonfinite_index(or_ctx* c);
/* newest version of a tracked block (resident slot, else host tier) */
int or_read_block(or_ctx* c, uint64_t k_global, float* theta, float* m, float* v);
uint32_t or_num_local_blocks(or_ctx* c);
uint32_t or_step_count(or_ctx* c, uint64_t k_global);

/* Level-2 fine filter (NEXT f1): I_t bits of a block of
 * A = R n K from its current slot theta and the last camera batch (R24).
 * words: ceil(B/32); blocks outside A give all-zero words. */
int or_fine_filter(or_ctx* c, uint64_t k_global, uint32_t* words);
/* the same as an or_mask_fn, user = the or_ctx itself */
void or_fine_filter_cb(void* ctx, uint64_t k_global, uint64_t t, uint32_t* words);
/* current bound (cx, cy, cz, r) of a global block of this shard */
int or_get_bound(or_ctx* c, uint64_t k_global, float* out4);
/* NEXT f2b (R26): Morton sort + blocking of n Gaussians given as (cx, cy, cz,
 * max log-scale) rows: perm[sorted position] = original index, bounds per
 * block of B consecutive sorted Gaussians (centroid, conservative radius). */
int or_build_layout(const float* cs, uint64_t n, uint32_t B, uint64_t* perm, float* bounds);
uint64_t or_morton3(uint32_t x, uint32_t y, uint32_t z);
/* the deterministic exp of R24 (exported for its pins) */
float or_exp_det(float x);

/* NEXT f3 -- the tier below the host (§3.4; readings R27,
 * R28 of DESIGN.md §3): an LRU CPU cache of cache_blocks (>= 2C) block records
 * with dirty bits over a log-structured store (immutable base segment +
 * append-only patch segments, Index[k] = (file_id, offset, size, version)).
 * Call after or_create, before the first activate.  dir != NULL: files are
 * written under dir (needs track_all); dir == NULL: metadata only (Index, LRU
 * and counters; no block may be tracked). */
int or_store_open(or_ctx* c, const char* dir, uint32_t cache_blocks, uint64_t segment_bytes);
/* R30 checkpoint/resume: a new session over the files of an earlier one
 * (after its barrier): Index recovered by scanning the segments (later
 * records win, a torn tail record dropped), empty cache; needs track_all. */
int or_store_reopen(or_ctx* c, const char* dir, uint32_t cache_blocks, uint64_t segment_bytes);
/* R31 compaction at a barrier (flush first; ESTATE otherwise): a new base
 * segment with every block's newest version replaces the old one, the patch
 * segments are removed, Index points into the base again (versions kept). */
int or_store_compact(or_ctx* c);
int or_store_index(or_ctx* c, uint64_t k_global, uint64_t* out4);
int or_store_stats(or_ctx* c, uint64_t* out10);
uint32_t or_store_lru(or_ctx* c, uint32_t* blocks, uint8_t* dirty, uint32_t cap);

/* NEXT f4 -- clustered-TSP view ordering (reading R29):
 * perm[M] = the order in which to present M views described by D <= 8
 * features each (feat: M x D doubles, e.g. camera centre and a point on the
 * optical axis); cluster (may be NULL) = k-means cluster of each view,
 * k_out = number of clusters, iters_out = Lloyd iterations. */
int or_order_views(const double* feat, uint32_t M, uint32_t D, uint32_t* perm,
                   uint32_t* cluster, uint32_t* k_out, uint32_t* iters_out);

/* cumulative wall time (ns) of the phases: [0] cull, [1] plan (selection, delta,
 * slots), [2] copies (write-back + gather of records), [3] Adam */
void or_phase_ns(or_ctx* o, uint64_t* out4);

/* timing aid (bench.py cpu_baseline only, never a parity check): track every
 * block from now on; resident untracked blocks take their initial rows */
int or_track_all_from_now(or_ctx* o);

/* CRC-32C of n bytes (the R28 format-2 record checksum), for the pins */
uint32_t or_crc32c(const void* data, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
