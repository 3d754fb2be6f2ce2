/*
 * tidegs.h -- C ABI of the B200-native TideGS working-set step.
 *
 * The library implements, for one shard of a block-virtualized Gaussian table,
 * the per-iteration working-set step of TideGS (arXiv 2605.20150):
 *
 *   a1  Level-1 block frustum culling of a camera batch        PAPER.md:196-208 (Eq. Kt_def)
 *   a2  differential delta  Omega = R_t n R_{t+1},
 *       S+ = R_{t+1} \ R_t,  S- = R_t \ R_{t+1}                 PAPER.md:280-288, Alg. 1 l.7-8
 *   a3  residency selection (score s(k), camera-balanced Top-C)
 *       and cache-slot allocation / eviction                   PAPER.md:268-278, Alg. 1 l.2-6
 *   a4  gather of S+ block records host tier -> slots and
 *       write-back of dirty S- records slots -> host tier
 *   a5  masked (sparse) Adam over the active rows              PAPER.md:717-727 (Eq. masked_update)
 *
 * Every silent or ambiguous point follows the readings R1..R22 of DESIGN.md §3
 * (the same ones the CPU oracle in oracle/ follows).  There is no CPU fallback:
 * every step of the path runs in CUDA kernels / copy engines of this library.
 *
 * Conventions
 *   - D = 59 fp32 attributes per Gaussian; a block is B rows
 *     (PAPER.md:180-187); K = ceil(N/B) global blocks, the last truncated.
 *   - Sharding (R17): global block k is owned by rank k % world_size and has
 *     local id k / world_size on that rank.  All lists returned below carry
 *     GLOBAL block ids, ascending.
 *   - A block "record" is B*59 fp32 (rows >= rows(k) are zero padding, R15).
 *     Slot layout on the device: [P slots][3][B][59] fp32 (theta | m | v),
 *     gradients separately [P][B][59].  Host tier: [K_loc][n_arr][B][59]
 *     with n_arr = 3 (persist: theta|m|v) or 1 (cold restart: theta only).
 *   - Status codes are returned; nothing throws across the ABI.  A CUDA error
 *     poisons the context (TGS_EPOISONED afterwards; only tgs_destroy is valid).
 *   - One host thread per context; one context per (rank, device).
 */
#ifndef TIDEGS_H
#define TIDEGS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGS_DIM 59

typedef struct tgs_ctx tgs_ctx;

typedef enum {
  TGS_OK = 0,
  TGS_EINVAL = 1,      /* bad argument / config; context state unchanged            */
  TGS_ESTATE = 2,      /* call order violated (see tgs_step_adam)                   */
  TGS_ENOMEM = 3,      /* host pinned or device allocation failed                   */
  TGS_ECUDA = 4,       /* CUDA runtime error; context poisoned                      */
  TGS_ENCCL = 5,       /* a collective of tgs_set_comm's transport failed (poisons)   */
  TGS_ENONFINITE = 6,  /* a non-finite gradient was seen in an active row (R20)     */
  TGS_EPOISONED = 7,   /* an earlier CUDA error poisoned this context               */
  TGS_EIO = 8          /* storage (f3 store tier) read/write failed; context poisoned */
} tgs_status;

typedef enum { TGS_MOMENTS_PERSIST = 0, TGS_MOMENTS_COLD_RESTART = 1 } tgs_moments;

typedef struct {
  uint64_t n_gaussians;  /* N >= 1, global                                          */
  uint32_t dim;          /* must be 59                               */
  uint32_t block_size;   /* B >= 4, B % 4 == 0 (4096 in the paper)   */
  uint32_t capacity;     /* C >= 1 resident blocks on this rank      */
  uint32_t pool_slots;   /* P >= C device slots; 0 -> 2C (R13)                      */
  uint32_t max_cameras;  /* J_max in [1, 256]                                       */
  uint32_t max_age;      /* A_max in [0, 1023]: Recency age saturation (R4)         */
  uint32_t quota_num, quota_den; /* beta = num/den in [0,1] (R10)                   */
  double lambda;         /* [0,1]                                */
  double gamma;          /* (0,1): Recency = gamma^age (R4)                         */
  int32_t moments;       /* tgs_moments (R6)                      */
  int32_t tide;          /* 1 = differential streaming; 0 = restage-all ablation    */
  int32_t world_size, rank; /* block k owned by rank k % world_size (R17)           */
  int32_t device;        /* CUDA device ordinal                                     */
  int32_t init_threads;  /* host threads used to build the host tier (0 -> auto)    */
  uint32_t staging_blocks; /* write-back staging ring, records per ring slot (3 slots;
                              0 -> C); an activate evicting more dirty records than
                              this writes them back straight from the slots instead */
  int32_t refresh_bounds; /* NEXT f2 (R25): after each update grow r_k to hold every
                             Gaussian of the block; the cull of batch t+2 sees it  */
  int32_t serialize;      /* ablation "w/o Overlap": activate returns
                             after its gather and write-back, step_adam after Adam  */
  int32_t level2;         /* NEXT f1: keep a 16-B extent sphere per resident row
                             (derived by the gather, updated by k_adam) so that
                             tgs_fine_filter reads 16 B per row instead of theta;
                             implied by refresh_bounds (whose per-row radius k_adam
                             then computes in its epilogue)                      */
  int32_t xfer;           /* a4 transfer mechanism (tgs_xfer; flat host tier only --
                             the store tier always uses TGS_XFER_KERNEL)          */
} tgs_config;

/* a4 transfer mechanism.
 * TGS_XFER_KERNEL: TMA bulk-copy kernels (k_xfer) read and write the pinned host
 *   tier over PCIe; no host decision needs the plan, so tgs_activate_async works.
 * TGS_XFER_COPY_ENGINE: the copy engines move the gather as runs of consecutive
 *   records (S+ runs host tier -> a device staging buffer, then k_commit places
 *   them in their slots); the dirty S- records go back from the write-back ring
 *   by the TMA kernel with 2 CTAs (environment TGS_WB_KERNEL=0: copy-engine runs
 *   issued by the library's I/O thread once the dirty list is known).  Needs the
 *   plan on the host: tgs_activate_async behaves as tgs_activate with it.  Why
 *   both mechanisms: copy-engine runs give the gather (which gates Adam) most of
 *   the link, the kernels need no plan readback (profiles/ab_xfer_r02.md,
 *   profiles/ab_wbk_r02.md). */
typedef enum { TGS_XFER_KERNEL = 0, TGS_XFER_COPY_ENGINE = 1 } tgs_xfer;

/* Optional device allocator hooks (PyTorch's caching allocator from Python).
 * NULL -> cudaMalloc / cudaFree. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, void* stream, void* user);
  void* user;
} tgs_allocator;

/* Host-tier filler: writes the B x 59 fp32 record of GLOBAL block k (padding
 * rows zero).  Called from several threads at once: must be thread-safe. */
typedef void (*tgs_fill_fn)(void* user, uint64_t k_global, float* out);

/* One camera = 6 frustum planes (nx, ny, nz, d0), unit normals, a point p is
 * inside iff n.p + d0 >= 0 (R1). */
typedef struct { float plane[6][4]; } tgs_camera;

typedef struct {
  /* host values, final on return (plan-synchronous, R14) */
  uint32_t n_visible;        /* |K_{t+1}|                                       */
  uint32_t n_resident;       /* |R_{t+1}|                                       */
  uint32_t n_active_blocks;  /* |R_{t+1} n K_{t+1}|                             */
  uint32_t n_stage_in;       /* |S+|                                            */
  uint32_t n_evict;          /* |S-|                                            */
  uint32_t n_evict_dirty;    /* |dirty S-| (0 until known, see tgs_get_stats)   */
  uint64_t h2d_bytes;        /* |S+| * record bytes * n_arr                     */
  /* device pointers, library-owned, valid until the next activate/flush/destroy */
  const uint32_t* d_active_blocks; /* [n_active_blocks] global ids, ascending   */
  const uint32_t* d_active_slots;  /* [n_active_blocks] slot of each            */
  float* d_params;           /* slot pool base: slot s at d_params + s*slot_stride */
  float* d_grads;            /* grad pool base: slot s at d_grads + s*grad_stride   */
  uint64_t slot_stride;      /* floats per slot in d_params (3*B*59)            */
  uint64_t grad_stride;      /* floats per slot in d_grads (B*59)               */
  void* ready;               /* cudaEvent_t: wait on it before touching slots   */
  /* C1 (multi-GPU, tgs_set_comm): the active sets A of every rank, [world_size]
   * rows of capacity entries each (rank-major, global ids ascending, padded with
   * 0xFFFFFFFF); device, library-owned, double-buffered by activate parity;
   * NULL without a comm.  global_ready (cudaEvent_t): wait before reading. */
  const uint32_t* d_global_active;
  uint32_t global_stride;    /* entries per rank row (= capacity C_g)           */
  void* global_ready;
  const uint32_t* d_n_active; /* device: |R n K| of this activate (valid in stream
                                 order after `ready`; the only count
                                 tgs_activate_async provides)                  */
} tgs_activation;

typedef struct {
  const float* lr;  /* [59] per-attribute learning rate (host, copied)         */
  float beta1, beta2, eps;
} tgs_adam;

typedef struct {
  uint64_t iter, n_visible, n_resident, n_active_blocks, n_stage_in, n_evict, n_evict_dirty,
      n_active_rows, h2d_bytes, d2h_bytes, flush_bytes, n_flush_blocks, readmissions,
      cold_restart_updates, total_updates, resident_streak_sum, streak_count,
      k_inter_sum, k_union_sum; /* sum over activates of |K_t n K_{t+1}| and |K_t u K_{t+1}|
                                  (consecutive-batch Jaccard of the visible sets, the
                                  PAPER.md:139 / 522,572 locality analog) */
} tgs_stats; /* cumulative */

typedef struct {
  /* device time of the library's kernels / copies, CUDA events on the stream
   * each is launched on; accumulated while profiling is enabled */
  double adam_ms, adam_prologue_ms, plan_ms, h2d_ms, d2h_ms, evict_ms, fine_ms;
  uint64_t adam_launches, plan_launches, h2d_batches, d2h_batches;
  uint64_t adam_rows;        /* active rows processed by the timed Adam launches */
  uint64_t adam_elems_quads; /* 4-row quads visited by the timed Adam launches   */
  uint64_t h2d_bytes, d2h_bytes; /* bytes moved by the timed copy batches        */
  uint64_t kernel_launches;  /* every kernel this library launched              */
  uint64_t copy_calls;       /* cudaMemcpyAsync calls issued (tgs_flush only; the
                              * per-step transfers are kernels, k_xfer) */
  /* cumulative since init (not only while profiling), for the algorithmic bytes
   * of k_adam under cold restart (R6): a block's first update after admission
   * reads no m, v and writes its whole m, v record */
  uint64_t fresh_active_rows; /* active rows of blocks updated for the first time */
  uint64_t fresh_blocks;      /* blocks updated for the first time since admission */
  /* cumulative: S+ records the gather took from the previous activate's
   * write-back ring in HBM (a block evicted dirty and re-admitted at once)
   * instead of over the host link */
  uint64_t h2d_ring_records;
} tgs_timing;

/* Transport of the two per-batch collectives of the sharded path (
 * reading R17: block k lives on rank k mod world_size, every rank runs the
 * whole step on its shard).  The library decides what is exchanged and when:
 *   C1  at the end of every tgs_activate, on the library's plan stream: the
 *       rank's A = R n K as global ids, padded to C_g, all-gathered into
 *       tgs_activation.d_global_active;
 *   C2  at the end of every tgs_step_adam, on the compute stream: the rank's
 *       cumulative tgs_stats counters, all-reduced (sum) into the buffer
 *       tgs_get_global_stats reads.
 * The caller supplies the transport: NCCL over NVLink on a B200 node
 * (ncclAllGather / ncclAllReduce(ncclUint64, ncclSum) enqueued on `stream`),
 * or torch.distributed (the Python binding's TorchComm).  Each function moves
 * device buffers and must be stream-ordered on `stream` (cudaStream_t) or
 * complete before returning; a non-zero return poisons the context and the
 * call reports TGS_ENCCL. */
typedef struct {
  /* d_recv[world_size * bytes] <- every rank's d_send[bytes], rank-major */
  int (*allgather)(void* user, const void* d_send, void* d_recv, size_t bytes, void* stream);
  /* d_buf[count] <- sum over ranks of d_buf[count] (uint64), in place */
  int (*allreduce_u64)(void* user, uint64_t* d_buf, size_t count, void* stream);
  void* user;
} tgs_comm;

/* ---------------------------------------------------------------- lifecycle */

/* Create the context for shard cfg->rank: validates cfg (EINVAL: dim != 59,
 * B % 4 != 0, C == 0, P < C, lambda/gamma/beta out of range, J_max outside
 * [1,256], max_age > 1023, non-finite or negative-radius bounds), allocates the
 * pinned host tier and copies this shard's blocks into it from EITHER
 * theta_rows (host, N x 59 fp32, global row order; may be freed afterwards) OR
 * fill (called per owned block; theta_rows must then be NULL), zeroes the host
 * moments, uploads bounds (host, K x 4 fp32 (cx,cy,cz,r) for ALL global
 * blocks) and allocates the device slot pool.
 * compute_stream (cudaStream_t, may be NULL = legacy default) is the stream
 * tgs_step_adam runs on and the stream callers order their gradient writes on. */
tgs_status tgs_init_table(const tgs_config* cfg, const float* theta_rows, tgs_fill_fn fill,
                          void* fill_user, const float* bounds, const tgs_allocator* alloc,
                          void* compute_stream, tgs_ctx** out);

tgs_status tgs_destroy(tgs_ctx* ctx);

/* Attach the collectives' transport (copied; comm->user must outlive the ctx).
 * Allowed once, before the first tgs_activate (ESTATE otherwise); EINVAL if a
 * function pointer is NULL.  Without it, a rank runs its shard alone. */
tgs_status tgs_set_comm(tgs_ctx* ctx, const tgs_comm* comm);
/* C2 result: every rank's tgs_stats summed, as of the last tgs_step_adam
 * (synchronising).  ESTATE without a comm. */
tgs_status tgs_get_global_stats(tgs_ctx* ctx, tgs_stats* out);

/* NEXT f3 -- the tier below the host tier (§3.4 "SSD
 * Storage, CPU Tiered Cache"; readings R27, R28 of DESIGN.md §3).  Instead of a
 * pinned host copy of the whole shard, the shard lives in a log-structured
 * store under dir: an immutable base segment (base.tdgs, written here from
 * theta_rows / fill, m = v = 0) and append-only patch segments
 * (patch-NNNNNN.tdgp) with a per-block Index[k] = (file_id, offset, size,
 * version).  Above it sits a CPU cache of cache_blocks
 * pinned block records (LRU with a dirty bit per entry),
 * inclusive of the GPU working set: the S+ gather reads from, and the dirty
 * S- write-back lands in, the block's entry; a dirty entry reaches the SSD
 * when the cache evicts it (LRU among blocks outside R_t u R_{t+1}) or at
 * tgs_flush.  Misses are read through Index[k] inside
 * tgs_activate (overlapping the previous Adam on the device).  File format:
 * little-endian, 4096-byte header pages, payloads page-aligned (R28).
 * Every other call behaves exactly as with tgs_init_table. */
typedef struct {
  const char* dir;         /* directory (created if absent; one store per dir: its stale
                              patch segments are removed); must not be NULL        */
  uint32_t cache_blocks;   /* H >= 2 * capacity block records (EINVAL otherwise)    */
  uint64_t segment_bytes;  /* patch segment rollover budget; 0 -> 1 GiB             */
  int32_t direct_io;       /* 1: O_DIRECT reads/writes (page cache bypassed)        */
  int32_t io_threads;      /* parallel SSD requests; 0 -> 8                         */
  int32_t reopen;          /* 1: resume the state of the last barrier an earlier session
                              left (checkpoint/resume, reading R30): no base is written
                              (theta_rows and fill may both be NULL); the barrier
                              manifest bounds the log, Index is recovered from the base
                              and the patch records up to it (later records win; every
                              record's CRC-32C checked), records appended after the
                              barrier are dropped, the Adam step counters come back from
                              the manifest; the cache starts empty, recency at zero;
                              TGS_EIO if the manifest or base does not describe this
                              shard or a durable record is corrupt                  */
  uint32_t prefetch_blocks; /* read-ahead buffers for tgs_prefetch (0: off); the pinned
                              pool then holds cache_blocks + prefetch_blocks records */
} tgs_store_config;

/* As tgs_init_table, with the store tier.  TGS_EIO: the store could not be
 * created (a message is printed to stderr; *out is not set). */
tgs_status tgs_init_table_store(const tgs_config* cfg, const tgs_store_config* store,
                                const float* theta_rows, tgs_fill_fn fill, void* fill_user,
                                const float* bounds, const tgs_allocator* alloc,
                                void* compute_stream, tgs_ctx** out);

typedef struct {
  uint64_t hits, misses;        /* CPU-cache lookups of S+ blocks                          */
  uint64_t evictions;           /* CPU-cache evictions (LRU victims)                       */
  uint64_t dirty_evictions;     /* victims appended to the patch log during training       */
  uint64_t flush_appends;       /* records appended by tgs_flush                           */
  uint64_t read_bytes;          /* SSD bytes read (misses x padded payload)                */
  uint64_t write_bytes;         /* SSD bytes appended (record + segment header pages incl.) */
  uint64_t segments;            /* patch segments created                                  */
  uint64_t cached, cached_dirty;/* current CPU-cache occupancy                             */
  double read_ms, write_ms;     /* host wall time spent in SSD reads / appends             */
  uint64_t read_calls;          /* vector reads issued (runs of neighbouring records)      */
  double read_busy_ms;          /* summed over the I/O threads: time inside the reads      */
  uint64_t prefetch_reads;      /* records read ahead (tgs_prefetch)                       */
  uint64_t prefetch_hits;       /* misses served from a read-ahead record (no SSD read then) */
  uint64_t prefetch_wasted;     /* read-ahead records recycled unused                      */
} tgs_store_stats;
/* ESTATE without a store.  Synchronising. */
tgs_status tgs_get_store_stats(tgs_ctx* ctx, tgs_store_stats* out);
/* NEXT f3 read-ahead ("Prefetch needed blocks into the CPU cache",
 * 253-259): announce the camera batch of the tgs_activate `ahead` calls from now
 * (1 = the next one; the trajectory is known ahead, and 2 lets the reads overlap
 * a whole step).  Its Level-1 visible set is culled on the GPU (k_probe, R1/R2
 * rule, no state changed), and the store's read-ahead threads read the newest
 * version of every such block that is not cached into free read-ahead buffers
 * while the steps before it run.  The CPU cache (R27) is not changed: that
 * activate's gather waits for the batches announced for it (or earlier) and, for a
 * miss whose read-ahead record is still the newest version, swaps that buffer into
 * the miss's entry instead of reading the SSD.  Returns once the reads are queued.
 * EINVAL also for ahead == 0.  No-op (TGS_OK) without a store or with prefetch_blocks = 0;
 * EINVAL on J > J_max or non-finite planes. */
tgs_status tgs_prefetch(tgs_ctx* ctx, const tgs_camera* cams, uint32_t J, uint32_t ahead);
/* Index[k] of global block k: out4 = (file_id, payload offset, payload bytes, version) */
tgs_status tgs_store_index(tgs_ctx* ctx, uint64_t k_global, uint64_t* out4);
/* Compaction ("Optional compaction can merge patch segments into a
 * new base segment, but this is outside the training critical path"; reading
 * R31): performs the tgs_flush barrier, then writes every block's newest version
 * into a new base segment (base.tdgs.tmp, made durable, renamed over base.tdgs),
 * removes the patch segments and points Index[k] into the base again (versions
 * kept; the next append opens patch segment 1).  ESTATE without a store; TGS_EIO
 * on an I/O failure (the old files stay valid until the rename). */
tgs_status tgs_store_compact(tgs_ctx* ctx);
/* cached global ids, least recently used first, and their dirty flags (either may
 * be NULL); returns the number cached (writes at most cap) */
uint32_t tgs_store_lru(tgs_ctx* ctx, uint32_t* blocks, uint8_t* dirty, uint32_t cap);

/* ------------------------------------------------------------ the hot path */

/* Activate the next camera batch (J = n_cams <= J_max; 0 is valid: K = {}).
 * Runs a1-a3 on the device, reads back the plan (one small host<->device
 * synchronisation that does NOT wait for the previous tgs_step_adam), issues
 * the H2D gather of S+ on its own stream (overlapping the previous Adam), and
 * the write-back of the dirty S- records after the previous Adam (tgs_xfer).
 * EINVAL: J > J_max, cams NULL with J > 0, non-finite plane.  Allowed after
 * init, after step_adam, after flush, and after another activate (R19). */
tgs_status tgs_activate(tgs_ctx* ctx, const tgs_camera* cams, uint32_t n_cams,
                        tgs_activation* out);

/* tgs_activate without the plan readback: the same a1-a4 work, enqueued and
 * returned at once, every count (|S+|, |S-|, |A|) read by the kernels from the
 * plan's device header -- the caller thread never waits for the GPU, so the
 * host runs ahead and small (latency-bound) steps are not bound by it.  Needs
 * the flat host tier, xfer = TGS_XFER_KERNEL, Tide on, pool_slots >= 2C (S+ never reuses an S- slot,
 * R13) and staging_blocks >= C (every S- fits the ring); otherwise it behaves as
 * tgs_activate.  out (may be NULL): the host counts are 0xFFFFFFFF (unknown),
 * the device pointers are valid, |A| is at d_n_active; tgs_get_stats /
 * tgs_get_stats_async give the counters, tgs_get_list the lists.  Errors as
 * tgs_activate. */
tgs_status tgs_activate_async(tgs_ctx* ctx, const tgs_camera* cams, uint32_t J,
                              tgs_activation* out);

/* Masked Adam (a5) over the rows of R n K of the last activate, on the compute
 * stream, after the activation's ready event.  d_row_mask: device
 * [P][ceil(B/32)] u32, bit r of slot s = row r active (I_t), or NULL = every
 * logical row active (R8).  Gradients are read from the grad pool (written by
 * the caller on the compute stream).  ESTATE unless the previous call was
 * tgs_activate.  Non-finite gradients: the row is skipped and the lowest
 * (gid*59 + attr) is reported by tgs_nonfinite_index (R20). */
tgs_status tgs_step_adam(tgs_ctx* ctx, const tgs_adam* hp, const uint32_t* d_row_mask);

/* Level-2 fine filter (NEXT f1): writes
 * the I_t row mask of every slot of R n K of the last activate into
 * d_row_mask (device [P][ceil(B/32)] u32, the layout tgs_step_adam reads):
 * bit r = row r's sphere (mu, 3*exp(max log-scale), R24 deterministic exp) is
 * kept by the Level-1 rule for at least one camera of the batch.  Runs on the
 * compute stream after the gather; call between tgs_activate and
 * tgs_step_adam (ESTATE otherwise), then pass the same mask to step_adam. */
tgs_status tgs_fine_filter(tgs_ctx* ctx, uint32_t* d_row_mask);

/* Consistency barrier: write every dirty resident record
 * back to the host tier, wait for all work, clear dirty bits.  Blocks stay
 * resident. */
tgs_status tgs_flush(tgs_ctx* ctx);

/* ------------------------------------------------------------- inspection
 * (synchronising; for tests, metrics and checkpoint export) */
tgs_status tgs_get_stats(tgs_ctx* ctx, tgs_stats* out);
tgs_status tgs_get_timing(tgs_ctx* ctx, tgs_timing* out);
/* Non-synchronising stats read: enqueues a device->host copy of the device
 * counters into out (must be pinned host memory, e.g. cudaHostAlloc) on the
 * compute stream, in stream order after the last tgs_step_adam; valid once
 * that stream is synchronised.  flush_bytes / n_flush_blocks are not included
 * (host-side; see tgs_get_stats). */
tgs_status tgs_get_stats_async(tgs_ctx* ctx, tgs_stats* out);
tgs_status tgs_set_profiling(tgs_ctx* ctx, int enabled); /* also resets tgs_timing */

/* Lists of the last activate, GLOBAL ids ascending: which = 0 K_{t+1},
 * 1 R_{t+1}, 2 S+, 3 S-, 4 Omega, 5 A = R n K.  slots[i] = slot of blocks[i]
 * after the activate (-1 for S-).  Returns the list length (writes at most cap
 * entries; blocks/slots may be NULL). */
uint32_t tgs_get_list(tgs_ctx* ctx, int which, uint32_t* blocks, int32_t* slots, uint32_t cap);
/* K_{t+1}^{(j)} of the last activate */
uint32_t tgs_get_percam(tgs_ctx* ctx, uint32_t j, uint32_t* blocks, uint32_t cap);
/* dirty members of S- written back by the last activate */
uint32_t tgs_get_evicted_dirty(tgs_ctx* ctx, uint32_t* blocks, uint32_t cap);
/* slot -> global block id (-1 free), P entries */
tgs_status tgs_get_slot_map(tgs_ctx* ctx, int64_t* slot_to_block);
/* lowest gid*59+attr of a non-finite active gradient so far, UINT64_MAX if none */
uint64_t tgs_nonfinite_index(tgs_ctx* ctx);
/* newest version of global block k: resident slot if resident, else host tier
 * (cold restart: m = v = 0 off the device).  Host buffers of B*59 fp32 each,
 * any may be NULL. */
tgs_status tgs_read_block(tgs_ctx* ctx, uint64_t k_global, float* theta, float* m, float* v);
uint32_t tgs_step_count(tgs_ctx* ctx, uint64_t k_global);
/* current Level-1 bound (cx, cy, cz, r) of global block k (host float[4]) */
tgs_status tgs_read_bound(tgs_ctx* ctx, uint64_t k_global, float* out4);
uint32_t tgs_num_local_blocks(const tgs_ctx* ctx);
uint32_t tgs_pool_slots(const tgs_ctx* ctx);

/* NEXT f2b -- Morton sort + blocking ("we Morton-sort
 * Gaussians by the codes of their centers before blocking", 375-376; SPEC.md:
 * 81-145; reading R26 in DESIGN.md §3).  cs: host [n][4] fp32 (cx, cy, cz,
 * max log-scale) of n <= 2^32-1 Gaussians in any order.  On the GPU: AABB,
 * 21-bit-per-axis quantisation in double, x-lowest bit interleave, stable radix
 * sort of the 63-bit codes (ties keep index order), then per block of
 * block_size consecutive sorted Gaussians: centroid (double, sorted order,
 * rounded to fp32) and radius max(|mu - c| (double) + 3*exp(max log-scale))
 * rounded up to fp32.  Outputs (host, caller-owned): perm[n] = original index
 * of sorted position i; bounds[ceil(n/B)][4] -- the tgs_init_table bounds of
 * the table whose row i is original row perm[i].  gpu_ms (may be NULL): device
 * time of the sort and bounds.  EINVAL: n == 0 or > 2^32-1, B == 0,
 * non-finite centre.  Stateless; allocates and frees its own device memory. */
tgs_status tgs_build_layout(const float* cs, uint64_t n, uint32_t block_size, int device,
                            uint64_t* perm, float* bounds, double* gpu_ms);

/* NEXT f4 -- clustered-TSP view ordering ("We use a clustered
 * TSP-ordered (no-shuffle) camera sequence to increase overlap between
 * consecutive block working sets", 709-712; reading R29 of DESIGN.md §3), on
 * the GPU.  feat: host [M][D] doubles (D in [1, 8]) describing each training
 * view's pose (e.g. camera centre and a point on its optical axis).  k =
 * ceil(sqrt(M)) k-means clusters (maximin initialisation from the
 * lexicographically smallest view, Lloyd iterations until no assignment
 * changes, at most 100), a nearest-neighbour tour over the cluster centres and
 * nearest-neighbour tours inside each cluster; every distance a
 * feature-ordered sum of squares in double without FMA, every tie to the
 * lowest index.  Outputs (host, caller-owned): perm[M] = the view to present
 * at position i; cluster[M] (may be NULL); k_out, iters_out (Lloyd passes that
 * changed something), gpu_ms (device time; each may be NULL).  EINVAL: M == 0,
 * D outside [1, 8], non-finite feature, k*D doubles over 200 KB.  Stateless. */
tgs_status tgs_order_views(const double* feat, uint32_t M, uint32_t D, int device, uint32_t* perm,
                           uint32_t* cluster, uint32_t* k_out, uint32_t* iters_out,
                           double* gpu_ms);

/* Frustum planes of a pinhole camera (R1): w2c row-major 4x4 world->camera
 * (camera +z forward, +x right, +y down), intrinsics fx, fy, cx, cy, image
 * width x height, near/far.  Computed in double, rounded to fp32. */
tgs_status tgs_frustum_planes(const double w2c[16], double fx, double fy, double cx, double cy,
                              uint32_t width, uint32_t height, double znear, double zfar,
                              tgs_camera* out);

const char* tgs_status_string(tgs_status s);
const char* tgs_last_error(const tgs_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TIDEGS_H */
