// tidegs_internal.h -- device-state layout and kernel launchers shared by
// tidegs_kernels.cu (sm_100a kernels) and tidegs_runtime.cu (host runtime).
// Nothing here is shared with oracle/ (the two sides share no code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tgs {

constexpr uint32_t kDim = 59;
constexpr int kRings = 5;                  // write-back ring slots, at most (activate T uses
                                           // T % nrings: 5 on the flat tier, 3 with the store)
constexpr uint32_t kFromHdr = 0xFFFFFFFFu; // count argument: read it from the device plan header
constexpr uint32_t kMaxCams = 256;
constexpr uint32_t kMaxAge = 1023;
constexpr uint32_t kMaxBuckets = 2 * 2 * (kMaxAge + 2);  // rank x (in R_t ? 0 : 1)


// cumulative counters, same order as tgs_stats
enum Stat : int {
  ST_ITER = 0, ST_VISIBLE, ST_RESIDENT, ST_ACTIVE_BLOCKS, ST_STAGE_IN, ST_EVICT, ST_EVICT_DIRTY,
  ST_ACTIVE_ROWS, ST_H2D, ST_D2H, ST_FLUSH_BYTES, ST_FLUSH_BLOCKS, ST_READMIT, ST_COLD_UPD,
  ST_TOTAL_UPD, ST_STREAK_SUM, ST_STREAK_CNT, ST_K_INTER, ST_K_UNION, ST_N,
  // internal (not in tgs_stats): fresh-update counts and the S+ records gathered
  // from the write-back ring instead of the host (tgs_timing)
  ST_FRESH_ROWS = ST_N, ST_FRESH_BLOCKS, ST_RING_READMIT, ST_ALL
};

// per-activate counters written by the cull kernel (zeroed before it)
enum Cnt : int { CNT_CAND = 0, CNT_K = 1, CNT_N = 4 };

// plan header: written by k_plan into host-mapped pinned memory (and a device copy)
struct PlanHdr {
  uint32_t nK, nR, nSp, nSm, nA, nOm, nfree, fallback;
  uint32_t n_dirty;   // written by k_evict
  uint32_t pad[7];
};

// per active (R n K) entry, written by k_adam_prologue
struct AdamEnt {
  uint32_t step;   // new step count, 0 = no active row (block untouched)
  uint16_t rows_hi_unused;
  uint16_t fresh;  // cold restart and first update since admission: m = v = 0 implicitly
  uint32_t rows;   // logical rows of the block
  float bc1;       // 1 - beta1^step   (R9)
  float ibs;       // 1 / sqrt(1 - beta2^step)
};

struct Dev {
  // sizes
  uint64_t N;
  uint32_t B, Kloc, W, P, PW, C, J_max, n_arr, G, rank, max_age, n_lut_cols;
  uint32_t quota_num, quota_den;
  int32_t tide, cold, refresh;
  uint64_t rec_floats;   // B*59
  // per local block
  float4* bounds;        // [Kloc] (cx,cy,cz,r)
  uint32_t* pend[2];     // [Kloc] R25 refreshed radius bits of the step of that parity (0 none)
  int32_t* last_access;  // [Kloc] -1 = never (R4)
  uint32_t* step;        // [Kloc] Adam step count (R7)
  int32_t* b2s;          // [Kloc] slot or -1
  uint8_t* ever;         // [Kloc] admitted at least once (k_plan only; readmissions)
  uint8_t* evicted;      // [Kloc] evicted at least once (k_evict only; cold-restart count)
  int32_t* admit;        // [Kloc] activate index of last admission
  // bitsets over local blocks, [W] words each
  uint32_t* percam[2];   // [J_max][W] per-camera K^(j) (parity: k_fine of t reads it
                         // while the plan of t+1 may already run)
  uint32_t *Kb, *cand, *Q, *Sp, *Sm, *Om, *Ab;
  uint32_t* R[2];        // R_t by parity
  // per slot
  int32_t* s2b;          // [P] local block or -1
  uint32_t *occ, *dirty, *rel;  // [PW]
  // plan outputs
  uint32_t *sp_blk[2], *sp_slot[2];    // [C] S+ ascending and its slots (parity)
  uint32_t *sm_blk[2], *sm_slot[2];    // [C] S- ascending and its slots (parity)
  uint32_t *a_blk[2], *a_slot[2], *a_gid[2];  // [C] A = R n K (parity)
  PlanHdr* hdr_dev[2];   // device copy of the header (parity: the gather of T reads it
                         // while the plan of T+1 may already run)
  PlanHdr* hdr_map;      // device alias of the mapped host header
  uint32_t* sp_map;      // mapped host [C][2] (local id, slot) of S+
  uint32_t* sm_map;      // mapped host [C] S- local ids (store mode only, else nullptr)
  // write-back state of activate T lives in ring slot T % kRings: the scatter of
  // T may still read it while the next two activates write theirs
  uint32_t* dirty_map[kRings];  // mapped host [C][2] (local id, slot) of dirty S- (ring slot)
  uint32_t* ndirty_map;    // mapped host [3] |dirty S-| (ring slot)
  uint32_t* ndirty_dev;    // [3] |dirty S-| (ring slot), read by k_pack and k_xfer
  uint32_t* dl_slot[kRings];  // [C] dirty S- slots (pack / direct write-back source)
  uint32_t* dl_blk[kRings];   // [C] dirty S- local ids (write-back destination)
  int32_t* wb_tag;       // [Kloc] activate index at which the block was packed (-1 never)
  uint32_t* wb_idx;      // [Kloc] its staging-ring index then
  float* staging[kRings];     // [S_max][n_arr][B][59] write-back staging rings (ring slot)
  float* stage_in;       // [C][n_arr][B][59] copy-engine gather staging: S+ record i at i
                         // (xfer = TGS_XFER_COPY_ENGINE, else nullptr; read by k_commit)
  uint32_t S_max;        // staging capacity in records
  int32_t nrings;        // ring slots in use: a block packed by one of the last nrings-1
                         // activates is re-admitted from its ring record
  float4* last_planes[2];  // [kMaxCams*6] camera batch of the activate of that parity
  const float4* planes_map[2];  // mapped pinned host staging of the camera batch (parity)
  // selection
  uint16_t* rank_lut;    // [2][max_age+2]
  uint32_t n_buckets;    // 2 * (number of distinct ranks)
  uint32_t* cnt;         // [CNT_N]
  unsigned long long* stats;      // [ST_N]
  unsigned long long* nonfinite;  // lowest gid*59+attr
  // Adam
  AdamEnt* ent;          // [C]
  uint32_t* adam_ctr;    // [1] dynamic quad-chunk counter of k_adam (count from the header)
  float *lut_bc1, *lut_ibs;  // [lut_cap]
  // host tier as the transfer kernels see it (device-mapped pinned memory)
  unsigned char* host_dev;  // flat tier: record l at l * host_stride; store tier: CPU-cache entries
  uint64_t host_stride;     // bytes between host records (n_arr*B*236, or the padded entry size)
  int32_t* ent_of;          // [Kloc] store tier: cache entry of each resident block (else nullptr)
  const uint32_t* sp_entry; // mapped host [C] store tier: cache entry of S+ block i (host-written)
  // f1 / f2 (cfg.level2 or cfg.refresh_bounds): per slot row, the 6 theta
  // attributes the Level-2 test and the bound refresh read -- centre (0..2) and
  // log-scales (52..54) -- packed as 24 B: written by the gather for admitted rows
  // and by k_adam for updated rows (R24, R25).  nullptr when off.
  float* geo6;           // [P][B][6]
  // pools
  float* params;         // [P][3][B][59]
  float* grads;          // [P][B][59]
};

struct AdamHyper {
  float lr[kDim];
  float b1, b2, omb1, omb2, eps;
};

// launchers (return cudaGetLastError())
cudaError_t launch_cull(const Dev& d, uint32_t J, int32_t T, int parity, cudaStream_t s);
cudaError_t launch_quota(const Dev& d, uint32_t J, int32_t T, int parity, cudaStream_t s);
cudaError_t launch_plan(const Dev& d, int32_t T, int parity, cudaStream_t s);
cudaError_t launch_pack(const Dev& d, uint32_t nSm, int ring, cudaStream_t s);
cudaError_t launch_evict_tagged(const Dev& d, uint32_t nSm, int parity, int ring, int32_t T,
                                bool tag, cudaStream_t s);
// a4 transfers (XferMode in tidegs_kernels.cu): 0 gather S+ (sel/n_sel: a host-
// selected subset, else all of hdr_dev->nSp), 1 scatter the ring, 2 scatter from
// the slots; n_hint > 0 is an upper bound of the records (sizes the grid);
// ctas CTAs of one warp, bufs 32 KB shared-memory buffers each (bufs-1 loads in flight)
cudaError_t launch_xfer(const Dev& d, int mode, int parity, int ring, int32_t T,
                        const uint32_t* sel, uint32_t n_sel, uint32_t n_hint, int ctas, int bufs,
                        cudaStream_t s);
cudaError_t launch_commit(const Dev& d, uint32_t nSp, int parity, int32_t T, cudaStream_t s);
cudaError_t launch_refresh(const Dev& d, uint32_t nA, int parity, cudaStream_t s);
cudaError_t launch_probe(const Dev& d, const float4* planes, uint32_t J, uint32_t* out,
                         cudaStream_t s);
cudaError_t launch_pad_active(uint32_t* gid, const PlanHdr* h, uint32_t C, cudaStream_t s);
cudaError_t launch_adam_prologue(const Dev& d, uint32_t nA, int parity, const uint32_t* mask,
                                 cudaStream_t s);
cudaError_t launch_adam(const Dev& d, uint32_t nA, int parity, const uint32_t* mask,
                        const AdamHyper& hp, int grid_ctas, cudaStream_t s);
cudaError_t launch_fine(const Dev& d, uint32_t nA, uint32_t J, int parity, uint32_t* mask,
                        cudaStream_t s);
int adam_grid(int device);

// NEXT f2b: Morton sort + blocking
struct LayoutBufs {
  float* cs;                      // [n][4] (cx, cy, cz, max log-scale)
  unsigned long long* k[2];       // [n] codes (ping-pong)
  uint32_t* v[2];                 // [n] indices (ping-pong)
  uint32_t* counts;               // [layout_scan_len(n)]
  uint32_t* sums;                 // [layout_nsums(n)]
  float* part;                    // [part_grid][6]
  float* bounds;                  // [K][4]
};
uint32_t layout_ntile(uint64_t n);
uint64_t layout_scan_len(uint64_t n);
uint32_t layout_nsums(uint64_t n);
cudaError_t layout_run(const LayoutBufs& b, uint64_t n, uint32_t B, cudaStream_t s, int part_grid,
                       int* perm_buf);

}  // namespace tgs
