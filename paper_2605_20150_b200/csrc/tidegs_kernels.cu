// tidegs_kernels.cu -- sm_100a kernels of the TideGS working-set step.
//
//   k_cull           a1  Level-1 sphere-vs-6-plane cull, per-camera bitsets by
//                        warp ballot, union K_{t+1}, candidate pool, recency stamp
//                        (PAPER.md:196-208 Eq. Kt_def; Alg. 1 l.1-3)
//   k_quota          a3  camera-balanced quota: top-q_j of K^{(j)} in score order
//                        (R10), one CTA per camera
//   k_plan           a2+a3  global Top-C fill, set differences S+/S-/Omega
//                        (Alg. 1 l.6-8), slot allocation /
//                        eviction (R13), active list A = R n K
//   k_evict          a4  dirty S- records -> write-back list
//   k_adam_prologue  a5  per-block active-row count, step, dirty bit
//   k_adam           a5  fused masked Adam, 128-bit coalesced (Eq. masked_update); a
//                        cold-restarted block's moments are zero until its first update
//                        (PAPER.md:327-328), which writes its whole m, v record
//
// Determinism: every choice (list order, Top-C, slot assignment) comes from
// prefix sums over id-ordered bitsets, never from atomic arrival order; atomics
// only carry commutative effects (or/and on bitmaps, integer adds, min).
// Floating point: IEEE RN intrinsics in the exact order DESIGN.md §3 (R2, R9)
// fixes; compiled without fast-math, FTZ off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "tidegs_internal.h"

namespace tgs {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// a count argument equal to kFromHdr is read from the activate's device plan
// header (tgs_activate_async: the host never reads the plan back)
__device__ __forceinline__ uint32_t count_or_hdr(uint32_t n, const PlanHdr* h, int which) {
  if (n != kFromHdr) return n;
  return which == 0 ? h->nA : h->nSm;
}

__device__ __forceinline__ uint32_t block_rows(const Dev& d, uint32_t l) {
  const uint64_t lo = ((uint64_t)l * d.G + d.rank) * d.B;
  if (lo >= d.N) return 0u;
  const uint64_t r = d.N - lo;
  return r < d.B ? (uint32_t)r : d.B;
}

// Exclusive block-wide scan of one u32 per thread.  NT threads; scratch >= 33 words.
template <int NT>
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t& total, uint32_t* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t y = lane < NT / 32 ? sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t z = __shfl_up_sync(kFull, y, o);
      if (lane >= o) y += z;
    }
    sh[lane] = y;
  }
  __syncthreads();
  const uint32_t pre = wid ? sh[wid - 1] : 0u;
  total = sh[NT / 32 - 1];
  __syncthreads();
  return pre + x - v;
}

template <int NT>
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* sh) {
  uint32_t t;
  block_scan<NT>(v, t, sh);
  return t;
}

// Selection key bucket of local block l (R4, R11): rank of (m, b) in descending
// score s(k) = lam*1[k in K_{t+1}] + (1-lam)*gamma^age (host LUT, exact double
// ties kept), then resident-first.  Ascending bucket, then ascending id, is the
// total key order of the oracle's comparator.
__device__ __forceinline__ uint32_t bucket_of(const Dev& d, uint32_t l, bool inK, bool inR,
                                              int32_t T) {
  const int32_t la = d.last_access[l];
  uint32_t b;
  if (la < 0) {
    b = d.max_age + 1;  // never accessed: Recency 0
  } else {
    const int32_t age = (T - 1) - la;
    b = (uint32_t)age > d.max_age ? d.max_age : (uint32_t)age;
  }
  const uint32_t r = d.rank_lut[(inK ? d.n_lut_cols : 0u) + b];
  return 2u * r + (inR ? 0u : 1u);
}

// CTA-wide Top-n over the candidate bits word(w), w in [0, nw), in key order
// (bucket asc, id asc).  emit(w, bits) is called once per word with a non-empty
// selection.  smem: hist[kMaxBuckets], sh[40].
template <int NT, class WordFn, class EmitFn>
__device__ void select_top(const Dev& d, uint32_t n, uint32_t nw, int32_t T, uint32_t* hist,
                           uint32_t* sh, const WordFn& word, const uint32_t* Rcur,
                           bool allK, const EmitFn& emit) {
  if (n == 0) return;
  const uint32_t NB = d.n_buckets;
  for (uint32_t i = threadIdx.x; i < NB; i += NT) hist[i] = 0;
  __syncthreads();
  for (uint32_t w = threadIdx.x; w < nw; w += NT) {
    uint32_t bits = word(w);
    const uint32_t rw = Rcur[w];
    const uint32_t kw = allK ? kFull : d.Kb[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t l = 32u * w + b;
      atomicAdd(&hist[bucket_of(d, l, (kw >> b) & 1u, (rw >> b) & 1u, T)], 1u);
    }
  }
  __syncthreads();
  // threshold bucket: first bucket whose inclusive prefix reaches n
  const uint32_t per = (NB + NT - 1) / NT;
  const uint32_t b0 = threadIdx.x * per;
  uint32_t mine = 0;
  for (uint32_t i = 0; i < per; ++i)
    if (b0 + i < NB) mine += hist[b0 + i];
  uint32_t total;
  uint32_t pre = block_scan<NT>(mine, total, sh);
  if (threadIdx.x == 0) {
    sh[34] = NB;  // threshold: all buckets < thr selected entirely
    sh[35] = 0;   // how many of bucket thr (lowest ids first)
  }
  __syncthreads();
  if (total > n) {
    for (uint32_t i = 0; i < per && b0 + i < NB; ++i) {
      const uint32_t h = hist[b0 + i];
      if (pre < n && n <= pre + h) {
        sh[34] = b0 + i;
        sh[35] = n - pre;
      }
      pre += h;
    }
  }
  __syncthreads();
  const uint32_t thr = sh[34], need = sh[35];
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nw; base += NT) {
    const uint32_t w = base + threadIdx.x;
    uint32_t sel = 0, tie = 0;
    if (w < nw) {
      uint32_t bits = word(w);
      const uint32_t rw = Rcur[w];
      const uint32_t kw = allK ? kFull : d.Kb[w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const uint32_t bk = bucket_of(d, 32u * w + b, (kw >> b) & 1u, (rw >> b) & 1u, T);
        if (bk < thr) sel |= 1u << b;
        else if (bk == thr) tie |= 1u << b;
      }
    }
    uint32_t tot;
    const uint32_t off = block_scan<NT>(__popc(tie), tot, sh);
    uint32_t start = carry + off;
    while (tie && start < need) {  // lowest ids of the threshold bucket
      const uint32_t bit = tie & (0u - tie);
      sel |= bit;
      tie ^= bit;
      ++start;
    }
    if (sel) emit(w, sel);
    carry += tot;
  }
  __syncthreads();
}

// ------------------------------------------------------------------- a1 cull
// one CTA: the camera batch from mapped pinned host memory (6 KB at J = 64)
// into device memory, so the plan never queues behind the gather on a copy engine
__global__ void __launch_bounds__(256) k_planes(Dev d, uint32_t J, int parity) {
  for (uint32_t i = threadIdx.x; i < J * 6; i += blockDim.x)
    d.last_planes[parity][i] = d.planes_map[parity][i];
}

__global__ void __launch_bounds__(256) k_cull(Dev d, uint32_t J, int32_t T, int parity) {
  __shared__ float4 pl[kMaxCams * 6];
  for (uint32_t i = threadIdx.x; i < J * 6; i += blockDim.x) pl[i] = d.last_planes[parity][i];
  __syncthreads();
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t w = l >> 5, lane = l & 31;
  const bool in = l < d.Kloc;
  float4 c = in ? d.bounds[l] : make_float4(0.f, 0.f, 0.f, 0.f);
  if (in && d.refresh) {  // R25: the refresh of the step two batches back enters now
    const uint32_t pv = d.pend[parity][l];
    if (pv) {
      if (pv > __float_as_uint(c.w)) {
        c.w = __uint_as_float(pv);
        d.bounds[l].w = c.w;
      }
      d.pend[parity][l] = 0u;
    }
  }
  // Alg. 1 l.2 (R12): blocks accessed by the previous batch (R_t n K_t) get age 0
  if (in && T > 0 && ((d.Ab[w] >> lane) & 1u)) d.last_access[l] = T - 1;
  const float nr = -c.w;
  uint32_t uni = 0;
  for (uint32_t j = 0; j < J; ++j) {
    bool vis = in;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const float4 n = pl[j * 6 + p];
      // R2: d = n.c + d0 as the fmaf chain x -> y -> z with d0 the first addend
      const float dist = __fmaf_rn(n.z, c.z, __fmaf_rn(n.y, c.y, __fmaf_rn(n.x, c.x, n.w)));
      if (dist < nr) vis = false;  // cull iff d < -r_k (NaN stays visible)
    }
    const uint32_t bits = __ballot_sync(kFull, vis);
    if (lane == 0 && w < d.W) d.percam[parity][(size_t)j * d.W + w] = bits;  // tail warps own no word
    uni |= bits;
  }
  if (lane == 0 && w < d.W) {
    const uint32_t kold = d.Kb[w];  // K_t (the previous activate's)
    if (kold | uni) {
      atomicAdd(&d.stats[ST_K_INTER], (unsigned long long)__popc(kold & uni));
      atomicAdd(&d.stats[ST_K_UNION], (unsigned long long)__popc(kold | uni));
    }
    d.Kb[w] = uni;  // Eq. Kt_def: K_{t+1} = U_j K^{(j)}
    const uint32_t cw = d.tide ? (d.R[parity][w] | uni) : uni;  // C_t = R_t u K_{t+1}
    d.cand[w] = cw;
    d.Q[w] = 0u;
    atomicAdd(&d.cnt[CNT_CAND], (uint32_t)__popc(cw));
    atomicAdd(&d.cnt[CNT_K], (uint32_t)__popc(uni));
  }
}

// ------------------------------------------------------ a3 camera quota (R10)
template <int NT>
__global__ void __launch_bounds__(NT) k_quota(Dev d, uint32_t J, int32_t T, int parity) {
  __shared__ uint32_t hist[kMaxBuckets];
  __shared__ uint32_t sh[40];
  if (d.cnt[CNT_CAND] <= d.C) return;  // #C_t <= C: nothing to select
  const uint32_t j = blockIdx.x;
  const uint32_t* pc = d.percam[parity] + (size_t)j * d.W;
  uint32_t mine = 0;
  for (uint32_t w = threadIdx.x; w < d.W; w += NT) mine += __popc(pc[w]);
  const uint32_t nj = block_sum<NT>(mine, sh);
  const uint64_t q = ((uint64_t)d.C * d.quota_num) / ((uint64_t)d.quota_den * J);
  const uint32_t qj = (uint32_t)(nj < q ? nj : q);
  select_top<NT>(
      d, qj, d.W, T, hist, sh, [&](uint32_t w) { return pc[w]; }, d.R[parity], true,
      [&](uint32_t w, uint32_t bits) { atomicOr(&d.Q[w], bits); });
}

// ------------------------------------- a2 + a3 fill, delta, slots, A list
// NT = 256 for bitsets of <= 1024 words (fits beside a running k_adam, whose
// CTAs leave too few registers for a 1024-thread CTA), 1024 above
template <int NT>
__global__ void __launch_bounds__(NT) k_plan(Dev d, int32_t T, int parity) {
  __shared__ uint32_t hist[kMaxBuckets];
  __shared__ uint32_t sh[40];
  __shared__ unsigned long long acc[4];
  const uint32_t tid = threadIdx.x;
  const uint32_t W = d.W;
  const uint32_t* R = d.R[parity];
  uint32_t* Rn = d.R[parity ^ 1];
  const uint32_t n_cand = d.cnt[CNT_CAND];
  if (tid < 4) acc[tid] = 0;

  // ---- Alg. 1 l.6: R_{t+1} = CameraBalancedTopC(...)
  if (n_cand <= d.C) {
    for (uint32_t w = tid; w < W; w += NT) Rn[w] = d.cand[w];
  } else {
    uint32_t mine = 0;
    for (uint32_t w = tid; w < W; w += NT) {
      const uint32_t q = d.Q[w];
      Rn[w] = q;
      mine += __popc(q);
    }
    const uint32_t nQ = block_sum<NT>(mine, sh);
    const uint32_t nfill = d.C - nQ;
    select_top<NT>(
        d, nfill, W, T, hist, sh, [&](uint32_t w) { return d.cand[w] & ~d.Q[w]; }, R, false,
        [&](uint32_t w, uint32_t bits) { Rn[w] |= bits; });
  }
  __syncthreads();

  // ---- Alg. 1 l.7-8: Omega, S+, S-; A = R_{t+1} n K_{t+1}
  uint32_t nR_mine = 0, nOm_mine = 0;
  for (uint32_t w = tid; w < W; w += NT) {
    const uint32_t r = R[w], rn = Rn[w];
    const uint32_t sp = d.tide ? (rn & ~r) : rn;
    const uint32_t sm = d.tide ? (r & ~rn) : r;
    const uint32_t om = d.tide ? (r & rn) : 0u;
    d.Sp[w] = sp;
    d.Sm[w] = sm;
    d.Om[w] = om;
    d.Ab[w] = rn & d.Kb[w];
    nR_mine += __popc(rn);
    nOm_mine += __popc(om);
  }
  const uint32_t nR = block_sum<NT>(nR_mine, sh);
  const uint32_t nOm = block_sum<NT>(nOm_mine, sh);

  // ---- compaction of S+ and S- (ascending ids) by prefix sums
  uint32_t* smb = d.sm_blk[parity];
  uint32_t* sms = d.sm_slot[parity];
  uint32_t* spb = d.sp_blk[parity];
  uint32_t* sps = d.sp_slot[parity];
  uint32_t cSp = 0, cSm = 0;
  for (uint32_t base = 0; base < W; base += NT) {
    const uint32_t w = base + tid;
    uint32_t sp = w < W ? d.Sp[w] : 0u, sm = w < W ? d.Sm[w] : 0u;
    uint32_t tp, tm;
    uint32_t op = cSp + block_scan<NT>(__popc(sp), tp, sh);
    uint32_t om = cSm + block_scan<NT>(__popc(sm), tm, sh);
    while (sp) {
      const int b = __ffs(sp) - 1;
      sp &= sp - 1;
      spb[op++] = 32u * w + b;
    }
    while (sm) {
      const int b = __ffs(sm) - 1;
      sm &= sm - 1;
      const uint32_t l = 32u * w + b;
      smb[om] = l;
      sms[om] = (uint32_t)d.b2s[l];
      ++om;
    }
    cSp += tp;
    cSm += tm;
  }
  const uint32_t nSp = cSp, nSm = cSm;
  __syncthreads();

  // ---- slot allocation (R13): the i-th S+ block takes the i-th lowest slot not
  //      held by R_t; if short, the slots S- releases, ascending.
  uint32_t nfree = 0;
  for (uint32_t base = 0; base < d.PW; base += NT) {
    const uint32_t w = base + tid;
    uint32_t fr = 0;
    if (w < d.PW) {
      const uint32_t valid = (32u * (w + 1) <= d.P) ? kFull : ((1u << (d.P - 32u * w)) - 1u);
      fr = ~d.occ[w] & valid;
    }
    uint32_t tot;
    uint32_t r = nfree + block_scan<NT>(__popc(fr), tot, sh);
    while (fr && r < nSp) {
      const int b = __ffs(fr) - 1;
      fr &= fr - 1;
      sps[r++] = 32u * w + b;
    }
    nfree += tot;
  }
  const uint32_t fallback = nfree < nSp ? 1u : 0u;
  if (fallback) {
    for (uint32_t w = tid; w < d.PW; w += NT) d.rel[w] = 0u;
    __syncthreads();
    for (uint32_t i = tid; i < nSm; i += NT) atomicOr(&d.rel[sms[i] >> 5], 1u << (sms[i] & 31));
    __syncthreads();
    uint32_t c = 0;
    for (uint32_t base = 0; base < d.PW; base += NT) {
      const uint32_t w = base + tid;
      uint32_t fr = w < d.PW ? d.rel[w] : 0u;
      uint32_t tot;
      uint32_t r = nfree + c + block_scan<NT>(__popc(fr), tot, sh);
      while (fr && r < nSp) {
        const int b = __ffs(fr) - 1;
        fr &= fr - 1;
        sps[r++] = 32u * w + b;
      }
      c += tot;
    }
  }
  __syncthreads();

  // ---- eviction bookkeeping (stage 4; dirty write-back decided after Adam(t))
  unsigned long long streak = 0;
  for (uint32_t i = tid; i < nSm; i += NT) {
    const uint32_t l = smb[i], s = sms[i];
    if (d.sm_map) d.sm_map[i] = l;  // f3: the host touches the CPU-cache entries of S-
    d.b2s[l] = -1;
    d.s2b[s] = -1;
    atomicAnd(&d.occ[s >> 5], ~(1u << (s & 31)));
    streak += (unsigned long long)(T - d.admit[l]);
  }
  __syncthreads();
  // ---- admission bookkeeping (stage 2); cold restart resets the step
  unsigned long long readmit = 0;
  for (uint32_t i = tid; i < nSp; i += NT) {
    const uint32_t l = spb[i], s = sps[i];
    d.b2s[l] = (int32_t)s;
    d.s2b[s] = (int32_t)l;
    atomicOr(&d.occ[s >> 5], 1u << (s & 31));
    if (d.ever[l]) ++readmit;
    d.ever[l] = 1;
    d.admit[l] = T;  // (cold restart resets step[l] in the gather: after the last Adam on l)
    d.sp_map[2 * i] = l;
    d.sp_map[2 * i + 1] = s;
  }
  if (streak) atomicAdd(&acc[0], streak);
  if (readmit) atomicAdd(&acc[1], readmit);
  __syncthreads();

  // ---- A = R_{t+1} n K_{t+1} with slots, ascending (what Adam and C1 consume)
  uint32_t* ab = d.a_blk[parity];
  uint32_t* as = d.a_slot[parity];
  uint32_t* ag = d.a_gid[parity];
  uint32_t cA = 0;
  for (uint32_t base = 0; base < W; base += NT) {
    const uint32_t w = base + tid;
    uint32_t a = w < W ? d.Ab[w] : 0u;
    uint32_t tot;
    uint32_t o = cA + block_scan<NT>(__popc(a), tot, sh);
    while (a) {
      const int b = __ffs(a) - 1;
      a &= a - 1;
      const uint32_t l = 32u * w + b;
      ab[o] = l;
      as[o] = (uint32_t)d.b2s[l];
      ag[o] = l * d.G + d.rank;
      ++o;
    }
    cA += tot;
  }
  if (tid == 0) {
    PlanHdr h{};
    h.nK = d.cnt[CNT_K];
    h.nR = nR;
    h.nSp = nSp;
    h.nSm = nSm;
    h.nA = cA;
    h.nOm = nOm;
    h.nfree = nfree;
    h.fallback = fallback;
    h.n_dirty = 0;
    *d.hdr_dev[parity] = h;
    *d.hdr_map = h;
    d.cnt[CNT_CAND] = 0u;  // ready for the next activate's cull
    d.cnt[CNT_K] = 0u;
    unsigned long long* st = d.stats;
    atomicAdd(&st[ST_ITER], 1ull);
    atomicAdd(&st[ST_VISIBLE], (unsigned long long)h.nK);
    atomicAdd(&st[ST_RESIDENT], (unsigned long long)nR);
    atomicAdd(&st[ST_ACTIVE_BLOCKS], (unsigned long long)cA);
    atomicAdd(&st[ST_STAGE_IN], (unsigned long long)nSp);
    atomicAdd(&st[ST_EVICT], (unsigned long long)nSm);
    atomicAdd(&st[ST_H2D], (unsigned long long)nSp * d.rec_floats * 4ull * d.n_arr);
    atomicAdd(&st[ST_STREAK_SUM], acc[0]);
    atomicAdd(&st[ST_STREAK_CNT], (unsigned long long)nSm);
    atomicAdd(&st[ST_READMIT], acc[1]);
  }
}

// ---------------------------------------- a4 dirty S- -> write-back list
template <int NT>
__global__ void __launch_bounds__(NT) k_evict(Dev d, uint32_t nSm, int parity, int ring,
                                              int32_t T, int tag) {
  __shared__ uint32_t sh[40];
  const uint32_t* smb = d.sm_blk[parity];
  const uint32_t* sms = d.sm_slot[parity];
  uint32_t c = 0;
  nSm = count_or_hdr(nSm, d.hdr_dev[parity], 1);
  for (uint32_t base = 0; base < nSm; base += NT) {
    const uint32_t i = base + threadIdx.x;
    uint32_t dirty = 0, l = 0, s = 0;
    if (i < nSm) {
      l = smb[i];
      s = sms[i];
      d.evicted[l] = 1;  // after Adam(t): the cold-restart counter of Adam(t) saw the old value
      dirty = (d.dirty[s >> 5] >> (s & 31)) & 1u;  // dirty only if updated
    }
    uint32_t tot;
    const uint32_t o = c + block_scan<NT>(dirty, tot, sh);
    if (dirty) {
      d.dirty_map[ring][2 * o] = l;
      d.dirty_map[ring][2 * o + 1] = s;
      d.dl_slot[ring][o] = s;
      d.dl_blk[ring][o] = l;
      if (tag) {  // packed into staging[ring][o]: a re-admission within nrings-1 batches reads it there
        d.wb_tag[l] = T;
        d.wb_idx[l] = o;
      } else {    // written back straight from its slot: an older ring record of l is stale
        d.wb_tag[l] = -1;
      }
      atomicAnd(&d.dirty[s >> 5], ~(1u << (s & 31)));
    }
    c += tot;
  }
  if (threadIdx.x == 0) {
    d.ndirty_map[ring] = c;
    d.ndirty_dev[ring] = c;
    atomicAdd(&d.stats[ST_EVICT_DIRTY], (unsigned long long)c);
    atomicAdd(&d.stats[ST_D2H], (unsigned long long)c * d.rec_floats * 4ull * d.n_arr);
  }
}

// ------------------- a4 pack: dirty S- records -> write-back staging ring
// grid (chunks, min(n_dirty, 65535)); entry i < n_dirty copies its slot's theta
// (| m | v when moments persist) into staging[ring][i] with 128-bit streaming
// loads and stores, so the slot is free for the next gather as soon as this
// kernel ends while k_xfer drains the ring to the host tier.
__global__ void __launch_bounds__(256, 6) k_pack(Dev d, int ring) {
  const uint32_t nd = d.ndirty_dev[ring];
  const size_t n4 = (size_t)d.n_arr * d.rec_floats / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.y; i < nd; i += gridDim.y) {  // grid.y is capped at 65535
    const uint32_t s = d.dl_slot[ring][i];
    const float4* src = reinterpret_cast<const float4*>(d.params + (size_t)s * 3 * d.rec_floats);
    float4* dst = reinterpret_cast<float4*>(d.staging[ring] + (size_t)i * d.n_arr * d.rec_floats);
    size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 1
    for (; e + 3 * stride < n4; e += 4 * stride) {  // 4 independent 16 B loads in flight
      const float4 a = __ldcs(src + e), b = __ldcs(src + e + stride);
      const float4 c = __ldcs(src + e + 2 * stride), f = __ldcs(src + e + 3 * stride);
      __stcs(dst + e, a);
      __stcs(dst + e + stride, b);
      __stcs(dst + e + 2 * stride, c);
      __stcs(dst + e + 3 * stride, f);
    }
#pragma unroll 1
    for (; e < n4; e += stride) __stcs(dst + e, __ldcs(src + e));
  }
}

// ------------------- a4 commit (xfer = TGS_XFER_COPY_ENGINE): staged S+ -> slots
// The copy engines have put S+ record i (host tier) at stage_in[i]; entry i goes
// to its slot, except a block packed by one of the last two activates (its host
// write-back may still be in flight), whose newest copy is its ring record --
// the same source rule as k_xfer's gather.  Cold restart resets the block's
// step here (after the last Adam that updated it, as in the gather); with f1/f2
// on, each theta row's centre and log-scales go to geo6 from the registers.
// grid (chunks, min(nSp, 4096)), 256 threads, 128-bit streaming loads/stores.
__global__ void __launch_bounds__(256, 6) k_commit(Dev d, int parity, int32_t T, uint32_t nSp) {
  const size_t n4 = (size_t)d.n_arr * d.rec_floats / 4;
  const size_t th4 = d.rec_floats / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.y; i < nSp; i += gridDim.y) {
    const uint32_t l = d.sp_blk[parity][i], slot = d.sp_slot[parity][i];
    const int32_t tg = d.wb_tag[l];
    const bool ring = tg >= 0 && tg >= T - (d.nrings - 1);
    const float4* src = reinterpret_cast<const float4*>(
        ring ? d.staging[tg % d.nrings] + (size_t)d.wb_idx[l] * d.n_arr * d.rec_floats
             : d.stage_in + (size_t)i * d.n_arr * d.rec_floats);
    float4* dst = reinterpret_cast<float4*>(d.params + (size_t)slot * 3 * d.rec_floats);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (d.cold) d.step[l] = 0u;
      if (ring) atomicAdd(&d.stats[ST_RING_READMIT], 1ull);
    }
    float* g6 = d.geo6 ? d.geo6 + (size_t)slot * d.B * 6 : nullptr;
#pragma unroll 1
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += stride) {
      const float4 v = __ldcs(src + e);
      __stcs(dst + e, v);
      if (g6 && e < th4) {  // theta floats 4e..4e+3: rows' attributes 0..2 and 52..54
        const uint32_t f0 = (uint32_t)(4 * e);
        uint32_t r = f0 / kDim, a = f0 - r * kDim;
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (a < 3u) g6[(size_t)r * 6 + a] = vv[q];
          else if (a >= 52u && a < 55u) g6[(size_t)r * 6 + a - 49u] = vv[q];
          if (++a == kDim) { a = 0; ++r; }
        }
      }
    }
  }
}

// R24 deterministic exp: k = rint(x log2 e) by the 1.5*2^23 trick, two-step
// Cody-Waite reduction, degree-7 Taylor polynomial by fma Horner, exact 2^k.
__device__ __forceinline__ float exp_det(float x) {
  if (x > 80.0f) x = 80.0f;
  if (x < -80.0f) x = -80.0f;
  const float t = __fmaf_rn(x, 1.44269504088896341f, 12582912.0f);
  const float kf = __fsub_rn(t, 12582912.0f);
  float r = __fmaf_rn(kf, -0.693145751953125f, x);
  r = __fmaf_rn(kf, -1.428606765330187045e-06f, r);
  float p = 1.98412698412698413e-04f;
  p = __fmaf_rn(p, r, 1.38888888888888889e-03f);
  p = __fmaf_rn(p, r, 8.33333333333333333e-03f);
  p = __fmaf_rn(p, r, 4.16666666666666667e-02f);
  p = __fmaf_rn(p, r, 1.66666666666666667e-01f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  const int k = (int)kf;
  return __fmul_rn(p, __int_as_float((k + 127) << 23));
}


// f1 / f2 per-row extent sphere (R24, R25): centre mu = attrs 0..2, extent
// 3 (x) exp_det(max of the log-scales 52..54), in the order both filters use
__device__ __forceinline__ float4 row_sphere(float x, float y, float z, float s0, float s1,
                                             float s2) {
  float sc = s0;
  if (s1 > sc) sc = s1;
  if (s2 > sc) sc = s2;
  return make_float4(x, y, z, __fmul_rn(3.0f, exp_det(sc)));
}

// R25 refreshed radius of a row around the fixed centre c_k, as fp32 bits
__device__ __forceinline__ uint32_t refresh_bits(const float4& sp, const float4& c) {
  const float dx = __fsub_rn(sp.x, c.x), dy = __fsub_rn(sp.y, c.y), dz = __fsub_rn(sp.z, c.z);
  const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
  return __float_as_uint(__fmul_rn(__fadd_rn(__fsqrt_rn(d2), sp.w), 1.0000019073486328f));
}

// ------------------------- a4 record transfer over the host link (TMA)
// One kernel per direction moves whole block records between pinned host
// memory (device-mapped, UVA) and HBM: a few CTAs of one warp each, whose lane 0
// streams 32 KB chunks through a ring of shared-memory buffers with bulk
// copies -- cp.async.bulk global->shared (completion on an mbarrier), then
// cp.async.bulk shared->global -- keeping kXferBufs-1 loads and one store in
// flight per CTA.  The copy engines are not used: each chunk is an SM-issued
// PCIe read (gather) or posted write (scatter), and a CTA occupies one SM's
// shared memory but almost none of its issue slots or load/store units, so the
// HBM-bound kernels beside it keep their bandwidth (profiles/linkbench2_r02.txt).
//
// XFER_GATHER   record i < n of S+ (or of the host-selected subset sel[0..n)):
//               l = sp_blk[i] -> slot sp_slot[i].  Source: host record of l
//               (flat tier: l * host_stride; store tier: entry sp_entry[i]), or,
//               for a block the previous activate packed into its write-back
//               ring (wb_tag[l] == T-1), that ring record in HBM -- its host
//               write-back may still be in flight and the ring copy is the newest.
// XFER_SCATTER  dirty record i < ndirty of this activate: write-back ring
//               (ring mode) or its slot (direct mode) -> host record of l
//               (flat: l * host_stride; store: entry ent_of[l]).
// A chunk is 128 whole rows (30,208 B = 32 x 944 B): a gather chunk of theta
// rows is complete in shared memory when its mbarrier fires, so with the f1/f2
// array on (d.geo6) the CTA's 32 lanes copy each admitted row's centre and
// log-scales from it there -- 24 B per row written, nothing re-read.
constexpr uint32_t kXferChunk = 128 * kDim * 4, kXferMaxBufs = 7;
enum XferMode : int { XFER_GATHER = 0, XFER_SCATTER_RING = 1, XFER_SCATTER_DIRECT = 2 };

__device__ __forceinline__ uint32_t smem_addr(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}

__global__ void __launch_bounds__(32) k_xfer(Dev d, int mode, int parity, int ring, int32_t T,
                                             const uint32_t* __restrict__ sel, uint32_t n_sel,
                                             uint32_t nbuf) {
  extern __shared__ __align__(128) unsigned char xbuf[];
  __shared__ __align__(8) unsigned long long bar[kXferMaxBufs];
  const bool leader = threadIdx.x == 0;
  const uint32_t n = mode == XFER_GATHER ? (sel ? n_sel : d.hdr_dev[parity]->nSp) : d.ndirty_dev[ring];
  const uint64_t rec_bytes = (uint64_t)d.n_arr * d.rec_floats * 4ull;
  const uint64_t theta_bytes = d.rec_floats * 4ull;
  const uint32_t per_rec = (uint32_t)((rec_bytes + kXferChunk - 1) / kXferChunk);
  const uint64_t total = (uint64_t)n * per_rec;
  if ((uint64_t)blockIdx.x >= total) return;
  const uint64_t mine = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const bool spheres = mode == XFER_GATHER && d.geo6 != nullptr;
  if (leader) {
    for (uint32_t b = 0; b < nbuf; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // chunk c of this CTA is global chunk blockIdx.x + c * gridDim.x
  auto geo = [&](uint64_t c, const unsigned char*& src, unsigned char*& dst, uint32_t& bytes,
                 uint32_t& slot, uint64_t& off) {
    const uint64_t g = blockIdx.x + c * gridDim.x;
    const uint32_t r = (uint32_t)(g / per_rec);
    off = (g - (uint64_t)r * per_rec) * kXferChunk;
    bytes = (uint32_t)(rec_bytes - off < kXferChunk ? rec_bytes - off : kXferChunk);
    if (mode == XFER_GATHER) {
      const uint32_t i = sel ? sel[r] : r;
      const uint32_t l = d.sp_blk[parity][i];
      slot = d.sp_slot[parity][i];
      const int32_t tg = d.wb_tag[l];
      if (tg >= 0 && tg >= T - (d.nrings - 1)) {  // packed by one of the last nrings-1 activates
        src = reinterpret_cast<const unsigned char*>(d.staging[tg % d.nrings]) +
              (uint64_t)d.wb_idx[l] * rec_bytes;
      } else {
        const uint64_t e = d.ent_of ? (uint64_t)d.sp_entry[i] : (uint64_t)l;
        src = d.host_dev + e * d.host_stride;
      }
      dst = reinterpret_cast<unsigned char*>(d.params + (size_t)slot * 3 * d.rec_floats);
      if (leader && off == 0) {
        // cold restart: the moments start over at step 0.  Done
        // here, not in the plan: the plan may run while an earlier Adam still
        // counts this block's last updates; the gather waits for that Adam
        if (d.cold) d.step[l] = 0u;
        if (d.ent_of) d.ent_of[l] = (int32_t)d.sp_entry[i];  // store tier: entry of a resident block
        if (tg >= 0 && tg >= T - (d.nrings - 1)) atomicAdd(&d.stats[ST_RING_READMIT], 1ull);
      }
    } else {
      const uint32_t l = d.dl_blk[ring][r];
      slot = d.dl_slot[ring][r];
      src = mode == XFER_SCATTER_RING
                ? reinterpret_cast<const unsigned char*>(d.staging[ring]) + (uint64_t)r * rec_bytes
                : reinterpret_cast<const unsigned char*>(d.params + (size_t)slot * 3 * d.rec_floats);
      const uint64_t e = d.ent_of ? (uint64_t)d.ent_of[l] : (uint64_t)l;
      dst = d.host_dev + e * d.host_stride;
    }
    src += off;
    dst += off;
  };
  auto load = [&](uint64_t c) {
    const uint32_t b = (uint32_t)(c % nbuf);
    const unsigned char* src;
    unsigned char* dst;
    uint32_t bytes, slot;
    uint64_t off;
    geo(c, src, dst, bytes, slot, off);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[b])),
                 "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(xbuf + (size_t)b * kXferChunk)),
        "l"(src), "r"(bytes), "r"(smem_addr(&bar[b])) : "memory");
  };
  // nbuf-1 loads in flight; buffer (c-1) % nbuf is refilled once its store has
  // read it (wait_group.read 1: all but the newest store group)
  uint64_t issued = 0;
  if (leader)
    for (; issued < mine && issued < nbuf - 1; ++issued) load(issued);
  uint32_t phase = 0;  // bit b: parity of buffer b's next completion
  for (uint64_t c = 0; c < mine; ++c) {
    const uint32_t b = (uint32_t)(c % nbuf);
    if (leader || spheres) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok) : "r"(smem_addr(&bar[b])), "r"((phase >> b) & 1u) : "memory");
    }
    phase ^= 1u << b;
    const unsigned char* src;
    unsigned char* dst;
    uint32_t bytes, slot;
    uint64_t off;
    if (leader || spheres) geo(c, src, dst, bytes, slot, off);
    if (leader) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"(smem_addr(xbuf + (size_t)b * kXferChunk)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (spheres && off < theta_bytes) {  // theta rows of an admitted block (R24, R25 inputs)
      const uint32_t row0 = (uint32_t)(off / (kDim * 4));
      const uint32_t nrow = d.B - row0 < 128u ? d.B - row0 : 128u;
      const float* rows = reinterpret_cast<const float*>(xbuf + (size_t)b * kXferChunk);
      float* out = d.geo6 + ((size_t)slot * d.B + row0) * 6;
      for (uint32_t e = threadIdx.x; e < 6 * nrow; e += 32) {  // coalesced 24-B rows
        const uint32_t j = e / 6, f = e - 6 * j;
        out[e] = rows[(size_t)j * kDim + (f < 3 ? f : f + 49)];
      }
    }
    __syncwarp();  // every lane is done reading buffer b before it can be refilled
    if (leader && issued < mine) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(issued++);
    }
  }
  if (leader) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    for (uint32_t b = 0; b < nbuf; ++b)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(&bar[b])));
  }
}

// ------------------------------------------------ a5 prologue (per block)
__global__ void __launch_bounds__(256) k_adam_prologue(Dev d, uint32_t nA, int parity,
                                                       const uint32_t* __restrict__ mask) {
  __shared__ unsigned long long acc[5];
  if (threadIdx.x < 5) acc[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  nA = count_or_hdr(nA, d.hdr_dev[parity], 0);
  if (blockIdx.x == 0 && threadIdx.x == 0) *d.adam_ctr = 0u;  // k_adam's dynamic chunk counter
  if (i < nA) {
    const uint32_t l = d.a_blk[parity][i], s = d.a_slot[parity][i];
    const uint32_t rows = block_rows(d, l);
    const uint32_t nw = (d.B + 31) / 32;
    uint32_t n = 0;
    for (uint32_t w = lane; w < nw; w += 32) {
      if (32u * w >= rows) break;
      const uint32_t valid = (32u * (w + 1) <= rows) ? kFull : ((1u << (rows - 32u * w)) - 1u);
      const uint32_t word = mask ? mask[(size_t)s * nw + w] : kFull;
      n += __popc(word & valid);
    }
    n = __reduce_add_sync(kFull, n);
    if (lane == 0) {
      AdamEnt e{};
      e.rows = rows;
      if (n > 0) {  // block holds rows of I_t: update, count, mark dirty
        const uint32_t before = d.step[l];
        const uint32_t ns = before + 1u;  // R7: per-block step counter
        d.step[l] = ns;
        atomicOr(&d.dirty[s >> 5], 1u << (s & 31));
        e.step = ns;
        // cold restart (R6): the moments of an admitted block are zero until its
        // first update; k_adam writes that block's whole m, v record then
        e.fresh = (d.cold && before == 0u) ? 1 : 0;
        e.bc1 = d.lut_bc1[ns];
        e.ibs = d.lut_ibs[ns];
        atomicAdd(&acc[0], 1ull);
        atomicAdd(&acc[1], (unsigned long long)n);
        if (d.cold && before == 0u && d.evicted[l]) atomicAdd(&acc[2], 1ull);
        if (e.fresh) {
          atomicAdd(&acc[3], (unsigned long long)n);
          atomicAdd(&acc[4], 1ull);
        }
      }
      d.ent[i] = e;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (acc[0]) atomicAdd(&d.stats[ST_TOTAL_UPD], acc[0]);
    if (acc[1]) atomicAdd(&d.stats[ST_ACTIVE_ROWS], acc[1]);
    if (acc[2]) atomicAdd(&d.stats[ST_COLD_UPD], acc[2]);
    if (acc[3]) atomicAdd(&d.stats[ST_FRESH_ROWS], acc[3]);
    if (acc[4]) atomicAdd(&d.stats[ST_FRESH_BLOCKS], acc[4]);
  }
}

// ------------------------------------------- f1 Level-2 fine filter -> I_t
// grid (ceil(B/256), nA): one thread per row of an A block.  The row's
// extent sphere (mu, 3 exp(max log-scale)) against every camera that sees the
// block at Level 1, with the Level-1 rule; a ballot per 32
// rows writes the I_t mask word of the slot.
__global__ void __launch_bounds__(256) k_fine(Dev d, uint32_t nA, uint32_t J, int parity,
                                              uint32_t* __restrict__ mask) {
  __shared__ float4 pl[kMaxCams * 6];
  __shared__ uint32_t cams[kMaxCams];
  __shared__ uint32_t wcount[8];
  const uint32_t nw = (d.B + 31) / 32;
  nA = count_or_hdr(nA, d.hdr_dev[parity], 0);
  for (uint32_t i = blockIdx.x; i < nA; i += gridDim.x) {  // one CTA per A block
    const uint32_t l = d.a_blk[parity][i], s = d.a_slot[parity][i];
    // cameras whose Level-1 set K^(j) holds block l (R24): camera j renders only
    // its own visible blocks; compacted in camera order by warp ballots
    const uint32_t j0 = threadIdx.x;  // blockDim 256 >= kMaxCams
    const bool has = j0 < J && ((d.percam[parity][(size_t)j0 * d.W + (l >> 5)] >> (l & 31)) & 1u);
    const uint32_t bal = __ballot_sync(kFull, has);
    if ((threadIdx.x & 31) == 0) wcount[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    uint32_t base = 0, ncam = 0;
    for (uint32_t w = 0; w < 8; ++w) {
      if (w < (threadIdx.x >> 5)) base += wcount[w];
      ncam += wcount[w];
    }
    if (has) {
      const uint32_t pos = base + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
      cams[pos] = j0;
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < ncam * 6; k += blockDim.x)
      pl[k] = d.last_planes[parity][cams[k / 6] * 6 + k % 6];
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < nw * 32; r += blockDim.x) {  // whole warps only
      bool vis = false;
      if (r < block_rows(d, l)) {
        float4 sp;
        if (d.geo6) {  // 24 B per row, kept current by the gather and k_adam
          const float* g6 = d.geo6 + ((size_t)s * d.B + r) * 6;
          sp = row_sphere(g6[0], g6[1], g6[2], g6[3], g6[4], g6[5]);
        } else {
          const float* row = d.params + (size_t)s * 3 * d.rec_floats + (size_t)r * kDim;
          sp = row_sphere(row[0], row[1], row[2], row[52], row[53], row[54]);
        }
        const float nr = -sp.w;
        for (uint32_t j = 0; j < ncam && !vis; ++j) {
          bool in = true;
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            const float4 n = pl[j * 6 + p];
            const float dist = __fmaf_rn(n.z, sp.z, __fmaf_rn(n.y, sp.y, __fmaf_rn(n.x, sp.x, n.w)));
            if (dist < nr) in = false;
          }
          vis = in;
        }
      }
      const uint32_t bits = __ballot_sync(kFull, vis);
      if ((threadIdx.x & 31) == 0) mask[(size_t)s * nw + (r >> 5)] = bits;
    }
    __syncthreads();  // the next block's cameras overwrite the shared lists
  }
}

// -------------------------------- f2 conservative bound refresh (R25)
// grid (ceil(B/256), min(nA, 65535)), after k_adam: every row of an updated
// block gives (|mu - c_k| + 3 exp(max log-scale)) * (1 + 2^-19) in fp32 RN from
// its packed centre / log-scales (24 B, written by the gather and k_adam); the
// block max (on the bit pattern: radii are >= 0) goes to pend[parity][l], which
// the cull of batch t+2 merges into r_k.
__global__ void __launch_bounds__(256) k_refresh(Dev d, uint32_t nA, int parity) {
  nA = count_or_hdr(nA, d.hdr_dev[parity], 0);
  for (uint32_t i = blockIdx.x; i < nA; i += gridDim.x) {  // one CTA per A block
    if (d.ent[i].step == 0u) continue;  // block not updated this step (uniform per CTA)
    const uint32_t l = d.a_blk[parity][i], s = d.a_slot[parity][i];
    const uint32_t rows = block_rows(d, l);
    const float4 ck = d.bounds[l];
    uint32_t bits = 0u;
    for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) {
      const float* g6 = d.geo6 + ((size_t)s * d.B + r) * 6;
      const uint32_t b = refresh_bits(row_sphere(g6[0], g6[1], g6[2], g6[3], g6[4], g6[5]), ck);
      bits = b > bits ? b : bits;
    }
    bits = __reduce_max_sync(kFull, bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicMax(&d.pend[parity][l], bits);
  }
}

// ------------------------------------------------------- a5 masked Adam
// A warp owns a contiguous range of 4-row quads (4 rows = 944 B = 59 float4
// per array); lane f and f+32 (< 59) load float4 #f of theta, m, v, g (128-bit,
// coalesced, streaming).  Element e = 4f+q of the quad belongs to row e/59 and
// attribute e%59, so the per-lane attribute / row maps are loop-invariant.
// Fast path (every row of the quad active, every gradient finite -- the
// NULL-mask steady state): no per-element row logic.  Slow path: partial
// quads, masked rows, non-finite rows (R20).
constexpr int kAdamNT = 256;
constexpr uint32_t kAdamQPW = 16;  // quads per warp (short CTA lifetime: the plan gets SMs)
constexpr uint32_t kAdamMinWaves = 4;  // small launches: fewer quads per warp, >= 4 waves
#ifndef TGS_ADAM_MINB
#define TGS_ADAM_MINB 3  // resident CTAs per SM the register budget targets
#endif

struct AdamConsts {
  float b1, b2, omb1, omb2, eps, ibs;
};

// Eq. masked_update with Adam's u_t (R9 prescribed order, IEEE RN, no contraction)
__device__ __forceinline__ void adam_elem(float& th, float& m, float& v, float g, float ss,
                                          const AdamConsts& k) {
  float mt = __fmul_rn(k.b1, m);
  mt = __fadd_rn(mt, __fmul_rn(k.omb1, g));
  const float g2 = __fmul_rn(g, g);
  float vt = __fmul_rn(k.b2, v);
  vt = __fadd_rn(vt, __fmul_rn(k.omb2, g2));
  m = mt;
  v = vt;
  float den = __fmul_rn(__fsqrt_rn(vt), k.ibs);
  den = __fadd_rn(den, k.eps);
  const float u = __fdiv_rn(mt, den);
  th = __fsub_rn(th, __fmul_rn(ss, u));
}

__device__ __forceinline__ void adam_f4(float4& t, float4& m, float4& v, const float4& g,
                                        const float* ss, const AdamConsts& k, uint32_t sel) {
  if (sel & 1u) adam_elem(t.x, m.x, v.x, g.x, ss[0], k);
  if (sel & 2u) adam_elem(t.y, m.y, v.y, g.y, ss[1], k);
  if (sel & 4u) adam_elem(t.z, m.z, v.z, g.z, ss[2], k);
  if (sel & 8u) adam_elem(t.w, m.w, v.w, g.w, ss[3], k);
}

__device__ __forceinline__ uint32_t nonfinite4(const float4& g) {
  const uint32_t e = 0x7f800000u;
  return ((__float_as_uint(g.x) & e) == e ? 1u : 0u) | ((__float_as_uint(g.y) & e) == e ? 2u : 0u) |
         ((__float_as_uint(g.z) & e) == e ? 4u : 0u) | ((__float_as_uint(g.w) & e) == e ? 8u : 0u);
}

// R20 slow path of k_adam (warp-collective; rare): the rows of the quad whose
// gradient has a non-finite component, and the lowest gid*59+attr among them
// reported to d.nonfinite.  Out of line so that the fast path keeps its
// registers (inlined, it spilled the loop state to local memory).
__device__ __noinline__ uint32_t adam_nonfinite(uint32_t nf0, uint32_t nf1, uint32_t rowsel0,
                                                uint32_t rowsel1, uint32_t lane, uint64_t gid0,
                                                unsigned long long* nonfinite) {
  uint32_t bad = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if ((nf0 >> q) & 1u) bad |= (rowsel0 >> (4 * q)) & 0xFu;
    if ((nf1 >> q) & 1u) bad |= (rowsel1 >> (4 * q)) & 0xFu;
  }
  bad = __reduce_or_sync(kFull, bad);
  unsigned long long best = ~0ull;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t e0 = 4 * lane + q, e1 = 4 * (lane + 32) + q;
    if ((nf0 >> q) & 1u) {
      const unsigned long long idx = (gid0 + e0 / 59) * 59ull + e0 % 59;
      best = idx < best ? idx : best;
    }
    if ((nf1 >> q) & 1u) {
      const unsigned long long idx = (gid0 + e1 / 59) * 59ull + e1 % 59;
      best = idx < best ? idx : best;
    }
  }
  if (best != ~0ull) atomicMin(nonfinite, best);
  return bad;
}

template <bool kSph>
__global__ void __launch_bounds__(kAdamNT, TGS_ADAM_MINB) k_adam(Dev d, uint32_t nA, int parity,
                                                     const uint32_t* __restrict__ mask,
                                                     AdamHyper hp, uint32_t qpw) {
  __shared__ float lr[kDim];
  if (threadIdx.x < kDim) lr[threadIdx.x] = hp.lr[threadIdx.x];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t QB = d.B / 4;
  // host-known count: a non-persistent grid, each warp a contiguous run of qpw
  // (<= kAdamQPW) quads, so CTAs retire continuously and the (high-priority)
  // plan of the next batch can be scheduled while this Adam is still running.
  // Count from the device header (tgs_activate_async): a resident grid whose
  // warps take qpw-quad chunks from a counter the prologue zeroed.
  const bool dynamic = nA == kFromHdr;
  if (dynamic) nA = d.hdr_dev[parity]->nA;
  const uint64_t total = (uint64_t)nA * QB;
  if (dynamic && qpw == 0) {
    qpw = kAdamQPW;
    // chunks small enough that every warp takes >= ~8 of them: with 16-quad
    // chunks a small A (the in-memory configs) left a tail of one chunk per warp.
    // (A static split -- warp w one contiguous range -- was slower still: the
    // warps then stream from ~3.5k scattered places instead of neighbouring ones)
    const uint64_t per = total / (8ull * gridDim.x * (kAdamNT / 32));
    qpw = per < 1 ? 1u : per < (uint64_t)qpw ? (uint32_t)per : qpw;
  }
  const uint64_t wid = (uint64_t)blockIdx.x * (kAdamNT / 32) + (threadIdx.x >> 5);
  uint64_t q0 = wid * qpw;
  uint64_t q1 = q0 + qpw < total ? q0 + qpw : total;
  if (!dynamic && q0 >= q1) return;

  // loop-invariant per-lane maps: rows of the 4 components of float4 #lane and #lane+32
  const bool has1 = lane + 32 < 59;
  uint32_t rowsel0 = 0, rowsel1 = 0;  // bit 4*q + r: component q belongs to row r
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t e0 = 4 * lane + q, e1 = 4 * (lane + 32) + q;
    rowsel0 |= 1u << (4 * q + e0 / 59);
    if (has1) rowsel1 |= 1u << (4 * q + e1 / 59);
  }
  AdamConsts K{hp.b1, hp.b2, hp.omb1, hp.omb2, hp.eps, 1.0f};
  const uint32_t nw = (d.B + 31) / 32;
  const size_t rf = d.rec_floats;

  uint32_t cur = 0xffffffffu;
  uint32_t step = 0, rows = 0, fresh = 0;
  // f1 / f2 (kSph, d.geo6 on): a lane whose float4 holds the centre (attrs
  // 0..2) or a log-scale (52..54) of an updated row also stores that component,
  // post-update, into the row's packed 24-B record: 6 predicated scalar stores
  // per quad, no extra loop state
  auto g6idx = [](uint32_t e) -> uint32_t {  // e in [0, 236) of a quad: row*6 + field, or 0xFF
    const uint32_t a = e % 59;
    const uint32_t f = a < 3 ? a : (a >= 52 && a <= 54) ? a - 49 : 0xFFu;
    return f == 0xFFu ? 0xFFu : (e / 59) * 6 + f;
  };
  float* pg6 = nullptr;
  // per-lane step sizes ss_a = lr[a] / (1 - beta1^s) of float4 #lane and
  // #lane+32, kept in shared memory (each lane reads back only what it wrote):
  // in registers they pushed the loop past the 80-register budget into spills
  __shared__ float4 ss_tab[kAdamNT / 32][64];
  float4* const my_ss = ss_tab[threadIdx.x >> 5];
  // one base pointer per block record: theta at pt, m at pt + rf4, v at
  // pt + 2 rf4 (registers: the loop runs at the 80-register budget of 3 CTAs/SM)
  float4* pt = nullptr;
  const float4* pg = nullptr;
  const uint32_t* pmask = nullptr;
  const size_t rf4 = rf / 4;

  for (;;) {
  if (dynamic) {
    uint32_t ch = 0;
    if (lane == 0) ch = atomicAdd(d.adam_ctr, 1u);
    ch = __shfl_sync(kFull, ch, 0);
    q0 = (uint64_t)ch * qpw;
    if (q0 >= total) break;
    q1 = q0 + qpw < total ? q0 + qpw : total;
  }
  uint32_t i = (uint32_t)(q0 / QB);
  uint32_t quad = (uint32_t)(q0 - (uint64_t)i * QB);
  const uint32_t nq = (uint32_t)(q1 - q0);  // <= qpw
  for (uint32_t k = 0; k < nq; ++k) {
    if (i != cur) {
      cur = i;
      const AdamEnt ent = d.ent[i];
      step = ent.step;
      rows = ent.rows;
      fresh = ent.fresh;
      K.ibs = ent.ibs;
      const uint32_t s = d.a_slot[parity][i];
      pt = reinterpret_cast<float4*>(d.params + (size_t)s * 3 * rf);
      pg = reinterpret_cast<const float4*>(d.grads + (size_t)s * rf);
      pmask = mask ? mask + (size_t)s * nw : nullptr;
      if (kSph) pg6 = d.geo6 + (size_t)s * d.B * 6;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // ss_a = lr[a] / (1 - beta1^s)  (R9)
        const uint32_t e0 = 4 * lane + q, e1 = 4 * (lane + 32) + q;
        reinterpret_cast<float*>(&my_ss[lane])[q] = __fdiv_rn(lr[e0 % 59], ent.bc1);
        reinterpret_cast<float*>(&my_ss[lane + 32])[q] = __fdiv_rn(lr[has1 ? e1 % 59 : 0], ent.bc1);
      }
    }
    const uint32_t r0 = 4u * quad;
    // advance (i, quad) for the next iteration
    if (++quad == QB) {
      quad = 0;
      ++i;
    }
    if (step == 0u) continue;  // no active row in this block: untouched
    const uint32_t valid = r0 >= rows ? 0u : (rows - r0) >= 4u ? 0xFu : ((1u << (rows - r0)) - 1u);
    uint32_t act = valid;
    if (pmask) act &= (pmask[r0 >> 5] >> (r0 & 31)) & 0xFu;
    if (act == 0u && !fresh) continue;  // warp-uniform
    const size_t f0 = (size_t)(r0 / 4) * 59 + lane, f1 = f0 + 32;
    // components of float4 #lane / #lane+32 whose row is active: lanes whose
    // float4s hold only inactive rows skip their loads and stores (masked I_t)
    uint32_t sel0 = 0, sel1 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if ((rowsel0 >> (4 * q)) & act) sel0 |= 1u << q;
      if ((rowsel1 >> (4 * q)) & act) sel1 |= 1u << q;
    }
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 g0 = z, t0 = z, m0 = z, v0 = z, g1 = z, t1 = z, m1 = z, v1 = z;
    if (sel0) {
      g0 = __ldcs(pg + f0);
      t0 = __ldcs(pt + f0);
      if (!fresh) {
        m0 = __ldcs(pt + rf4 + f0);
        v0 = __ldcs(pt + 2 * rf4 + f0);
      }
    }
    if (sel1) {
      g1 = __ldcs(pg + f1);
      t1 = __ldcs(pt + f1);
      if (!fresh) {
        m1 = __ldcs(pt + rf4 + f1);
        v1 = __ldcs(pt + 2 * rf4 + f1);
      }
    }
    const uint32_t nf0 = nonfinite4(g0) & sel0, nf1 = nonfinite4(g1) & sel1;
    uint32_t upd = act;  // rows updated by this quad
    (void)upd;
    if (__any_sync(kFull, (nf0 | nf1) != 0u)) {  // R20: rows with a non-finite g are skipped
      const uint32_t bad = adam_nonfinite(nf0, nf1, rowsel0, rowsel1, lane,
                                          (uint64_t)d.a_gid[parity][cur] * d.B + r0, d.nonfinite);
      upd = act & ~bad;  // Eq. masked_update: unchanged off I_t
      sel0 = sel1 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((rowsel0 >> (4 * q)) & upd) sel0 |= 1u << q;
        if ((rowsel1 >> (4 * q)) & upd) sel1 |= 1u << q;
      }
    }
    // a fresh (cold-restarted) block gets its whole m, v record written: the
    // computed moments of updated rows, zeros for every other row
    if (sel0) {
      const float4 s4 = my_ss[lane];
      const float ss0[4] = {s4.x, s4.y, s4.z, s4.w};
      adam_f4(t0, m0, v0, g0, ss0, K, sel0);
      __stcs(pt + f0, t0);
    }
    if (sel0 || fresh) {
      __stcs(pt + rf4 + f0, m0);
      __stcs(pt + 2 * rf4 + f0, v0);
    }
    if (sel1) {
      const float4 s4 = my_ss[lane + 32];
      const float ss1[4] = {s4.x, s4.y, s4.z, s4.w};
      adam_f4(t1, m1, v1, g1, ss1, K, sel1);
      __stcs(pt + f1, t1);
    }
    if (sel1 || (fresh && has1)) {
      __stcs(pt + rf4 + f1, m1);
      __stcs(pt + 2 * rf4 + f1, v1);
    }
    if (kSph) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((sel0 >> q) & 1u) {
          const uint32_t c0 = g6idx(4 * lane + q);
          if (c0 != 0xFFu) pg6[(size_t)r0 * 6 + c0] = reinterpret_cast<const float*>(&t0)[q];
        }
        if ((sel1 >> q) & 1u) {
          const uint32_t c1 = g6idx(4 * (lane + 32) + q);
          if (c1 != 0xFFu) pg6[(size_t)r0 * 6 + c1] = reinterpret_cast<const float*>(&t1)[q];
        }
      }
    }
  }
  if (!dynamic) break;
  }
}


// ============================================================================
// NEXT f2b: Morton sort + blocking (
// reading R26).  Input: n Gaussians as (cx, cy, cz, max log-scale).
// ============================================================================
constexpr int kRsNT = 256, kRsItems = 16, kRsTile = kRsNT * kRsItems;

__global__ void __launch_bounds__(256) k_lay_aabb(const float4* __restrict__ cs, uint64_t n,
                                                  float* __restrict__ part) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float4 c = cs[i];
    lo[0] = fminf(lo[0], c.x); lo[1] = fminf(lo[1], c.y); lo[2] = fminf(lo[2], c.z);
    hi[0] = fmaxf(hi[0], c.x); hi[1] = fmaxf(hi[1], c.y); hi[2] = fmaxf(hi[2], c.z);
  }
  __shared__ float sh[6][256];
  for (int a = 0; a < 3; ++a) {
    sh[a][threadIdx.x] = lo[a];
    sh[3 + a][threadIdx.x] = hi[a];
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int a = 0; a < 3; ++a) {
        sh[a][threadIdx.x] = fminf(sh[a][threadIdx.x], sh[a][threadIdx.x + w]);
        sh[3 + a][threadIdx.x] = fmaxf(sh[3 + a][threadIdx.x], sh[3 + a][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

__device__ __forceinline__ uint64_t spread3(uint32_t v) {  // 21 bits -> every third bit
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

// R26 quantisation: q = min(2^21-1, floor(((double)p - lo) * inv)), in double
__device__ __forceinline__ uint32_t quant(float p, double lo, double inv) {
  double t = floor(__dmul_rn(__dsub_rn((double)p, lo), inv));
  t = t > 2097151.0 ? 2097151.0 : (t < 0.0 ? 0.0 : t);
  return (uint32_t)t;
}

__global__ void __launch_bounds__(256) k_lay_codes(const float4* __restrict__ cs, uint64_t n,
                                                   double lx, double ly, double lz, double ix,
                                                   double iy, double iz,
                                                   unsigned long long* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 c = cs[i];
  keys[i] = spread3(quant(c.x, lx, ix)) | (spread3(quant(c.y, ly, iy)) << 1) |
            (spread3(quant(c.z, lz, iz)) << 2);
  vals[i] = (uint32_t)i;
}

// LSD radix sort pass, 8-bit digit: per-tile digit histogram (digit-major layout)
__global__ void __launch_bounds__(kRsNT) k_rs_hist(const unsigned long long* __restrict__ keys,
                                                   uint64_t n, int shift, uint32_t ntile,
                                                   uint32_t* __restrict__ counts) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    const uint64_t i = base + (uint64_t)r * kRsNT + threadIdx.x;
    if (i < n) atomicAdd(&h[(uint32_t)(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[(size_t)threadIdx.x * ntile + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of m u32 values: per-CTA scan of kRsTile, block sums, fix-up
__global__ void __launch_bounds__(kRsNT) k_scan_local(uint32_t* __restrict__ v, uint64_t m,
                                                      uint32_t* __restrict__ sums) {
  __shared__ uint32_t sh[40];
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile + (uint64_t)threadIdx.x * kRsItems;
  uint32_t loc[kRsItems], acc = 0;
#pragma unroll
  for (int k = 0; k < kRsItems; ++k) {
    const uint64_t i = base + k;
    loc[k] = i < m ? v[i] : 0u;
    const uint32_t x = loc[k];
    loc[k] = acc;
    acc += x;
  }
  uint32_t tot;
  const uint32_t pre = block_scan<kRsNT>(acc, tot, sh);
#pragma unroll
  for (int k = 0; k < kRsItems; ++k)
    if (base + k < m) v[base + k] = pre + loc[k];
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t* __restrict__ sums, uint32_t m) {
  __shared__ uint32_t sh[40];
  uint32_t carry = 0;
  for (uint32_t b = 0; b < m; b += 1024) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t x = i < m ? sums[i] : 0u;
    uint32_t tot;
    const uint32_t pre = block_scan<1024>(x, tot, sh);
    if (i < m) sums[i] = carry + pre;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kRsNT) k_scan_add(uint32_t* __restrict__ v, uint64_t m,
                                                    const uint32_t* __restrict__ sums) {
  const uint32_t add = sums[blockIdx.x];
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int k = 0; k < kRsItems; ++k) {
    const uint64_t i = base + (uint64_t)k * kRsNT + threadIdx.x;
    if (i < m) v[i] += add;
  }
}

// stable scatter: items of a tile in index order; the rank among equal digits
// comes from __match_any_sync within a warp, per-warp counts across warps and
// a running count across the tile's rounds
__global__ void __launch_bounds__(kRsNT) k_rs_scatter(
    const unsigned long long* __restrict__ kin, const uint32_t* __restrict__ vin,
    unsigned long long* __restrict__ kout, uint32_t* __restrict__ vout, uint64_t n, int shift,
    uint32_t ntile, const uint32_t* __restrict__ offs) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kRsNT / 32][256];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  run[threadIdx.x] = 0;
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    for (int w = 0; w < kRsNT / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const uint64_t i = base + (uint64_t)r * kRsNT + threadIdx.x;
    const bool valid = i < n;
    unsigned long long key = 0;
    uint32_t val = 0, dig = 256 + lane;  // invalid lanes never match a real digit
    if (valid) {
      key = kin[i];
      val = vin[i];
      dig = (uint32_t)(key >> shift) & 255u;
    }
    const uint32_t peers = __match_any_sync(kFull, dig);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) wcnt[warp][dig] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pre = 0;
      for (uint32_t w = 0; w < warp; ++w) pre += wcnt[w][dig];
      const uint32_t pos = offs[(size_t)dig * ntile + blockIdx.x] + run[dig] + pre + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    uint32_t add = 0;
    for (int w = 0; w < kRsNT / 32; ++w) add += wcnt[w][threadIdx.x];
    run[threadIdx.x] += add;
    __syncthreads();
  }
}

// one thread per block: centroid (double, sorted order) and conservative radius
__global__ void __launch_bounds__(128) k_lay_bounds(const float4* __restrict__ cs, uint64_t n,
                                                    uint32_t B, const uint32_t* __restrict__ perm,
                                                    float4* __restrict__ bounds, uint64_t K) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  const uint64_t a0 = k * B, a1 = a0 + B < n ? a0 + B : n;
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (uint64_t p = a0; p < a1; ++p) {
    const float4 c = cs[perm[p]];
    sx = __dadd_rn(sx, (double)c.x);
    sy = __dadd_rn(sy, (double)c.y);
    sz = __dadd_rn(sz, (double)c.z);
  }
  const double cnt = (double)(a1 - a0);
  const float cx = __double2float_rn(__ddiv_rn(sx, cnt)), cy = __double2float_rn(__ddiv_rn(sy, cnt)),
              cz = __double2float_rn(__ddiv_rn(sz, cnt));
  double rad = 0.0;
  for (uint64_t p = a0; p < a1; ++p) {
    const float4 c = cs[perm[p]];
    const double dx = __dsub_rn((double)c.x, (double)cx), dy = __dsub_rn((double)c.y, (double)cy),
                 dz = __dsub_rn((double)c.z, (double)cz);
    const double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                             __dmul_rn(dz, dz)));
    const double e = __dadd_rn(dist, (double)__fmul_rn(3.0f, exp_det(c.w)));
    if (e > rad) rad = e;
  }
  float rf = __double2float_rn(rad);
  if ((double)rf < rad) rf = nextafterf(rf, INFINITY);
  bounds[k] = make_float4(cx, cy, cz, rf);
}

}  // namespace

// ------------------------------------------------------------- launchers
cudaError_t launch_cull(const Dev& d, uint32_t J, int32_t T, int parity, cudaStream_t s) {
  if (d.Kloc == 0) return cudaSuccess;
  if (J) k_planes<<<1, 256, 0, s>>>(d, J, parity);
  const uint32_t grid = (d.Kloc + 255) / 256;
  k_cull<<<grid, 256, 0, s>>>(d, J, T, parity);
  return cudaGetLastError();
}

cudaError_t launch_quota(const Dev& d, uint32_t J, int32_t T, int parity, cudaStream_t s) {
  if (J == 0 || d.Kloc == 0) return cudaSuccess;
  if (d.W <= 1024)
    k_quota<256><<<J, 256, 0, s>>>(d, J, T, parity);
  else
    k_quota<512><<<J, 512, 0, s>>>(d, J, T, parity);
  return cudaGetLastError();
}

cudaError_t launch_plan(const Dev& d, int32_t T, int parity, cudaStream_t s) {
  if (d.W <= 1024 && d.PW <= 1024)
    k_plan<256><<<1, 256, 0, s>>>(d, T, parity);
  else
    k_plan<1024><<<1, 1024, 0, s>>>(d, T, parity);
  return cudaGetLastError();
}

cudaError_t launch_evict_tagged(const Dev& d, uint32_t nSm, int parity, int ring, int32_t T,
                                bool tag, cudaStream_t s) {
  if (nSm <= 1024)  // (kFromHdr > 1024: the count comes from the header)
    k_evict<256><<<1, 256, 0, s>>>(d, nSm, parity, ring, T, tag ? 1 : 0);
  else
    k_evict<1024><<<1, 1024, 0, s>>>(d, nSm, parity, ring, T, tag ? 1 : 0);
  return cudaGetLastError();
}

// grid for a per-A-block kernel: one CTA per block, or a resident-sized
// grid-stride grid when the count is read from the device header
static uint32_t per_block_grid(uint32_t nA) {
  return nA == kFromHdr ? 148u * 4u : (nA < 148u * 64u ? nA : 148u * 64u);
}

// C1 send buffer: the A list's global ids padded to C with 0xFFFFFFFF
__global__ void __launch_bounds__(256) k_pad_active(uint32_t* gid, const PlanHdr* h, uint32_t C) {
  for (uint32_t i = h->nA + blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x)
    gid[i] = 0xFFFFFFFFu;
}

// f3 read-ahead: the Level-1 union of an announced camera batch (the R2 rule of
// k_cull), written to mapped host memory; nothing else is touched
__global__ void __launch_bounds__(256) k_probe(Dev d, const float4* __restrict__ planes, uint32_t J,
                                               uint32_t* __restrict__ out) {
  __shared__ float4 pl[kMaxCams * 6];
  for (uint32_t i = threadIdx.x; i < J * 6; i += blockDim.x) pl[i] = planes[i];
  __syncthreads();
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = l < d.Kloc;
  const float4 c = in ? d.bounds[l] : make_float4(0.f, 0.f, 0.f, 0.f);
  bool any = false;
  for (uint32_t j = 0; j < J && in; ++j) {
    bool vis = true;
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      const float4 n = pl[j * 6 + p];
      const float dist = __fmaf_rn(n.z, c.z, __fmaf_rn(n.y, c.y, __fmaf_rn(n.x, c.x, n.w)));
      if (dist < -c.w) vis = false;
    }
    any = any || vis;
  }
  const uint32_t bits = __ballot_sync(kFull, any);
  if ((threadIdx.x & 31) == 0 && (l >> 5) < d.W) out[l >> 5] = bits;
}

cudaError_t launch_probe(const Dev& d, const float4* planes, uint32_t J, uint32_t* out,
                         cudaStream_t s) {
  k_probe<<<(d.Kloc + 255) / 256, 256, 0, s>>>(d, planes, J, out);
  return cudaGetLastError();
}

cudaError_t launch_refresh(const Dev& d, uint32_t nA, int parity, cudaStream_t s) {
  if (nA == 0) return cudaSuccess;
  k_refresh<<<per_block_grid(nA), 256, 0, s>>>(d, nA, parity);
  return cudaGetLastError();
}

cudaError_t launch_pad_active(uint32_t* gid, const PlanHdr* h, uint32_t C, cudaStream_t s) {
  k_pad_active<<<(C + 255) / 256 < 64 ? (C + 255) / 256 : 64, 256, 0, s>>>(gid, h, C);
  return cudaGetLastError();
}

cudaError_t launch_xfer(const Dev& d, int mode, int parity, int ring, int32_t T,
                        const uint32_t* sel, uint32_t n_sel, uint32_t n_hint, int ctas, int bufs,
                        cudaStream_t s) {
  if (n_hint == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_xfer, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(kXferChunk * kXferMaxBufs));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const uint32_t nbuf = (uint32_t)std::max(2, std::min(bufs, (int)kXferMaxBufs));
  const uint64_t per_rec = ((uint64_t)d.n_arr * d.rec_floats * 4ull + kXferChunk - 1) / kXferChunk;
  const uint64_t chunks = (uint64_t)n_hint * per_rec;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)ctas, chunks));
  k_xfer<<<grid, 32, kXferChunk * nbuf, s>>>(d, mode, parity, ring, T, sel, n_sel, nbuf);
  return cudaGetLastError();
}

cudaError_t launch_pack(const Dev& d, uint32_t nSm, int ring, cudaStream_t s) {
  if (nSm == 0) return cudaSuccess;
  // grid-stride over the dirty records (count from the header: 64 rows of CTAs)
  dim3 grid(16, nSm == kFromHdr ? 64u : (nSm < 4096u ? nSm : 4096u));
  k_pack<<<grid, 256, 0, s>>>(d, ring);
  return cudaGetLastError();
}

cudaError_t launch_commit(const Dev& d, uint32_t nSp, int parity, int32_t T, cudaStream_t s) {
  if (nSp == 0) return cudaSuccess;
  dim3 grid(16, nSp < 4096u ? nSp : 4096u);
  k_commit<<<grid, 256, 0, s>>>(d, parity, T, nSp);
  return cudaGetLastError();
}

cudaError_t launch_adam_prologue(const Dev& d, uint32_t nA, int parity, const uint32_t* mask,
                                 cudaStream_t s) {
  if (nA == 0) return cudaSuccess;
  const uint32_t grid = ((nA == kFromHdr ? d.C : nA) + 7) / 8;
  k_adam_prologue<<<grid, 256, 0, s>>>(d, nA, parity, mask);
  return cudaGetLastError();
}

cudaError_t launch_adam(const Dev& d, uint32_t nA, int parity, const uint32_t* mask,
                        const AdamHyper& hp, int grid_ctas, cudaStream_t s) {
  if (nA == 0) return cudaSuccess;
  if (nA == kFromHdr) {  // count on the device: resident grid, dynamic chunks (<= 16 quads)
    const unsigned grid = (unsigned)std::max(grid_ctas, 1);
    // TGS_ADAM_DYNQPW=1: chunks sized on the device (0); default fixed 16-quad
    // chunks (same-box A/B at 11m: 0.177 vs 0.182 ms/step, profiles/ab_qpw_r02.md)
    static const uint32_t qd = [] {
      const char* e = getenv("TGS_ADAM_DYNQPW");
      return (e && atoi(e) == 1) ? 0u : kAdamQPW;
    }();
    if (d.geo6)
      k_adam<true><<<grid, kAdamNT, 0, s>>>(d, nA, parity, mask, hp, qd);
    else
      k_adam<false><<<grid, kAdamNT, 0, s>>>(d, nA, parity, mask, hp, qd);
    return cudaGetLastError();
  }
  const uint64_t quads = (uint64_t)nA * (d.B / 4);
  // grid_ctas = resident CTAs of the device: a small launch (the in-memory
  // configs) gets fewer quads per warp so that it still spans several waves
  uint32_t qpw = kAdamQPW;
  auto ctas = [&](uint32_t q) { return (quads + (uint64_t)(kAdamNT / 32) * q - 1) /
                                       ((uint64_t)(kAdamNT / 32) * q); };
  while (qpw > 1 && ctas(qpw) < (uint64_t)kAdamMinWaves * (uint64_t)std::max(grid_ctas, 1))
    qpw /= 2;
  const unsigned grid = (unsigned)ctas(qpw);
  if (d.geo6)
    k_adam<true><<<grid, kAdamNT, 0, s>>>(d, nA, parity, mask, hp, qpw);
  else
    k_adam<false><<<grid, kAdamNT, 0, s>>>(d, nA, parity, mask, hp, qpw);
  return cudaGetLastError();
}

cudaError_t launch_fine(const Dev& d, uint32_t nA, uint32_t J, int parity, uint32_t* mask,
                        cudaStream_t s) {
  if (nA == 0) return cudaSuccess;
  k_fine<<<per_block_grid(nA), 256, 0, s>>>(d, nA, J, parity, mask);
  return cudaGetLastError();
}


uint32_t layout_ntile(uint64_t n) { return (uint32_t)((n + kRsTile - 1) / kRsTile); }
uint64_t layout_scan_len(uint64_t n) { return 256ull * layout_ntile(n); }
uint32_t layout_nsums(uint64_t n) { return (uint32_t)((layout_scan_len(n) + kRsTile - 1) / kRsTile); }

// The whole GPU part of tgs_build_layout: AABB (partials reduced on the host,
// exact and order-free), codes, 8 stable 8-bit LSD radix passes over the
// 63-bit codes (ties keep index order), per-block bounds.  *perm_buf returns
// which of b.v[0], b.v[1] holds the sorted indices.
cudaError_t layout_run(const LayoutBufs& b, uint64_t n, uint32_t B, cudaStream_t s,
                       int part_grid, int* perm_buf) {
  k_lay_aabb<<<part_grid, 256, 0, s>>>(reinterpret_cast<const float4*>(b.cs), n, b.part);
  std::vector<float> part((size_t)part_grid * 6);
  cudaError_t e = cudaMemcpyAsync(part.data(), b.part, sizeof(float) * part.size(),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int g = 0; g < part_grid; ++g)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::fmin(lo[a], part[6 * g + a]);
      hi[a] = std::fmax(hi[a], part[6 * g + 3 + a]);
    }
  double inv[3];
  for (int a = 0; a < 3; ++a)
    inv[a] = hi[a] > lo[a] ? 2097151.0 / ((double)hi[a] - (double)lo[a]) : 0.0;
  const unsigned gridn = (unsigned)((n + 255) / 256);
  k_lay_codes<<<gridn, 256, 0, s>>>(reinterpret_cast<const float4*>(b.cs), n, lo[0], lo[1],
                                    lo[2], inv[0], inv[1], inv[2], b.k[0], b.v[0]);
  const uint32_t ntile = layout_ntile(n);
  const uint64_t m = layout_scan_len(n);
  const uint32_t nsums = layout_nsums(n);
  int cur = 0;
  for (int shift = 0; shift < 64; shift += 8) {
    k_rs_hist<<<ntile, kRsNT, 0, s>>>(b.k[cur], n, shift, ntile, b.counts);
    k_scan_local<<<nsums, kRsNT, 0, s>>>(b.counts, m, b.sums);
    k_scan_sums<<<1, 1024, 0, s>>>(b.sums, nsums);
    k_scan_add<<<nsums, kRsNT, 0, s>>>(b.counts, m, b.sums);
    k_rs_scatter<<<ntile, kRsNT, 0, s>>>(b.k[cur], b.v[cur], b.k[cur ^ 1], b.v[cur ^ 1], n,
                                         shift, ntile, b.counts);
    cur ^= 1;
  }
  const uint64_t K = (n + B - 1) / B;
  k_lay_bounds<<<(unsigned)((K + 127) / 128), 128, 0, s>>>(
      reinterpret_cast<const float4*>(b.cs), n, B, b.v[cur], reinterpret_cast<float4*>(b.bounds), K);
  *perm_buf = cur;
  return cudaGetLastError();
}

int adam_grid(int device) {
  int sms = 148, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_adam<false>, kAdamNT, 0);
  if (per < 1) per = 1;
  return sms * per;
}

}  // namespace tgs
