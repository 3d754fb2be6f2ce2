// tidegs_order.cu -- NEXT f4: clustered-TSP view ordering on the GPU
// ("We use a clustered TSP-ordered (no-shuffle) camera sequence";
// 709-712 "applying a clustered traveling-salesperson (TSP) ordering over
// camera poses"; reading R29 of DESIGN.md §3).
//
// M views, each a point of D <= 8 double features.  Every distance is
// d2(a, b) = sum_i (a_i - b_i)^2 accumulated in feature order with explicit
// round-to-nearest double intrinsics (no FMA contraction), every choice an
// argmin/argmax with ties to the lowest index, every mean a sequential sum in
// ascending view index -- so the GPU reaches the same integers as any
// sequential evaluation of R29.
//
//   k_lex          : lexicographically smallest view v0 (grid argmin + last-CTA finish)
//   k_init_step x k: maximin initialisation, one centre per launch
//   Lloyd          : k_assign (grid, centres in smem, change flag), then a stable
//                    counting sort of the views by cluster (k_chunk_count, k_chunk_scan,
//                    k_offsets, k_scatter: ascending member lists) and k_update_lists (warp per
//                    cluster: each member in ascending view index added in turn -> means)
//   k_cluster_tour : one CTA, nearest-neighbour over the non-empty centres
//   k_inner_tour   : one CTA per cluster, nearest-neighbour over its members
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "tidegs.h"

namespace {

constexpr int kMaxD = 8;
constexpr int kNT = 256;

__device__ __forceinline__ double d2(const double* a, const double* b, int D) {
  double s = 0.0;
  for (int i = 0; i < D; ++i) {
    const double t = __dsub_rn(a[i], b[i]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// (value, index) pairs: "better" = smaller value, then smaller index (argmin);
// argmax uses the negated comparison on the value only
struct Best {
  double v;
  uint32_t i;
};
__device__ __forceinline__ bool better_min(const Best& a, const Best& b) {
  return a.v < b.v || (a.v == b.v && a.i < b.i);
}
__device__ __forceinline__ bool better_max(const Best& a, const Best& b) {
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}

template <bool MAX>
__device__ Best block_best(Best x) {
  __shared__ double sv[32];
  __shared__ uint32_t si[32];
  auto pick = [](const Best& a, const Best& b) { return (MAX ? better_max(b, a) : better_min(b, a)) ? b : a; };
  for (int o = 16; o; o >>= 1) {
    Best y{__shfl_down_sync(0xffffffffu, x.v, o), __shfl_down_sync(0xffffffffu, x.i, o)};
    x = pick(x, y);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sv[w] = x.v, si[w] = x.i;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    x = lane < nw ? Best{sv[lane], si[lane]} : Best{MAX ? -1.0 : __longlong_as_double(0x7ff0000000000000ll), 0xffffffffu};
    for (int o = 16; o; o >>= 1) {
      Best y{__shfl_down_sync(0xffffffffu, x.v, o), __shfl_down_sync(0xffffffffu, x.i, o)};
      x = pick(x, y);
    }
    if (lane == 0) sv[0] = x.v, si[0] = x.i;
  }
  __syncthreads();
  Best r{sv[0], si[0]};
  __syncthreads();
  return r;
}

struct Ctl {
  uint32_t v0;          // lexicographically smallest view
  uint32_t changed;     // Lloyd: an assignment changed in this pass
  uint32_t done_ctas;   // last-CTA-done counter
  uint32_t n_tour;      // non-empty clusters in the tour
  uint32_t stop;        // Lloyd converged
  uint32_t iters;       // Lloyd passes that changed an assignment
};

__device__ __forceinline__ bool lex_less(const double* f, int D, uint32_t a, uint32_t b) {
  for (int i = 0; i < D; ++i) {
    const double x = f[(size_t)a * D + i], y = f[(size_t)b * D + i];
    if (x < y) return true;
    if (x > y) return false;
  }
  return a < b;
}

// v0 = lexicographic argmin: per-CTA candidate, the last CTA reduces them
__global__ void k_lex(const double* f, uint32_t M, int D, uint32_t* part, Ctl* ctl) {
  __shared__ uint32_t sb[kNT];
  uint32_t best = UINT32_MAX;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < M; v += gridDim.x * blockDim.x)
    if (best == UINT32_MAX || lex_less(f, D, v, best)) best = v;
  // tree reduction of the lexicographic minimum inside the CTA
  sb[threadIdx.x] = best;
  __syncthreads();
  for (int w = kNT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const uint32_t a = sb[threadIdx.x], c = sb[threadIdx.x + w];
      if (c != UINT32_MAX && (a == UINT32_MAX || lex_less(f, D, c, a))) sb[threadIdx.x] = c;
    }
    __syncthreads();
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sb[0];
    __threadfence();
    last = atomicAdd(&ctl->done_ctas, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  const volatile uint32_t* vp = part;
  uint32_t g = UINT32_MAX;
  for (uint32_t c = threadIdx.x; c < gridDim.x; c += blockDim.x) {
    const uint32_t x = vp[c];
    if (x != UINT32_MAX && (g == UINT32_MAX || lex_less(f, D, x, g))) g = x;
  }
  sb[threadIdx.x] = g;
  __syncthreads();
  for (int w = kNT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const uint32_t a = sb[threadIdx.x], c = sb[threadIdx.x + w];
      if (c != UINT32_MAX && (a == UINT32_MAX || lex_less(f, D, c, a))) sb[threadIdx.x] = c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctl->v0 = sb[0];
    ctl->done_ctas = 0;
  }
}

// maximin step j: fold centre j-1 into mind, then centre j = argmax mind
__global__ void k_init_step(const double* f, uint32_t M, int D, double* mind, double* cen,
                            uint32_t j, Best* part, Ctl* ctl) {
  __shared__ double c[kMaxD];
  if (threadIdx.x < D) {
    const uint32_t src = (j == 0) ? ctl->v0 : 0u;
    c[threadIdx.x] = (j == 0) ? f[(size_t)src * D + threadIdx.x] : cen[(size_t)(j - 1) * D + threadIdx.x];
  }
  __syncthreads();
  if (j == 0) {  // centre 0 = v0
    if (blockIdx.x == 0 && threadIdx.x < D) cen[threadIdx.x] = c[threadIdx.x];
    return;
  }
  Best b{-1.0, UINT32_MAX};
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < M; v += gridDim.x * blockDim.x) {
    const double e = d2(f + (size_t)v * D, c, D);
    double m = (j == 1) ? e : mind[v];
    if (e < m) m = e;
    mind[v] = m;
    const Best x{m, v};
    if (better_max(x, b)) b = x;
  }
  b = block_best<true>(b);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(&ctl->done_ctas, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // the last CTA reduces the per-CTA candidates with all its threads
  const volatile Best* vp = part;
  Best g{-1.0, UINT32_MAX};
  for (uint32_t q = threadIdx.x; q < gridDim.x; q += blockDim.x) {
    const Best x{vp[q].v, vp[q].i};
    if (better_max(x, g)) g = x;
  }
  g = block_best<true>(g);
  if (threadIdx.x < D) cen[(size_t)j * D + threadIdx.x] = f[(size_t)g.i * D + threadIdx.x];
  if (threadIdx.x == 0) ctl->done_ctas = 0;
}

// Lloyd assignment: nearest centre (ties lowest), change flag.  Every Lloyd
// pass is enqueued up front; once a pass changes nothing (ctl->stop) the
// remaining launches return at once, so the host never waits per pass.
__global__ void k_assign(const double* f, uint32_t M, int D, const double* cen, uint32_t k,
                         uint32_t* asg, Ctl* ctl) {
  if (ctl->stop) return;
  extern __shared__ double sc[];
  for (uint32_t i = threadIdx.x; i < k * D; i += blockDim.x) sc[i] = cen[i];
  __syncthreads();
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < M; v += gridDim.x * blockDim.x) {
    double p[kMaxD];
    for (int i = 0; i < D; ++i) p[i] = f[(size_t)v * D + i];
    uint32_t bj = 0;
    double bd = d2(p, sc, D);
    for (uint32_t j = 1; j < k; ++j) {
      const double e = d2(p, sc + (size_t)j * D, D);
      if (e < bd) bd = e, bj = j;
    }
    if (asg[v] != bj) ch = true;
    asg[v] = bj;
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(&ctl->changed, 1u);
}

// end of a pass: stop when nothing changed, else count the pass and re-arm
__global__ void k_lloyd_check(Ctl* ctl) {
  if (ctl->stop) return;
  if (!ctl->changed) {
    ctl->stop = 1u;
  } else {
    ctl->iters += 1;
    ctl->changed = 0u;
  }
}

// ---- stable counting sort of the views by cluster (chunks of kChunk views)
constexpr int kChunk = 256;
constexpr uint32_t kMaxK = 8192;

// per chunk: how many of its views each cluster holds
__global__ void k_chunk_count(uint32_t M, uint32_t k, const uint32_t* asg, uint32_t* chunk_cnt,
                              const Ctl* ctl) {
  if (ctl->stop) return;
  extern __shared__ uint32_t sc_cnt[];
  for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) sc_cnt[j] = 0;
  __syncthreads();
  const uint32_t v = blockIdx.x * kChunk + threadIdx.x;
  if (v < M) atomicAdd(&sc_cnt[asg[v]], 1u);  // a count: order-free
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < k; j += blockDim.x)
    chunk_cnt[(size_t)blockIdx.x * k + j] = sc_cnt[j];
}

// per cluster: exclusive scan over the chunks (in place) and the cluster size
__global__ void k_chunk_scan(uint32_t nchunks, uint32_t k, uint32_t* chunk_cnt, uint32_t* cnt,
                             const Ctl* ctl) {
  if (ctl->stop) return;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  uint32_t run = 0;
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint32_t x = chunk_cnt[(size_t)c * k + j];
    chunk_cnt[(size_t)c * k + j] = run;
    run += x;
  }
  cnt[j] = run;
}

// cluster offsets: exclusive scan of the sizes (one CTA of 1024)
__global__ void k_offsets(uint32_t k, const uint32_t* cnt, uint32_t* off, const Ctl* ctl) {
  if (ctl->stop) return;
  __shared__ uint32_t part[1024];
  const uint32_t per = (k + blockDim.x - 1) / blockDim.x;
  const uint32_t a = threadIdx.x * per, b = min(k, a + per);
  uint32_t sum = 0;
  for (uint32_t j = a; j < b; ++j) sum += cnt[j];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (uint32_t w = 1; w < blockDim.x; w <<= 1) {  // inclusive Hillis-Steele scan
    const uint32_t x = threadIdx.x >= w ? part[threadIdx.x - w] : 0u;
    __syncthreads();
    part[threadIdx.x] += x;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - sum;
  for (uint32_t j = a; j < b; ++j) {
    off[j] = run;
    run += cnt[j];
  }
}

// each chunk places its views in ascending order (one thread walks the chunk,
// so equal clusters keep index order): member lists ascending per cluster
__global__ void k_scatter(uint32_t M, uint32_t k, const uint32_t* asg, const uint32_t* chunk_off,
                          const uint32_t* off, uint32_t* mem, const Ctl* ctl) {
  if (ctl->stop) return;
  extern __shared__ uint32_t sc_pos[];
  for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) sc_pos[j] = 0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t v0 = blockIdx.x * kChunk, v1 = min(M, v0 + kChunk);
  for (uint32_t v = v0; v < v1; ++v) {
    const uint32_t j = asg[v];
    mem[off[j] + chunk_off[(size_t)blockIdx.x * k + j] + sc_pos[j]++] = v;
  }
}

// Lloyd update from the member lists: warp per cluster, lane i (< D) adds
// feature i of each member in ascending view index (R29's sequential sum)
__global__ void k_update_lists(const double* f, int D, double* cen, uint32_t k,
                               const uint32_t* cnt, const uint32_t* off, const uint32_t* mem,
                               const Ctl* ctl) {
  if (ctl->stop) return;
  const uint32_t j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (j >= k || lane >= (uint32_t)D) return;
  const uint32_t n = cnt[j], o = off[j];
  if (n == 0) return;
  double s = 0.0;
  for (uint32_t m = 0; m < n; ++m) s = __dadd_rn(s, f[(size_t)mem[o + m] * D + lane]);
  cen[(size_t)j * D + lane] = __ddiv_rn(s, (double)n);
}

// nearest-neighbour tour over the non-empty centres from the cluster of v0
__global__ void k_cluster_tour(const double* cen, int D, uint32_t k, const uint32_t* cnt,
                               const uint32_t* asg, uint32_t* tour, uint8_t* used, Ctl* ctl) {
  for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) used[j] = cnt[j] == 0;
  __syncthreads();
  uint32_t cur = asg[ctl->v0];
  uint32_t n = 0;
  if (threadIdx.x == 0) used[cur] = 1, tour[0] = cur;
  n = 1;
  __syncthreads();
  for (;;) {
    Best b{__longlong_as_double(0x7ff0000000000000ll), UINT32_MAX};
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
      if (used[j]) continue;
      const Best x{d2(cen + (size_t)cur * D, cen + (size_t)j * D, D), j};
      if (better_min(x, b)) b = x;
    }
    b = block_best<false>(b);
    if (b.i == UINT32_MAX) break;
    if (threadIdx.x == 0) used[b.i] = 1, tour[n] = b.i;
    ++n;
    cur = b.i;
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->n_tour = n;
}

// one CTA per tour position: nearest-neighbour over the cluster's members,
// from v0 (first cluster) or the member nearest to the preceding centre
__global__ void k_inner_tour(const double* f, int D, const double* cen, const uint32_t* tour,
                             const uint32_t* cnt, const uint32_t* off, const uint32_t* mem,
                             const uint32_t* tour_off, uint8_t* used_all, uint32_t* perm,
                             const Ctl* ctl) {
  const uint32_t ci = blockIdx.x;
  if (ci >= ctl->n_tour) return;
  const uint32_t j = tour[ci];
  const uint32_t n = cnt[j];
  const uint32_t* ms = mem + off[j];
  uint8_t* used = used_all + off[j];
  uint32_t* out = perm + tour_off[ci];
  for (uint32_t m = threadIdx.x; m < n; m += blockDim.x) used[m] = 0;
  __syncthreads();
  Best b{__longlong_as_double(0x7ff0000000000000ll), UINT32_MAX};
  if (ci == 0) {
    for (uint32_t m = threadIdx.x; m < n; m += blockDim.x)
      if (ms[m] == ctl->v0) b = Best{0.0, m};
  } else {
    const double* pc = cen + (size_t)tour[ci - 1] * D;
    for (uint32_t m = threadIdx.x; m < n; m += blockDim.x) {
      const Best x{d2(f + (size_t)ms[m] * D, pc, D), m};
      if (better_min(x, b)) b = x;
    }
  }
  b = block_best<false>(b);
  uint32_t cur = b.i;
  for (uint32_t step = 0; step < n; ++step) {
    if (threadIdx.x == 0) used[cur] = 1, out[step] = ms[cur];
    __syncthreads();
    if (step + 1 == n) break;
    Best nb{__longlong_as_double(0x7ff0000000000000ll), UINT32_MAX};
    const double* pcur = f + (size_t)ms[cur] * D;
    for (uint32_t m = threadIdx.x; m < n; m += blockDim.x) {
      if (used[m]) continue;
      const Best x{d2(f + (size_t)ms[m] * D, pcur, D), m};
      if (better_min(x, nb)) nb = x;
    }
    nb = block_best<false>(nb);
    cur = nb.i;
  }
}

}  // namespace

extern "C" tgs_status tgs_order_views(const double* feat, uint32_t M, uint32_t D, int device,
                                      uint32_t* perm, uint32_t* cluster, uint32_t* k_out,
                                      uint32_t* iters_out, double* gpu_ms) {
  if (!feat || !perm || M == 0 || D == 0 || D > kMaxD) return TGS_EINVAL;
  for (size_t i = 0; i < (size_t)M * D; ++i)
    if (!(feat[i] - feat[i] == 0.0)) return TGS_EINVAL;  // non-finite
  uint32_t k = 1;
  while ((uint64_t)k * k < M) ++k;  // R29 step 1
  if ((size_t)k * D * sizeof(double) > 200 * 1024 || k > kMaxK) return TGS_EINVAL;  // smem
  if (cudaSetDevice(device) != cudaSuccess) return TGS_ECUDA;
  const int grid = (int)std::min<uint64_t>(148 * 4, ((uint64_t)M + kNT - 1) / kNT);
  std::vector<void*> allocs;
  bool ok = true;
  auto get = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) {
      ok = false;
      return nullptr;
    }
    allocs.push_back(p);
    return p;
  };
  double* d_f = (double*)get((size_t)M * D * 8);
  double* d_mind = (double*)get((size_t)M * 8);
  double* d_cen = (double*)get((size_t)k * D * 8);
  uint32_t* d_asg = (uint32_t*)get((size_t)M * 4);
  uint32_t* d_cnt = (uint32_t*)get((size_t)k * 4);
  uint32_t* d_off = (uint32_t*)get((size_t)k * 4);
  uint32_t* d_mem = (uint32_t*)get((size_t)M * 4);
  uint32_t* d_tour = (uint32_t*)get((size_t)k * 4);
  uint32_t* d_toff = (uint32_t*)get((size_t)k * 4);
  uint8_t* d_used = (uint8_t*)get((size_t)M + k);
  uint32_t* d_perm = (uint32_t*)get((size_t)M * 4);
  const uint32_t nchunks = (M + kChunk - 1) / kChunk;
  uint32_t* d_chunk = (uint32_t*)get((size_t)nchunks * k * 4);
  uint32_t* d_part = (uint32_t*)get((size_t)grid * 16);
  Ctl* d_ctl = (Ctl*)get(sizeof(Ctl));
  Ctl* h_ctl = nullptr;
  auto release = [&]() {
    for (void* p : allocs) cudaFree(p);
    if (h_ctl) cudaFreeHost(h_ctl);
    cudaGetLastError();
  };
  if (!ok || cudaHostAlloc((void**)&h_ctl, sizeof(Ctl), cudaHostAllocDefault) != cudaSuccess) {
    release();
    return TGS_ENOMEM;
  }
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  tgs_status st = TGS_OK;
  uint32_t it = 0;
  const size_t smem = (size_t)k * D * 8;
#define CKO(x) do { if ((x) != cudaSuccess) { st = TGS_ECUDA; goto out; } } while (0)
  CKO(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CKO(cudaEventCreate(&e0));
  CKO(cudaEventCreate(&e1));
  CKO(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CKO(cudaMemcpyAsync(d_f, feat, (size_t)M * D * 8, cudaMemcpyHostToDevice, s));
  CKO(cudaMemsetAsync(d_ctl, 0, sizeof(Ctl), s));
  CKO(cudaMemsetAsync(d_asg, 0xff, (size_t)M * 4, s));
  CKO(cudaEventRecord(e0, s));
  k_lex<<<grid, kNT, 0, s>>>(d_f, M, (int)D, d_part, d_ctl);
  for (uint32_t j = 0; j < k; ++j)  // R29 step 2
    k_init_step<<<grid, kNT, 0, s>>>(d_f, M, (int)D, d_mind, d_cen, j, (Best*)d_part, d_ctl);
  CKO(cudaGetLastError());
  for (uint32_t pass = 0; pass < 100; ++pass) {  // R29 step 3, no host round trip per pass
    k_assign<<<grid, kNT, smem, s>>>(d_f, M, (int)D, d_cen, k, d_asg, d_ctl);
    k_lloyd_check<<<1, 1, 0, s>>>(d_ctl);
    // members of every cluster in ascending index, then the ordered-sum means;
    // after the last pass that changed something these lists are the final ones
    k_chunk_count<<<nchunks, kChunk, k * 4, s>>>(M, k, d_asg, d_chunk, d_ctl);
    k_chunk_scan<<<(k + 127) / 128, 128, 0, s>>>(nchunks, k, d_chunk, d_cnt, d_ctl);
    k_offsets<<<1, 1024, 0, s>>>(k, d_cnt, d_off, d_ctl);
    k_scatter<<<nchunks, kChunk, k * 4, s>>>(M, k, d_asg, d_chunk, d_off, d_mem, d_ctl);
    k_update_lists<<<(k + 7) / 8, 256, 0, s>>>(d_f, (int)D, d_cen, k, d_cnt, d_off, d_mem, d_ctl);
  }
  CKO(cudaGetLastError());
  {
    // cluster tour, tours inside clusters (member lists of the final assignment)
    std::vector<uint32_t> cnt(k);
    CKO(cudaMemcpyAsync(cnt.data(), d_cnt, k * 4, cudaMemcpyDeviceToHost, s));
    k_cluster_tour<<<1, 1024, 0, s>>>(d_cen, (int)D, k, d_cnt, d_asg, d_tour, d_used + M, d_ctl);
    std::vector<uint32_t> tour(k);
    CKO(cudaMemcpyAsync(tour.data(), d_tour, k * 4, cudaMemcpyDeviceToHost, s));
    CKO(cudaMemcpyAsync(h_ctl, d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    CKO(cudaStreamSynchronize(s));
    it = h_ctl->iters;
    std::vector<uint32_t> toff(k, 0);
    uint32_t acc = 0;
    for (uint32_t c = 0; c < h_ctl->n_tour; ++c) toff[c] = acc, acc += cnt[tour[c]];
    CKO(cudaMemcpyAsync(d_toff, toff.data(), k * 4, cudaMemcpyHostToDevice, s));
    k_inner_tour<<<h_ctl->n_tour, 256, 0, s>>>(d_f, (int)D, d_cen, d_tour, d_cnt, d_off, d_mem,
                                               d_toff, d_used, d_perm, d_ctl);
    CKO(cudaGetLastError());
    CKO(cudaEventRecord(e1, s));
    CKO(cudaMemcpyAsync(perm, d_perm, (size_t)M * 4, cudaMemcpyDeviceToHost, s));
    if (cluster) CKO(cudaMemcpyAsync(cluster, d_asg, (size_t)M * 4, cudaMemcpyDeviceToHost, s));
    CKO(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (gpu_ms) *gpu_ms = ms;
    if (k_out) *k_out = k;
    if (iters_out) *iters_out = it;
  }
out:
#undef CKO
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  release();
  return st;
}
