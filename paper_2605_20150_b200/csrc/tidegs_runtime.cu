// tidegs_runtime.cu -- host runtime behind the C ABI of include/tidegs.h.
//
// Owns the pinned host tier (one shard of Theta, M, V as block records), the
// device slot pool, the streams/events of the pipeline, the plan readback and
// an I/O thread for the write-back.  Per activate t (parity p = t & 1;
// DESIGN.md §2):
//
//   plan stream    : [lists of p free: Adam/evict/gather of t-2 done]
//                    k_cull -> k_quota -> k_plan                       (a1-a3)
//   host           : wait for the plan only (never for an Adam)
//   h2d stream     : [slots freed by t-1, host records written by t-2]
//                    k_xfer gather: S+ records host tier -> slots over PCIe
//                    (a block packed by t-1 comes from its ring record instead)
//                    -> ready[p]   (cold-restart zeros are folded into k_adam)
//   compute stream : [after Adam(t-1)] k_evict (dirty S-) -> k_pack (slots ->
//                    staging ring p) -> evict[p]                        (a4)
//   d2h stream     : [evict[p]] k_xfer scatter: ring p -> host tier -> d2h[p]
//   step_adam      : compute waits ready[p]; k_adam_prologue; k_adam   (a5)
//
// S+ always lands in slots that R_t does not hold (R13), so the gather of
// batch t overlaps Adam of batch t-1; the write-back of t is decided after
// Adam(t-1) (R14) without blocking the caller: every step of the chain is a
// GPU-side dependency, the host waits only for the plan.  The host link is
// driven by the transfer kernels (TMA bulk copies to / from device-mapped
// pinned memory), not by the copy engines.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "tidegs.h"
#include "tidegs_internal.h"
#include "tidegs_store.h"

using namespace tgs;

namespace {

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  bool armed = false;
};

}  // namespace

struct tgs_ctx {
  tgs_config cfg{};
  Dev d{};
  uint64_t K = 0;                 // global blocks
  uint64_t rec_bytes = 0;         // B*59*4
  int device = 0;
  // allocator
  tgs_allocator alloc{};
  bool has_alloc = false;
  std::vector<void*> dev_allocs;
  // host tier: [Kloc][n_arr][B][59]; or (NEXT f3) a CPU cache of H records over
  // the log-structured store on SSD
  float* host = nullptr;
  size_t host_bytes = 0;
  tgs::BlockStore* store = nullptr;
  // A = R n K lists of the last three activates (index T % 3): the plan of t+2
  // may then overwrite its parity's other lists while Adam(t) still reads its A
  uint32_t *a3_blk[3] = {}, *a3_slot[3] = {}, *a3_gid[3] = {};
  char* cache_pool = nullptr;     // [H][S] pinned (store mode)
  uint32_t* sm_map = nullptr;     // mapped host [C] S- local ids (store mode, written by k_plan)
  // mapped pinned
  PlanHdr* hdr = nullptr;         // host view
  uint32_t* sp_map = nullptr;     // host view
  uint32_t* dirty_map[kRings] = {};  // host views (ring slot T % nrings)
  uint32_t* ndirty = nullptr;     // host view [kRings]
  float* planes_pinned = nullptr; // [3][kMaxCams*24] mapped staging: camera batches (parity), prefetch
  uint32_t* probe_map = nullptr;  // mapped host [W] Level-1 union of an announced batch (prefetch)
  cudaEvent_t ev_probe = nullptr;
  // streams / events (ev_*[p]: last record by an activate of parity p)
  cudaStream_t compute = nullptr, plan = nullptr, h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_plan = nullptr;
  // lists of activate T (S+, S-, K^(j), header, camera batch, A) live in list slot
  // T % 3: the plan of T+3 reuses them once their consumers of T are done
  cudaEvent_t ev_ready[3] = {}, ev_lists[3] = {};
  cudaEvent_t ev_refresh[2] = {};  // R25: the refresh of the step of that parity done
  cudaEvent_t ev_planes[3] = {};   // k_planes of the activate of that list slot done
  bool rec_planes[3] = {};
  bool rec_refresh[2] = {};
  uint32_t *l3_percam[3] = {}, *l3_sp_blk[3] = {}, *l3_sp_slot[3] = {}, *l3_sm_blk[3] = {},
           *l3_sm_slot[3] = {};
  PlanHdr* l3_hdr[3] = {};
  float4* l3_planes[3] = {};
  const float4* l3_planes_map[3] = {};
  cudaEvent_t ev_evict[kRings] = {}, ev_d2h[kRings] = {};  // by ring slot T % nrings
  // write-back ring slots in use: 5 on the flat tier (a churn burst's write-backs may
  // lag four activates before a gather or a pack waits for them), 3 with the store tier
  // (whose CPU-cache bookkeeping waits for write-backs of at most T-4)
  int nrings = 3;
  cudaEvent_t ev_job[4] = {};      // write-back of activate J done: ev_job[J & 3] (store mode)
  bool rec_ready[3] = {}, rec_lists[3] = {}, rec_evict[kRings] = {};
  int32_t d2h_job[kRings] = {-1, -1, -1, -1, -1};  // activate whose write-back last used ring slot k
  bool ring_direct[kRings] = {};   // ... and whether it wrote back straight from its slots
  int last_evict_ring = -1;        // ring slot of the most recent write-back kernels
  // a4 transfer kernels: CTAs of the gather (h2d) and the write-back (d2h)
  // (TGS_GATHER_CTAS / TGS_SCATTER_CTAS; defaults from profiles/linkbench2_r02.txt)
  int gather_ctas = 8, scatter_ctas = 4, gather_bufs = 4, scatter_bufs = 4;
  // xfer = TGS_XFER_COPY_ENGINE (flat tier): runs of consecutive records move by
  // copy-engine copies; the write-backs are issued by the I/O thread
  bool ce = false;
  cudaStream_t cm = nullptr;            // k_commit (high priority)
  // TGS_CE_STREAMS=2: the run copies of each direction alternate between two
  // streams (two copy engines), joined by an event (ev_fork / ev_join per direction)
  int ce_streams = 1;
  // TGS_WB_KERNEL (copy-engine mode): the write-back as the TMA kernel with N CTAs
  // (default 2: the gather, which gates Adam, keeps more of the link;
  // profiles/ab_wbk_r02.md), 0 = copy-engine runs from the I/O thread, -n = n CTAs
  // while the write-backs keep up and scatter_ctas when the previous one is late
  int wb_kernel = 2;
  int last_d2h_ring = -1;    // ring slot of the newest kernel write-back
  cudaStream_t h2d2 = nullptr, d2h2 = nullptr;
  cudaEvent_t ev_hfork = nullptr, ev_hjoin = nullptr, ev_dfork = nullptr, ev_djoin = nullptr;
  cudaEvent_t ev_copies = nullptr, ev_commit[2] = {};  // stage_in buffer T & 1 copied / read
  bool rec_commit[2] = {};
  // store tier, per parity (the host fills them while the other parity's gather may still run):
  uint32_t* sel_map[2][2] = {};               // mapped host [C]: S+ subsets (hits, misses)
  uint32_t* sp_entry_map[2] = {};             // mapped host [C]: cache entry of S+ block i
  int32_t h2d_prof = -1;           // pending timer of the last gather (bytes known after the readback)
  // C1 / C2 collectives (tgs_set_comm)
  tgs_comm comm{};
  bool has_comm = false;
  uint32_t* c1_recv[3] = {};  // [G][C] gathered A lists (list slot)
  unsigned long long* c2_buf = nullptr;       // [ST_N] summed cumulative counters
  cudaEvent_t ev_c1[3] = {};
  // I/O thread (store tier: marks the CPU-cache entries of each write-back dirty)
  struct Job { int32_t T; int parity; bool direct; };
  std::thread io;
  std::mutex mu;
  std::condition_variable cv_job, cv_done;
  std::deque<Job> jobs;
  int32_t inflight = -1;
  bool stop = false;
  std::atomic<bool> io_failed{false};
  std::string io_err;
  uint32_t last_ndirty = 0;
  std::mutex prof_mu;
  // (the list slot of activate T is released once Adam(T) -- and its refresh --
  // is done: with three list slots the plan of T+3 is what waits for it)
  // Adam LUT (bias corrections, R9)
  std::vector<float> lut_bc1_h, lut_ibs_h;
  float* lut_pinned = nullptr;     // [2][lut_cap]
  uint32_t lut_cap = 0, lut_n = 0;
  float lut_b1 = NAN, lut_b2 = NAN;
  int adam_grid = 0;
  // state
  int32_t T = 0;                  // activates so far
  int parity = 0;                 // parity of R_t (current)
  int last_parity = 0;            // parity the last activate wrote lists into
  bool can_step = false;
  bool poisoned = false;
  PlanHdr last{};                 // header of the last activate (when last_known)
  bool last_known = false;        // false after tgs_activate_async: counts are on the device
  uint32_t last_J = 0;            // batch size of the last activate
  uint64_t n_steps = 0;
  uint64_t host_flush_bytes = 0, host_flush_blocks = 0;
  std::string err;
  // profiling
  bool prof = false;
  tgs_timing tm{};
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { cudaEvent_t a, b; int kind; uint64_t bytes; int32_t iter; };
  std::vector<Pending> pending;
  bool trace = false;             // TGS_TRACE=1: print every timed span (stderr)
  cudaEvent_t trace_base = nullptr;
};

namespace {

void set_err(tgs_ctx* c, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      c->poisoned = true;                                                             \
      set_err(c, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return TGS_ECUDA;                                                               \
    }                                                                                 \
  } while (0)

void* dalloc(tgs_ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~(size_t)255;
  void* p = nullptr;
  if (c->has_alloc) {
    p = c->alloc.alloc(bytes, (void*)c->compute, c->alloc.user);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
  }
  if (p) c->dev_allocs.push_back(p);
  return p;
}

template <class T>
T* dalloc_t(tgs_ctx* c, size_t n, bool& ok) {
  T* p = static_cast<T*>(dalloc(c, n * sizeof(T)));
  if (!p) ok = false;
  return p;
}

cudaEvent_t prof_event(tgs_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// kinds: 0 adam, 1 prologue, 2 plan, 3 h2d, 4 d2h, 5 evict
void prof_begin(tgs_ctx* c, cudaStream_t s, Timer& t) {
  if (!c->prof) return;
  std::lock_guard<std::mutex> g(c->prof_mu);
  t.a = prof_event(c);
  t.b = prof_event(c);
  cudaEventRecord(t.a, s);
  t.armed = true;
}
int32_t prof_end(tgs_ctx* c, cudaStream_t s, Timer& t, int kind, uint64_t bytes = 0) {
  if (!t.armed) return -1;
  std::lock_guard<std::mutex> g(c->prof_mu);
  cudaEventRecord(t.b, s);
  c->pending.push_back({t.a, t.b, kind, bytes, c->T});
  return (int32_t)c->pending.size() - 1;
}
void prof_collect(tgs_ctx* c) {
  std::lock_guard<std::mutex> g(c->prof_mu);
  static const char* names[] = {"adam", "prologue", "plan", "h2d", "d2h", "evict+pack", "commit", "-", "fine"};
  for (auto& p : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) != cudaSuccess) ms = 0.f;
    if (c->trace && c->trace_base) {
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, c->trace_base, p.a);
      fprintf(stderr, "[tgs trace] it %d %-10s %9.3f .. %9.3f ms (%7.3f) %llu B\n", p.iter,
              names[p.kind], t0, t0 + ms, ms, (unsigned long long)p.bytes);
    }
    switch (p.kind) {
      case 0: c->tm.adam_ms += ms; c->tm.adam_launches++; break;
      case 1: c->tm.adam_prologue_ms += ms; break;
      case 2: c->tm.plan_ms += ms; c->tm.plan_launches++; break;
      case 3: c->tm.h2d_ms += ms; c->tm.h2d_batches++; c->tm.h2d_bytes += p.bytes; break;
      case 4: c->tm.d2h_ms += ms; c->tm.d2h_batches++; c->tm.d2h_bytes += p.bytes; break;
      case 5: c->tm.evict_ms += ms; break;
      case 6: case 7: break;
      case 8: c->tm.fine_ms += ms; break;
    }
    c->ev_pool.push_back(p.a);
    c->ev_pool.push_back(p.b);
  }
  c->pending.clear();
  cudaGetLastError();
}

// Host LUT of the selection key (R4, R5, R11): rank of every (m, b) pair by
// descending score s = lam*m + (1-lam)*gamma^b, evaluated in double with
// gamma^b by repeated multiplication; b = max_age+1 means never accessed
// (Recency 0).  Pairs with equal doubles share a rank.
void build_rank_lut(const tgs_config& g, std::vector<uint16_t>& lut, uint32_t& n_ranks) {
  const uint32_t cols = g.max_age + 2;
  std::vector<double> score(2 * cols);
  for (uint32_t m = 0; m < 2; ++m) {
    double rec = 1.0;
    for (uint32_t b = 0; b < cols; ++b) {
      const double recency = (b == cols - 1) ? 0.0 : rec;
      score[m * cols + b] = g.lambda * (double)m + (1.0 - g.lambda) * recency;
      rec *= g.gamma;
    }
  }
  std::vector<double> uniq(score);
  std::sort(uniq.begin(), uniq.end(), [](double a, double b) { return a > b; });
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  lut.resize(2 * cols);
  for (uint32_t i = 0; i < 2 * cols; ++i)
    lut[i] = (uint16_t)(std::lower_bound(uniq.begin(), uniq.end(), score[i],
                                         [](double a, double b) { return a > b; }) -
                        uniq.begin());
  n_ranks = (uint32_t)uniq.size();
}

// bias-correction LUT entry s (R9): 1 - beta^s evaluated in double, rounded to fp32
void lut_entry(float b1, float b2, uint32_t s, float& bc1, float& ibs) {
  bc1 = (float)(1.0 - std::pow((double)b1, (double)s));
  const float bc2 = (float)(1.0 - std::pow((double)b2, (double)s));
  ibs = 1.0f / std::sqrt(bc2);
}

tgs_status ensure_lut(tgs_ctx* c, float b1, float b2, uint32_t need) {
  // need: entries [0, need) must be valid
  if (need > c->lut_cap) {
    uint32_t cap = std::max<uint32_t>(c->lut_cap * 2, 1u << 16);
    while (cap < need) cap *= 2;
    CK(cudaStreamSynchronize(c->compute));
    float *bc = nullptr, *ib = nullptr;
    bool ok = true;
    bc = dalloc_t<float>(c, cap, ok);
    ib = dalloc_t<float>(c, cap, ok);
    if (!ok) return TGS_ENOMEM;
    if (c->lut_pinned) cudaFreeHost(c->lut_pinned);
    CK(cudaHostAlloc((void**)&c->lut_pinned, sizeof(float) * 2 * cap, cudaHostAllocDefault));
    c->d.lut_bc1 = bc;
    c->d.lut_ibs = ib;
    c->lut_cap = cap;
    c->lut_n = 0;  // re-upload
  }
  if (!(b1 == c->lut_b1) || !(b2 == c->lut_b2)) {
    CK(cudaStreamSynchronize(c->compute));  // pending uploads read the pinned mirror
    c->lut_n = 0;
    c->lut_b1 = b1;
    c->lut_b2 = b2;
  }
  if (need > c->lut_n) {
    // fill the whole capacity at once: one upload per (re)build, none per step
    for (uint32_t s = c->lut_n; s < c->lut_cap; ++s)
      lut_entry(b1, b2, s, c->lut_pinned[s], c->lut_pinned[c->lut_cap + s]);
    const size_t n = c->lut_cap - c->lut_n;
    CK(cudaMemcpyAsync(c->d.lut_bc1 + c->lut_n, c->lut_pinned + c->lut_n, n * sizeof(float),
                       cudaMemcpyHostToDevice, c->compute));
    CK(cudaMemcpyAsync(c->d.lut_ibs + c->lut_n, c->lut_pinned + c->lut_cap + c->lut_n,
                       n * sizeof(float), cudaMemcpyHostToDevice, c->compute));
    c->lut_n = c->lut_cap;
  }
  return TGS_OK;
}

// the device state as the kernels of activate T (parity p) see it: its lists
// (the kernels index them by parity) come from list slot T % 3; R and the
// pending refresh radii stay parity-indexed
inline Dev dev_for(const tgs_ctx* c, int p, int32_t T) {
  Dev x = c->d;
  const int r = (int)(((uint32_t)T) % 3u);
  x.a_blk[p] = c->a3_blk[r];
  x.a_slot[p] = c->a3_slot[r];
  x.a_gid[p] = c->a3_gid[r];
  x.percam[p] = c->l3_percam[r];
  x.sp_blk[p] = c->l3_sp_blk[r];
  x.sp_slot[p] = c->l3_sp_slot[r];
  x.sm_blk[p] = c->l3_sm_blk[r];
  x.sm_slot[p] = c->l3_sm_slot[r];
  x.hdr_dev[p] = c->l3_hdr[r];
  x.last_planes[p] = c->l3_planes[r];
  x.planes_map[p] = c->l3_planes_map[r];
  return x;
}

inline float* host_rec(tgs_ctx* c, uint32_t l) {
  if (c->store) return c->store->entry_of(l);  // cached by inclusion whenever it moves (R27)
  return c->host + (size_t)l * c->d.n_arr * c->d.rec_floats;
}
inline float* slot_rec(tgs_ctx* c, uint32_t s) {
  return c->d.params + (size_t)s * 3 * c->d.rec_floats;
}

// A list of 1-D copies; adjacent copies merge when both sides are contiguous.
struct CopyBatch {
  std::vector<void*> dst;
  std::vector<void*> src;
  std::vector<size_t> size;
  uint64_t bytes = 0;
  size_t max_merge = SIZE_MAX;  // largest merged copy (bytes)
  void add(void* d, const void* s, size_t n) {
    bytes += n;
    if (!dst.empty() && size.back() + n <= max_merge &&
        (char*)dst.back() + size.back() == (char*)d &&
        (char*)src.back() + size.back() == (const char*)s) {
      size.back() += n;
      return;
    }
    dst.push_back(d);
    src.push_back(const_cast<void*>(s));
    size.push_back(n);
  }
};

// copies alternate between s and s2 (s2 forked from s and joined back into s)
cudaError_t submit_split(tgs_ctx* c, CopyBatch& b, cudaStream_t s, cudaStream_t s2,
                         cudaEvent_t fork, cudaEvent_t join) {
  cudaError_t e = cudaSuccess;
  const bool two = s2 && b.dst.size() > 1;
  if (two) {
    e = cudaEventRecord(fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, fork, 0);
  }
  for (size_t i = 0; i < b.dst.size() && e == cudaSuccess; ++i)
    e = cudaMemcpyAsync(b.dst[i], b.src[i], b.size[i], cudaMemcpyDefault, (two && (i & 1)) ? s2 : s);
  if (two && e == cudaSuccess) {
    e = cudaEventRecord(join, s2);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, join, 0);
  }
  std::lock_guard<std::mutex> g(c->mu);
  c->tm.copy_calls += b.dst.size();
  return e;
}

tgs_status submit(tgs_ctx* c, CopyBatch& b, cudaStream_t s) {
  if (b.dst.empty()) return TGS_OK;
  for (size_t i = 0; i < b.dst.size(); ++i)
    CK(cudaMemcpyAsync(b.dst[i], b.src[i], b.size[i], cudaMemcpyDefault, s));
  {
    std::lock_guard<std::mutex> g(c->mu);  // the I/O thread counts its copies too
    c->tm.copy_calls += b.dst.size();
  }
  return TGS_OK;
}

// Records of (local id, slot) pairs between the host tier and the slots
// (theta only when moments cold-restart: the slot keeps m, v behind theta).
void add_records(tgs_ctx* c, CopyBatch& b, const uint32_t* pairs, uint32_t n, bool to_device) {
  const size_t w = (size_t)c->d.n_arr * c->rec_bytes;
  for (uint32_t i = 0; i < n; ++i) {
    float* h = host_rec(c, pairs[2 * i]);
    float* d = slot_rec(c, pairs[2 * i + 1]);
    if (to_device)
      b.add(d, h, w);
    else
      b.add(h, d, w);
  }
}

tgs_status issue_copies(tgs_ctx* c, const uint32_t* pairs, uint32_t n, bool to_device,
                        cudaStream_t s) {
  CopyBatch b;
  add_records(c, b, pairs, n, to_device);
  return submit(c, b, s);
}

// initial record of local block l: theta from the caller's rows or fill, m = v = 0
void fill_record(tgs_ctx* c, const float* rows, tgs_fill_fn fill, void* user, uint32_t l,
                 float* dst) {
  const size_t rf = c->d.rec_floats;
  const uint32_t B = c->d.B;
  const uint64_t k = (uint64_t)l * c->cfg.world_size + c->cfg.rank;
  if (rows) {
    const uint64_t lo = k * B;
    const uint64_t nr = std::min<uint64_t>(B, c->cfg.n_gaussians - lo);
    std::memcpy(dst, rows + lo * kDim, nr * kDim * sizeof(float));
    std::memset(dst + nr * kDim, 0, (rf - nr * kDim) * sizeof(float));
  } else {
    fill(user, k, dst);
  }
  if (c->d.n_arr == 3) std::memset(dst + rf, 0, 2 * rf * sizeof(float));  // m = v = 0
}

void fill_host_tier(tgs_ctx* c, const float* rows, tgs_fill_fn fill, void* user, int nthreads) {
  const uint32_t Kloc = c->d.Kloc;
  std::atomic<uint32_t> next{0};
  auto work = [&]() {
    for (;;) {
      const uint32_t l0 = next.fetch_add(16);
      if (l0 >= Kloc) break;
      for (uint32_t l = l0; l < std::min<uint32_t>(l0 + 16, Kloc); ++l)
        fill_record(c, rows, fill, user, l, host_rec(c, l));
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < nthreads; ++i) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

// ---------------------------------------------------------------- I/O thread
// Issues the write-back of each activate once its k_evict/k_pack finished:
// the dirty decision depends on Adam(t-1) (R14), so the caller's thread never
// waits for it.  Jobs run in activate order.
void io_process(tgs_ctx* c, const tgs_ctx::Job& j) {
  const int p = j.parity;  // the job's ring slot
  cudaError_t e = cudaEventSynchronize(c->ev_evict[p]);
  if (e != cudaSuccess) {
    std::lock_guard<std::mutex> g(c->mu);
    c->io_err = std::string("io: cudaEventSynchronize(evict): ") + cudaGetErrorString(e);
    c->io_failed = true;
    return;
  }
  const uint32_t nd = c->ndirty[p];
  const uint32_t* dl = c->dirty_map[p];
  if (c->ce) {
    // copy-engine write-back (flat tier): dirty record k sits at ring index k
    // (ascending local id, k_evict / k_pack), so a run of consecutive ids is one
    // contiguous copy on both sides; a direct write-back copies from the slots
    const size_t w = (size_t)c->d.n_arr * c->rec_bytes;
    CopyBatch b;
    for (uint32_t k = 0; k < nd; ++k) {
      const char* src = j.direct ? reinterpret_cast<const char*>(slot_rec(c, dl[2 * k + 1]))
                                 : reinterpret_cast<const char*>(c->d.staging[p]) + (size_t)k * w;
      b.add(host_rec(c, dl[2 * k]), src, w);
    }
    Timer td;
    prof_begin(c, c->d2h, td);
    e = submit_split(c, b, c->d2h, c->d2h2, c->ev_dfork, c->ev_djoin);
    prof_end(c, c->d2h, td, 4, b.bytes);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_d2h[p], c->d2h);
    std::lock_guard<std::mutex> g(c->mu);
    if (e != cudaSuccess) {
      c->io_err = std::string("io: write-back copies: ") + cudaGetErrorString(e);
      c->io_failed = true;
    }
    c->last_ndirty = nd;
    return;
  }
  for (uint32_t k = 0; k < nd; ++k) c->store->mark_dirty(dl[2 * k], j.T);  // R27 (a): inserted dirty
  std::lock_guard<std::mutex> g(c->mu);
  c->last_ndirty = nd;
}

void io_main(tgs_ctx* c) {
  cudaSetDevice(c->device);
  for (;;) {
    tgs_ctx::Job j;
    {
      std::unique_lock<std::mutex> g(c->mu);
      c->cv_job.wait(g, [&] { return c->stop || !c->jobs.empty(); });
      if (c->jobs.empty()) return;  // stop requested and drained
      j = c->jobs.front();
      c->jobs.pop_front();
      c->inflight = j.T;
    }
    if (!c->io_failed) io_process(c, j);
    {
      std::lock_guard<std::mutex> g(c->mu);
      c->inflight = -1;
    }
    c->cv_done.notify_all();
  }
}

void io_submit(tgs_ctx* c, const tgs_ctx::Job& j) {
  {
    std::lock_guard<std::mutex> g(c->mu);
    c->jobs.push_back(j);
  }
  c->cv_job.notify_one();
}

// Wait until every write-back job of an activate <= T has been issued (its
// d2h event recorded), so a cudaStreamWaitEvent on it refers to that record.
void io_join(tgs_ctx* c, int32_t T) {
  std::unique_lock<std::mutex> g(c->mu);
  c->cv_done.wait(g, [&] {
    return (c->jobs.empty() || c->jobs.front().T > T) && (c->inflight < 0 || c->inflight > T);
  });
}

tgs_status check(tgs_ctx* c) {
  if (!c) return TGS_EINVAL;
  if (c->io_failed && !c->poisoned) {
    std::lock_guard<std::mutex> g(c->mu);
    c->poisoned = true;
    c->err = c->io_err;
  }
  if (c->poisoned) return TGS_EPOISONED;
  return TGS_OK;
}

tgs_status sync_all(tgs_ctx* c) {
  io_join(c, INT32_MAX);
  if (c->io_failed) {
    check(c);
    return TGS_ECUDA;
  }
  CK(cudaStreamSynchronize(c->plan));
  CK(cudaStreamSynchronize(c->h2d));
  CK(cudaStreamSynchronize(c->compute));
  if (c->cm) CK(cudaStreamSynchronize(c->cm));
  for (cudaStream_t s2 : {c->h2d2, c->d2h2})
    if (s2) CK(cudaStreamSynchronize(s2));
  CK(cudaStreamSynchronize(c->d2h));
  prof_collect(c);
  return TGS_OK;
}

void destroy_impl(tgs_ctx* c) {
  if (!c) return;
  if (c->io.joinable()) {
    {
      std::lock_guard<std::mutex> g(c->mu);
      c->stop = true;
    }
    c->cv_job.notify_all();
    c->io.join();
  }
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (void* p : c->dev_allocs) {
    if (c->has_alloc)
      c->alloc.free(p, (void*)c->compute, c->alloc.user);
    else
      cudaFree(p);
  }
  if (c->host) cudaFreeHost(c->host);
  delete c->store;
  if (c->cache_pool) cudaFreeHost(c->cache_pool);
  if (c->sm_map) cudaFreeHost(c->sm_map);
  for (int q = 0; q < 2; ++q)
    for (void* h : {(void*)c->sel_map[q][0], (void*)c->sel_map[q][1], (void*)c->sp_entry_map[q]})
      if (h) cudaFreeHost(h);
  for (void* h : c->dirty_map)
    if (h) cudaFreeHost(h);
  for (void* h : {(void*)c->hdr, (void*)c->sp_map, (void*)c->ndirty, (void*)c->planes_pinned,
                  (void*)c->lut_pinned, (void*)c->probe_map})
    if (h) cudaFreeHost(h);
  for (cudaEvent_t e : c->ev_job)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->ev_c1)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_copies, c->ev_commit[0], c->ev_commit[1], c->ev_hfork, c->ev_hjoin,
                        c->ev_dfork, c->ev_djoin})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_plan, c->ev_probe, c->ev_ready[0], c->ev_ready[1], c->ev_ready[2],
                        c->ev_evict[0], c->ev_evict[1], c->ev_evict[2], c->ev_evict[3],
                        c->ev_evict[4], c->ev_d2h[0], c->ev_d2h[1], c->ev_d2h[2], c->ev_d2h[3],
                        c->ev_d2h[4], c->ev_lists[0], c->ev_lists[1], c->ev_lists[2],
                        c->ev_refresh[0], c->ev_refresh[1], c->ev_planes[0], c->ev_planes[1],
                        c->ev_planes[2], c->trace_base})
    if (e) cudaEventDestroy(e);
  for (auto& p : c->pending) c->ev_pool.push_back(p.a), c->ev_pool.push_back(p.b);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaStream_t s : {c->plan, c->h2d, c->d2h, c->cm, c->h2d2, c->d2h2}) if (s) cudaStreamDestroy(s);
  cudaGetLastError();
  delete c;
}

}  // namespace

extern "C" {

const char* tgs_status_string(tgs_status s) {
  switch (s) {
    case TGS_OK: return "ok";
    case TGS_EINVAL: return "invalid argument";
    case TGS_ESTATE: return "invalid call order";
    case TGS_ENOMEM: return "out of memory";
    case TGS_ECUDA: return "CUDA error";
    case TGS_ENCCL: return "NCCL error";
    case TGS_ENONFINITE: return "non-finite gradient";
    case TGS_EPOISONED: return "context poisoned by an earlier CUDA error";
    case TGS_EIO: return "storage I/O error";
  }
  return "unknown status";
}

const char* tgs_last_error(const tgs_ctx* c) { return c ? c->err.c_str() : "null context"; }

}  // extern "C"

namespace {

tgs_status init_impl(const tgs_config* cfg, const tgs_store_config* scfg, const float* theta_rows,
                     tgs_fill_fn fill, void* fill_user, const float* bounds,
                     const tgs_allocator* alloc, void* compute_stream, tgs_ctx** out) {
  if (!cfg || !out || !bounds) return TGS_EINVAL;
  const tgs_config& g = *cfg;
  if (g.dim != kDim || g.block_size < 4 || g.block_size % 4 != 0 || g.capacity == 0 ||
      g.n_gaussians == 0)
    return TGS_EINVAL;
  if (!(g.lambda >= 0.0 && g.lambda <= 1.0) || !(g.gamma > 0.0 && g.gamma < 1.0))
    return TGS_EINVAL;
  if (g.quota_den == 0 || g.quota_num > g.quota_den) return TGS_EINVAL;
  if (g.world_size < 1 || g.rank < 0 || g.rank >= g.world_size) return TGS_EINVAL;
  if (g.moments != TGS_MOMENTS_PERSIST && g.moments != TGS_MOMENTS_COLD_RESTART) return TGS_EINVAL;
  if (g.max_cameras < 1 || g.max_cameras > kMaxCams || g.max_age > kMaxAge) return TGS_EINVAL;
  if (g.xfer != TGS_XFER_KERNEL && g.xfer != TGS_XFER_COPY_ENGINE) return TGS_EINVAL;
  const bool reopen = scfg && scfg->reopen;
  if (!reopen && (theta_rows == nullptr) == (fill == nullptr)) return TGS_EINVAL;
  if (reopen && theta_rows && fill) return TGS_EINVAL;
  const uint32_t P = g.pool_slots ? g.pool_slots : 2u * g.capacity;
  if (P < g.capacity) return TGS_EINVAL;
  if (scfg && (!scfg->dir || scfg->cache_blocks < 2ull * g.capacity)) return TGS_EINVAL;  // R27
  const uint64_t K = (g.n_gaussians + g.block_size - 1) / g.block_size;
  const uint64_t Kloc64 = K > (uint64_t)g.rank ? (K - g.rank + g.world_size - 1) / g.world_size : 0;
  if (Kloc64 > (1ull << 31) / 32) return TGS_EINVAL;
  for (uint64_t k = 0; k < K; ++k) {
    if (k % g.world_size != (uint64_t)g.rank) continue;
    for (int i = 0; i < 4; ++i)
      if (!std::isfinite(bounds[4 * k + i])) return TGS_EINVAL;
    if (bounds[4 * k + 3] < 0.0f) return TGS_EINVAL;
  }

  tgs_ctx* c = new tgs_ctx();
  c->cfg = g;
  c->device = g.device;
  c->K = K;
  if (alloc && alloc->alloc && alloc->free) {
    c->alloc = *alloc;
    c->has_alloc = true;
  }
  Dev& d = c->d;
  d.N = g.n_gaussians;
  d.B = g.block_size;
  d.Kloc = (uint32_t)Kloc64;
  d.W = (d.Kloc + 31) / 32;
  d.P = P;
  d.PW = (P + 31) / 32;
  d.C = g.capacity;
  d.J_max = g.max_cameras;
  d.n_arr = g.moments == TGS_MOMENTS_PERSIST ? 3u : 1u;
  d.G = (uint32_t)g.world_size;
  d.rank = (uint32_t)g.rank;
  d.max_age = g.max_age;
  d.n_lut_cols = g.max_age + 2;
  d.quota_num = g.quota_num;
  d.quota_den = g.quota_den;
  d.tide = g.tide ? 1 : 0;
  d.cold = g.moments == TGS_MOMENTS_COLD_RESTART ? 1 : 0;
  d.refresh = g.refresh_bounds ? 1 : 0;
  d.rec_floats = (uint64_t)d.B * kDim;
  c->rec_bytes = d.rec_floats * sizeof(float);

  auto fail = [&](tgs_status st) {
    destroy_impl(c);
    return st;
  };
  if (cudaSetDevice(g.device) != cudaSuccess) return fail(TGS_ECUDA);
  c->compute = (cudaStream_t)compute_stream;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  // the plan is latency-critical (the host waits for it): highest priority
  // (TGS_PLAN_PRIO=0: default priority, for A/B measurements)
  const char* pp = getenv("TGS_PLAN_PRIO");
  const int plan_prio = (pp && atoi(pp) == 0) ? prio_lo : prio_hi;
  if (cudaStreamCreateWithPriority(&c->plan, cudaStreamNonBlocking, plan_prio) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) != cudaSuccess)
    return fail(TGS_ECUDA);
  if (const char* cs = getenv("TGS_CE_STREAMS")) c->ce_streams = atoi(cs) == 2 ? 2 : 1;
  if (const char* wk = getenv("TGS_WB_KERNEL")) c->wb_kernel = atoi(wk);
  if (g.xfer == TGS_XFER_COPY_ENGINE && c->ce_streams == 2 &&
      (cudaStreamCreateWithFlags(&c->h2d2, cudaStreamNonBlocking) != cudaSuccess ||
       cudaStreamCreateWithFlags(&c->d2h2, cudaStreamNonBlocking) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_hfork, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_hjoin, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_dfork, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_djoin, cudaEventDisableTiming) != cudaSuccess))
    return fail(TGS_ECUDA);
  if (g.xfer == TGS_XFER_COPY_ENGINE &&
      (cudaStreamCreateWithPriority(&c->cm, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_copies, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_commit[0], cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&c->ev_commit[1], cudaEventDisableTiming) != cudaSuccess))
    return fail(TGS_ECUDA);
  for (cudaEvent_t* e : {&c->ev_plan, &c->ev_probe, &c->ev_ready[0], &c->ev_ready[1],
                         &c->ev_ready[2], &c->ev_evict[0], &c->ev_evict[1], &c->ev_evict[2],
                         &c->ev_evict[3], &c->ev_evict[4], &c->ev_d2h[0], &c->ev_d2h[1],
                         &c->ev_d2h[2], &c->ev_d2h[3], &c->ev_d2h[4], &c->ev_lists[0],
                         &c->ev_lists[1], &c->ev_lists[2], &c->ev_refresh[0], &c->ev_refresh[1],
                         &c->ev_planes[0], &c->ev_planes[1], &c->ev_planes[2],
                         &c->ev_job[0], &c->ev_job[1], &c->ev_job[2],
                         &c->ev_job[3]})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return fail(TGS_ECUDA);

  // ---- host tier (pinned, block records)
  int nth = g.init_threads > 0 ? g.init_threads : (int)std::thread::hardware_concurrency();
  nth = std::max(1, std::min(nth, 128));
  if (scfg) {
    // NEXT f3: CPU cache of H records over the log-structured store
    const uint64_t S = (d.n_arr * c->rec_bytes + 4095) / 4096 * 4096;
    if (cudaHostAlloc((void**)&c->cache_pool, ((size_t)scfg->cache_blocks + scfg->prefetch_blocks) * S,
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      c->cache_pool = nullptr;
      cudaGetLastError();
      return fail(TGS_ENOMEM);
    }
    tgs::BlockStore::Geometry geo{d.N, d.B, d.n_arr, d.G, d.rank, d.Kloc, c->rec_bytes};
    c->store = new tgs::BlockStore();
    const int io_threads = scfg->io_threads > 0 ? std::min(scfg->io_threads, 64) : 8;
    const std::string e = c->store->open(
        scfg->dir, geo, scfg->cache_blocks, c->cache_pool,
        scfg->segment_bytes ? scfg->segment_bytes : (1ull << 30), scfg->direct_io != 0,
        io_threads,
        [&](uint32_t l, float* dst) { fill_record(c, theta_rows, fill, fill_user, l, dst); },
        reopen);
    if (!e.empty()) {
      fprintf(stderr, "tidegs: store: %s\n", e.c_str());  // the context is gone on return
      return fail(TGS_EIO);
    }
    c->store->start_prefetch(scfg->prefetch_blocks, io_threads);
  } else {
    c->host_bytes = (size_t)d.Kloc * d.n_arr * c->rec_bytes;
    if (c->host_bytes &&
        cudaHostAlloc((void**)&c->host, c->host_bytes,
                      cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
      c->host = nullptr;
      cudaGetLastError();
      return fail(TGS_ENOMEM);
    }
    fill_host_tier(c, theta_rows, fill, fill_user, nth);
  }

  // ---- mapped pinned plan readback
  const size_t list_bytes = sizeof(uint32_t) * 2 * (size_t)std::max(d.C, 1u);
  if (cudaHostAlloc((void**)&c->hdr, sizeof(PlanHdr), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->sp_map, list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->dirty_map[0], list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->dirty_map[1], list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->dirty_map[2], list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->dirty_map[3], list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->dirty_map[4], list_bytes, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->ndirty, sizeof(uint32_t) * kRings, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->planes_pinned, sizeof(float) * 4 * kMaxCams * 24,
                    cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void**)&c->probe_map, sizeof(uint32_t) * std::max(d.W, 1u),
                    cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return fail(TGS_ENOMEM);
  }
  if (c->store) {
    const size_t cb = sizeof(uint32_t) * std::max(d.C, 1u);
    bool okm = cudaHostAlloc((void**)&c->sm_map, cb, cudaHostAllocMapped) == cudaSuccess;
    for (int q = 0; q < 2; ++q)
      for (uint32_t** m : {&c->sel_map[q][0], &c->sel_map[q][1], &c->sp_entry_map[q]})
        okm = okm && cudaHostAlloc((void**)m, cb, cudaHostAllocMapped) == cudaSuccess;
    if (!okm) {
      cudaGetLastError();
      return fail(TGS_ENOMEM);
    }
    cudaHostGetDevicePointer((void**)&d.sm_map, c->sm_map, 0);
    cudaHostGetDevicePointer((void**)&d.host_dev, c->cache_pool, 0);
    d.host_stride = c->store->entry_bytes();
  } else {
    if (c->host) cudaHostGetDevicePointer((void**)&d.host_dev, c->host, 0);
    d.host_stride = (uint64_t)d.n_arr * c->rec_bytes;
  }
  std::memset(c->hdr, 0, sizeof(PlanHdr));
  std::memset(c->ndirty, 0, sizeof(uint32_t) * kRings);
  cudaHostGetDevicePointer((void**)&d.hdr_map, c->hdr, 0);
  cudaHostGetDevicePointer((void**)&d.sp_map, c->sp_map, 0);
  for (int k = 0; k < kRings; ++k)
    cudaHostGetDevicePointer((void**)&d.dirty_map[k], c->dirty_map[k], 0);
  cudaHostGetDevicePointer((void**)&d.ndirty_map, c->ndirty, 0);
  for (int r = 0; r < 3; ++r) {
    float* dp = nullptr;
    cudaHostGetDevicePointer((void**)&dp, c->planes_pinned + (size_t)r * kMaxCams * 24, 0);
    c->l3_planes_map[r] = reinterpret_cast<const float4*>(dp);
  }

  // ---- device state
  bool ok = true;
  const uint32_t Kl = std::max(d.Kloc, 1u), Wd = std::max(d.W, 1u), Cc = std::max(d.C, 1u);
  d.bounds = dalloc_t<float4>(c, Kl, ok);
  d.last_access = dalloc_t<int32_t>(c, Kl, ok);
  d.step = dalloc_t<uint32_t>(c, Kl, ok);
  d.b2s = dalloc_t<int32_t>(c, Kl, ok);
  d.ever = dalloc_t<uint8_t>(c, Kl, ok);
  d.evicted = dalloc_t<uint8_t>(c, Kl, ok);
  d.admit = dalloc_t<int32_t>(c, Kl, ok);
  for (int r = 0; r < 3; ++r) c->l3_percam[r] = dalloc_t<uint32_t>(c, (size_t)d.J_max * Wd, ok);
  for (uint32_t** p : {&d.Kb, &d.cand, &d.Q, &d.Sp, &d.Sm, &d.Om, &d.Ab, &d.R[0], &d.R[1]})
    *p = dalloc_t<uint32_t>(c, Wd, ok);
  d.s2b = dalloc_t<int32_t>(c, P, ok);
  d.occ = dalloc_t<uint32_t>(c, d.PW, ok);
  d.dirty = dalloc_t<uint32_t>(c, d.PW, ok);
  d.rel = dalloc_t<uint32_t>(c, d.PW, ok);
  for (int r = 0; r < 3; ++r) {
    c->l3_sp_blk[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->l3_sp_slot[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->l3_sm_blk[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->l3_sm_slot[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->l3_hdr[r] = dalloc_t<PlanHdr>(c, 1, ok);
    c->l3_planes[r] = dalloc_t<float4>(c, kMaxCams * 6, ok);
  }
  for (int p = 0; p < 2; ++p) {
    d.percam[p] = d.sp_blk[p] = d.sp_slot[p] = d.sm_blk[p] = d.sm_slot[p] = nullptr;  // per launch
    d.hdr_dev[p] = nullptr;
    d.last_planes[p] = nullptr;
    d.planes_map[p] = nullptr;
    d.a_blk[p] = d.a_slot[p] = d.a_gid[p] = nullptr;  // per launch, from the ring below
  }
  d.cnt = dalloc_t<uint32_t>(c, CNT_N, ok);
  d.stats = dalloc_t<unsigned long long>(c, ST_ALL, ok);
  d.nonfinite = dalloc_t<unsigned long long>(c, 1, ok);
  for (int r = 0; r < 3; ++r) {
    c->a3_blk[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->a3_slot[r] = dalloc_t<uint32_t>(c, Cc, ok);
    c->a3_gid[r] = dalloc_t<uint32_t>(c, Cc, ok);
  }
  d.ent = dalloc_t<AdamEnt>(c, Cc, ok);
  d.adam_ctr = dalloc_t<uint32_t>(c, 1, ok);
  for (int k = 0; k < kRings; ++k) {
    d.dl_slot[k] = dalloc_t<uint32_t>(c, Cc, ok);
    d.dl_blk[k] = dalloc_t<uint32_t>(c, Cc, ok);
  }
  if (c->store) d.ent_of = dalloc_t<int32_t>(c, Kl, ok);
  d.pend[0] = dalloc_t<uint32_t>(c, Kl, ok);
  d.pend[1] = dalloc_t<uint32_t>(c, Kl, ok);
  d.ndirty_dev = dalloc_t<uint32_t>(c, kRings, ok);
  d.wb_tag = dalloc_t<int32_t>(c, Kl, ok);
  d.wb_idx = dalloc_t<uint32_t>(c, Kl, ok);
  // default ring = C records: any S- fits, so no write-back ever has to come
  // straight from the slots (and tgs_activate_async needs no plan readback)
  d.S_max = g.staging_blocks ? g.staging_blocks : std::max(1u, d.C);
  c->nrings = c->store ? 3 : kRings;
  d.nrings = c->nrings;
  for (int k = 0; k < kRings; ++k)
    d.staging[k] = k < c->nrings ? dalloc_t<float>(c, (size_t)d.S_max * d.n_arr * d.rec_floats, ok)
                                 : nullptr;
  c->ce = g.xfer == TGS_XFER_COPY_ENGINE && !c->store;
  d.stage_in = c->ce ? dalloc_t<float>(c, 2 * (size_t)Cc * d.n_arr * d.rec_floats, ok) : nullptr;
  std::vector<uint16_t> lut;
  uint32_t n_ranks = 0;
  build_rank_lut(g, lut, n_ranks);
  d.n_buckets = 2 * n_ranks;
  d.rank_lut = dalloc_t<uint16_t>(c, lut.size(), ok);
  const size_t pool_floats = (size_t)P * 3 * d.rec_floats, grad_floats = (size_t)P * d.rec_floats;
  d.params = dalloc_t<float>(c, pool_floats, ok);
  if (g.level2 || g.refresh_bounds) d.geo6 = dalloc_t<float>(c, (size_t)P * d.B * 6, ok);
  d.grads = dalloc_t<float>(c, grad_floats, ok);
  if (!ok) return fail(TGS_ENOMEM);

  // ---- initial contents
  std::vector<float4> bl(Kl);
  for (uint32_t l = 0; l < d.Kloc; ++l) {
    const float* b = bounds + 4 * ((uint64_t)l * g.world_size + g.rank);
    bl[l] = make_float4(b[0], b[1], b[2], b[3]);
  }
  cudaStream_t s0 = c->plan;
#define CKI(x) do { if ((x) != cudaSuccess) { set_err(c, "%s", #x); return fail(TGS_ECUDA); } } while (0)
  CKI(cudaMemcpyAsync(d.bounds, bl.data(), sizeof(float4) * Kl, cudaMemcpyHostToDevice, s0));
  CKI(cudaMemcpyAsync(d.rank_lut, lut.data(), sizeof(uint16_t) * lut.size(), cudaMemcpyHostToDevice, s0));
  CKI(cudaMemsetAsync(d.last_access, 0xff, sizeof(int32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.step, 0, sizeof(uint32_t) * Kl, s0));
  if (c->store && reopen && d.Kloc)  // R30: step counters of the barrier resumed from
    CKI(cudaMemcpyAsync(d.step, c->store->barrier_steps().data(), sizeof(uint32_t) * d.Kloc,
                        cudaMemcpyHostToDevice, s0));
  CKI(cudaMemsetAsync(d.b2s, 0xff, sizeof(int32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.ever, 0, Kl, s0));
  CKI(cudaMemsetAsync(d.evicted, 0, Kl, s0));
  CKI(cudaMemsetAsync(d.admit, 0, sizeof(int32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.wb_tag, 0xff, sizeof(int32_t) * Kl, s0));
  if (d.ent_of) CKI(cudaMemsetAsync(d.ent_of, 0xff, sizeof(int32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.pend[0], 0, sizeof(uint32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.pend[1], 0, sizeof(uint32_t) * Kl, s0));
  CKI(cudaMemsetAsync(d.ndirty_dev, 0, sizeof(uint32_t) * kRings, s0));
  for (uint32_t* p : {d.Kb, d.cand, d.Q, d.Sp, d.Sm, d.Om, d.Ab, d.R[0], d.R[1]})
    CKI(cudaMemsetAsync(p, 0, sizeof(uint32_t) * Wd, s0));
  for (int r = 0; r < 3; ++r) {
    CKI(cudaMemsetAsync(c->l3_percam[r], 0, sizeof(uint32_t) * (size_t)d.J_max * Wd, s0));
    CKI(cudaMemsetAsync(c->l3_hdr[r], 0, sizeof(PlanHdr), s0));
  }
  CKI(cudaMemsetAsync(d.s2b, 0xff, sizeof(int32_t) * P, s0));
  CKI(cudaMemsetAsync(d.occ, 0, sizeof(uint32_t) * d.PW, s0));
  CKI(cudaMemsetAsync(d.dirty, 0, sizeof(uint32_t) * d.PW, s0));
  CKI(cudaMemsetAsync(d.stats, 0, sizeof(unsigned long long) * ST_ALL, s0));
  CKI(cudaMemsetAsync(d.cnt, 0, sizeof(uint32_t) * CNT_N, s0));  // k_plan re-zeroes it after use
  CKI(cudaMemsetAsync(d.nonfinite, 0xff, sizeof(unsigned long long), s0));
  CKI(cudaMemsetAsync(d.params, 0, sizeof(float) * pool_floats, s0));
  CKI(cudaMemsetAsync(d.grads, 0, sizeof(float) * grad_floats, s0));
  if (d.geo6) CKI(cudaMemsetAsync(d.geo6, 0, sizeof(float) * (size_t)P * d.B * 6, s0));
  CKI(cudaStreamSynchronize(s0));
#undef CKI
  int dev = g.device;
  c->adam_grid = adam_grid(dev);
  if (const char* m = getenv("TGS_GATHER_CTAS")) c->gather_ctas = std::max(1, atoi(m));
  if (const char* m = getenv("TGS_SCATTER_CTAS")) c->scatter_ctas = std::max(1, atoi(m));
  if (const char* m = getenv("TGS_GATHER_BUFS")) c->gather_bufs = atoi(m);
  if (const char* m = getenv("TGS_SCATTER_BUFS")) c->scatter_bufs = atoi(m);
  // store tier: CPU-cache dirty marks; copy-engine transfers: the write-back
  // copies (the flat tier with the transfer kernels has no host work per write-back)
  if (c->store || c->ce) c->io = std::thread(io_main, c);
  *out = c;
  return TGS_OK;
}

// a5: k_adam_prologue, k_adam (+ k_refresh, f2) of the last activate's A list
tgs_status adam_launches(tgs_ctx* c, int p, uint32_t nA, const AdamHyper& h,
                         const uint32_t* d_row_mask) {
  const Dev dk = dev_for(c, p, c->T - 1);
  Timer t1, t2;
  prof_begin(c, c->compute, t1);
  CK(launch_adam_prologue(dk, nA, p, d_row_mask, c->compute));
  prof_end(c, c->compute, t1, 1);
  // Adam and the refresh read the A lists and header of list slot m: the plan
  // of T+3, which rewrites them, waits for ev_lists[m] recorded after them
  const int m = (int)(((uint32_t)c->T + 2) % 3u);  // list slot of the last activate
  prof_begin(c, c->compute, t2);
  CK(launch_adam(dk, nA, p, d_row_mask, h, c->adam_grid, c->compute));
  prof_end(c, c->compute, t2, 0);
  c->tm.kernel_launches += 2;
  if (c->d.refresh) {  // R25 from the packed centre / log-scales k_adam just wrote
    CK(launch_refresh(dk, nA, p, c->compute));
    c->tm.kernel_launches++;
  }
  CK(cudaEventRecord(c->ev_lists[m], c->compute));  // lists in use until here
  if (c->d.refresh) {  // the cull two batches later merges these radii (R25)
    CK(cudaEventRecord(c->ev_refresh[p], c->compute));
    c->rec_refresh[p] = true;
  }
  return TGS_OK;
}

}  // namespace

extern "C" {

tgs_status tgs_init_table(const tgs_config* cfg, const float* theta_rows, tgs_fill_fn fill,
                          void* fill_user, const float* bounds, const tgs_allocator* alloc,
                          void* compute_stream, tgs_ctx** out) {
  return init_impl(cfg, nullptr, theta_rows, fill, fill_user, bounds, alloc, compute_stream, out);
}

tgs_status tgs_init_table_store(const tgs_config* cfg, const tgs_store_config* store,
                                const float* theta_rows, tgs_fill_fn fill, void* fill_user,
                                const float* bounds, const tgs_allocator* alloc,
                                void* compute_stream, tgs_ctx** out) {
  if (!store) return TGS_EINVAL;
  return init_impl(cfg, store, theta_rows, fill, fill_user, bounds, alloc, compute_stream, out);
}

tgs_status tgs_destroy(tgs_ctx* c) {
  if (!c) return TGS_EINVAL;
  destroy_impl(c);
  return TGS_OK;
}

static tgs_status activate_impl(tgs_ctx* c, const tgs_camera* cams, uint32_t J,
                                tgs_activation* out, bool want_async);

tgs_status tgs_activate(tgs_ctx* c, const tgs_camera* cams, uint32_t J, tgs_activation* out) {
  return activate_impl(c, cams, J, out, false);
}

tgs_status tgs_activate_async(tgs_ctx* c, const tgs_camera* cams, uint32_t J,
                              tgs_activation* out) {
  return activate_impl(c, cams, J, out, true);
}

static tgs_status activate_impl(tgs_ctx* c, const tgs_camera* cams, uint32_t J,
                                tgs_activation* out, bool want_async) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (J > c->d.J_max || (J > 0 && !cams)) return TGS_EINVAL;
  for (uint32_t j = 0; j < J; ++j)
    for (int p = 0; p < 6; ++p)
      for (int i = 0; i < 4; ++i)
        if (!std::isfinite(cams[j].plane[p][i])) return TGS_EINVAL;
  Dev& d = c->d;
  const int p = c->parity;  // parity of R_t (R and the pending refresh radii)
  const int32_t T = c->T;
  const int m = (int)(((uint32_t)T) % 3u), mq = (int)(((uint32_t)T + 2) % 3u);  // list slots T, T-1

  // ---- plan stream: a1 cull, a3 quota + fill, a2 delta, slots, A list.
  //      List slot m is free once activate T-3's consumers are done (Adam or its
  //      prologue, the Level-2 filter, the write-back kernels, the gather):
  //      GPU-side waits only, so the plan may run up to two batches ahead of
  //      Adam.  With the bound refresh on, the cull merges the radii of the step
  //      two batches back (R25): it waits for that refresh.  The camera batch is
  //      read from mapped pinned memory by k_planes: nothing here queues behind
  //      a copy engine.
  if (c->rec_lists[m]) CK(cudaStreamWaitEvent(c->plan, c->ev_lists[m], 0));
  if (c->rec_ready[m]) CK(cudaStreamWaitEvent(c->plan, c->ev_ready[m], 0));
  if (d.refresh && c->rec_refresh[p]) CK(cudaStreamWaitEvent(c->plan, c->ev_refresh[p], 0));
  Timer tp;
  // the staging buffer of slot m held the batch of T-3: its k_planes must have
  // copied it (free after a plan readback; with tgs_activate_async the host may
  // be up to three plans ahead of the plan stream)
  if (c->rec_planes[m]) CK(cudaEventSynchronize(c->ev_planes[m]));
  if (J) std::memcpy(c->planes_pinned + (size_t)m * kMaxCams * 24, cams, sizeof(float) * 24 * J);
  prof_begin(c, c->plan, tp);
  const Dev dk = dev_for(c, p, T);
  CK(launch_cull(dk, J, T, p, c->plan));
  CK(cudaEventRecord(c->ev_planes[m], c->plan));
  c->rec_planes[m] = true;
  CK(launch_quota(dk, J, T, p, c->plan));
  CK(launch_plan(dk, T, p, c->plan));
  prof_end(c, c->plan, tp, 2);
  c->tm.kernel_launches += (d.Kloc ? 1 : 0) + ((J && d.Kloc) ? 2 : 0) + 1;
  CK(cudaEventRecord(c->ev_plan, c->plan));

  // ---- a4 gather of S+ into free slots (k_xfer on the h2d stream).  Hazards
  //      (GPU-side waits only): slots freed by t-1 (its pack, or its direct
  //      write-back, done), host records written back by t-2 landed.  With the
  //      default pool (P >= 2C) and Tide on, S+ never takes a slot S- frees in
  //      the same activate (R13), so the gather is enqueued before the host even
  //      reads the plan: it starts the moment k_plan ends.
  Dev dg = dev_for(c, p, T);
  uint32_t* const* sel = c->sel_map[p];
  uint32_t* spe = c->sp_entry_map[p];
  if (c->store) CK(cudaHostGetDevicePointer((void**)&dg.sp_entry, spe, 0));
  //      Write-back state: activate T uses ring slot T % nrings.  A block packed
  //      by T-1 .. T-nrings+1 is re-admitted from its ring record (the host write-back
  //      may still be in flight); one written back by T-nrings or earlier from the host,
  //      whose write-back (serial on the d2h stream) is waited for here.
  const int NR = c->nrings;
  const int k = (int)(((uint32_t)T) % (uint32_t)NR);
  auto gather_waits = [&]() -> tgs_status {
    CK(cudaStreamWaitEvent(c->h2d, c->ev_plan, 0));
    // every slot this gather may fill was freed by an earlier write-back, whose
    // k_evict / k_pack ran after the last Adam on it: wait for the newest one
    // (copy engines: the copies only write stage_in -- k_commit, which fills the
    // slots, waits for it on its own stream)
    if (c->last_evict_ring >= 0 && !c->ce)
      CK(cudaStreamWaitEvent(c->h2d, c->ev_evict[c->last_evict_ring], 0));
    // (copy-engine write-backs: the I/O thread records ev_d2h -- join it first)
    for (int back = 1; back < NR; ++back) {  // a direct write-back (T-1 .. T-NR+1) has no
      const int r = (int)(((uint32_t)(T - back)) % (uint32_t)NR);  // ring copy: wait for it
      if (T - back >= 0 && c->d2h_job[r] >= 0 && c->ring_direct[r]) {
        if (c->ce) io_join(c, c->d2h_job[r]);
        CK(cudaStreamWaitEvent(c->h2d, c->ev_d2h[r], 0));
      }
    }
    if (c->d2h_job[k] >= 0 && c->d2h_job[k] <= T - NR) {
      if (c->ce) io_join(c, c->d2h_job[k]);
      CK(cudaStreamWaitEvent(c->h2d, c->ev_d2h[k], 0));
    }
    if (c->io_failed) return check(c);
    return TGS_OK;
  };
  auto gather_flat = [&](uint32_t n_hint) -> tgs_status {
    tgs_status gs = gather_waits();
    if (gs != TGS_OK) return gs;
    Timer th;
    prof_begin(c, c->h2d, th);
    if (c->ce) {
      // copy engines (the plan is on the host): S+ record i from the host tier to
      // stage_in[i] -- one copy per run of consecutive local ids -- then k_commit
      // places each in its slot (or takes a ring re-admission from HBM)
      // stage_in is double-buffered (buffer T & 1), k_commit runs on its own
      // stream: the next gather's copies start as soon as these end, while
      // k_commit waits for the newest evict / pack (the slots it fills)
      const int sb = T & 1;
      const size_t w = (size_t)d.n_arr * c->rec_bytes;
      char* const stage = reinterpret_cast<char*>(d.stage_in) + (size_t)sb * d.C * w;
      if (c->rec_commit[sb]) CK(cudaStreamWaitEvent(c->h2d, c->ev_commit[sb], 0));
      CopyBatch b;
      for (uint32_t i = 0; i < n_hint; ++i)
        b.add(stage + (size_t)i * w, host_rec(c, c->sp_map[2 * i]), w);
      CK(submit_split(c, b, c->h2d, c->h2d2, c->ev_hfork, c->ev_hjoin));
      prof_end(c, c->h2d, th, 3, b.bytes);
      CK(cudaEventRecord(c->ev_copies, c->h2d));
      CK(cudaStreamWaitEvent(c->cm, c->ev_copies, 0));
      if (c->last_evict_ring >= 0)
        CK(cudaStreamWaitEvent(c->cm, c->ev_evict[c->last_evict_ring], 0));
      Timer tc;
      prof_begin(c, c->cm, tc);
      Dev dc = dg;
      dc.stage_in = reinterpret_cast<float*>(stage);
      CK(launch_commit(dc, n_hint, p, T, c->cm));
      prof_end(c, c->cm, tc, 6);
      CK(cudaEventRecord(c->ev_commit[sb], c->cm));
      c->rec_commit[sb] = true;
      c->tm.kernel_launches++;
      CK(cudaEventRecord(c->ev_ready[m], c->cm));
      c->rec_ready[m] = true;
      return TGS_OK;
    } else {
      CK(launch_xfer(dg, 0, p, k, T, nullptr, 0, n_hint, c->gather_ctas, c->gather_bufs, c->h2d));
      c->h2d_prof = prof_end(c, c->h2d, th, 3);
    }
    c->tm.kernel_launches++;
    CK(cudaEventRecord(c->ev_ready[m], c->h2d));
    c->rec_ready[m] = true;
    return TGS_OK;
  };
  const bool early = !c->store && !c->ce && d.tide && d.P >= 2u * d.C;
  // asynchronous activate: no host decision needs the plan -- S+ never reuses an
  // S- slot (P >= 2C) and the ring holds any S- (S_max >= C), so every count is
  // read from the device header by the kernels themselves
  const bool async = want_async && early && d.S_max >= d.C;
  if (early) {
    st = gather_flat(d.C);
    if (st != TGS_OK) return st;
  }
  PlanHdr h{};
  if (async) {
    h.nSm = kFromHdr;
    c->last_known = false;
  } else {
    CK(cudaEventSynchronize(c->ev_plan));  // the one plan readback (R14)
    h = *c->hdr;
    c->last = h;
    c->last_known = true;
  }
  c->last_J = J;
  if (c->h2d_prof >= 0 && !async) {  // the timed gather's algorithmic bytes
    std::lock_guard<std::mutex> g(c->prof_mu);
    if ((size_t)c->h2d_prof < c->pending.size())
      c->pending[c->h2d_prof].bytes = (uint64_t)h.nSp * d.n_arr * c->rec_bytes;
    c->h2d_prof = -1;
  }

  // ---- a4 write-back of dirty S-, enqueued on the compute stream after
  //      Adam(t-1) (the dirty decision).  Normal path: k_evict compacts the
  //      dirty list and k_pack copies those records into staging ring p, so
  //      their slots are free at once; k_xfer then drains the ring to the host
  //      tier on the d2h stream.  Direct path (this activate's S+ may reuse S-
  //      slots, or the ring is too small): k_xfer reads the slots themselves.
  const bool reuse_now = !async && (!d.tide || h.fallback);
  const bool direct = !async && (reuse_now || h.nSm > d.S_max);
  auto writeback = [&]() -> tgs_status {
    Timer te, td;
    CK(cudaStreamWaitEvent(c->compute, c->ev_plan, 0));
    // ring slot k held T-nrings' records, which the previous activate's gather may
    // re-admit from: it must be done
    if (c->rec_ready[mq]) CK(cudaStreamWaitEvent(c->compute, c->ev_ready[mq], 0));
    if (c->d2h_job[k] >= 0) {
      // the write-back of T-nrings must be done with ring slot k (its ring, dirty
      // lists; store tier: the I/O job's read of dirty_map[k] / ndirty[k])
      if (c->store || c->ce) io_join(c, c->d2h_job[k]);
      if (c->io_failed) return check(c);
      CK(cudaStreamWaitEvent(c->compute, c->ev_d2h[k], 0));
    }
    prof_begin(c, c->compute, te);
    CK(launch_evict_tagged(dg, h.nSm, p, k, T, !direct, c->compute));
    if (!direct) CK(launch_pack(dg, h.nSm, k, c->compute));
    prof_end(c, c->compute, te, 5);
    c->tm.kernel_launches += direct ? 1 : 2;
    CK(cudaEventRecord(c->ev_evict[k], c->compute));
    c->rec_evict[k] = true;
    c->last_evict_ring = k;
    // copy-engine mode: the write-back of a ring goes either as copy-engine runs
    // (the I/O thread) or, with TGS_WB_KERNEL, as the TMA kernel: N CTAs, or -n =
    // n CTAs while the write-backs keep up (the gather, on the critical path,
    // then gets most of the link) and scatter_ctas when the previous one is late
    int wb_ctas = c->scatter_ctas;
    const bool ce_runs = c->ce && c->wb_kernel == 0;
    if (c->ce && !ce_runs) {
      wb_ctas = c->wb_kernel > 0 ? c->wb_kernel : -c->wb_kernel;
      if (c->wb_kernel < 0 && c->last_d2h_ring >= 0 &&
          cudaEventQuery(c->ev_d2h[c->last_d2h_ring]) == cudaErrorNotReady)
        wb_ctas = c->scatter_ctas;
      cudaGetLastError();
    }
    if (ce_runs) {  // the I/O thread copies the dirty runs once k_evict / k_pack are done
      c->d2h_job[k] = T;
      c->ring_direct[k] = direct;
      io_submit(c, {T, k, direct});
      return TGS_OK;
    }
    CK(cudaStreamWaitEvent(c->d2h, c->ev_evict[k], 0));
    prof_begin(c, c->d2h, td);
    CK(launch_xfer(dg, direct ? 2 : 1, p, k, T, nullptr, 0, async ? d.C : h.nSm, wb_ctas,
                   c->scatter_bufs, c->d2h));
    prof_end(c, c->d2h, td, 4);
    c->tm.kernel_launches++;
    CK(cudaEventRecord(c->ev_d2h[k], c->d2h));
    c->last_d2h_ring = k;
    if (c->store) {
      CK(cudaEventRecord(c->ev_job[T & 3], c->d2h));
      io_submit(c, {T, k, direct});
    }
    c->d2h_job[k] = T;
    c->ring_direct[k] = direct;
    return TGS_OK;
  };
  if (reuse_now && h.nSm) {
    st = writeback();
    if (st != TGS_OK) return st;
    if (c->store || c->ce) io_join(c, T);
    if (c->io_failed) return check(c);
    CK(cudaStreamWaitEvent(c->h2d, c->ev_d2h[k], 0));
  }

  if (!early && !c->store) {
    st = gather_flat(h.nSp);
    if (st != TGS_OK) return st;
  } else if (c->store) {
    // NEXT f3, R27 (b): S+ records come from their CPU-cache entries; misses
    // are read from SSD through Index[k] after a dirty LRU victim (if any) is
    // appended to the patch log.  Needs the dirty marks of activate T-1.  The
    // hits move over PCIe (k_xfer from their entries) while the SSD reads the
    // misses; then a second k_xfer moves the misses.
    st = gather_waits();
    if (st != TGS_OK) return st;
    io_join(c, T - 1);
    if (c->io_failed) return check(c);
    auto wait_d2h = [&](int32_t job) {
      // the plan of T waited (GPU-side) for the gather of T-2, which waited
      // for the write-back of T-4: older jobs have landed
      if (job + 4 <= T) return;
      io_join(c, job);
      cudaEventSynchronize(c->ev_job[job & 3]);
    };
    uint32_t n_sel[2] = {0, 0};
    tgs_status hst = TGS_OK;
    auto launch_subset = [&](int which) -> tgs_status {
      if (!n_sel[which]) return TGS_OK;
      Timer t1;
      prof_begin(c, c->h2d, t1);
      uint32_t* sel_dev = nullptr;
      CK(cudaHostGetDevicePointer((void**)&sel_dev, sel[which], 0));
      CK(launch_xfer(dg, 0, p, k, T, sel_dev, n_sel[which], n_sel[which], c->gather_ctas,
                     c->gather_bufs, c->h2d));
      prof_end(c, c->h2d, t1, 3, (uint64_t)n_sel[which] * d.n_arr * c->rec_bytes);
      c->tm.kernel_launches++;
      return TGS_OK;
    };
    auto hits_ready = [&](const std::vector<uint8_t>& miss) {
      for (uint32_t i = 0; i < h.nSp; ++i) {
        const int w = miss[i] ? 1 : 0;
        sel[w][n_sel[w]++] = i;
        if (!miss[i]) spe[i] = (uint32_t)c->store->entry_index(c->sp_map[2 * i]);
      }
      hst = launch_subset(0);
    };
    const std::string e = c->store->gather(c->sp_map, h.nSp, T, wait_d2h, hits_ready);
    if (!e.empty()) {
      c->poisoned = true;
      set_err(c, "store: %s", e.c_str());
      return TGS_EIO;
    }
    if (hst != TGS_OK) return hst;
    for (uint32_t k = 0; k < n_sel[1]; ++k) {
      const uint32_t i = sel[1][k];
      spe[i] = (uint32_t)c->store->entry_index(c->sp_map[2 * i]);
    }
    st = launch_subset(1);
    if (st != TGS_OK) return st;
    CK(cudaEventRecord(c->ev_ready[m], c->h2d));
    c->rec_ready[m] = true;
    // R27 (c): the blocks that left the GPU are accesses of the CPU cache too
    if (h.nSm) c->store->touch_evicted(c->sm_map, h.nSm, T);
  }

  if (!reuse_now && h.nSm) {  // (async: always; the kernels read |S-| themselves)
    st = writeback();
    if (st != TGS_OK) return st;
  }
  // lists of parity p stay in use until this batch's write-back kernels (and
  // its Adam, which re-records this event) are done
  CK(cudaEventRecord(c->ev_lists[m], c->compute));
  c->rec_lists[m] = true;

  // ---- C1: the active set of every rank, on the plan stream
  //      after k_plan; every rank calls it once per activate
  if (c->has_comm) {
    uint32_t* send = c->a3_gid[(uint32_t)T % 3u];
    CK(launch_pad_active(send, dk.hdr_dev[p], d.C, c->plan));
    c->tm.kernel_launches++;
    if (c->comm.allgather(c->comm.user, send, c->c1_recv[m], sizeof(uint32_t) * d.C,
                          (void*)c->plan) != 0) {
      c->poisoned = true;
      set_err(c, "C1 all-gather failed (activate %d)", T);
      return TGS_ENCCL;
    }
    CK(cudaEventRecord(c->ev_c1[m], c->plan));
  }
  c->last_parity = p;
  c->parity = p ^ 1;
  c->T = T + 1;
  c->can_step = true;
  if (c->cfg.serialize) {  // ablation w/o Overlap: I/O completes before compute starts
    st = sync_all(c);
    if (st != TGS_OK) return st;
  }
  if (out) {
    const uint32_t unknown = 0xFFFFFFFFu;
    out->n_visible = async ? unknown : h.nK;
    out->n_resident = async ? unknown : h.nR;
    out->n_active_blocks = async ? unknown : h.nA;
    out->n_stage_in = async ? unknown : h.nSp;
    out->n_evict = async ? unknown : h.nSm;
    out->n_evict_dirty = 0;  // decided after the previous Adam; see tgs_get_stats
    out->h2d_bytes = async ? ~0ull : (uint64_t)h.nSp * d.n_arr * c->rec_bytes;
    out->d_n_active = &dev_for(c, p, T).hdr_dev[p]->nA;
    out->d_active_blocks = c->a3_gid[(uint32_t)T % 3u];
    out->d_active_slots = c->a3_slot[(uint32_t)T % 3u];
    out->d_params = d.params;
    out->d_grads = d.grads;
    out->slot_stride = 3 * d.rec_floats;
    out->grad_stride = d.rec_floats;
    out->ready = (void*)c->ev_ready[m];
    out->d_global_active = c->has_comm ? c->c1_recv[m] : nullptr;
    out->global_stride = d.C;
    out->global_ready = c->has_comm ? (void*)c->ev_c1[m] : nullptr;
  }
  return TGS_OK;
}

tgs_status tgs_step_adam(tgs_ctx* c, const tgs_adam* hp, const uint32_t* d_row_mask) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!c->can_step) return TGS_ESTATE;
  if (!hp || !hp->lr) return TGS_EINVAL;
  c->can_step = false;
  const int p = c->last_parity;
  const uint32_t nA = c->last_known ? c->last.nA : kFromHdr;  // async: read on the device
  st = ensure_lut(c, hp->beta1, hp->beta2, (uint32_t)std::min<uint64_t>(c->n_steps + 2, 0xffffffffu));
  if (st != TGS_OK) return st;
  c->n_steps++;
  AdamHyper h{};
  for (uint32_t a = 0; a < kDim; ++a) h.lr[a] = hp->lr[a];
  h.b1 = hp->beta1;
  h.b2 = hp->beta2;
  h.omb1 = 1.0f - hp->beta1;
  h.omb2 = 1.0f - hp->beta2;
  h.eps = hp->eps;
  CK(cudaStreamWaitEvent(c->compute, c->ev_plan, 0));
  CK(cudaStreamWaitEvent(c->compute, c->ev_ready[((uint32_t)c->T + 2) % 3u], 0));
  st = nA ? adam_launches(c, p, nA, h, d_row_mask) : TGS_OK;
  if (st != TGS_OK) return st;
  // ---- C2: every rank's cumulative counters summed, after this
  //      step's Adam on the compute stream; every rank calls it once per step
  if (c->has_comm) {
    CK(cudaMemcpyAsync(c->c2_buf, c->d.stats, sizeof(unsigned long long) * ST_N,
                       cudaMemcpyDeviceToDevice, c->compute));
    if (c->comm.allreduce_u64(c->comm.user, reinterpret_cast<uint64_t*>(c->c2_buf), ST_N,
                              (void*)c->compute) != 0) {
      c->poisoned = true;
      set_err(c, "C2 all-reduce failed (step %llu)", (unsigned long long)c->n_steps);
      return TGS_ENCCL;
    }
  }
  if (c->cfg.serialize) CK(cudaStreamSynchronize(c->compute));  // ablation w/o Overlap
  return TGS_OK;
}

tgs_status tgs_fine_filter(tgs_ctx* c, uint32_t* d_row_mask) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!c->can_step) return TGS_ESTATE;
  if (!d_row_mask) return TGS_EINVAL;
  const int p = c->last_parity;
  // reads theta of every A slot: after the plan and the gather of this batch
  CK(cudaStreamWaitEvent(c->compute, c->ev_plan, 0));
  const int m = (int)(((uint32_t)c->T + 2) % 3u);  // list slot of the last activate
  CK(cudaStreamWaitEvent(c->compute, c->ev_ready[m], 0));
  if ((c->last_known && c->last.nA == 0) || c->d.Kloc == 0) return TGS_OK;
  Timer tf;
  prof_begin(c, c->compute, tf);
  CK(launch_fine(dev_for(c, p, c->T - 1), c->last_known ? c->last.nA : kFromHdr, c->last_J, p,
                 d_row_mask, c->compute));
  prof_end(c, c->compute, tf, 8);
  c->tm.kernel_launches++;
  CK(cudaEventRecord(c->ev_lists[m], c->compute));  // k_fine reads this slot's K^(j)
  return TGS_OK;
}

tgs_status tgs_flush(tgs_ctx* c) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  Dev& d = c->d;
  std::vector<uint32_t> dirty(d.PW);
  std::vector<int32_t> s2b(d.P);
  CK(cudaMemcpy(dirty.data(), d.dirty, sizeof(uint32_t) * d.PW, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(s2b.data(), d.s2b, sizeof(int32_t) * d.P, cudaMemcpyDeviceToHost));
  std::vector<std::pair<uint32_t, uint32_t>> list;  // (local id, slot), ascending id
  for (uint32_t s = 0; s < d.P; ++s)
    if (((dirty[s >> 5] >> (s & 31)) & 1u) && s2b[s] >= 0) list.push_back({(uint32_t)s2b[s], s});
  std::sort(list.begin(), list.end());
  std::vector<uint32_t> pairs;
  for (auto& e : list) pairs.push_back(e.first), pairs.push_back(e.second);
  st = issue_copies(c, pairs.data(), (uint32_t)list.size(), false, c->d2h);
  if (st != TGS_OK) return st;
  CK(cudaStreamSynchronize(c->d2h));
  CK(cudaMemset(d.dirty, 0, sizeof(uint32_t) * d.PW));
  CK(cudaDeviceSynchronize());
  if (c->store) {
    // NEXT f3: the barrier reaches the SSD too: the dirty
    // residents just landed in their entries, then every dirty entry is appended
    for (auto& e : list) c->store->mark_dirty(e.first, -1);
    // R30: the manifest carries the Adam step counters of this barrier
    std::vector<uint32_t> steps(std::max(d.Kloc, 1u));
    CK(cudaMemcpy(steps.data(), d.step, sizeof(uint32_t) * d.Kloc, cudaMemcpyDeviceToHost));
    const std::string e = c->store->flush_all([](int32_t) {}, steps.data());
    if (!e.empty()) {
      c->poisoned = true;
      set_err(c, "store: %s", e.c_str());
      return TGS_EIO;
    }
  }
  c->host_flush_blocks += list.size();
  c->host_flush_bytes += (uint64_t)list.size() * d.n_arr * c->rec_bytes;
  c->can_step = false;
  return TGS_OK;
}

tgs_status tgs_set_comm(tgs_ctx* c, const tgs_comm* comm) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!comm || !comm->allgather || !comm->allreduce_u64) return TGS_EINVAL;
  if (c->T != 0 || c->has_comm) return TGS_ESTATE;
  bool ok = true;
  const size_t rows = (size_t)c->cfg.world_size * std::max(c->d.C, 1u);
  for (int r = 0; r < 3; ++r) c->c1_recv[r] = dalloc_t<uint32_t>(c, rows, ok);
  c->c2_buf = dalloc_t<unsigned long long>(c, ST_N, ok);
  if (!ok) return TGS_ENOMEM;
  for (cudaEvent_t* e : {&c->ev_c1[0], &c->ev_c1[1], &c->ev_c1[2]})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  CK(cudaMemsetAsync(c->c2_buf, 0, sizeof(unsigned long long) * ST_N, c->compute));
  CK(cudaStreamSynchronize(c->compute));
  c->comm = *comm;
  c->has_comm = true;
  return TGS_OK;
}

tgs_status tgs_get_global_stats(tgs_ctx* c, tgs_stats* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  if (!c->has_comm) return TGS_ESTATE;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  CK(cudaMemcpy(out, c->c2_buf, sizeof(uint64_t) * ST_N, cudaMemcpyDeviceToHost));
  return TGS_OK;
}

tgs_status tgs_get_stats(tgs_ctx* c, tgs_stats* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  unsigned long long v[ST_N];
  CK(cudaMemcpy(v, c->d.stats, sizeof v, cudaMemcpyDeviceToHost));
  v[ST_FLUSH_BYTES] += c->host_flush_bytes;
  v[ST_FLUSH_BLOCKS] += c->host_flush_blocks;
  static_assert(sizeof(tgs_stats) == sizeof(uint64_t) * ST_N, "tgs_stats layout");
  std::memcpy(out, v, sizeof v);
  return TGS_OK;
}

tgs_status tgs_get_stats_async(tgs_ctx* c, tgs_stats* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  CK(cudaMemcpyAsync(out, c->d.stats, sizeof(unsigned long long) * ST_N, cudaMemcpyDeviceToHost,
                     c->compute));
  return TGS_OK;
}

tgs_status tgs_set_profiling(tgs_ctx* c, int enabled) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  c->prof = enabled != 0;
  c->tm = tgs_timing{};
  const char* tr = getenv("TGS_TRACE");
  c->trace = c->prof && tr && tr[0] == '1';
  if (c->trace) {
    if (!c->trace_base) cudaEventCreate(&c->trace_base);
    cudaEventRecord(c->trace_base, c->compute);
  }
  return TGS_OK;
}

tgs_status tgs_get_timing(tgs_ctx* c, tgs_timing* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  *out = c->tm;
  unsigned long long fr[3] = {0, 0, 0};
  CK(cudaMemcpy(fr, c->d.stats + ST_FRESH_ROWS, sizeof(fr), cudaMemcpyDeviceToHost));
  out->fresh_active_rows = fr[0];
  out->fresh_blocks = fr[1];
  out->h2d_ring_records = fr[2];
  return TGS_OK;
}

uint32_t tgs_get_list(tgs_ctx* c, int which, uint32_t* blocks, int32_t* slots, uint32_t cap) {
  if (check(c) != TGS_OK || which < 0 || which > 5) return 0;
  if (sync_all(c) != TGS_OK) return 0;
  Dev& d = c->d;
  const uint32_t Wd = std::max(d.W, 1u);
  std::vector<uint32_t> bits(Wd, 0u);
  uint32_t* src = nullptr;
  switch (which) {
    case 0: src = d.Kb; break;
    case 1: src = d.R[c->parity]; break;  // R_{t+1} (parity flipped after activate)
    case 2: src = d.Sp; break;
    case 3: src = d.Sm; break;
    case 4: src = d.Om; break;
    case 5: src = d.Ab; break;
  }
  if (c->T == 0) return 0;
  if (cudaMemcpy(bits.data(), src, sizeof(uint32_t) * Wd, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  std::vector<int32_t> b2s(std::max(d.Kloc, 1u));
  if (slots && cudaMemcpy(b2s.data(), d.b2s, sizeof(int32_t) * b2s.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  uint32_t n = 0;
  for (uint32_t w = 0; w < d.W; ++w) {
    uint32_t x = bits[w];
    while (x) {
      const int b = __builtin_ctz(x);
      x &= x - 1;
      const uint32_t l = 32 * w + b;
      if (n < cap) {
        if (blocks) blocks[n] = l * c->cfg.world_size + c->cfg.rank;
        if (slots) slots[n] = which == 3 ? -1 : b2s[l];
      }
      ++n;
    }
  }
  return n;
}

uint32_t tgs_get_percam(tgs_ctx* c, uint32_t j, uint32_t* blocks, uint32_t cap) {
  if (check(c) != TGS_OK || j >= c->d.J_max || c->T == 0) return 0;
  if (sync_all(c) != TGS_OK) return 0;
  Dev& d = c->d;
  std::vector<uint32_t> bits(std::max(d.W, 1u));
  if (cudaMemcpy(bits.data(), c->l3_percam[((uint32_t)c->T - 1) % 3u] + (size_t)j * d.W,
                 sizeof(uint32_t) * d.W,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  uint32_t n = 0;
  for (uint32_t w = 0; w < d.W; ++w)
    for (uint32_t x = bits[w]; x; x &= x - 1) {
      if (n < cap && blocks) blocks[n] = (32 * w + __builtin_ctz(x)) * c->cfg.world_size + c->cfg.rank;
      ++n;
    }
  return n;
}

uint32_t tgs_get_evicted_dirty(tgs_ctx* c, uint32_t* blocks, uint32_t cap) {
  if (check(c) != TGS_OK) return 0;
  if (sync_all(c) != TGS_OK) return 0;
  const int k = c->T > 0 ? (int)(((uint32_t)c->T - 1) % (uint32_t)c->nrings) : 0;  // the last activate's slot
  // (after an asynchronous activate the write-back kernels always ran)
  const uint32_t n = (c->T > 0 && (!c->last_known || c->last.nSm)) ? c->ndirty[k] : 0;
  for (uint32_t i = 0; i < n && i < cap; ++i)
    if (blocks) blocks[i] = c->dirty_map[k][2 * i] * c->cfg.world_size + c->cfg.rank;
  return n;
}

tgs_status tgs_get_slot_map(tgs_ctx* c, int64_t* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  std::vector<int32_t> s2b(c->d.P);
  CK(cudaMemcpy(s2b.data(), c->d.s2b, sizeof(int32_t) * c->d.P, cudaMemcpyDeviceToHost));
  for (uint32_t s = 0; s < c->d.P; ++s)
    out[s] = s2b[s] < 0 ? -1 : (int64_t)s2b[s] * c->cfg.world_size + c->cfg.rank;
  return TGS_OK;
}

uint64_t tgs_nonfinite_index(tgs_ctx* c) {
  if (check(c) != TGS_OK || sync_all(c) != TGS_OK) return ~0ull;
  unsigned long long v = ~0ull;
  if (cudaMemcpy(&v, c->d.nonfinite, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) return ~0ull;
  return v;
}

tgs_status tgs_read_block(tgs_ctx* c, uint64_t kg, float* theta, float* m, float* v) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (kg % c->cfg.world_size != (uint64_t)c->cfg.rank) return TGS_EINVAL;
  const uint64_t l = kg / c->cfg.world_size;
  if (l >= c->d.Kloc) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  int32_t s = -1;
  uint32_t stp = 0;
  CK(cudaMemcpy(&s, c->d.b2s + l, sizeof s, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&stp, c->d.step + l, sizeof stp, cudaMemcpyDeviceToHost));
  // cold restart: a resident block not updated since admission has m = v = 0
  // (k_adam writes its moment record at the first update)
  const bool zero_moments = c->d.cold && s >= 0 && stp == 0;
  const size_t rb = c->rec_bytes, rf = c->d.rec_floats;
  float* outs[3] = {theta, m, v};
  std::vector<float> stored;
  const float* hrec = nullptr;
  if (s < 0 && c->store) {  // f3: CPU-cache entry, else the newest version through Index[k]
    stored.resize((size_t)c->d.n_arr * rf);
    const std::string e = c->store->read_block((uint32_t)l, stored.data());
    if (!e.empty()) {
      set_err(c, "store: %s", e.c_str());
      return TGS_EIO;
    }
    hrec = stored.data();
  } else if (s < 0) {
    hrec = host_rec(c, (uint32_t)l);
  }
  for (int a = 0; a < 3; ++a) {
    if (!outs[a]) continue;
    if (s >= 0 && a > 0 && zero_moments) {
      std::memset(outs[a], 0, rb);
    } else if (s >= 0) {
      CK(cudaMemcpy(outs[a], slot_rec(c, (uint32_t)s) + a * rf, rb, cudaMemcpyDeviceToHost));
    } else if (a < (int)c->d.n_arr) {
      std::memcpy(outs[a], hrec + a * rf, rb);
    } else {
      std::memset(outs[a], 0, rb);  // cold restart: moments do not exist off the device
    }
  }
  return TGS_OK;
}

uint32_t tgs_step_count(tgs_ctx* c, uint64_t kg) {
  if (check(c) != TGS_OK || kg % c->cfg.world_size != (uint64_t)c->cfg.rank) return 0;
  const uint64_t l = kg / c->cfg.world_size;
  if (l >= c->d.Kloc || sync_all(c) != TGS_OK) return 0;
  uint32_t s = 0;
  cudaMemcpy(&s, c->d.step + l, sizeof s, cudaMemcpyDeviceToHost);
  return s;
}

tgs_status tgs_read_bound(tgs_ctx* c, uint64_t kg, float* out4) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out4 || kg % c->cfg.world_size != (uint64_t)c->cfg.rank) return TGS_EINVAL;
  const uint64_t l = kg / c->cfg.world_size;
  if (l >= c->d.Kloc) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  CK(cudaMemcpy(out4, c->d.bounds + l, sizeof(float4), cudaMemcpyDeviceToHost));
  return TGS_OK;
}

uint32_t tgs_num_local_blocks(const tgs_ctx* c) { return c ? c->d.Kloc : 0; }
uint32_t tgs_pool_slots(const tgs_ctx* c) { return c ? c->d.P : 0; }

tgs_status tgs_build_layout(const float* cs, uint64_t n, uint32_t block_size, int device,
                            uint64_t* perm, float* bounds, double* gpu_ms) {
  if (!cs || n == 0 || n > 0xffffffffull || block_size == 0 || !perm || !bounds)
    return TGS_EINVAL;
  for (uint64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a)
      if (!std::isfinite(cs[4 * i + a])) return TGS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TGS_ECUDA;
  const uint64_t K = (n + block_size - 1) / block_size;
  const int part_grid = 592;
  LayoutBufs b{};
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
  b.cs = (float*)get(n * 16);
  b.k[0] = (unsigned long long*)get(n * 8);
  b.k[1] = (unsigned long long*)get(n * 8);
  b.v[0] = (uint32_t*)get(n * 4);
  b.v[1] = (uint32_t*)get(n * 4);
  b.counts = (uint32_t*)get(layout_scan_len(n) * 4);
  b.sums = (uint32_t*)get((size_t)layout_nsums(n) * 4);
  b.part = (float*)get((size_t)part_grid * 6 * 4);
  b.bounds = (float*)get(K * 16);
  auto release = [&]() {
    for (void* p : allocs) cudaFree(p);
    cudaGetLastError();
  };
  if (!ok) {
    release();
    return TGS_ENOMEM;
  }
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  tgs_status st = TGS_OK;
  int cur = 0;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess ||
      cudaMemcpyAsync(b.cs, cs, n * 16, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaEventRecord(e0, s) != cudaSuccess ||
      layout_run(b, n, block_size, s, part_grid, &cur) != cudaSuccess ||
      cudaEventRecord(e1, s) != cudaSuccess) {
    st = TGS_ECUDA;
  }
  std::vector<uint32_t> p32;
  if (st == TGS_OK) {
    p32.resize(n);
    if (cudaMemcpyAsync(p32.data(), b.v[cur], n * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(bounds, b.bounds, K * 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      st = TGS_ECUDA;
  }
  if (st == TGS_OK) {
    for (uint64_t i = 0; i < n; ++i) perm[i] = p32[i];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (gpu_ms) *gpu_ms = ms;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  release();
  return st;
}

tgs_status tgs_frustum_planes(const double w2c[16], double fx, double fy, double cx, double cy,
                              uint32_t width, uint32_t height, double znear, double zfar,
                              tgs_camera* out) {
  if (!w2c || !out || !(fx > 0) || !(fy > 0) || width == 0 || height == 0 || !(znear > 0) ||
      !(zfar > znear))
    return TGS_EINVAL;
  // camera-space planes (inside iff n.pc + d >= 0): x >= -cx z/fx, x <= (w-cx) z/fx, ...
  const double pc[6][4] = {
      {fx, 0.0, cx, 0.0},  {-fx, 0.0, (double)width - cx, 0.0},
      {0.0, fy, cy, 0.0},  {0.0, -fy, (double)height - cy, 0.0},
      {0.0, 0.0, 1.0, -znear}, {0.0, 0.0, -1.0, zfar},
  };
  // world plane: n_w = R^T n_c, d_w = n_c . t + d_c   (pc = R p + t)
  for (int p = 0; p < 6; ++p) {
    const double nn = std::sqrt(pc[p][0] * pc[p][0] + pc[p][1] * pc[p][1] + pc[p][2] * pc[p][2]);
    double n[3] = {pc[p][0] / nn, pc[p][1] / nn, pc[p][2] / nn};
    double dc = pc[p][3] / nn;
    double nw[3];
    for (int i = 0; i < 3; ++i) nw[i] = n[0] * w2c[0 * 4 + i] + n[1] * w2c[1 * 4 + i] + n[2] * w2c[2 * 4 + i];
    const double dw = n[0] * w2c[3] + n[1] * w2c[7] + n[2] * w2c[11] + dc;
    const double len = std::sqrt(nw[0] * nw[0] + nw[1] * nw[1] + nw[2] * nw[2]);
    for (int i = 0; i < 3; ++i) out->plane[p][i] = (float)(nw[i] / len);
    out->plane[p][3] = (float)(dw / len);
  }
  return TGS_OK;
}

// ---- NEXT f3 inspection
tgs_status tgs_prefetch(tgs_ctx* c, const tgs_camera* cams, uint32_t J, uint32_t ahead) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (J > c->d.J_max || (J > 0 && !cams) || ahead == 0) return TGS_EINVAL;
  for (uint32_t j = 0; j < J; ++j)
    for (int p = 0; p < 6; ++p)
      for (int i = 0; i < 4; ++i)
        if (!std::isfinite(cams[j].plane[p][i])) return TGS_EINVAL;
  if (!c->store || J == 0 || c->d.Kloc == 0) return TGS_OK;
  // the third staging buffer: k_probe reads it on the plan stream, and the host
  // waits for that before returning, so the next prefetch may reuse it
  float* pl = c->planes_pinned + (size_t)3 * kMaxCams * 24;
  std::memcpy(pl, cams, sizeof(float) * 24 * J);
  float* pl_dev = nullptr;
  uint32_t* out_dev = nullptr;
  CK(cudaHostGetDevicePointer((void**)&pl_dev, pl, 0));
  CK(cudaHostGetDevicePointer((void**)&out_dev, c->probe_map, 0));
  CK(launch_probe(c->d, reinterpret_cast<const float4*>(pl_dev), J, out_dev, c->plan));
  c->tm.kernel_launches++;
  CK(cudaEventRecord(c->ev_probe, c->plan));
  CK(cudaEventSynchronize(c->ev_probe));
  std::vector<uint32_t> blocks;
  for (uint32_t w = 0; w < c->d.W; ++w)
    for (uint32_t bits = c->probe_map[w]; bits; bits &= bits - 1)
      blocks.push_back(32u * w + (uint32_t)__builtin_ctz(bits));
  c->store->prefetch(blocks, c->T + (int32_t)ahead - 1);
  return TGS_OK;
}

tgs_status tgs_get_store_stats(tgs_ctx* c, tgs_store_stats* out) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!out) return TGS_EINVAL;
  if (!c->store) return TGS_ESTATE;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  c->store->settle();  // no read-ahead batch in flight
  const tgs::StoreCounters& k = c->store->counters();
  out->hits = k.hits;
  out->misses = k.misses;
  out->evictions = k.evictions;
  out->dirty_evictions = k.dirty_evictions;
  out->flush_appends = k.flush_appends;
  out->read_bytes = k.read_bytes;
  out->write_bytes = k.write_bytes;
  out->segments = k.segments;
  out->cached = c->store->cached();
  out->cached_dirty = c->store->cached_dirty();
  out->read_ms = k.read_ms;
  out->write_ms = k.write_ms;
  out->read_calls = k.read_calls;
  out->read_busy_ms = k.read_busy_ms;
  out->prefetch_reads = k.prefetch_reads;
  out->prefetch_hits = k.prefetch_hits;
  out->prefetch_wasted = k.prefetch_wasted;
  return TGS_OK;
}

tgs_status tgs_store_index(tgs_ctx* c, uint64_t kg, uint64_t* out4) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!c->store) return TGS_ESTATE;
  if (!out4 || kg % c->cfg.world_size != (uint64_t)c->cfg.rank) return TGS_EINVAL;
  const uint64_t l = kg / c->cfg.world_size;
  if (l >= c->d.Kloc) return TGS_EINVAL;
  st = sync_all(c);
  if (st != TGS_OK) return st;
  const tgs::StoreIndex& ix = c->store->index((uint32_t)l);
  out4[0] = ix.file_id;
  out4[1] = ix.offset;
  out4[2] = ix.size;
  out4[3] = ix.version;
  return TGS_OK;
}

tgs_status tgs_store_compact(tgs_ctx* c) {
  tgs_status st = check(c);
  if (st != TGS_OK) return st;
  if (!c->store) return TGS_ESTATE;
  st = tgs_flush(c);  // the barrier
  if (st != TGS_OK) return st;
  const std::string e = c->store->compact();
  if (!e.empty()) {
    c->poisoned = true;
    set_err(c, "store: %s", e.c_str());
    return TGS_EIO;
  }
  return TGS_OK;
}

uint32_t tgs_store_lru(tgs_ctx* c, uint32_t* blocks, uint8_t* dirty, uint32_t cap) {
  if (check(c) != TGS_OK || !c->store || sync_all(c) != TGS_OK) return 0;
  std::vector<uint32_t> b;
  std::vector<uint8_t> d;
  c->store->lru_order(b, d);
  for (uint32_t i = 0; i < b.size() && i < cap; ++i) {
    if (blocks) blocks[i] = b[i] * c->cfg.world_size + c->cfg.rank;
    if (dirty) dirty[i] = d[i];
  }
  return (uint32_t)b.size();
}

}  // extern "C"
