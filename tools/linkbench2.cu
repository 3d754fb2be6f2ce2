// linkbench2.cu -- one step's host-link traffic (the default 300m bench: ~382 S+
// records in, ~228 dirty S- records out, 966,656 B each), moved by candidate
// a4 mechanisms: SM zero-copy gather/scatter kernels (plain 16-B loads, deeper
// unrolled loads, TMA bulk copies through shared memory), per-record copy-engine
// copies, and copy-engine copies of contiguous runs.  Reports each direction's
// rate and the time until both are done, alone and beside a many-wave HBM-bound
// kernel (the Adam stand-in), whose rate is reported too.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/linkbench2 tools/linkbench2.cu
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr uint32_t kRec = 4096 * 59 * 4;  // 966,656 B
constexpr uint32_t kRec4 = kRec / 16;

// element e of a list of records: record r = e / rec4 is list[r] on the indirect side
template <int U>
__global__ void zc_move(float4* __restrict__ dst, const float4* __restrict__ src,
                        const uint32_t* __restrict__ list, uint32_t n, int gather) {
  const uint64_t total = (uint64_t)n * kRec4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto at = [&](uint64_t e, bool is_src) -> uint64_t {
    const uint64_t r = e / kRec4, f = e - r * kRec4;
    const bool ind = (gather != 0) == is_src;
    return (ind ? (uint64_t)list[r] : r) * kRec4 + f;
  };
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < total; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + at(i + u * stride, true));
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + at(i + u * stride, false), v[u]);
  }
  for (; i < total; i += stride) __stcs(dst + at(i, false), __ldcs(src + at(i, true)));
}

// TMA bulk gather: one elected thread per CTA streams chunks of the CTA's records
// host -> smem (cp.async.bulk + mbarrier) -> device (cp.async.bulk.global.shared)
constexpr uint32_t kChunk = 32768, kNbuf = 6;
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__global__ void __launch_bounds__(32) tma_gather(char* __restrict__ dst, const char* __restrict__ src,
                                                 const uint32_t* __restrict__ list, uint32_t n,
                                                 int gather) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t bar[kNbuf];
  if (threadIdx.x != 0) return;
  for (uint32_t b = 0; b < kNbuf; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t per_rec = (kRec + kChunk - 1) / kChunk;
  const uint64_t nchunks = (uint64_t)n * per_rec;
  uint32_t phase[kNbuf] = {};
  // chunk c of this CTA: global chunk id blockIdx.x + c * gridDim.x
  auto geo = [&](uint64_t g, const char*& s, char*& d, uint32_t& bytes) {
    const uint64_t r = g / per_rec, k = g - r * per_rec;
    const uint64_t off = k * kChunk;
    bytes = (uint32_t)((kRec - off) < kChunk ? (kRec - off) : kChunk);
    const uint64_t rs = gather ? list[r] : r, rd = gather ? r : list[r];
    s = src + rs * kRec + off;
    d = dst + rd * kRec + off;
  };
  uint64_t issued = 0, done = 0;
  const uint64_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](uint64_t c) {
    const uint32_t b = (uint32_t)(c % kNbuf);
    const char* s; char* d; uint32_t bytes;
    geo(blockIdx.x + c * gridDim.x, s, d, bytes);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[b])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(buf + (size_t)b * kChunk)), "l"(s), "r"(bytes), "r"(smem_u32(&bar[b])) : "memory");
  };
  for (; issued < mine && issued < kNbuf; ++issued) issue(issued);
  for (; done < mine; ++done) {
    const uint32_t b = (uint32_t)(done % kNbuf);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&bar[b])), "r"(phase[b]) : "memory");
    phase[b] ^= 1u;
    const char* s; char* d; uint32_t bytes;
    geo(blockIdx.x + done * gridDim.x, s, d, bytes);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(d), "r"(smem_u32(buf + (size_t)b * kChunk)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < mine) {
      // the store of the oldest buffer must have read it before it is refilled
      asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(kNbuf - 1) : "memory");
      issue(issued++);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// many short CTAs, each streaming a 256 KB piece (Adam-like occupancy behaviour)
__global__ void __launch_bounds__(256) hbm_pieces(float4* __restrict__ dst, const float4* __restrict__ src) {
  const size_t base = (size_t)blockIdx.x * (262144 / 16);
  for (uint32_t i = threadIdx.x; i < 262144 / 16; i += 256) __stcs(dst + base + i, __ldcs(src + base + i));
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) { float m; cudaEventElapsedTime(&m, a, b); return m; }

int main(int argc, char** argv) {
  const bool tma_only = argc > 1 && !strcmp(argv[1], "tma");
  const bool dma_only = argc > 1 && !strcmp(argv[1], "dma");
  const bool graph_only = argc > 1 && !strcmp(argv[1], "graph");
  const int nh = 382, nd = 228;
  // LB_HOST_RECS: size of the pinned host tier in records (default 8192 = 7.9 GB;
  // the 300m bench's is 73,243 = 70.8 GB)
  const size_t host_recs = getenv("LB_HOST_RECS") ? (size_t)atoll(getenv("LB_HOST_RECS")) : 8192;
  char* h_tier;
  CK(cudaHostAlloc((void**)&h_tier, (size_t)kRec * host_recs, cudaHostAllocMapped));
  for (size_t i = 0; i < (size_t)kRec * host_recs; i += 4096) h_tier[i] = 1;
  char *d_slots, *d_ring;
  CK(cudaMalloc(&d_slots, (size_t)kRec * nh));
  CK(cudaMalloc(&d_ring, (size_t)kRec * nd));
  CK(cudaMemset(d_ring, 0, (size_t)kRec * nd));
  std::vector<uint32_t> perm(host_recs);
  for (size_t i = 0; i < host_recs; ++i) perm[i] = (uint32_t)i;
  uint64_t st = 88172645463325252ull;
  for (size_t i = host_recs - 1; i > 0; --i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    std::swap(perm[i], perm[st % (i + 1)]);
  }
  std::vector<uint32_t> src_l(perm.begin(), perm.begin() + nh), dst_l(perm.begin() + nh, perm.begin() + nh + nd);
  // runs of R consecutive host records for the run-length d2h variants
  const uint32_t run0 = perm[nh + nd] % (uint32_t)(host_recs - 16 * nd);
  uint32_t *d_src_l, *d_dst_l;
  CK(cudaMalloc(&d_src_l, nh * 4));
  CK(cudaMalloc(&d_dst_l, nd * 4));
  CK(cudaMemcpy(d_src_l, src_l.data(), nh * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_dst_l, dst_l.data(), nd * 4, cudaMemcpyHostToDevice));
  char* h_dev;
  CK(cudaHostGetDevicePointer((void**)&h_dev, h_tier, 0));
  cudaStream_t hs, ds, fork, hb;
  CK(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&fork, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&hb, cudaStreamNonBlocking));
  cudaEvent_t e0, eh, ed, ehb;
  for (cudaEvent_t* ev : {&e0, &eh, &ed, &ehb}) CK(cudaEventCreate(ev));
  const size_t hbm_bytes = (size_t)4 << 30;
  char *x, *y;
  CK(cudaMalloc(&x, hbm_bytes));
  CK(cudaMalloc(&y, hbm_bytes));
  CK(cudaMemset(x, 0, hbm_bytes));
  CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, kChunk * kNbuf));

  using Fn = std::function<void(void)>;
  auto h_zc = [&](int g, int u) -> Fn {
    return [=] {
      if (u == 8) zc_move<8><<<g, 512, 0, hs>>>((float4*)d_slots, (const float4*)h_dev, d_src_l, nh, 1);
      else zc_move<4><<<g, 512, 0, hs>>>((float4*)d_slots, (const float4*)h_dev, d_src_l, nh, 1);
    };
  };
  auto h_tma = [&](int g) -> Fn {
    return [=] { tma_gather<<<g, 32, kChunk * kNbuf, hs>>>(d_slots, h_dev, d_src_l, nh, 1); };
  };
  auto h_dma = [&]() -> Fn {
    return [=, &src_l] { for (int i = 0; i < nh; ++i) cudaMemcpyAsync(d_slots + (size_t)i * kRec, h_tier + (size_t)src_l[i] * kRec, kRec, cudaMemcpyHostToDevice, hs); };
  };
  auto d_zc = [&](int g) -> Fn {
    return [=] { zc_move<4><<<g, 512, 0, ds>>>((float4*)h_dev, (const float4*)d_ring, d_dst_l, nd, 0); };
  };
  auto d_tma = [&](int g) -> Fn {
    return [=] { tma_gather<<<g, 32, kChunk * kNbuf, ds>>>(h_dev, d_ring, d_dst_l, nd, 0); };
  };
  auto d_dma = [&]() -> Fn {
    return [=, &dst_l] { for (int i = 0; i < nd; ++i) cudaMemcpyAsync(h_tier + (size_t)dst_l[i] * kRec, d_ring + (size_t)i * kRec, kRec, cudaMemcpyDeviceToHost, ds); };
  };
  auto d_runs = [&](int R) -> Fn {  // contiguous runs of R records (a log-structured append)
    return [=] { for (int i = 0; i < nd; i += R) cudaMemcpyAsync(h_tier + (size_t)(run0 + i) * kRec, d_ring + (size_t)i * kRec, (size_t)std::min(R, nd - i) * kRec, cudaMemcpyDeviceToHost, ds); };
  };
  // copy-engine copies spread round-robin over S streams per direction, joined back
  // into hs / ds by events (several copies in flight per direction)
  cudaStream_t hsx[8], dsx[8];
  cudaEvent_t ejh[8], ejd[8], efk;
  for (int i = 0; i < 8; ++i) {
    CK(cudaStreamCreateWithFlags(&hsx[i], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&dsx[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ejh[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ejd[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&efk, cudaEventDisableTiming));
  auto h_dma_s = [&](int S) -> Fn {
    return [=, &src_l] {
      CK(cudaEventRecord(efk, hs));
      for (int k = 0; k < S; ++k) CK(cudaStreamWaitEvent(hsx[k], efk, 0));
      for (int i = 0; i < nh; ++i) cudaMemcpyAsync(d_slots + (size_t)i * kRec, h_tier + (size_t)src_l[i] * kRec, kRec, cudaMemcpyHostToDevice, hsx[i % S]);
      for (int k = 0; k < S; ++k) { CK(cudaEventRecord(ejh[k], hsx[k])); CK(cudaStreamWaitEvent(hs, ejh[k], 0)); }
    };
  };
  auto d_dma_s = [&](int S) -> Fn {
    return [=, &dst_l] {
      CK(cudaEventRecord(efk, ds));
      for (int k = 0; k < S; ++k) CK(cudaStreamWaitEvent(dsx[k], efk, 0));
      for (int i = 0; i < nd; ++i) cudaMemcpyAsync(h_tier + (size_t)dst_l[i] * kRec, d_ring + (size_t)i * kRec, kRec, cudaMemcpyDeviceToHost, dsx[i % S]);
      for (int k = 0; k < S; ++k) { CK(cudaEventRecord(ejd[k], dsx[k])); CK(cudaStreamWaitEvent(ds, ejd[k], 0)); }
    };
  };
  auto h_runs = [&](int R) -> Fn {  // h2d copies of contiguous host runs of R records
    return [=] { for (int i = 0; i < nh; i += R) cudaMemcpyAsync(d_slots + (size_t)i * kRec, h_tier + (size_t)(run0 + i) * kRec, (size_t)std::min(R, nh - i) * kRec, cudaMemcpyHostToDevice, hs); };
  };
  auto hbm = [&]() { hbm_pieces<<<(unsigned)(hbm_bytes / 262144), 256, 0, hb>>>((float4*)y, (const float4*)x); };

  auto run = [&](const char* name, Fn h, Fn d, bool with_hbm = false) {
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, fork));
      for (cudaStream_t s : {hs, ds, hb}) CK(cudaStreamWaitEvent(s, e0, 0));
      if (with_hbm) { hbm(); hbm(); }
      if (h) h();
      if (d) d();
      CK(cudaEventRecord(eh, hs));
      CK(cudaEventRecord(ed, ds));
      CK(cudaEventRecord(ehb, hb));
      CK(cudaDeviceSynchronize());
      if (rep < 2) continue;
      const float th = ms_between(e0, eh), td = ms_between(e0, ed);
      printf("%-44s", name);
      if (h) printf(" h2d %6.2f", (double)kRec * nh / (th * 1e6));
      if (d) printf(" d2h %6.2f", (double)kRec * nd / (td * 1e6));
      printf(" GB/s  done %6.3f ms", std::max(h ? th : 0.f, d ? td : 0.f));
      if (with_hbm) printf("  | HBM %.0f GB/s", 2 * 2.0 * hbm_bytes / (ms_between(e0, ehb) * 1e6));
      printf("\n");
    }
  };
  printf("# one step: %d records in (h2d), %d out (d2h), %u B each\n", nh, nd, kRec);
  // CUDA graphs of per-record memcpy nodes (independent, or chained), instantiated
  // once and re-launched; plus the host cost of re-pointing every node
  auto make_graph = [&](bool h2d, bool chain, cudaGraphExec_t& ge, std::vector<cudaGraphNode_t>& nodes) {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    const int n = h2d ? nh : nd;
    nodes.assign(n, nullptr);
    for (int i = 0; i < n; ++i) {
      void* dst = h2d ? (void*)(d_slots + (size_t)i * kRec) : (void*)(h_tier + (size_t)dst_l[i] * kRec);
      const void* src = h2d ? (const void*)(h_tier + (size_t)src_l[i] * kRec) : (const void*)(d_ring + (size_t)i * kRec);
      CK(cudaGraphAddMemcpyNode1D(&nodes[i], g, (chain && i) ? &nodes[i - 1] : nullptr, (chain && i) ? 1 : 0,
                                  dst, src, kRec, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
    }
    CK(cudaGraphInstantiate(&ge, g, 0));
  };
  if (graph_only) {
    for (int chain = 0; chain < 2; ++chain) {
      cudaGraphExec_t gh, gd;
      std::vector<cudaGraphNode_t> nhv, ndv;
      auto t0 = std::chrono::steady_clock::now();
      make_graph(true, chain, gh, nhv);
      auto t1 = std::chrono::steady_clock::now();
      make_graph(false, chain, gd, ndv);
      printf("# graph build+instantiate (%s): h2d %.2f ms for %d nodes\n", chain ? "chained" : "independent",
             std::chrono::duration<double, std::milli>(t1 - t0).count(), nh);
      // re-point every node (what a per-step update costs on the host)
      t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < nh; ++i)
        CK(cudaGraphExecMemcpyNodeSetParams1D(gh, nhv[i], d_slots + (size_t)i * kRec, h_tier + (size_t)src_l[(i + 1) % nh] * kRec, kRec, cudaMemcpyHostToDevice));
      t1 = std::chrono::steady_clock::now();
      printf("# SetParams1D x %d: %.3f ms host\n", nh, std::chrono::duration<double, std::milli>(t1 - t0).count());
      char nm[96];
      snprintf(nm, sizeof nm, "h2d graph %s alone", chain ? "chained" : "indep");
      run(nm, [=] { cudaGraphLaunch(gh, hs); }, nullptr);
      snprintf(nm, sizeof nm, "d2h graph %s alone", chain ? "chained" : "indep");
      run(nm, nullptr, [=] { cudaGraphLaunch(gd, ds); });
      snprintf(nm, sizeof nm, "h2d graph %s || d2h graph", chain ? "chained" : "indep");
      run(nm, [=] { cudaGraphLaunch(gh, hs); }, [=] { cudaGraphLaunch(gd, ds); });
      snprintf(nm, sizeof nm, "h2d graph %s || d2h graph || HBM", chain ? "chained" : "indep");
      run(nm, [=] { cudaGraphLaunch(gh, hs); }, [=] { cudaGraphLaunch(gd, ds); }, true);
    }
    run("h2d DMA x1 || d2h DMA x1 (per record, stream)", h_dma_s(1), d_dma_s(1));
    run("h2d DMA runs of 8 || d2h DMA runs of 8", h_runs(8), d_runs(8));
    return 0;
  }
  if (argc > 1 && !strcmp(argv[1], "mix")) {  // copy-engine runs in, TMA kernel out (and back)
    for (int g : {1, 2, 4, 8}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d DMA runs of 6 || d2h TMA %d", g);
      run(nm, h_runs(6), d_tma(g));
      snprintf(nm, sizeof nm, "h2d DMA runs of 6 || d2h TMA %d || HBM", g);
      run(nm, h_runs(6), d_tma(g), true);
    }
    run("h2d DMA runs of 6 || d2h DMA runs of 8", h_runs(6), d_runs(8));
    run("h2d DMA runs of 6 || d2h DMA runs of 8 || HBM", h_runs(6), d_runs(8), true);
    return 0;
  }
  if (dma_only) {
    run("h2d DMA runs of all (one copy)", h_runs(nh), nullptr);
    run("d2h DMA runs of all (one copy)", nullptr, d_runs(nd));
    run("h2d DMA runs of all || d2h DMA runs of all", h_runs(nh), d_runs(nd));
    run("h2d DMA runs of 8 || d2h DMA runs of 8", h_runs(8), d_runs(8));
    for (int S : {1, 2, 3, 4, 6, 8}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d DMA x%d streams", S);
      run(nm, h_dma_s(S), nullptr);
      snprintf(nm, sizeof nm, "d2h DMA x%d streams", S);
      run(nm, nullptr, d_dma_s(S));
      snprintf(nm, sizeof nm, "h2d DMA x%d || d2h DMA x%d", S, S);
      run(nm, h_dma_s(S), d_dma_s(S));
      snprintf(nm, sizeof nm, "h2d DMA x%d || d2h DMA x%d || HBM", S, S);
      run(nm, h_dma_s(S), d_dma_s(S), true);
    }
    for (int S : {2, 4}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d TMA 8 || d2h DMA x%d", S);
      run(nm, h_tma(8), d_dma_s(S));
      snprintf(nm, sizeof nm, "h2d DMA x%d || d2h TMA 4", S);
      run(nm, h_dma_s(S), d_tma(4));
      snprintf(nm, sizeof nm, "h2d DMA x%d || d2h TMA 4 || HBM", S);
      run(nm, h_dma_s(S), d_tma(4), true);
    }
    run("h2d TMA 8 || d2h TMA 4", h_tma(8), d_tma(4));
    run("h2d TMA 8 || d2h TMA 4 || HBM", h_tma(8), d_tma(4), true);
    return 0;
  }
  if (tma_only) {
    for (int g : {1, 2, 4, 8, 16, 32}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d TMA gather grid %d", g);
      run(nm, h_tma(g), nullptr);
    }
    for (int g : {4, 8, 16}) {
      char nm[96];
      snprintf(nm, sizeof nm, "d2h TMA scatter grid %d", g);
      run(nm, nullptr, d_tma(g));
      snprintf(nm, sizeof nm, "h2d TMA %d || d2h ZC 16", g);
      run(nm, h_tma(g), d_zc(16));
      snprintf(nm, sizeof nm, "h2d TMA %d || d2h TMA %d", g, g);
      run(nm, h_tma(g), d_tma(g));
      snprintf(nm, sizeof nm, "h2d TMA %d || d2h runs of all", g);
      run(nm, h_tma(g), d_runs(nd));
      snprintf(nm, sizeof nm, "h2d TMA %d || d2h ZC 16 || HBM", g);
      run(nm, h_tma(g), d_zc(16), true);
    }
    return 0;
  }
  run("HBM pieces alone", nullptr, nullptr, true);
  run("h2d DMA per record || d2h DMA per record", h_dma(), d_dma());
  run("h2d DMA per record || d2h DMA per record || HBM", h_dma(), d_dma(), true);
  for (int g : {8, 16, 32, 64, 148}) {
    for (int g2 : {8, 16, 32}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d ZC %d || d2h ZC %d", g, g2);
      run(nm, h_zc(g, 4), d_zc(g2));
    }
  }
  for (int g : {4, 8, 16}) {
    char nm[96];
    snprintf(nm, sizeof nm, "h2d ZC-u8 %d || d2h ZC 16", g);
    run(nm, h_zc(g, 8), d_zc(16));
  }
  for (int g : {16, 32, 64}) {
    for (int R : {1, 4, 8, 16, 228}) {
      char nm[96];
      snprintf(nm, sizeof nm, "h2d ZC %d || d2h DMA runs of %d", g, R);
      run(nm, h_zc(g, 4), R == 1 ? d_dma() : d_runs(R));
    }
  }
  run("h2d ZC 32 || d2h ZC 16 || HBM", h_zc(32, 4), d_zc(16), true);
  run("h2d ZC 32 || d2h ZC 8 || HBM", h_zc(32, 4), d_zc(8), true);
  run("h2d ZC 16 || d2h ZC 8 || HBM", h_zc(16, 4), d_zc(8), true);
  run("h2d ZC 32 || d2h runs of 8 || HBM", h_zc(32, 4), d_runs(8), true);
  return 0;
}
