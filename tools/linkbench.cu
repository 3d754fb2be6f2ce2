// linkbench.cu -- host<->device link microbenchmark for the a4 gather / write-back
// design without batched copy submission: per-record copy-engine copies spread
// over several streams, SM zero-copy gather/scatter kernels over a record list,
// and one large contiguous copy (the write-back into a log-structured host tier),
// each alone and with the opposite direction running concurrently.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/linkbench tools/linkbench.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

// one CTA-stride loop over (record, float4) of a list of records: dst[i] <- src[list[i]]
// (gather) or dst[list[i]] <- src[i] (scatter); 4 independent 16-B loads in flight per thread
__global__ void zc_move(float4* __restrict__ dst, const float4* __restrict__ src,
                        const uint32_t* __restrict__ list, uint32_t n, uint32_t rec4, int gather) {
  const uint64_t total = (uint64_t)n * rec4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto at = [&](uint64_t e, bool is_src) -> uint64_t {
    const uint64_t r = e / rec4, f = e - r * rec4;
    const bool indirect = (gather != 0) == is_src;
    return (indirect ? (uint64_t)list[r] : r) * rec4 + f;
  };
  for (; i + 3 * stride < total; i += 4 * stride) {
    float4 a = __ldcs(src + at(i, true)), b = __ldcs(src + at(i + stride, true));
    float4 c = __ldcs(src + at(i + 2 * stride, true)), d = __ldcs(src + at(i + 3 * stride, true));
    __stcs(dst + at(i, false), a);
    __stcs(dst + at(i + stride, false), b);
    __stcs(dst + at(i + 2 * stride, false), c);
    __stcs(dst + at(i + 3 * stride, false), d);
  }
  for (; i < total; i += stride) __stcs(dst + at(i, false), __ldcs(src + at(i, true)));
}

__global__ void hbm_copy(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
    __stcs(dst + i, __ldcs(src + i));
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) { float m; cudaEventElapsedTime(&m, a, b); return m; }

int main(int argc, char** argv) {
  const size_t rec = 4096 * 59 * 4;  // 966,656 B
  const int n = argc > 1 ? atoi(argv[1]) : 370;
  const size_t bytes = rec * n;
  const size_t host_recs = 8192;     // 7.9 GB pinned host region, records scattered in it
  char *h_tier;
  CK(cudaHostAlloc((void**)&h_tier, rec * host_recs, cudaHostAllocMapped));
  for (size_t i = 0; i < rec * host_recs; i += 4096) h_tier[i] = 1;
  char *d_slots, *d_ring;
  CK(cudaMalloc(&d_slots, bytes * 2));
  CK(cudaMalloc(&d_ring, bytes));
  CK(cudaMemset(d_slots, 0, bytes * 2));
  CK(cudaMemset(d_ring, 0, bytes));
  // S+ sources and write-back destinations: distinct random host records
  std::vector<uint32_t> perm(host_recs);
  for (size_t i = 0; i < host_recs; ++i) perm[i] = (uint32_t)i;
  uint64_t st = 88172645463325252ull;
  for (size_t i = host_recs - 1; i > 0; --i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    std::swap(perm[i], perm[st % (i + 1)]);
  }
  std::vector<uint32_t> src_l(perm.begin(), perm.begin() + n), dst_l(perm.begin() + n, perm.begin() + 2 * n);
  const uint32_t run0 = perm[2 * n] % (uint32_t)(host_recs - n);  // contiguous append target
  uint32_t *d_src_l, *d_dst_l;
  CK(cudaMalloc(&d_src_l, n * 4));
  CK(cudaMalloc(&d_dst_l, n * 4));
  CK(cudaMemcpy(d_src_l, src_l.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_dst_l, dst_l.data(), n * 4, cudaMemcpyHostToDevice));
  char* h_dev;
  CK(cudaHostGetDevicePointer((void**)&h_dev, h_tier, 0));

  const int NS = 8;
  cudaStream_t hs[NS], ds[NS], fork, hb_s;
  for (int i = 0; i < NS; ++i) {
    CK(cudaStreamCreateWithFlags(&hs[i], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ds[i], cudaStreamNonBlocking));
  }
  CK(cudaStreamCreateWithFlags(&fork, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&hb_s, cudaStreamNonBlocking));
  cudaEvent_t e0, eh[NS], ed[NS], ehb;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&ehb));
  for (int i = 0; i < NS; ++i) { CK(cudaEventCreate(&eh[i])); CK(cudaEventCreate(&ed[i])); }

  // H2D variants: per-record DMA over k streams, zero-copy gather with grid g
  using Fn = std::function<void(void)>;
  auto h2d_dma = [&](int k) -> Fn {
    return [=, &src_l] { for (int i = 0; i < n; ++i) cudaMemcpyAsync(d_slots + i * rec, h_tier + (size_t)src_l[i] * rec, rec, cudaMemcpyHostToDevice, hs[i % k]); };
  };
  auto h2d_zc = [&](int g) -> Fn {
    return [=] { zc_move<<<g, 512, 0, hs[0]>>>((float4*)d_slots, (const float4*)h_dev, d_src_l, n, rec / 16, 1); };
  };
  auto h2d_big = [&]() -> Fn { return [=] { cudaMemcpyAsync(d_slots, h_tier, bytes, cudaMemcpyHostToDevice, hs[0]); }; };
  auto d2h_dma = [&](int k) -> Fn {
    return [=, &dst_l] { for (int i = 0; i < n; ++i) cudaMemcpyAsync(h_tier + (size_t)dst_l[i] * rec, d_ring + i * rec, rec, cudaMemcpyDeviceToHost, ds[i % k]); };
  };
  auto d2h_zc = [&](int g) -> Fn {
    return [=] { zc_move<<<g, 512, 0, ds[0]>>>((float4*)h_dev, (const float4*)d_ring, d_dst_l, n, rec / 16, 0); };
  };
  auto d2h_big = [&]() -> Fn { return [=] { cudaMemcpyAsync(h_tier + (size_t)run0 * rec, d_ring, bytes, cudaMemcpyDeviceToHost, ds[0]); }; };
  auto d2h_big_k = [&](int k) -> Fn {  // the append split into k equal pieces on k streams
    return [=] {
      const size_t per = (size_t)(n + k - 1) / k;
      for (int i = 0; i < k; ++i) {
        const size_t a = i * per, b = std::min<size_t>(n, a + per);
        if (a < b) cudaMemcpyAsync(h_tier + (run0 + a) * rec, d_ring + a * rec, (b - a) * rec, cudaMemcpyDeviceToHost, ds[i]);
      }
    };
  };
  const size_t hbm_bytes = (size_t)4 << 30;
  char *x = nullptr, *y = nullptr;
  CK(cudaMalloc(&x, hbm_bytes));
  CK(cudaMalloc(&y, hbm_bytes));
  CK(cudaMemset(x, 0, hbm_bytes));
  auto hbm = [&](int reps) { for (int r = 0; r < reps; ++r) hbm_copy<<<148 * 4, 512, 0, hb_s>>>((float4*)y, (const float4*)x, hbm_bytes / 16); };

  // run h (may be null) and d (may be null) concurrently, optionally with the HBM kernel
  auto run = [&](const char* name, Fn h, Fn d, int hbm_reps = 0) {
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, fork));
      for (int i = 0; i < NS; ++i) { cudaStreamWaitEvent(hs[i], e0, 0); cudaStreamWaitEvent(ds[i], e0, 0); }
      cudaStreamWaitEvent(hb_s, e0, 0);
      if (hbm_reps) hbm(hbm_reps);
      if (h) h();
      if (d) d();
      for (int i = 0; i < NS; ++i) { cudaEventRecord(eh[i], hs[i]); cudaEventRecord(ed[i], ds[i]); }
      cudaEventRecord(ehb, hb_s);
      CK(cudaDeviceSynchronize());
      if (rep < 2) continue;
      float th = 0, td = 0;
      for (int i = 0; i < NS; ++i) { th = std::max(th, ms_between(e0, eh[i])); td = std::max(td, ms_between(e0, ed[i])); }
      printf("%-46s", name);
      if (h) printf(" h2d %6.2f", bytes / (th * 1e6));
      if (d) printf(" d2h %6.2f", bytes / (td * 1e6));
      if (h && d) printf(" sum %6.2f GB/s (both done %.3f ms)", 2 * bytes / (std::max(th, td) * 1e6), std::max(th, td));
      else printf(" GB/s");
      if (hbm_reps) printf("  | HBM kernel %.1f GB/s", hbm_reps * 2.0 * hbm_bytes / (ms_between(e0, ehb) * 1e6));
      printf("\n");
    }
  };
  printf("# %d records of %zu B, host records scattered over %zu pinned records\n", n, rec, host_recs);
  run("HBM kernel alone", nullptr, nullptr, 4);
  run("h2d one copy", h2d_big(), nullptr);
  run("d2h one copy", nullptr, d2h_big());
  run("h2d one || d2h one", h2d_big(), d2h_big());
  for (int k : {1, 2, 4, 8}) {
    char nm[96];
    snprintf(nm, sizeof nm, "h2d per-record DMA, %d streams", k);
    run(nm, h2d_dma(k), nullptr);
    snprintf(nm, sizeof nm, "d2h per-record DMA, %d streams", k);
    run(nm, nullptr, d2h_dma(k));
    snprintf(nm, sizeof nm, "h2d DMA %d st || d2h DMA %d st", k, k);
    run(nm, h2d_dma(k), d2h_dma(k));
    snprintf(nm, sizeof nm, "h2d DMA %d st || d2h one copy", k);
    run(nm, h2d_dma(k), d2h_big());
    snprintf(nm, sizeof nm, "h2d DMA %d st || d2h append in %d pieces", k, k);
    run(nm, h2d_dma(k), d2h_big_k(k));
  }
  for (int g : {4, 8, 16, 32, 148}) {
    char nm[96];
    snprintf(nm, sizeof nm, "h2d ZC gather grid %d", g);
    run(nm, h2d_zc(g), nullptr);
    snprintf(nm, sizeof nm, "d2h ZC scatter grid %d", g);
    run(nm, nullptr, d2h_zc(g));
    snprintf(nm, sizeof nm, "h2d ZC %d || d2h one copy", g);
    run(nm, h2d_zc(g), d2h_big());
    snprintf(nm, sizeof nm, "h2d ZC %d || d2h ZC %d", g, g);
    run(nm, h2d_zc(g), d2h_zc(g));
    snprintf(nm, sizeof nm, "h2d ZC %d || d2h DMA 4 st", g);
    run(nm, h2d_zc(g), d2h_dma(4));
  }
  // contention with an HBM-bound kernel (Adam stand-in)
  run("h2d DMA 4 st || d2h one copy || HBM", h2d_dma(4), d2h_big(), 4);
  run("h2d ZC 16 || d2h one copy || HBM", h2d_zc(16), d2h_big(), 4);
  run("h2d ZC 16 || d2h ZC 16 || HBM", h2d_zc(16), d2h_zc(16), 4);
  run("h2d DMA 4 st || d2h DMA 4 st || HBM", h2d_dma(4), d2h_dma(4), 4);
  return 0;
}
