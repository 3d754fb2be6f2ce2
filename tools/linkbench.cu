// linkbench.cu -- host<->device link microbenchmark for the a4 gather/write-back
// design (copy engines vs SM zero-copy, 1-D vs pitched, one vs both directions).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/linkbench tools/linkbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void zc_copy(float4* __restrict__ dst, const float4* __restrict__ src, size_t n4) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}

static float ms_between(cudaEvent_t a, cudaEvent_t b) { float m; cudaEventElapsedTime(&m, a, b); return m; }

int main() {
  const size_t rec = 4096 * 59 * 4;  // 966,656 B
  const int n = 370;
  const size_t bytes = rec * n;
  char *h_src, *h_dst;
  CK(cudaHostAlloc((void**)&h_src, bytes * 3, cudaHostAllocMapped));
  CK(cudaHostAlloc((void**)&h_dst, bytes * 3, cudaHostAllocMapped));
  for (size_t i = 0; i < bytes * 3; i += 4096) h_src[i] = 1, h_dst[i] = 2;
  char *d_a, *d_b;
  CK(cudaMalloc(&d_a, bytes * 3));
  CK(cudaMalloc(&d_b, bytes * 3));
  cudaStream_t s1, s2, s3;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  cudaEvent_t e[8];
  for (auto& x : e) CK(cudaEventCreate(&x));
  char *hs_dev, *hd_dev;
  CK(cudaHostGetDevicePointer((void**)&hs_dev, h_src, 0));
  CK(cudaHostGetDevicePointer((void**)&hd_dev, h_dst, 0));

  auto h2d_1d = [&](cudaStream_t s) { for (int i = 0; i < n; ++i) cudaMemcpyAsync(d_a + i * rec, h_src + i * rec, rec, cudaMemcpyHostToDevice, s); };
  auto h2d_2d = [&](cudaStream_t s) { for (int i = 0; i < n; ++i) cudaMemcpy2DAsync(d_a + 3 * i * rec, 3 * rec, h_src + i * rec, rec, rec, 1, cudaMemcpyHostToDevice, s); };
  auto h2d_one = [&](cudaStream_t s) { cudaMemcpyAsync(d_a, h_src, bytes, cudaMemcpyHostToDevice, s); };
  auto d2h_1d = [&](cudaStream_t s) { for (int i = 0; i < n; ++i) cudaMemcpyAsync(h_dst + i * rec, d_b + i * rec, rec, cudaMemcpyDeviceToHost, s); };
  auto d2h_one = [&](cudaStream_t s) { cudaMemcpyAsync(h_dst, d_b, bytes, cudaMemcpyDeviceToHost, s); };
  auto zc_h2d = [&](cudaStream_t s, int g) { zc_copy<<<g, 512, 0, s>>>((float4*)d_a, (const float4*)hs_dev, bytes / 16); };
  auto zc_d2h = [&](cudaStream_t s, int g) { zc_copy<<<g, 512, 0, s>>>((float4*)hd_dev, (const float4*)d_b, bytes / 16); };

  auto one = [&](const char* name, auto f) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e[0], s1);
      f(s1);
      cudaEventRecord(e[1], s1);
      CK(cudaDeviceSynchronize());
      if (rep) printf("%-34s %7.2f GB/s\n", name, bytes / (ms_between(e[0], e[1]) * 1e6));
    }
  };
  auto two = [&](const char* name, auto f, auto g) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e[0], s1);
      cudaStreamWaitEvent(s2, e[0], 0);
      f(s1);
      g(s2);
      cudaEventRecord(e[1], s1);
      cudaEventRecord(e[2], s2);
      CK(cudaDeviceSynchronize());
      float a = ms_between(e[0], e[1]), b = ms_between(e[0], e[2]);
      if (rep) printf("%-34s A %7.2f GB/s  B %7.2f GB/s  total %7.2f GB/s\n", name, bytes / (a * 1e6), bytes / (b * 1e6), 2 * bytes / (std::max(a, b) * 1e6));
    }
  };
  one("h2d one copy", h2d_one);
  one("h2d 370 x 1D", h2d_1d);
  one("h2d 370 x 2D pitched", h2d_2d);
  one("d2h one copy", d2h_one);
  one("d2h 370 x 1D", d2h_1d);
  for (int g : {16, 32, 64, 148, 296, 592}) {
    char nm[64];
    snprintf(nm, sizeof nm, "zero-copy h2d kernel grid %d", g);
    one(nm, [&](cudaStream_t s) { zc_h2d(s, g); });
    snprintf(nm, sizeof nm, "zero-copy d2h kernel grid %d", g);
    one(nm, [&](cudaStream_t s) { zc_d2h(s, g); });
  }
  two("DMA h2d 1D || DMA d2h 1D", h2d_1d, d2h_1d);
  two("DMA h2d 2D || DMA d2h 1D", h2d_2d, d2h_1d);
  two("DMA h2d one || DMA d2h one", h2d_one, d2h_one);
  two("DMA h2d || ZC d2h 148", h2d_1d, [&](cudaStream_t s) { zc_d2h(s, 148); });
  two("ZC h2d 148 || DMA d2h", [&](cudaStream_t s) { zc_h2d(s, 148); }, d2h_1d);
  two("ZC h2d 148 || ZC d2h 148", [&](cudaStream_t s) { zc_h2d(s, 148); }, [&](cudaStream_t s) { zc_d2h(s, 148); });
  two("DMA h2d halves 2 streams (per-stream half bytes)", [&](cudaStream_t s) { for (int i = 0; i < n; i += 2) cudaMemcpyAsync(d_a + i * rec, h_src + i * rec, rec, cudaMemcpyHostToDevice, s); },
      [&](cudaStream_t s) { for (int i = 1; i < n; i += 2) cudaMemcpyAsync(d_a + i * rec, h_src + i * rec, rec, cudaMemcpyHostToDevice, s); });
  for (int L : {1, 2, 4, 8, 16, 37}) {
    char nm[96];
    snprintf(nm, sizeof nm, "runs of %d: DMA h2d || DMA d2h", L);
    two(nm, [&](cudaStream_t s) { for (int i = 0; i < n; i += L) cudaMemcpyAsync(d_a + i * rec, h_src + i * rec, rec * std::min(L, n - i), cudaMemcpyHostToDevice, s); },
        [&](cudaStream_t s) { for (int i = 0; i < n; i += L) cudaMemcpyAsync(h_dst + i * rec, d_b + i * rec, rec * std::min(L, n - i), cudaMemcpyDeviceToHost, s); });
  }
  // cudaMemcpyBatchAsync of 370 single records per direction
  std::vector<void*> hd(n), hs(n), dd(n), ds(n);
  std::vector<size_t> sz(n, rec);
  for (int i = 0; i < n; ++i) { hd[i] = d_a + i * rec; hs[i] = h_src + i * rec; dd[i] = h_dst + i * rec; ds[i] = d_b + i * rec; }
  cudaMemcpyAttributes at{};
  at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  at.flags = cudaMemcpyFlagPreferOverlapWithCompute;
  size_t aidx = 0, fail = 0;
  auto b_h2d = [&](cudaStream_t s) { CK(cudaMemcpyBatchAsync(hd.data(), hs.data(), sz.data(), n, &at, &aidx, 1, &fail, s)); };
  auto b_d2h = [&](cudaStream_t s) { CK(cudaMemcpyBatchAsync(dd.data(), ds.data(), sz.data(), n, &at, &aidx, 1, &fail, s)); };
  one("batch h2d 370", b_h2d);
  one("batch d2h 370", b_d2h);
  two("batch h2d || batch d2h", b_h2d, b_d2h);
  at.flags = 0;
  one("batch(noflag) h2d 370", b_h2d);
  two("batch(noflag) h2d || d2h", b_h2d, b_d2h);

  // (1) the same batches while an HBM-saturating kernel runs on a third stream
  const size_t hb = (size_t)8 << 30;
  char *x, *y;
  CK(cudaMalloc(&x, hb));
  CK(cudaMalloc(&y, hb));
  auto hbm = [&](cudaStream_t s) { for (int r = 0; r < 6; ++r) zc_copy<<<148 * 4, 512, 0, s>>>((float4*)y, (const float4*)x, hb / 16); };
  {
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e[0], s3);
    hbm(s3);
    cudaEventRecord(e[1], s3);
    CK(cudaDeviceSynchronize());
    printf("%-34s %7.1f GB/s (r+w)\n", "HBM copy kernel alone", 6 * 2.0 * hb / (ms_between(e[0], e[1]) * 1e6));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e[0], s3);
      cudaStreamWaitEvent(s1, e[0], 0);
      cudaStreamWaitEvent(s2, e[0], 0);
      hbm(s3);
      b_h2d(s1);
      b_d2h(s2);
      cudaEventRecord(e[1], s1);
      cudaEventRecord(e[2], s2);
      cudaEventRecord(e[3], s3);
      CK(cudaDeviceSynchronize());
      if (rep) printf("%-34s h2d %6.2f d2h %6.2f GB/s, HBM kernel %.2f ms\n", "batch || batch || HBM kernel",
                      bytes / (ms_between(e[0], e[1]) * 1e6), bytes / (ms_between(e[0], e[2]) * 1e6), ms_between(e[0], e[3]));
    }
  }
  CK(cudaFree(x));
  CK(cudaFree(y));
  // (2) records scattered over a large pinned host region (host-tier-like)
  const size_t big = (size_t)64 << 30;
  char* hbig;
  if (cudaHostAlloc((void**)&hbig, big, cudaHostAllocDefault) == cudaSuccess) {
    for (size_t i = 0; i < big; i += 4096) hbig[i] = 0;
    const size_t nrec = big / rec;
    std::vector<void*> bs(n), bd(n);
    uint64_t st = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
      st ^= st << 13; st ^= st >> 7; st ^= st << 17;
      char* r = hbig + (st % nrec) * rec;
      bs[i] = r;
      bd[i] = r;
    }
    auto s_h2d = [&](cudaStream_t s) { CK(cudaMemcpyBatchAsync(hd.data(), bs.data(), sz.data(), n, &at, &aidx, 1, &fail, s)); };
    auto s_d2h = [&](cudaStream_t s) { CK(cudaMemcpyBatchAsync(bd.data(), ds.data(), sz.data(), n, &at, &aidx, 1, &fail, s)); };
    one("scattered-64GB batch h2d", s_h2d);
    one("scattered-64GB batch d2h", s_d2h);
    two("scattered-64GB batch h2d || d2h", s_h2d, s_d2h);
    cudaFreeHost(hbig);
  } else {
    printf("64 GB pinned alloc failed\n");
  }
  return 0;
}
