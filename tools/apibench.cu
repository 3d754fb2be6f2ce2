// apibench.cu -- host cost of the CUDA runtime calls one step issues (kernel launch,
// event record, stream wait, small async copy, event sync), and the GPU-side
// back-to-back launch gap, on this pool's driver stack.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/apibench tools/apibench.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k() {}
int main() {
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e, a, b;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int* d; int* h;
  cudaMalloc(&d, 4096);
  cudaHostAlloc((void**)&h, 4096, cudaHostAllocMapped);
  const int N = 20000;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto t0, auto t1) { return std::chrono::duration<double, std::micro>(t1 - t0).count(); };
  for (int i = 0; i < 1000; ++i) empty_k<<<1, 32, 0, s>>>();
  cudaDeviceSynchronize();
  auto t0 = now();
  cudaEventRecord(a, s);
  for (int i = 0; i < N; ++i) empty_k<<<1, 32, 0, s>>>();
  cudaEventRecord(b, s);
  auto t1 = now();
  cudaDeviceSynchronize();
  float gms; cudaEventElapsedTime(&gms, a, b);
  printf("kernel launch: host %.2f us/call, GPU %.2f us/kernel back to back\n", us(t0, t1) / N, gms * 1e3 / N);
  t0 = now(); for (int i = 0; i < N; ++i) cudaEventRecord(e, s); t1 = now();
  cudaDeviceSynchronize();
  printf("cudaEventRecord: %.2f us/call\n", us(t0, t1) / N);
  t0 = now(); for (int i = 0; i < N; ++i) cudaStreamWaitEvent(s2, e, 0); t1 = now();
  cudaDeviceSynchronize();
  printf("cudaStreamWaitEvent: %.2f us/call\n", us(t0, t1) / N);
  t0 = now(); for (int i = 0; i < N; ++i) cudaMemcpyAsync(d, h, 64, cudaMemcpyHostToDevice, s); t1 = now();
  cudaDeviceSynchronize();
  printf("cudaMemcpyAsync 64 B: %.2f us/call\n", us(t0, t1) / N);
  t0 = now(); for (int i = 0; i < N / 10; ++i) { cudaEventRecord(e, s); cudaEventSynchronize(e); } t1 = now();
  printf("record + cudaEventSynchronize (idle stream): %.2f us/pair\n", us(t0, t1) / (N / 10));
  t0 = now(); for (int i = 0; i < N / 10; ++i) { empty_k<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); } t1 = now();
  printf("launch + cudaStreamSynchronize round trip: %.2f us\n", us(t0, t1) / (N / 10));
  // dependent chain across two streams: kernel on s, event, wait on s2, kernel on s2
  cudaEventRecord(a, s);
  t0 = now();
  for (int i = 0; i < N / 10; ++i) {
    empty_k<<<1, 32, 0, s>>>();
    cudaEventRecord(e, s);
    cudaStreamWaitEvent(s2, e, 0);
    empty_k<<<1, 32, 0, s2>>>();
    cudaEventRecord(e, s2);
    cudaStreamWaitEvent(s, e, 0);
  }
  cudaEventRecord(b, s);
  t1 = now();
  cudaDeviceSynchronize();
  cudaEventElapsedTime(&gms, a, b);
  printf("ping-pong 2 streams: host %.2f us/iter, GPU %.2f us/iter (2 kernels + 2 cross-stream deps)\n", us(t0, t1) / (N / 10), gms * 1e3 / (N / 10));
  // graph of the same 20-kernel chain
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) empty_k<<<1, 32, 0, s>>>();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaDeviceSynchronize();
  cudaEventRecord(a, s);
  t0 = now();
  for (int i = 0; i < N / 20; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  t1 = now();
  cudaDeviceSynchronize();
  cudaEventElapsedTime(&gms, a, b);
  printf("graph of 20 kernels: host %.2f us/launch, GPU %.2f us/kernel\n", us(t0, t1) / (N / 20), gms * 1e3 / N);
  return 0;
}
