// tgs_workload_cuda.cu -- CUDA twin of the counter-based gradient / row-mask
// input generators in tgs_workload.c (bit-identical: integer hashing plus an
// exact int->float conversion and a power-of-two scale).  These kernels stand
// in for the renderer's backward pass (out of scope, SURVEY.md §8d "Gradients")
// and are harness code: they are not part of the working-set step library.
#include <cstdint>
#include <cuda_runtime.h>

#define WL_DIM 59
#define PHI1 0x9E3779B97F4A7C15ull
#define PHI2 0xC2B2AE3D27D4EB4Full
#define PHI3 0x165667B19E3779F9ull

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float grad_of(uint64_t seed, uint64_t gid, uint32_t a, uint64_t t) {
  uint64_t x = sm64(seed ^ (PHI1 * (gid * WL_DIM + a)) ^ (PHI2 * t));
  int32_t q = (int32_t)(x >> 40) - (1 << 23);
  return __fmul_rn(__int2float_rn(q), 0x1p-33f);
}

// grid: (ceil(B*59/4 / 256), n_blocks); one float4 per thread.  d_n (may be
// NULL): the block count on the device (an asynchronous activate's |A|)
__global__ void wl_grad_kernel(float* __restrict__ grads, uint64_t slot_stride,
                               const uint32_t* __restrict__ blocks,
                               const uint32_t* __restrict__ slots, uint32_t B, uint64_t N,
                               uint64_t seed, uint64_t t, const uint32_t* __restrict__ d_n) {
  const uint32_t i = blockIdx.y;
  if (d_n && i >= *d_n) return;
  const uint64_t k = blocks[i];
  const uint64_t lo = k * B;
  const uint32_t rows = lo >= N ? 0u : (uint32_t)((N - lo) < B ? (N - lo) : B);
  const uint32_t n4 = B * WL_DIM / 4;
  const uint32_t e4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (e4 >= n4) return;
  float v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t e = 4 * e4 + q;
    uint32_t r = e / WL_DIM, a = e - r * WL_DIM;
    v[q] = r < rows ? grad_of(seed, lo + r, a, t) : 0.0f;
  }
  float4* dst = reinterpret_cast<float4*>(grads + (uint64_t)slots[i] * slot_stride);
  dst[e4] = make_float4(v[0], v[1], v[2], v[3]);
}

// grid: (ceil(nw/32)... ) one thread per mask word
__global__ void wl_mask_kernel(uint32_t* __restrict__ mask, uint32_t words_per_slot,
                               const uint32_t* __restrict__ blocks,
                               const uint32_t* __restrict__ slots, uint32_t B, uint64_t N,
                               uint64_t seed, uint64_t t, uint32_t p32) {
  const uint32_t i = blockIdx.y;
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words_per_slot) return;
  const uint64_t k = blocks[i];
  const uint64_t lo = k * B;
  const uint32_t rows = lo >= N ? 0u : (uint32_t)((N - lo) < B ? (N - lo) : B);
  uint32_t word = 0;
  for (uint32_t b = 0; b < 32; ++b) {
    uint32_t r = w * 32 + b;
    if (r < rows) {
      uint64_t x = sm64(seed ^ (PHI3 * (lo + r)) ^ (PHI2 * t));
      if ((uint32_t)(x >> 32) < p32) word |= 1u << b;
    }
  }
  mask[(uint64_t)slots[i] * words_per_slot + w] = word;
}

extern "C" int wl_cuda_synth_grads(float* d_grads, uint64_t slot_stride, const uint32_t* d_blocks,
                                   const uint32_t* d_slots, uint32_t n, uint32_t B, uint64_t N,
                                   uint64_t seed, uint64_t t, void* stream) {
  if (n == 0) return 0;
  uint32_t n4 = B * WL_DIM / 4;
  dim3 grid((n4 + 255) / 256, n);
  wl_grad_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_grads, slot_stride, d_blocks, d_slots,
                                                         B, N, seed, t, nullptr);
  return (int)cudaGetLastError();
}

// the same with the block count on the device (n_max: an upper bound)
extern "C" int wl_cuda_synth_grads_devn(float* d_grads, uint64_t slot_stride,
                                        const uint32_t* d_blocks, const uint32_t* d_slots,
                                        const uint32_t* d_n, uint32_t n_max, uint32_t B,
                                        uint64_t N, uint64_t seed, uint64_t t, void* stream) {
  if (n_max == 0) return 0;
  uint32_t n4 = B * WL_DIM / 4;
  dim3 grid((n4 + 255) / 256, n_max);
  wl_grad_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d_grads, slot_stride, d_blocks, d_slots,
                                                         B, N, seed, t, d_n);
  return (int)cudaGetLastError();
}

extern "C" int wl_cuda_synth_mask(uint32_t* d_mask, uint32_t words_per_slot,
                                  const uint32_t* d_blocks, const uint32_t* d_slots, uint32_t n,
                                  uint32_t B, uint64_t N, uint64_t seed, uint64_t t, uint32_t p32,
                                  void* stream) {
  if (n == 0) return 0;
  dim3 grid((words_per_slot + 127) / 128, n);
  wl_mask_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(d_mask, words_per_slot, d_blocks, d_slots,
                                                         B, N, seed, t, p32);
  return (int)cudaGetLastError();
}

// test hook: overwrite one device float in stream order (fault injection)
__global__ void wl_poke_kernel(float* p, float v) { *p = v; }

extern "C" int wl_cuda_poke(float* p, float v, void* stream) {
  wl_poke_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(p, v);
  return (int)cudaGetLastError();
}
