// Host-only read benchmark of the f3 store tier (tidegs_store.cpp) on this
// box's disk: a K-record base segment, then gathers of `misses` blocks per
// step whose ids follow a sliding window (like the aerial path entering new
// territory), reading into a pinned-or-pageable cache.  Prints the SSD GB/s the
// store's own read path reaches, per thread count.
//   g++ -O2 -std=c++17 -pthread -I/usr/local/cuda/include tools/store_readbench.cpp \
//       paper_2605_20150_b200/csrc/tidegs_store.cpp -L/usr/local/cuda/lib64 -lcudart
//   ./a.out DIR K MISSES STEPS THREADS [direct=1] [pinned=0] [run=1] [H]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <sys/mman.h>

#include <cuda_runtime.h>

#include "../paper_2605_20150_b200/csrc/tidegs_store.h"

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const std::string dir = argv[1];
  const uint32_t K = std::atoi(argv[2]), misses = std::atoi(argv[3]), steps = std::atoi(argv[4]);
  const int threads = std::atoi(argv[5]);
  const int direct = argc > 6 ? std::atoi(argv[6]) : 1;
  const int pinned = argc > 7 ? std::atoi(argv[7]) : 0;  // cudaHostAlloc cache, as the library
  const uint32_t run = argc > 8 ? std::atoi(argv[8]) : 1;   // neighbouring misses per run
  const uint32_t B = 4096;
  const uint32_t H = argc > 9 ? std::atoi(argv[9]) : misses * 4 + 64;  // cache records
  tgs::BlockStore::Geometry geo{(uint64_t)B * K, B, 1, 1, 0, K, (uint64_t)B * 59 * 4};
  const uint64_t S = (geo.rec_bytes + 4095) / 4096 * 4096;
  // pinned: 1 cudaHostAlloc, 2 THP-backed anonymous memory + cudaHostRegister, 3 THP only
  char* pool = nullptr;
  const size_t bytes = ((size_t)H * S + (2u << 20) - 1) / (2u << 20) * (2u << 20);
  if (pinned == 1) {
    if (cudaHostAlloc((void**)&pool, bytes, cudaHostAllocPortable) != cudaSuccess) return 3;
  } else if (pinned >= 2) {
    pool = (char*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (pool == MAP_FAILED) return 3;
    madvise(pool, bytes, MADV_HUGEPAGE);
    std::memset(pool, 0, bytes);
    if (pinned == 2 && cudaHostRegister(pool, bytes, cudaHostRegisterPortable) != cudaSuccess) return 3;
  } else if (posix_memalign((void**)&pool, 4096, bytes) != 0) {
    return 3;
  }
  std::memset(pool, getenv("SRB_FILL") ? atoi(getenv("SRB_FILL")) : 0, bytes);
  tgs::BlockStore st;
  auto t0 = std::chrono::steady_clock::now();
  std::string err = st.open(dir, geo, H, pool, 1ull << 30, direct != 0, threads,
                            [&](uint32_t l, float* dst) { dst[0] = (float)l; });
  if (!err.empty()) {
    std::fprintf(stderr, "%s\n", err.c_str());
    return 4;
  }
  const double wsec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("base: %u records, %.1f GB written in %.1f s (%.2f GB/s)\n", K, K * S / 1e9, wsec,
              K * S / 1e9 / wsec);
  std::vector<uint32_t> resident;
  uint32_t window = 0;
  auto noop = [](int32_t) {};
  double read_ms0 = 0;
  uint64_t read_b0 = 0;
  for (uint32_t t = 0; t < steps; ++t) {
    // S+ = `misses` never-seen blocks from a window sliding over the id space
    // (spread like a Morton-ordered strip edge), S- = the previous batch
    std::vector<uint32_t> sp;
    for (uint32_t i = 0; i < misses; ++i) {  // runs of `run` neighbouring records
      const uint32_t l = (window + (i / run) * 7 * run + i % run) % K;
      if (std::find(sp.begin(), sp.end(), l) == sp.end()) sp.push_back(l);
    }
    window = (window + misses * 7) % K;
    std::sort(sp.begin(), sp.end());
    std::vector<uint32_t> pairs;
    for (uint32_t l : sp)
      if (!std::binary_search(resident.begin(), resident.end(), l)) pairs.push_back(l), pairs.push_back(0);
    err = st.gather(pairs.data(), (uint32_t)pairs.size() / 2, (int32_t)t, noop);
    if (!err.empty()) {
      std::fprintf(stderr, "%s\n", err.c_str());
      return 5;
    }
    std::vector<uint32_t> sm;
    for (uint32_t l : resident)
      if (!std::binary_search(sp.begin(), sp.end(), l)) sm.push_back(l);
    st.touch_evicted(sm.data(), (uint32_t)sm.size(), (int32_t)t);
    resident = sp;
    if (t == 4) {  // warm-up excluded
      read_ms0 = st.counters().read_ms;
      read_b0 = st.counters().read_bytes;
    }
  }
  const double ms = st.counters().read_ms - read_ms0;
  const double gb = (st.counters().read_bytes - read_b0) / 1e9;
  std::printf("H %u threads %d direct %d pinned %d run %u: %u misses/step, %.2f ms/step in reads, "
              "%.2f GB/s, %.1f read calls/step\n", H, threads, direct, pinned, run, misses,
              ms / (steps - 5), gb / (ms / 1e3), (double)st.counters().read_calls / steps);
  if (pinned == 1) cudaFreeHost(pool);
  else if (pinned >= 2) { if (pinned == 2) cudaHostUnregister(pool); munmap(pool, bytes); }
  else free(pool);
  return 0;
}
