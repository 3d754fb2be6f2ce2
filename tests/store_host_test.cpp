// Host-only stress test of the f3 store tier's native code (no GPU): the I/O
// thread pool and the BlockStore data paths (base write, coalesced preadv
// reads, pwritev appends across segment rollover, LRU victims, barrier), with
// every record's content checked against the value it must hold.  Built and
// run by tests/test_store_host.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "../paper_2605_20150_b200/csrc/tidegs_store.h"

using tgs::BlockStore;

static int fails = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::fprintf(stderr, "CHECK failed %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                       \
    }                                                                \
  } while (0)

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp/tgs_store_host_test";
  const int direct = argc > 2 ? std::atoi(argv[2]) : 0;

  // ---- the pool: many generations of tiny tasks (a late worker must never
  //      run a generation with the previous one's function)
  {
    tgs::IoPool pool(8);
    std::mt19937 rng(1);
    for (int g = 0; g < 20000; ++g) {
      const uint32_t n = rng() % 5;
      std::vector<int> hit(n, 0);
      std::function<void(uint32_t)> fn = [&](uint32_t i) { hit[i] += 1; };
      pool.parallel_for(n, fn);
      for (uint32_t i = 0; i < n; ++i) CHECK(hit[i] == 1);
    }
  }

  // ---- the store: K blocks of B rows; value of (block l, version v, float i)
  const uint32_t B = 8, K = 40, H = 12;
  BlockStore::Geometry geo{(uint64_t)B * K, B, 1, 1, 0, K, (uint64_t)B * 59 * 4};
  const uint64_t S = (geo.rec_bytes + 4095) / 4096 * 4096;
  char* pool = nullptr;
  if (posix_memalign((void**)&pool, 4096, H * S) != 0) return 2;
  auto val = [](uint32_t l, uint32_t ver, uint32_t i) { return (float)(l * 1000 + ver * 7) + i * 1e-3f; };
  BlockStore st;
  std::string err = st.open(dir, geo, H, pool, 4096 + 3 * (4096 + S), direct != 0, 6,
                            [&](uint32_t l, float* dst) {
                              for (uint32_t i = 0; i < B * 59; ++i) dst[i] = val(l, 0, i);
                            });
  CHECK(err.empty());
  if (!err.empty()) std::fprintf(stderr, "%s\n", err.c_str());
  std::map<uint32_t, uint32_t> ver;  // newest version written into the cache per block
  std::mt19937 rng(7);
  std::vector<uint32_t> resident;
  auto noop = [](int32_t) {};
  for (int t = 0; t < 300; ++t) {
    // next resident set: 4 random blocks (sorted); S+ = new ones, S- = leaving ones
    std::vector<uint32_t> next;
    while (next.size() < 4) {
      const uint32_t l = rng() % K;
      if (std::find(next.begin(), next.end(), l) == next.end()) next.push_back(l);
    }
    std::sort(next.begin(), next.end());
    std::vector<uint32_t> sp, sm;
    for (uint32_t l : next)
      if (!std::binary_search(resident.begin(), resident.end(), l)) sp.push_back(l), sp.push_back(0);
    for (uint32_t l : resident)
      if (!std::binary_search(next.begin(), next.end(), l)) sm.push_back(l);
    err = st.gather(sp.data(), (uint32_t)sp.size() / 2, t, noop);
    CHECK(err.empty());
    for (size_t i = 0; i < sp.size(); i += 2) {  // the gathered record holds the newest version
      const uint32_t l = sp[i];
      const float* e = st.entry_of(l);
      CHECK(e != nullptr);
      if (!e) continue;
      const uint32_t v = ver.count(l) ? ver[l] : 0;
      for (uint32_t k = 0; k < B * 59; k += 97) CHECK(e[k] == val(l, v, k));
    }
    st.touch_evicted(sm.data(), (uint32_t)sm.size(), t);
    // "write back" half of the leaving blocks as a new version (dirty)
    for (uint32_t l : sm)
      if (rng() & 1) {
        float* e = st.entry_of(l);
        CHECK(e != nullptr);
        if (!e) continue;
        const uint32_t v = ++ver[l];
        for (uint32_t i = 0; i < B * 59; ++i) e[i] = val(l, v, i);
        st.mark_dirty(l, t);
      }
    resident = next;
  }
  err = st.flush_all(noop);
  CHECK(err.empty());
  CHECK(st.cached_dirty() == 0);
  CHECK(st.counters().dirty_evictions > 20 && st.counters().segments > 3);
  std::vector<float> buf(B * 59);
  for (uint32_t l = 0; l < K; ++l) {  // every block's newest version, through Index or the cache
    err = st.read_block(l, buf.data());
    CHECK(err.empty());
    const uint32_t v = ver.count(l) ? ver[l] : 0;
    CHECK(st.index(l).version <= v);
    for (uint32_t k = 0; k < B * 59; k += 13) CHECK(buf[k] == val(l, v, k));
  }
  // ---- R30 resume: a second store over the same files recovers every Index
  //      entry and serves the same newest versions
  {
    char* pool2 = nullptr;
    if (posix_memalign((void**)&pool2, 4096, H * S) != 0) return 2;
    BlockStore st2;
    err = st2.open(dir, geo, H, pool2, 4096 + 3 * (4096 + S), direct != 0, 3,
                   [](uint32_t, float*) {}, true);
    CHECK(err.empty());
    if (!err.empty()) std::fprintf(stderr, "%s\n", err.c_str());
    for (uint32_t l = 0; l < K; ++l) {
      const tgs::StoreIndex a = st.index(l), b = st2.index(l);
      CHECK(a.file_id == b.file_id && a.offset == b.offset && a.size == b.size &&
            a.version == b.version);
      err = st2.read_block(l, buf.data());
      CHECK(err.empty());
      const uint32_t v = ver.count(l) ? ver[l] : 0;
      for (uint32_t k = 0; k < B * 59; k += 13) CHECK(buf[k] == val(l, v, k));
    }
    free(pool2);
  }
  std::printf("store host test: %d failures; hits %llu misses %llu dirty evictions %llu segments %llu\n",
              fails, (unsigned long long)st.counters().hits, (unsigned long long)st.counters().misses,
              (unsigned long long)st.counters().dirty_evictions,
              (unsigned long long)st.counters().segments);
  free(pool);
  return fails ? 1 : 0;
}
