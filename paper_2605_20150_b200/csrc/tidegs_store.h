// tidegs_store.h -- NEXT f3: the tier below the host tier (PAPER.md:224-251,
// §3.4 "Out-of-Core Engine: SSD Storage, CPU Tiered Cache"), host-side C++.
//
//   * log-structured store: an immutable base segment written once at init and
//     append-only patch segments; Index[k] = (file_id, offset, size, version)
//     points at the newest version of each block;
//   * CPU cache: H pinned block records with an LRU order and a dirty bit per
//     entry, inclusive of the GPU working set (reading R27): the entry of a
//     block in R_t u R_{t+1} is never evicted, so the H2D gather reads straight
//     from it and the D2H write-back lands straight in it;
//   * two-step write-back VRAM -> CPU cache -> SSD: a dirty
//     entry reaches the SSD only when the cache evicts it, or at the barrier.
//
// Segment format: reading R28.  Reads and appends use O_DIRECT
// (optional) straight from / into the pinned entries (page-aligned payloads),
// issued by a small thread pool so the device sees queue depth.  Nothing here
// is shared with oracle/.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace tgs {

// a fixed pool of threads running one parallel_for at a time
class IoPool {
 public:
  explicit IoPool(int n);
  ~IoPool();
  // runs fn(i) for i in [0, n) on the pool (and the caller); returns when all are done
  void parallel_for(uint32_t n, const std::function<void(uint32_t)>& fn);

 private:
  void worker();
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(uint32_t)>* fn_ = nullptr;
  uint32_t n_ = 0;
  std::atomic<uint32_t> next_{0};
  size_t acked_ = 0;  // workers done with the current generation
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct StoreIndex {  // PAPER.md:233 "Index[k] = (file_id, offset, size, version)"
  uint32_t file_id = 0;
  uint64_t offset = 0;
  uint64_t size = 0;
  uint64_t version = 0;
};

struct StoreCounters {
  uint64_t hits = 0, misses = 0, evictions = 0, dirty_evictions = 0, flush_appends = 0,
           read_bytes = 0, write_bytes = 0, segments = 0;
  double read_ms = 0.0, write_ms = 0.0;  // wall time of the SSD phases
  uint64_t read_calls = 0;               // vector reads issued (runs of neighbouring records)
  double read_busy_ms = 0.0;             // sum over threads of time inside preadv
  uint64_t prefetch_reads = 0, prefetch_hits = 0, prefetch_wasted = 0;  // read-ahead records
};

class BlockStore {
 public:
  static constexpr uint64_t kPage = 4096;

  // geometry of the shard (header fields of R28)
  struct Geometry {
    uint64_t N;
    uint32_t B, n_arr, G, rank, Kloc;
    uint64_t rec_bytes;  // B*59*4
  };

  BlockStore() = default;
  ~BlockStore();

  // Creates dir/base.tdgs from fill(l, dst) (dst: n_arr*B*59 floats, zeroed
  // beyond what fill writes) and sets up an empty cache over pool (H entries
  // of entry_bytes(), pinned, page-aligned; owned by the caller).  Returns an
  // error string or "".
  // reopen (R30): no base is written; Index is recovered from the files.
  std::string open(const std::string& dir, const Geometry& g, uint32_t H, char* pool,
                   uint64_t seg_budget, bool direct, int threads,
                   const std::function<void(uint32_t, float*)>& fill, bool reopen = false);
  uint64_t entry_bytes() const { return S_; }
  uint64_t payload_bytes() const { return payload_; }

  // R27 (b): S+ (local ids, ascending) of activate T.  wait_d2h(job) must
  // return once the write-back of that activate into the cache has landed.
  // hits_ready(miss flags per S+ entry), if set, is called once the cache
  // decisions are made and before any SSD I/O: the hits' entries are final.
  std::string gather(const uint32_t* sp_pairs /* (l, slot) */, uint32_t n, int32_t T,
                     const std::function<void(int32_t)>& wait_d2h,
                     const std::function<void(const std::vector<uint8_t>&)>& hits_ready = nullptr);
  // R27 (c): S- of activate T, ascending (after gather of the same activate)
  void touch_evicted(const uint32_t* sm, uint32_t n, int32_t T);
  // R27 (a): the D2H write-back of activate T put block l's dirty record into its entry
  void mark_dirty(uint32_t l, int32_t T);
  // the barrier: append every dirty entry (ascending id), clear dirty, fdatasync,
  // then the manifest (R30) with the Adam step counters `steps` [Kloc] (NULL:
  // those of the last barrier)
  std::string flush_all(const std::function<void(int32_t)>& wait_d2h,
                        const uint32_t* steps = nullptr);
  // R30: the Adam step counters of the barrier a reopened store resumed from
  const std::vector<uint32_t>& barrier_steps() const { return steps_; }
  // R31: merge the patch segments into a new base (after flush_all)
  std::string compact();

  // host address of block l's cached record, nullptr if not cached
  float* entry_of(uint32_t l) const {
    const int32_t e = ent_of_[l];
    return e < 0 ? nullptr : reinterpret_cast<float*>(pool_ + (uint64_t)buf_of_[e] * S_);
  }
  // physical buffer of block l's cache entry (its record sits at pool + index *
  // entry_bytes()), -1 if not cached
  int32_t entry_index(uint32_t l) const { return ent_of_[l] < 0 ? -1 : (int32_t)buf_of_[ent_of_[l]]; }
  // read-ahead (prefetch): X extra pool buffers (pool holds H + X) and threads
  void start_prefetch(uint32_t X, int threads);
  // the blocks activate `target` may need (its Level-1 visible set); returns at once
  void prefetch(const std::vector<uint32_t>& blocks, int32_t target);
  // waits for the read-ahead batch in flight (counters are then settled)
  void settle() { pf_join(); }
  // newest version of block l (cache, else SSD) into dst (payload bytes)
  std::string read_block(uint32_t l, void* dst);

  const StoreIndex& index(uint32_t l) const { return index_[l]; }
  const StoreCounters& counters() const { return cnt_; }
  uint32_t cached() const { return H_ - (uint32_t)free_.size(); }
  uint32_t cached_dirty() const;
  // cached local ids ordered by last access (least recent first) + dirty flags
  void lru_order(std::vector<uint32_t>& blocks, std::vector<uint8_t>& dirty) const;

 private:
  struct Ent {
    int32_t blk = -1;
    bool dirty = false;
    bool resident = false;     // block in the GPU working set (not evictable)
    int32_t admitted = -1;     // activate that last admitted the block to the GPU
    int32_t wb_job = -1;       // activate whose write-back last wrote this entry
    uint64_t stamp = 0;        // LRU clock of the last access
    int32_t prev = -1, next = -1;
    bool listed = false;       // in the evictable list (cached, not pinned)
  };
  void unlink(int32_t e);
  void push_mru(int32_t e);
  int fd_of(uint32_t fid);
  std::string new_segment();
  std::string recover();
  std::string write_manifest();
  void init_buffers();
  void pf_main();
  uint64_t pf_wait(uint64_t upto);
  void pf_join();
  // reserves the next record of the patch log for block l: (fd, file offset of the record)
  std::string reserve_append(uint32_t l, int& fd, uint64_t& rec_off);
  std::string write_records(const std::vector<std::pair<uint32_t, int32_t>>& recs /* (l, entry) */);
  std::string read_records(const std::vector<std::pair<uint32_t, int32_t>>& recs /* (l, entry) */);

  Geometry g_{};
  std::string dir_;
  uint32_t H_ = 0;
  char* pool_ = nullptr;
  uint64_t payload_ = 0, S_ = 0, seg_budget_ = 0;
  bool direct_ = false;
  std::vector<StoreIndex> index_;
  std::vector<int32_t> ent_of_;
  std::vector<Ent> ents_;
  std::vector<int32_t> free_;
  int32_t head_ = -1, tail_ = -1;  // evictable list: head = least recently used
  uint64_t clock_ = 0;
  std::vector<int> fds_;           // by file id (-1 not open)
  uint32_t cur_file_ = 0;
  uint64_t cur_size_ = 0;
  StoreCounters cnt_{};
  IoPool* pool_io_ = nullptr;
  char* hdr_pages_ = nullptr;      // aligned record header pages (grown on demand)
  uint64_t epoch_ = 0;             // manifests written (barriers, compactions, the initial base)
  std::vector<uint64_t> base_version_;  // version of each block's base record (R31)
  std::vector<uint32_t> steps_;    // Adam step counters of the last barrier (R30)
  // physical buffers: entry e's record is buffer buf_of_[e]; read-ahead buffers
  std::vector<uint32_t> buf_of_;
  uint32_t X_ = 0;                 // read-ahead buffers (0: no prefetch)
  std::vector<uint32_t> ra_free_;
  std::vector<int32_t> ra_buf_;    // [Kloc] read-ahead buffer of block l, -1 none
  std::vector<uint64_t> ra_ver_;   // [Kloc] Index version it was read at
  std::vector<uint64_t> ra_seq_;   // [Kloc] read-ahead batch it belongs to
  std::deque<uint32_t> ra_fifo_;   // blocks in read-ahead, oldest first
  IoPool* pf_pool_ = nullptr;
  std::thread pf_thread_;
  std::mutex pf_mu_;
  std::condition_variable pf_cv_;
  struct PfItem { uint32_t buf; int fd; uint64_t off; };
  std::deque<std::pair<uint64_t, std::vector<PfItem>>> pf_q_;  // batches waiting / in flight
  uint64_t pf_issued_ = 0, pf_done_ = 0;  // batches announced / read completely
  std::deque<std::pair<uint64_t, int32_t>> pf_target_;  // (batch, activate it targets)
  std::vector<uint8_t> pf_badbuf_;        // [H + X] a read-ahead read into it failed
  bool pf_stop_ = false;
  size_t hdr_cap_ = 0;
};

}  // namespace tgs
