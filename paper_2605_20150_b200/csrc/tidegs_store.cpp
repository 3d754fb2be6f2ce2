// tidegs_store.cpp -- NEXT f3 store tier (see tidegs_store.h; PAPER.md:224-251,
// readings R27/R28 of DESIGN.md §3).
#include "tidegs_store.h"

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include <dirent.h>
#include <fcntl.h>
#include <nmmintrin.h>
#include <sys/stat.h>
#include <sys/uio.h>
#include <unistd.h>

namespace tgs {

// ------------------------------------------------------------------ IoPool
IoPool::IoPool(int n) {
  for (int i = 1; i < n; ++i) th_.emplace_back([this] { worker(); });
}

IoPool::~IoPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : th_) t.join();
}

// Every worker takes part in every generation and acknowledges it; the caller
// returns only after all of them have, so no worker can still hold the
// previous generation's function when the next parallel_for starts.
void IoPool::worker() {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(uint32_t)>* fn;
    uint32_t n;
    {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      fn = fn_;
      n = n_;
    }
    for (uint32_t i; (i = next_.fetch_add(1)) < n;) (*fn)(i);
    {
      std::lock_guard<std::mutex> g(mu_);
      ++acked_;
    }
    done_cv_.notify_all();
  }
}

void IoPool::parallel_for(uint32_t n, const std::function<void(uint32_t)>& fn) {
  if (n == 0) return;
  {
    std::lock_guard<std::mutex> g(mu_);
    fn_ = &fn;
    n_ = n;
    next_ = 0;
    acked_ = 0;
    ++gen_;
  }
  cv_.notify_all();
  for (uint32_t i; (i = next_.fetch_add(1)) < n;) fn(i);
  std::unique_lock<std::mutex> g(mu_);
  done_cv_.wait(g, [&] { return acked_ == th_.size(); });
  fn_ = nullptr;
}

// -------------------------------------------------------------- helpers
namespace {

void put32(unsigned char* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (unsigned char)(v >> (8 * i));
}
void put64(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (unsigned char)(v >> (8 * i));
}

char* aligned_pages(size_t bytes) {
  void* p = nullptr;
  if (posix_memalign(&p, BlockStore::kPage, std::max<size_t>(bytes, BlockStore::kPage)) != 0)
    return nullptr;
  return static_cast<char*>(p);
}

std::string errno_str(const char* what) {
  return std::string(what) + ": " + std::strerror(errno);
}

// full-length positional I/O (short counts retried)
bool pwrite_all(int fd, const void* p, uint64_t n, uint64_t off) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t w = ::pwrite(fd, c, n, (off_t)off);
    if (w <= 0) {
      if (w < 0 && errno == EINTR) continue;
      return false;
    }
    c += w, n -= (uint64_t)w, off += (uint64_t)w;
  }
  return true;
}
bool pread_all(int fd, void* p, uint64_t n, uint64_t off) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t r = ::pread(fd, c, n, (off_t)off);
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      return false;
    }
    c += r, n -= (uint64_t)r, off += (uint64_t)r;
  }
  return true;
}

uint32_t get32(const unsigned char* p) {
  uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
uint64_t get64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// CRC-32C of the R28 format-2 records and of the manifest, with the SSE4.2
// crc32 instruction (8 bytes per step; ~10x the table form): a 2.9 MB persist
// record costs ~0.2 ms of one I/O thread.
__attribute__((target("sse4.2"))) uint32_t crc32c(const void* data, uint64_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t c = 0xFFFFFFFFu;
  for (; n >= 8; n -= 8, p += 8) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    c = _mm_crc32_u64(c, w);
  }
  uint32_t c32 = (uint32_t)c;
  for (; n; --n, ++p) c32 = _mm_crc32_u8(c32, *p);
  return c32 ^ 0xFFFFFFFFu;
}

// durable rename: fsync of the directory that holds the entry
bool fsync_dir(const std::string& dir) {
  const int fd = ::open(dir.c_str(), O_RDONLY | O_DIRECTORY);
  if (fd < 0) return false;
  const bool ok = ::fsync(fd) == 0;
  ::close(fd);
  return ok;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ---------------------------------------------------------------- BlockStore
BlockStore::~BlockStore() {
  if (pf_thread_.joinable()) {
    {
      std::lock_guard<std::mutex> g(pf_mu_);
      pf_stop_ = true;
    }
    pf_cv_.notify_all();
    pf_thread_.join();
  }
  delete pf_pool_;
  delete pool_io_;
  for (int fd : fds_)
    if (fd >= 0) ::close(fd);
  free(hdr_pages_);
}

int BlockStore::fd_of(uint32_t fid) {
  if (fid < fds_.size() && fds_[fid] >= 0) return fds_[fid];
  char name[64];
  std::snprintf(name, sizeof name, fid == 0 ? "/base.tdgs" : "/patch-%06u.tdgp", fid);
  const int fd = ::open((dir_ + name).c_str(), O_RDWR | (direct_ ? O_DIRECT : 0));
  if (fid >= fds_.size()) fds_.resize(fid + 1, -1);
  fds_[fid] = fd;
  return fd;
}

// R28 segment header page: magic, format 1, file id, n_arr, N, D, B, G, rank, Kloc
static void segment_header(unsigned char* h, uint32_t fid, const BlockStore::Geometry& g) {
  std::memset(h, 0, BlockStore::kPage);
  std::memcpy(h, fid == 0 ? "TDGS" : "TDGP", 4);
  put32(h + 4, 1);
  put32(h + 8, fid);
  put32(h + 12, g.n_arr);
  put64(h + 16, g.N);
  put32(h + 24, 59);
  put32(h + 28, g.B);
  put32(h + 32, g.G);
  put32(h + 36, g.rank);
  put32(h + 40, g.Kloc);
}

std::string BlockStore::open(const std::string& dir, const Geometry& g, uint32_t H, char* pool,
                             uint64_t seg_budget, bool direct, int threads,
                             const std::function<void(uint32_t, float*)>& fill, bool reopen) {
  g_ = g;
  dir_ = dir;
  H_ = H;
  pool_ = pool;
  direct_ = direct;
  payload_ = (uint64_t)g.n_arr * g.rec_bytes;
  S_ = (payload_ + kPage - 1) / kPage * kPage;
  seg_budget_ = seg_budget;
  if (seg_budget_ < 2 * kPage + S_) return "segment budget below one record";
  if (reopen) {
    pool_io_ = new IoPool(std::max(1, threads));
    std::string err = recover();
    if (!err.empty()) return err;
    ent_of_.assign(g.Kloc, -1);
    ents_.assign(H, Ent{});
    free_.clear();
    for (uint32_t e = H; e-- > 0;) free_.push_back((int32_t)e);
    init_buffers();
    return "";
  }
  if (::mkdir(dir.c_str(), 0755) != 0 && errno != EEXIST) return errno_str("mkdir");
  // the directory holds one store: stale patch segments of an earlier store go
  if (DIR* dp = ::opendir(dir.c_str())) {
    while (dirent* e = ::readdir(dp)) {
      const std::string n = e->d_name;
      if (n.size() == 17 && n.compare(0, 6, "patch-") == 0 && n.compare(12, 5, ".tdgp") == 0)
        ::unlink((dir + "/" + n).c_str());
    }
    ::closedir(dp);
  }
  pool_io_ = new IoPool(std::max(1, threads));
  // the base segment is built by every host core (generation is CPU work); the
  // training reads and appends use the `threads` of pool_io_ (queue depth)
  IoPool build_pool(std::max(threads, std::min<int>(32, (int)std::thread::hardware_concurrency())));

  // "The initial model is written once as an immutable base segment"
  // (PAPER.md:228): header page, record l at 4096 + l*S; Index[l] = (0, off, size, 0)
  int fd = ::open((dir + "/base.tdgs").c_str(),
                  O_RDWR | O_CREAT | O_TRUNC | (direct ? O_DIRECT : 0), 0644);
  if (fd < 0 && direct && errno == EINVAL) {  // e.g. tmpfs: no O_DIRECT, use the page cache
    std::fprintf(stderr, "tidegs: store: %s does not support O_DIRECT; using buffered I/O\n",
                 dir.c_str());
    direct_ = false;
    fd = ::open((dir + "/base.tdgs").c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
  }
  if (fd < 0) return errno_str("open base.tdgs");
  fds_.assign(1, fd);
  std::unique_ptr<char, decltype(&free)> hp(aligned_pages(kPage), &free);
  segment_header(reinterpret_cast<unsigned char*>(hp.get()), 0, g);
  if (!pwrite_all(fd, hp.get(), kPage, 0)) return errno_str("write base header");
  std::atomic<bool> bad{false};
  build_pool.parallel_for(g.Kloc, [&](uint32_t l) {
    thread_local std::unique_ptr<char, decltype(&free)> buf(nullptr, &free);
    thread_local uint64_t cap = 0;
    if (cap < S_) {
      buf.reset(aligned_pages(S_));
      cap = S_;
    }
    std::memset(buf.get(), 0, S_);
    fill(l, reinterpret_cast<float*>(buf.get()));
    if (!pwrite_all(fd, buf.get(), S_, kPage + (uint64_t)l * S_)) bad = true;
  });
  if (bad) return errno_str("write base record");
  if (::fdatasync(fd) != 0) return errno_str("fdatasync base");
  index_.resize(g.Kloc);
  for (uint32_t l = 0; l < g.Kloc; ++l) index_[l] = {0, kPage + (uint64_t)l * S_, payload_, 0};
  base_version_.assign(g.Kloc, 0);
  steps_.assign(g.Kloc, 0);
  epoch_ = 0;
  std::string merr = write_manifest();  // epoch 1: the base alone
  if (!merr.empty()) return merr;
  ent_of_.assign(g.Kloc, -1);
  ents_.assign(H, Ent{});
  free_.clear();
  for (uint32_t e = H; e-- > 0;) free_.push_back((int32_t)e);
  init_buffers();
  return "";
}

// entry e's record sits in physical buffer buf_of_[e]; buffers H .. H+X-1 start
// as the read-ahead pool (X = prefetch_blocks)
void BlockStore::init_buffers() {
  buf_of_.resize(H_);
  for (uint32_t e = 0; e < H_; ++e) buf_of_[e] = e;
  ra_free_.clear();
  for (uint32_t b = H_ + X_; b-- > H_;) ra_free_.push_back(b);
  ra_buf_.assign(g_.Kloc, -1);
  ra_ver_.assign(g_.Kloc, 0);
  ra_seq_.assign(g_.Kloc, 0);
  ra_fifo_.clear();
}

// ------------------------------------------------------ read-ahead (prefetch)
// PAPER.md:150 "Prefetch needed blocks into the CPU cache", 253-259 (SSD reads
// overlapped with compute).  The caller announces the blocks the next batch
// may need; those not cached get their newest version read into free
// read-ahead buffers by the prefetch thread.  The cache itself (R27: which
// blocks are cached, the LRU order, dirty bits, Index) is not touched: the next
// gather, for a miss whose read-ahead record still holds the newest version,
// swaps that buffer into the miss's entry instead of reading the SSD.
void BlockStore::prefetch(const std::vector<uint32_t>& blocks, int32_t target) {
  if (!X_) return;
  uint64_t done;
  {
    std::lock_guard<std::mutex> g(pf_mu_);
    done = pf_done_;
  }
  const uint64_t seq = pf_issued_ + 1;
  std::vector<PfItem> batch;
  for (uint32_t l : blocks) {
    if (ent_of_[l] >= 0 || ra_buf_[l] >= 0) continue;  // cached, or already read ahead
    if (ra_free_.empty()) {  // recycle the oldest completed read-ahead record
      while (!ra_fifo_.empty() && ra_buf_[ra_fifo_.front()] < 0) ra_fifo_.pop_front();
      if (ra_fifo_.empty() || ra_seq_[ra_fifo_.front()] > done) break;  // all still in flight
      const uint32_t o = ra_fifo_.front();
      ra_fifo_.pop_front();
      ra_free_.push_back((uint32_t)ra_buf_[o]);
      ra_buf_[o] = -1;
      cnt_.prefetch_wasted += 1;
    }
    const uint32_t b = ra_free_.back();
    ra_free_.pop_back();
    ra_buf_[l] = (int32_t)b;
    ra_ver_[l] = index_[l].version;
    ra_seq_[l] = seq;
    ra_fifo_.push_back(l);
    // the file and offset are taken here, on the caller's thread (segments are
    // opened and Index changes only there)
    batch.push_back({b, fd_of(index_[l].file_id), index_[l].offset});
  }
  if (batch.empty()) return;
  pf_issued_ = seq;
  pf_target_.push_back({seq, target});
  {
    std::lock_guard<std::mutex> g(pf_mu_);
    pf_q_.push_back({seq, std::move(batch)});
  }
  pf_cv_.notify_all();
}

// batches are read in order; pf_done_ = the last batch read completely
void BlockStore::pf_main() {
  for (;;) {
    uint64_t seq;
    std::vector<PfItem> batch;
    {
      std::unique_lock<std::mutex> g(pf_mu_);
      pf_cv_.wait(g, [&] { return pf_stop_ || !pf_q_.empty(); });
      if (pf_stop_) return;
      seq = pf_q_.front().first;
      batch = pf_q_.front().second;
    }
    std::vector<uint8_t> bad(batch.size(), 0);
    pf_pool_->parallel_for((uint32_t)batch.size(), [&](uint32_t i) {
      const PfItem& it = batch[i];
      if (it.fd < 0 || !pread_all(it.fd, pool_ + (uint64_t)it.buf * S_, S_, it.off)) bad[i] = 1;
    });
    {
      std::lock_guard<std::mutex> g(pf_mu_);
      for (size_t i = 0; i < batch.size(); ++i)
        if (bad[i]) pf_badbuf_[batch[i].buf] = 1;  // dropped at use; the gather reads itself
      cnt_.prefetch_reads += batch.size();
      pf_q_.pop_front();
      pf_done_ = seq;
    }
    pf_cv_.notify_all();
  }
}

// waits until every read-ahead batch up to `upto` has been read; returns the
// last completed batch
uint64_t BlockStore::pf_wait(uint64_t upto) {
  if (!X_) return 0;
  std::unique_lock<std::mutex> g(pf_mu_);
  pf_cv_.wait(g, [&] { return pf_done_ >= upto; });
  return pf_done_;
}

void BlockStore::pf_join() { pf_wait(pf_issued_); }

void BlockStore::start_prefetch(uint32_t X, int threads) {
  X_ = X;
  ra_free_.clear();  // buffers H .. H+X-1 of the pool
  for (uint32_t b = H_ + X_; b-- > H_;) ra_free_.push_back(b);
  pf_badbuf_.assign((size_t)H_ + X_, 0);
  if (!X_) return;
  pf_pool_ = new IoPool(std::max(1, threads));
  pf_thread_ = std::thread([this] { pf_main(); });
}

// R30 barrier manifest (manifest.tdgm): "TDGM", format 1, epoch, the last patch
// segment and the length it had at the barrier (the durable end of the log),
// the shard geometry, then per local block the version of its base record
// (R31) and its Adam step counter, then a CRC-32C of all of it.  Written under
// a temporary name, made durable, renamed, directory synced: a crash leaves
// either this barrier's manifest or the previous one.
std::string BlockStore::write_manifest() {
  epoch_ += 1;
  const uint64_t K = g_.Kloc;
  std::vector<unsigned char> m(64 + 12 * K + 4, 0);
  std::memcpy(m.data(), "TDGM", 4);
  put32(&m[4], 1);
  put64(&m[8], epoch_);
  put32(&m[16], cur_file_);
  put64(&m[24], cur_file_ ? cur_size_ : 0);
  put32(&m[32], g_.n_arr);
  put64(&m[40], g_.N);
  put32(&m[48], g_.B);
  put32(&m[52], g_.G);
  put32(&m[56], g_.rank);
  put32(&m[60], g_.Kloc);
  for (uint64_t l = 0; l < K; ++l) {
    put64(&m[64 + 8 * l], base_version_[l]);
    put32(&m[64 + 8 * K + 4 * l], steps_[l]);
  }
  put32(&m[m.size() - 4], crc32c(m.data(), m.size() - 4));
  const std::string tmp = dir_ + "/manifest.tdgm.tmp", dst = dir_ + "/manifest.tdgm";
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return errno_str("open manifest");
  const bool ok = pwrite_all(fd, m.data(), m.size(), 0) && ::fdatasync(fd) == 0;
  ::close(fd);
  if (!ok) return errno_str("write manifest");
  if (::rename(tmp.c_str(), dst.c_str()) != 0 || !fsync_dir(dir_)) return errno_str("rename manifest");
  return "";
}

// R30 checkpoint/resume: the state of the last barrier.  Its manifest must
// describe this shard and pass its CRC; Index starts from the base records
// (with the versions the manifest carries) and takes every patch record up to
// the durable end in file_id order, later records winning.  Those records were
// durable at the barrier, so a bad header or payload CRC there is corruption
// (an error), not a torn tail.  Whatever was appended after the barrier -- the
// tail of the last segment and any later segment -- is cut off / removed, and
// the Adam step counters come back from the manifest.
std::string BlockStore::recover() {
  std::unique_ptr<char, decltype(&free)> want(aligned_pages(kPage), &free), got(aligned_pages(kPage), &free);
  if (fd_of(0) < 0 && direct_ && errno == EINVAL) {  // no O_DIRECT here: page cache
    direct_ = false;
    fds_.clear();
  }
  if (fd_of(0) < 0) return errno_str("open base.tdgs");
  segment_header(reinterpret_cast<unsigned char*>(want.get()), 0, g_);
  if (!pread_all(fds_[0], got.get(), kPage, 0) || std::memcmp(want.get(), got.get(), kPage) != 0)
    return "base.tdgs does not hold this shard (header mismatch)";
  // the manifest
  const uint64_t K = g_.Kloc, msize = 64 + 12 * K + 4;
  std::vector<unsigned char> m(msize);
  {
    const int fd = ::open((dir_ + "/manifest.tdgm").c_str(), O_RDONLY);
    if (fd < 0) return errno_str("open manifest.tdgm (no barrier state)");
    struct stat sb;
    const bool ok = ::fstat(fd, &sb) == 0 && (uint64_t)sb.st_size == msize &&
                    pread_all(fd, m.data(), msize, 0);
    ::close(fd);
    if (!ok) return "manifest.tdgm: wrong size for this shard";
  }
  if (std::memcmp(m.data(), "TDGM", 4) != 0 || get32(&m[4]) != 1 ||
      get32(&m[msize - 4]) != crc32c(m.data(), msize - 4))
    return "manifest.tdgm: bad magic, format or CRC";
  if (get32(&m[32]) != g_.n_arr || get64(&m[40]) != g_.N || get32(&m[48]) != g_.B ||
      get32(&m[52]) != g_.G || get32(&m[56]) != g_.rank || get32(&m[60]) != g_.Kloc)
    return "manifest.tdgm does not describe this shard";
  epoch_ = get64(&m[8]);
  const uint32_t last = get32(&m[16]);
  const uint64_t end = get64(&m[24]);
  index_.resize(K);
  base_version_.resize(K);
  steps_.resize(K);
  for (uint64_t l = 0; l < K; ++l) {
    base_version_[l] = get64(&m[64 + 8 * l]);
    steps_[l] = get32(&m[64 + 8 * K + 4 * l]);
    index_[l] = {0, kPage + l * S_, payload_, base_version_[l]};
  }
  std::unique_ptr<char, decltype(&free)> pay(aligned_pages(S_), &free);
  for (uint32_t fid = 1; fid <= last; ++fid) {
    char name[64];
    std::snprintf(name, sizeof name, "/patch-%06u.tdgp", fid);
    struct stat sb;
    if (::stat((dir_ + name).c_str(), &sb) != 0) return std::string("missing ") + (name + 1);
    const int fd = fd_of(fid);
    if (fd < 0) return errno_str("open patch segment");
    segment_header(reinterpret_cast<unsigned char*>(want.get()), fid, g_);
    if (!pread_all(fd, got.get(), kPage, 0) || std::memcmp(want.get(), got.get(), kPage) != 0)
      return std::string("patch segment header mismatch: ") + (name + 1);
    const uint64_t limit = fid == last ? end : (uint64_t)sb.st_size;
    const uint64_t rec = kPage + S_;
    if (limit > (uint64_t)sb.st_size || limit < kPage || (limit - kPage) % rec != 0)
      return std::string("segment shorter than the barrier recorded: ") + (name + 1);
    for (uint64_t off = kPage; off < limit; off += rec) {
      if (!pread_all(fd, got.get(), kPage, off) || !pread_all(fd, pay.get(), S_, off + kPage))
        return errno_str("read record");
      const unsigned char* r = reinterpret_cast<const unsigned char*>(got.get());
      const uint64_t gid = get64(r + 8);
      if (std::memcmp(r, "TREC", 4) != 0 || get32(r + 4) != 2 || get64(r + 24) != payload_ ||
          gid % g_.G != g_.rank || gid / g_.G >= g_.Kloc || get32(r + 36) != crc32c(r, 36) ||
          get32(r + 32) != crc32c(pay.get(), payload_))
        return std::string("corrupt record inside the barrier's log: ") + (name + 1) + " @" +
               std::to_string(off);
      index_[gid / g_.G] = {fid, off + kPage, payload_, get64(r + 16)};
    }
  }
  // appends after the barrier are not part of its state
  if (last && ::ftruncate(fds_[last], (off_t)end) != 0) return errno_str("truncate after barrier");
  for (uint32_t fid = last + 1;; ++fid) {
    char name[64];
    std::snprintf(name, sizeof name, "/patch-%06u.tdgp", fid);
    if (::unlink((dir_ + name).c_str()) != 0) break;
  }
  fsync_dir(dir_);
  cur_file_ = last;
  cur_size_ = last ? end : 0;
  return "";
}

// R31 compaction, at a barrier: every block's newest version
// is copied to base.tdgs.tmp at the base offsets (reads through Index, writes
// in parallel), which is made durable and renamed over the base; the patch
// segments are removed and Index points into the base again.
std::string BlockStore::compact() {
  pf_join();
  for (const Ent& e : ents_)
    if (e.blk >= 0 && ent_of_[e.blk] >= 0 && e.dirty) return "compact: dirty entries (barrier first)";
  const std::string tmp = dir_ + "/base.tdgs.tmp";
  int fd = ::open(tmp.c_str(), O_RDWR | O_CREAT | O_TRUNC | (direct_ ? O_DIRECT : 0), 0644);
  if (fd < 0) return errno_str("open base.tdgs.tmp");
  std::unique_ptr<char, decltype(&free)> hp(aligned_pages(kPage), &free);
  segment_header(reinterpret_cast<unsigned char*>(hp.get()), 0, g_);
  if (!pwrite_all(fd, hp.get(), kPage, 0)) {
    ::close(fd);
    return errno_str("write base header");
  }
  for (uint32_t f = 0; f <= cur_file_; ++f)
    if (fd_of(f) < 0) {
      ::close(fd);
      return errno_str("open segment");
    }
  std::atomic<bool> bad{false};
  pool_io_->parallel_for(g_.Kloc, [&](uint32_t l) {
    thread_local std::unique_ptr<char, decltype(&free)> buf(nullptr, &free);
    thread_local uint64_t cap = 0;
    if (cap < S_) {
      buf.reset(aligned_pages(S_));
      cap = S_;
    }
    const StoreIndex& ix = index_[l];
    std::memset(buf.get(), 0, S_);
    if (!pread_all(fds_[ix.file_id], buf.get(), S_, ix.offset) ||
        !pwrite_all(fd, buf.get(), S_, kPage + (uint64_t)l * S_))
      bad = true;
  });
  if (bad || ::fdatasync(fd) != 0) {
    ::close(fd);
    return errno_str("write compacted base");
  }
  // crash order: new base durable under its name, then a manifest that points
  // at it alone, then the patches go (an older manifest over the new base and
  // the old patches still recovers the same newest versions)
  if (::rename(tmp.c_str(), (dir_ + "/base.tdgs").c_str()) != 0 || !fsync_dir(dir_)) {
    ::close(fd);
    return errno_str("rename compacted base");
  }
  const uint32_t old_last = cur_file_;
  for (uint32_t l = 0; l < g_.Kloc; ++l) {
    index_[l].file_id = 0;
    index_[l].offset = kPage + (uint64_t)l * S_;
    base_version_[l] = index_[l].version;
  }
  cur_file_ = 0;
  cur_size_ = 0;
  std::string merr = write_manifest();
  if (!merr.empty()) {
    ::close(fd);
    return merr;
  }
  for (uint32_t f = 0; f < fds_.size(); ++f)
    if (fds_[f] >= 0) ::close(fds_[f]);
  for (uint32_t f = 1; f <= old_last; ++f) {
    char name[64];
    std::snprintf(name, sizeof name, "/patch-%06u.tdgp", f);
    ::unlink((dir_ + name).c_str());
  }
  fsync_dir(dir_);
  fds_.assign(1, fd);
  return "";
}

void BlockStore::unlink(int32_t e) {
  Ent& x = ents_[e];
  if (!x.listed) return;
  if (x.prev >= 0) ents_[x.prev].next = x.next; else head_ = x.next;
  if (x.next >= 0) ents_[x.next].prev = x.prev; else tail_ = x.prev;
  x.prev = x.next = -1;
  x.listed = false;
}

void BlockStore::push_mru(int32_t e) {
  Ent& x = ents_[e];
  x.prev = tail_;
  x.next = -1;
  if (tail_ >= 0) ents_[tail_].next = e; else head_ = e;
  tail_ = e;
  x.listed = true;
}

std::string BlockStore::new_segment() {
  cur_file_ += 1;
  char name[64];
  std::snprintf(name, sizeof name, "/patch-%06u.tdgp", cur_file_);
  const int fd = ::open((dir_ + name).c_str(), O_RDWR | O_CREAT | O_TRUNC | (direct_ ? O_DIRECT : 0),
                        0644);
  if (fd < 0) return errno_str("open patch segment");
  if (cur_file_ >= fds_.size()) fds_.resize(cur_file_ + 1, -1);
  fds_[cur_file_] = fd;
  std::unique_ptr<char, decltype(&free)> hp(aligned_pages(kPage), &free);
  segment_header(reinterpret_cast<unsigned char*>(hp.get()), cur_file_, g_);
  if (!pwrite_all(fd, hp.get(), kPage, 0)) return errno_str("write patch header");
  cur_size_ = kPage;
  cnt_.segments += 1;
  cnt_.write_bytes += kPage;
  return "";
}

// updated blocks are appended to patch segments, never
// written in place; Index[k] then points to the latest location.  R28: a new
// segment starts when the record would push a non-empty segment past the budget.
std::string BlockStore::reserve_append(uint32_t l, int& fd, uint64_t& rec_off) {
  const uint64_t rec = kPage + S_;
  if (cur_file_ == 0 || (cur_size_ > kPage && cur_size_ + rec > seg_budget_)) {
    std::string err = new_segment();
    if (!err.empty()) return err;
  }
  fd = fds_[cur_file_];
  rec_off = cur_size_;
  StoreIndex& ix = index_[l];
  ix = {cur_file_, rec_off + kPage, payload_, ix.version + 1};
  cur_size_ += rec;
  cnt_.write_bytes += rec;
  return "";
}

// appends the given (block, entry) records in order: offsets are reserved
// sequentially, then the header page + payload of every record is written in
// parallel (pwritev straight from the pinned entry).
std::string BlockStore::write_records(const std::vector<std::pair<uint32_t, int32_t>>& recs) {
  if (recs.empty()) return "";
  const size_t need = recs.size() * kPage;
  if (hdr_cap_ < need) {
    free(hdr_pages_);
    hdr_pages_ = aligned_pages(need);
    hdr_cap_ = need;
  }
  std::vector<int> fd(recs.size());
  std::vector<uint64_t> off(recs.size());
  for (size_t i = 0; i < recs.size(); ++i) {
    std::string err = reserve_append(recs[i].first, fd[i], off[i]);
    if (!err.empty()) return err;
    unsigned char* h = reinterpret_cast<unsigned char*>(hdr_pages_ + i * kPage);
    std::memset(h, 0, kPage);
    std::memcpy(h, "TREC", 4);
    put32(h + 4, 2);
    put64(h + 8, (uint64_t)recs[i].first * g_.G + g_.rank);
    put64(h + 16, index_[recs[i].first].version);
    put64(h + 24, payload_);
    // CRCs (h + 32 payload, h + 36 header) are filled by the writing thread
  }
  // consecutive records of one segment form one pwritev (header page +
  // payload per record, up to 16 MiB); the runs are spread over the pool
  constexpr uint64_t kRunBytes = 16ull << 20;
  constexpr size_t kMaxRec = 64;
  std::vector<std::pair<size_t, size_t>> runs;
  for (size_t i = 0; i < recs.size();) {
    size_t j = i + 1;
    while (j < recs.size() && j - i < kMaxRec && fd[j] == fd[i] &&
           off[j] == off[j - 1] + kPage + S_ && (j - i + 1) * (kPage + S_) <= kRunBytes)
      ++j;
    runs.push_back({i, j});
    i = j;
  }
  std::atomic<bool> bad{false};
  pool_io_->parallel_for((uint32_t)runs.size(), [&](uint32_t r) {
    const size_t b = runs[r].first, e = runs[r].second;
    for (size_t i = b; i < e; ++i) {  // R28 format 2 integrity
      unsigned char* h = reinterpret_cast<unsigned char*>(hdr_pages_ + i * kPage);
      put32(h + 32, crc32c(pool_ + (uint64_t)buf_of_[recs[i].second] * S_, payload_));
      put32(h + 36, crc32c(h, 36));
    }
    iovec iov[2 * kMaxRec];
    int n = 0;
    for (size_t i = b; i < e; ++i) {
      iov[n].iov_base = hdr_pages_ + i * kPage;
      iov[n++].iov_len = kPage;
      iov[n].iov_base = pool_ + (uint64_t)buf_of_[recs[i].second] * S_;
      iov[n++].iov_len = S_;
    }
    const uint64_t total = (uint64_t)(e - b) * (kPage + S_);
    ssize_t w;
    do {
      w = ::pwritev(fd[b], iov, n, (off_t)off[b]);
    } while (w < 0 && errno == EINTR);
    if (w == (ssize_t)total) return;
    for (size_t i = b; i < e; ++i)  // short or failed vector write: record by record
      if (!pwrite_all(fd[i], hdr_pages_ + i * kPage, kPage, off[i]) ||
          !pwrite_all(fd[i], pool_ + (uint64_t)buf_of_[recs[i].second] * S_, S_, off[i] + kPage))
        bad = true;
  });
  return bad ? errno_str("append patch record") : "";
}

std::string BlockStore::gather(const uint32_t* sp, uint32_t n, int32_t T,
                               const std::function<void(int32_t)>& wait_d2h,
                               const std::function<void(const std::vector<uint8_t>&)>& hits_ready) {
  // the read-ahead batches announced for this activate or earlier have landed
  // (batches for later activates may still be reading)
  uint64_t upto = 0;
  while (!pf_target_.empty() && pf_target_.front().second <= T) {
    upto = pf_target_.front().first;
    pf_target_.pop_front();
  }
  const uint64_t pf_done = pf_wait(upto);
  // every S+ block is in R_{t+1}: its entry (if cached) is not evictable (R27)
  for (uint32_t i = 0; i < n; ++i) {
    const int32_t e = ent_of_[sp[2 * i]];
    if (e >= 0) unlink(e);
  }
  std::vector<std::pair<uint32_t, int32_t>> victims, misses;  // (block, entry)
  std::vector<int32_t> jobs;
  std::vector<uint8_t> miss(n, 0);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t l = sp[2 * i];
    int32_t e = ent_of_[l];
    if (e >= 0) {
      cnt_.hits += 1;
    } else {
      cnt_.misses += 1;
      miss[i] = 1;
      if (!free_.empty()) {
        e = free_.back();
        free_.pop_back();
      } else {
        e = head_;  // least recently used entry outside R_t u R_{t+1}
        if (e < 0) return "CPU cache: no evictable entry (cache_blocks < 2C?)";
        unlink(e);
        Ent& v = ents_[e];
        cnt_.evictions += 1;
        if (v.dirty) {  // two-step write-back, step 2
          cnt_.dirty_evictions += 1;
          victims.push_back({(uint32_t)v.blk, e});
          if (v.wb_job >= 0) jobs.push_back(v.wb_job);
        }
        ent_of_[v.blk] = -1;
      }
      ent_of_[l] = e;
      misses.push_back({l, e});
      ents_[e].dirty = false;
      ents_[e].wb_job = -1;
    }
    Ent& x = ents_[e];
    x.blk = (int32_t)l;
    x.resident = true;
    x.admitted = T;
    x.stamp = ++clock_;
  }
  // the hits' records are final: the caller can start moving them while the
  // victims are appended and the misses read
  if (hits_ready) hits_ready(miss);
  if (!victims.empty()) {
    const auto t0 = std::chrono::steady_clock::now();
    std::sort(jobs.begin(), jobs.end());
    jobs.erase(std::unique(jobs.begin(), jobs.end()), jobs.end());
    for (int32_t j : jobs) wait_d2h(j);  // the victim's newest record has landed
    std::string err = write_records(victims);
    if (!err.empty()) return err;
    cnt_.write_ms += ms_since(t0);
  }
  if (!misses.empty()) {  // fetched through Index[k]
    cnt_.read_bytes += misses.size() * S_;
    // a miss read ahead at its newest version takes that buffer (the victims
    // written above no longer need the entry's old one); the rest is read now
    std::vector<std::pair<uint32_t, int32_t>> rest;
    for (auto& m : misses) {
      const int32_t b = ra_buf_[m.first];
      const bool complete = b >= 0 && ra_seq_[m.first] <= pf_done;
      bool bad = false;
      if (complete) {
        std::lock_guard<std::mutex> g(pf_mu_);
        bad = pf_badbuf_[b] != 0;
        pf_badbuf_[b] = 0;
      }
      if (complete && !bad && ra_ver_[m.first] == index_[m.first].version) {
        ra_free_.push_back(buf_of_[m.second]);
        buf_of_[m.second] = (uint32_t)b;
        ra_buf_[m.first] = -1;
        cnt_.prefetch_hits += 1;
      } else {
        if (complete) {  // stale or failed: released; an in-flight one finishes first
          ra_free_.push_back((uint32_t)b);
          ra_buf_[m.first] = -1;
          cnt_.prefetch_wasted += 1;
        }
        rest.push_back(m);
      }
    }
    if (!rest.empty()) {
      const auto t0 = std::chrono::steady_clock::now();
      std::string err = read_records(rest);
      if (!err.empty()) return err;
      cnt_.read_ms += ms_since(t0);
    }
  }
  return "";
}

// Reads the newest version of each (block, entry) into its entry.  Records
// that are neighbours in one segment (consecutive base records, or patch
// records separated only by their header page) are read by one preadv into
// the scattered entries (header pages into a scratch page), up to kRunBytes,
// so the device sees large requests; the runs are spread over the pool.
std::string BlockStore::read_records(const std::vector<std::pair<uint32_t, int32_t>>& recs) {
  // TGS_STORE_READ_RUN=<MiB> caps a coalesced read.  Default 1 MiB, i.e. one
  // record per request: on this box's virtio disk 8 parallel single-record
  // reads beat coalesced 3- and 8-record reads (5.6 vs 5.4 / 5.0 GB/s,
  // profiles/store_r01.md)
  static const uint64_t kRunBytes = [] {
    const char* v = getenv("TGS_STORE_READ_RUN");
    return v ? (uint64_t)std::max(1, atoi(v)) * (1ull << 20) : (1ull << 20);
  }();
  constexpr int kMaxIov = 256;
  struct Item { uint32_t fid; uint64_t off; int32_t e; };
  std::vector<Item> it(recs.size());
  for (size_t i = 0; i < recs.size(); ++i) {
    const StoreIndex& ix = index_[recs[i].first];
    it[i] = {ix.file_id, ix.offset, recs[i].second};
    if (fd_of(ix.file_id) < 0) return errno_str("open segment");  // opened serially
  }
  std::sort(it.begin(), it.end(), [](const Item& a, const Item& b) {
    return a.fid != b.fid ? a.fid < b.fid : a.off < b.off;
  });
  std::vector<std::pair<size_t, size_t>> runs;  // [begin, end) into it
  for (size_t i = 0; i < it.size();) {
    size_t j = i + 1;
    uint64_t end = it[i].off + S_;
    int iov = 1;
    while (j < it.size() && it[j].fid == it[i].fid && end - it[i].off + S_ + kPage <= kRunBytes &&
           iov + 2 <= kMaxIov && (it[j].off == end || it[j].off == end + kPage)) {
      iov += it[j].off == end ? 1 : 2;
      end = it[j].off + S_;
      ++j;
    }
    runs.push_back({i, j});
    i = j;
  }
  std::atomic<bool> bad{false};
  std::mutex busy_mu;
  double busy = 0.0;
  cnt_.read_calls += runs.size();
  pool_io_->parallel_for((uint32_t)runs.size(), [&](uint32_t r) {
    thread_local std::unique_ptr<char, decltype(&free)> scratch(aligned_pages(kPage), &free);
    const size_t b = runs[r].first, e = runs[r].second;
    const int fd = fds_[it[b].fid];
    iovec iov[kMaxIov];
    int n = 0;
    uint64_t total = 0, pos = it[b].off;
    for (size_t i = b; i < e; ++i) {
      if (it[i].off != pos) {  // a patch record's header page between two payloads
        iov[n].iov_base = scratch.get();
        iov[n++].iov_len = kPage;
        total += kPage;
      }
      iov[n].iov_base = pool_ + (uint64_t)buf_of_[it[i].e] * S_;
      iov[n++].iov_len = S_;
      total += S_;
      pos = it[i].off + S_;
    }
    ssize_t got;
    const auto t0 = std::chrono::steady_clock::now();
    do {
      got = ::preadv(fd, iov, n, (off_t)it[b].off);
    } while (got < 0 && errno == EINTR);
    {
      std::lock_guard<std::mutex> g(busy_mu);
      busy += ms_since(t0);
    }
    if (got == (ssize_t)total) return;
    for (size_t i = b; i < e; ++i)  // short or failed vector read: record by record
      if (!pread_all(fd, pool_ + (uint64_t)buf_of_[it[i].e] * S_, S_, it[i].off)) bad = true;
  });
  cnt_.read_busy_ms += busy;
  return bad ? errno_str("read block record") : "";
}

void BlockStore::touch_evicted(const uint32_t* sm, uint32_t n, int32_t T) {
  for (uint32_t i = 0; i < n; ++i) {
    const int32_t e = ent_of_[sm[i]];
    if (e < 0) continue;  // cannot happen (inclusion)
    Ent& x = ents_[e];
    x.stamp = ++clock_;
    if (x.admitted == T) continue;  // re-admitted by this activate (tide off): still pinned
    x.resident = false;
    unlink(e);
    push_mru(e);
  }
}

void BlockStore::mark_dirty(uint32_t l, int32_t T) {
  const int32_t e = ent_of_[l];
  if (e < 0) return;
  ents_[e].dirty = true;
  ents_[e].wb_job = T;
}

std::string BlockStore::flush_all(const std::function<void(int32_t)>& wait_d2h,
                                  const uint32_t* steps) {
  pf_join();  // no read-ahead in flight while segments change
  std::vector<std::pair<uint32_t, int32_t>> recs;
  for (uint32_t l = 0; l < g_.Kloc; ++l) {
    const int32_t e = ent_of_[l];
    if (e >= 0 && ents_[e].dirty) {
      recs.push_back({l, e});
      if (ents_[e].wb_job >= 0) wait_d2h(ents_[e].wb_job);
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  std::string err = write_records(recs);
  if (!err.empty()) return err;
  for (auto& r : recs) {
    ents_[r.second].dirty = false;
    ents_[r.second].wb_job = -1;
  }
  cnt_.flush_appends += recs.size();
  for (int fd : fds_)  // a consistency barrier: durable on return
    if (fd >= 0 && ::fdatasync(fd) != 0) return errno_str("fdatasync");
  if (steps) std::memcpy(steps_.data(), steps, sizeof(uint32_t) * g_.Kloc);
  err = write_manifest();  // R30: the durable end of the log
  if (!err.empty()) return err;
  cnt_.write_ms += ms_since(t0);
  return "";
}

std::string BlockStore::read_block(uint32_t l, void* dst) {
  if (const float* p = entry_of(l)) {
    std::memcpy(dst, p, payload_);
    return "";
  }
  std::unique_ptr<char, decltype(&free)> buf(aligned_pages(S_), &free);
  const StoreIndex& ix = index_[l];
  const int fd = fd_of(ix.file_id);
  if (fd < 0 || !pread_all(fd, buf.get(), S_, ix.offset)) return errno_str("read block record");
  std::memcpy(dst, buf.get(), payload_);
  return "";
}

uint32_t BlockStore::cached_dirty() const {
  uint32_t n = 0;
  for (const Ent& e : ents_) n += (e.blk >= 0 && ent_of_[e.blk] >= 0 && e.dirty) ? 1 : 0;
  return n;
}

void BlockStore::lru_order(std::vector<uint32_t>& blocks, std::vector<uint8_t>& dirty) const {
  std::vector<std::pair<uint64_t, int32_t>> v;
  for (uint32_t l = 0; l < g_.Kloc; ++l)
    if (ent_of_[l] >= 0) v.push_back({ents_[ent_of_[l]].stamp, ent_of_[l]});
  std::sort(v.begin(), v.end());
  blocks.clear();
  dirty.clear();
  for (auto& x : v) {
    blocks.push_back((uint32_t)ents_[x.second].blk);
    dirty.push_back(ents_[x.second].dirty ? 1 : 0);
  }
}

}  // namespace tgs
