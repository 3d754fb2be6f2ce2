// tgs_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see tgs_oracle.h).
//
// Plain single-threaded C++17, compiled with -O2 -ffp-contract=off and no
// fast-math, default MXCSR (no FTZ/DAZ).  Every step follows the paper in its
// order and notation; every silent point follows a DESIGN.md reading (R#).
#include "tgs_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>
#include <limits>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

namespace {

constexpr uint32_t D = 59;  // PAPER.md:101-103 "D = 59"


// ---- NEXT f3: the tier below the host (§3.4), readings
// R27 (cache events) and R28 (segment format) of DESIGN.md §3.
struct IndexEntry {     // PAPER.md:233 "Index[k] = (file_id, offset, size, version)"
  uint32_t file_id = 0;  // 0 = base segment
  uint64_t offset = 0;   // byte offset of the payload in that file
  uint64_t size = 0;     // payload bytes (n_arr * B * 59 * 4)
  uint64_t version = 0;  // 0 = base, +1 per appended version
};
struct CacheEntry {     // PAPER.md:239-240 "an LRU cache over blocks together with a per-block dirty bit"
  std::vector<float> payload;  // theta | m | v (persist) or theta; empty in metadata-only mode
  bool dirty = false;
  uint64_t stamp = 0;          // LRU clock of the last access
};
struct Store {
  bool on = false;
  bool data = false;           // files written / read (needs every block tracked)
  std::string dir;
  uint32_t H = 0;              // cache capacity in block records
  uint64_t seg_budget = 0;     // patch segment rollover budget (bytes)
  uint64_t S = 0;              // payload bytes padded to 4096 (record slot)
  uint64_t payload = 0;        // n_arr * rec_bytes
  std::vector<IndexEntry> index;   // per local block
  std::map<uint32_t, CacheEntry> cache;
  uint64_t clock = 0;
  uint32_t cur_file = 0;       // 0 = no patch segment open yet
  uint64_t cur_size = 0;       // bytes in the current patch segment
  uint64_t epoch = 0;          // barriers (and compactions) written to the manifest
  std::vector<uint64_t> base_version;  // version of each block's base record (R31)
  uint64_t hits = 0, misses = 0, evictions = 0, dirty_evictions = 0, flush_appends = 0,
           read_bytes = 0, write_bytes = 0, segments = 0;
};

struct Ctx {
  or_config cfg{};
  uint64_t K = 0;       // global blocks, K = ceil(N/B)
  uint32_t Kloc = 0;    // blocks owned by this shard (R17: k % G == rank)
  uint32_t P = 0;       // slots
  std::vector<float> bounds;  // Kloc x 4 (c_k, r_k)
  or_fill_fn fill = nullptr;
  void* fill_user = nullptr;
  bool track_all = false;
  std::vector<char> tracked;

  // per local block state
  std::vector<int64_t> last_access;  // -1 = never accessed (R4)
  std::vector<uint32_t> step;        // Adam step counter (R7)
  std::vector<int32_t> slot_of;      // -1 = not resident
  std::vector<char> ever_resident, evicted_once;
  std::vector<int64_t> admit_iter;

  // per slot state
  std::vector<int64_t> block_of;     // local id or -1
  std::vector<char> dirty;

  // data (tracked blocks only): host tier record and slot contents
  std::unordered_map<uint32_t, std::vector<float>> host;  // theta|m|v (persist) or theta
  std::unordered_map<int32_t, std::vector<float>> slot_data;  // theta|m|v

  // sets, as sorted vectors of local ids
  std::vector<float> planes;              // camera batch of the last activate (J x 6 x 4)
  std::vector<float> pend[2];             // R25: refreshed radii of the step of that parity
  std::vector<uint32_t> R;                // R_t
  std::vector<uint32_t> A_prev;           // R_t n K_t
  std::vector<std::vector<uint32_t>> percam;
  std::vector<uint32_t> Kset, Rnew, Splus, Sminus, Omega, A, evicted_dirty;

  int64_t t = 0;          // number of activates so far
  bool can_step = false;  // one step_adam per activate
  uint64_t nonfinite = std::numeric_limits<uint64_t>::max();
  or_stats st{};
  Store sto;
  // phase timers (SURVEY §8c timing hooks): cull, plan (selection, delta,
  // slots), copies (write-back + gather of records), Adam -- nanoseconds
  uint64_t phase_ns[4] = {0, 0, 0, 0};

  uint64_t gid_block(uint32_t l) const { return (uint64_t)l * cfg.world_size + cfg.rank; }
  uint32_t rows(uint32_t l) const {
    uint64_t lo = gid_block(l) * cfg.block_size;
    if (lo >= cfg.n_gaussians) return 0;
    uint64_t r = cfg.n_gaussians - lo;
    return (uint32_t)std::min<uint64_t>(r, cfg.block_size);
  }
  size_t rec_floats() const { return (size_t)cfg.block_size * D; }
  uint32_t n_arr() const { return cfg.moments == OR_PERSIST ? 3u : 1u; }
  uint64_t rec_bytes() const { return (uint64_t)rec_floats() * 4u; }
  bool is_tracked(uint32_t l) const { return track_all || tracked[l]; }

  std::vector<float>& host_rec(uint32_t l) {
    auto it = host.find(l);
    if (it != host.end()) return it->second;
    std::vector<float> v((size_t)n_arr() * rec_floats(), 0.0f);  // m = v = 0 initially
    if (fill) fill(fill_user, gid_block(l), v.data());
    return host.emplace(l, std::move(v)).first->second;
  }
};

// Level-1 test: cull iff d < -r_k for some plane; R2: d is
// the fmaf chain x -> y -> z with d0 as the first addend.
bool sphere_visible(const float* b, const float* pl /* 6x4 */) {
  for (int p = 0; p < 6; ++p) {
    const float* n = pl + 4 * p;
    float d = std::fmaf(n[2], b[2], std::fmaf(n[1], b[1], std::fmaf(n[0], b[0], n[3])));
    if (d < -b[3]) return false;
  }
  return true;
}

// R24: deterministic exp for the Level-2 extent, written out so that any
// IEEE machine with a correctly rounded fma gives the same bits: k = rint(x
// log2 e) by the 1.5*2^23 trick, Cody-Waite reduction r = x - k ln2 (two fma
// steps), degree-7 Taylor polynomial in Horner form (fma), exact scaling 2^k.
// Valid for x in [-80, 80] (the generator's log-scales are in [-12, 5]).
float exp_det(float x) {
  if (x > 80.0f) x = 80.0f;
  if (x < -80.0f) x = -80.0f;
  const float t = std::fmaf(x, 1.44269504088896341f, 12582912.0f);
  const float kf = t - 12582912.0f;
  float r = std::fmaf(kf, -0.693145751953125f, x);
  r = std::fmaf(kf, -1.428606765330187045e-06f, r);
  float p = 1.98412698412698413e-04f;                 // 1/5040
  p = std::fmaf(p, r, 1.38888888888888889e-03f);      // 1/720
  p = std::fmaf(p, r, 8.33333333333333333e-03f);      // 1/120
  p = std::fmaf(p, r, 4.16666666666666667e-02f);      // 1/24
  p = std::fmaf(p, r, 1.66666666666666667e-01f);      // 1/6
  p = std::fmaf(p, r, 0.5f);
  p = std::fmaf(p, r, 1.0f);
  p = std::fmaf(p, r, 1.0f);
  const int k = (int)kf;
  uint32_t bits = (uint32_t)(k + 127) << 23;
  float two_k;
  std::memcpy(&two_k, &bits, 4);
  return p * two_k;
}

// Level-2 test of one Gaussian (R24): the
// sphere (mu_i, 3 * exp(max log-scale)) against the cameras whose Level-1 set
// K^(j) holds its block -- camera j renders only its visible blocks -- with the
// Level-1 rule (cull iff d < -r on some plane, R2); visible if one keeps it.
bool gaussian_visible(const float* row, const std::vector<float>& planes,
                      const std::vector<uint32_t>& cams) {
  float s = row[52];
  if (row[53] > s) s = row[53];
  if (row[54] > s) s = row[54];
  const float ext = 3.0f * exp_det(s);
  const float b[4] = {row[0], row[1], row[2], ext};
  for (uint32_t j : cams)
    if (sphere_visible(b, planes.data() + 24 * j)) return true;
  return false;
}

uint32_t fbits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
}

// R25 (NEXT f2, "we conservatively refresh each affected block
// bound as centers move"): radius that holds Gaussian row i around the fixed
// centre c_k: (|mu_i - c_k| + 3 exp(max log-scale_i)) inflated by 2^-19
// relative so fp32 rounding cannot make it smaller than the real value.
float refresh_radius(const float* row, const float* c) {
  const float dx = row[0] - c[0], dy = row[1] - c[1], dz = row[2] - c[2];
  const float d2 = std::fmaf(dz, dz, std::fmaf(dy, dy, dx * dx));
  const float dist = std::sqrt(d2);
  float s = row[52];
  if (row[53] > s) s = row[53];
  if (row[54] > s) s = row[54];
  const float ext = 3.0f * exp_det(s);
  return (dist + ext) * 1.0000019073486328f;
}

std::vector<uint32_t> set_union(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> o;
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}
std::vector<uint32_t> set_inter(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> o;
  std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}
std::vector<uint32_t> set_minus(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  std::vector<uint32_t> o;
  std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(o));
  return o;
}
bool contains(const std::vector<uint32_t>& s, uint32_t x) {
  return std::binary_search(s.begin(), s.end(), x);
}


// ---- NEXT f3 store tier helpers (R28 format: little-endian, every header a
// 4096-byte page so payloads start page-aligned -- PAPER.md:187-188 "236
// contiguous 4 KB pages ... aligns the dominant block records with common
// filesystem/page-cache granularities").
constexpr uint64_t kPage = 4096;
uint64_t pad_page(uint64_t x) { return (x + kPage - 1) / kPage * kPage; }

// CRC-32C (Castagnoli, reflected polynomial 0x82F63B78, init and final xor
// 0xFFFFFFFF): the textbook byte-table form, the table being the bitwise
// division of each byte value by the polynomial (check value of "123456789":
// 0xE3069283).  R28 format 2: integrity of every record.
uint32_t crc32c(const void* data, uint64_t n) {
  static const std::vector<uint32_t> table = [] {
    std::vector<uint32_t> t(256);
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ (0x82F63B78u & (0u - (c & 1u)));
      t[i] = c;
    }
    return t;
  }();
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint32_t crc = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) crc = (crc >> 8) ^ table[(crc ^ p[i]) & 0xFFu];
  return crc ^ 0xFFFFFFFFu;
}

void put32(unsigned char* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (unsigned char)(v >> (8 * i));
}
void put64(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (unsigned char)(v >> (8 * i));
}

std::string seg_path(const Store& s, uint32_t fid) {
  char b[64];
  if (fid == 0)
    std::snprintf(b, sizeof b, "/base.tdgs");
  else
    std::snprintf(b, sizeof b, "/patch-%06u.tdgp", fid);
  return s.dir + b;
}

// segment header page: magic, format 1, file id, n_arr, N, D, B, G, rank, Kloc
std::vector<unsigned char> segment_header(const Ctx& c, uint32_t fid) {
  std::vector<unsigned char> h(kPage, 0);
  std::memcpy(h.data(), fid == 0 ? "TDGS" : "TDGP", 4);
  put32(&h[4], 1);
  put32(&h[8], fid);
  put32(&h[12], c.n_arr());
  put64(&h[16], c.cfg.n_gaussians);
  put32(&h[24], D);
  put32(&h[28], c.cfg.block_size);
  put32(&h[32], (uint32_t)c.cfg.world_size);
  put32(&h[36], (uint32_t)c.cfg.rank);
  put32(&h[40], c.Kloc);
  return h;
}

void write_at(const std::string& path, uint64_t off, const void* p, uint64_t n, bool create) {
  FILE* f = std::fopen(path.c_str(), create ? "w+b" : "r+b");
  if (!f) return;
  std::fseek(f, (long)off, SEEK_SET);
  std::fwrite(p, 1, n, f);
  std::fclose(f);
}

void read_at(const std::string& path, uint64_t off, void* p, uint64_t n) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return;
  std::fseek(f, (long)off, SEEK_SET);
  size_t got = std::fread(p, 1, n, f);
  (void)got;
  std::fclose(f);
}

// "updated blocks are written sequentially into patch
// segments rather than overwriting existing block locations in place"; Index[k]
// then points to the latest location.  R28: a record is a
// header page ("TREC", format 2, global id, version, payload bytes, CRC-32C of
// the payload, CRC-32C of header bytes [0, 36)) followed by the payload padded
// to whole pages; a new segment starts when the record would push a non-empty
// segment past the byte budget.
void append_version(Ctx& c, uint32_t l, const CacheEntry& e) {
  Store& s = c.sto;
  const uint64_t rec = kPage + s.S;
  if (s.cur_file == 0 || (s.cur_size > kPage && s.cur_size + rec > s.seg_budget)) {
    s.cur_file += 1;
    s.segments += 1;
    s.cur_size = kPage;
    s.write_bytes += kPage;
    if (s.data) {
      std::vector<unsigned char> h = segment_header(c, s.cur_file);
      write_at(seg_path(s, s.cur_file), 0, h.data(), kPage, true);
    }
  }
  IndexEntry& ix = s.index[l];
  const uint64_t off = s.cur_size;
  const uint64_t version = ix.version + 1;
  if (s.data) {
    std::vector<unsigned char> r(rec, 0);
    std::memcpy(&r[0], "TREC", 4);
    put32(&r[4], 2);
    put64(&r[8], c.gid_block(l));
    put64(&r[16], version);
    put64(&r[24], s.payload);
    std::memcpy(&r[kPage], e.payload.data(), s.payload);
    put32(&r[32], crc32c(&r[kPage], s.payload));
    put32(&r[36], crc32c(&r[0], 36));
    write_at(seg_path(s, s.cur_file), off, r.data(), rec, false);
  }
  ix.file_id = s.cur_file;
  ix.offset = off + kPage;
  ix.size = s.payload;
  ix.version = version;
  s.cur_size += rec;
  s.write_bytes += rec;
}

// R30 barrier manifest ("manifest.tdgm"), written at every barrier and after a
// compaction: "TDGM", format 1, epoch, the last patch segment and its length
// as of the barrier (the durable end of the log), the shard geometry, then per
// local block the version of its base record (R31) and its Adam step counter,
// then a CRC-32C of everything before.  Written to a temporary name and
// renamed, so a crash leaves the previous barrier's manifest.
void write_manifest(Ctx& c) {
  Store& s = c.sto;
  s.epoch += 1;
  std::vector<unsigned char> m(64 + 12 * (size_t)c.Kloc + 4, 0);
  std::memcpy(&m[0], "TDGM", 4);
  put32(&m[4], 1);
  put64(&m[8], s.epoch);
  put32(&m[16], s.cur_file);
  put64(&m[24], s.cur_file ? s.cur_size : 0);
  put32(&m[32], c.n_arr());
  put64(&m[40], c.cfg.n_gaussians);
  put32(&m[48], c.cfg.block_size);
  put32(&m[52], (uint32_t)c.cfg.world_size);
  put32(&m[56], (uint32_t)c.cfg.rank);
  put32(&m[60], c.Kloc);
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    put64(&m[64 + 8 * (size_t)l], s.base_version[l]);
    put32(&m[64 + 8 * (size_t)c.Kloc + 4 * (size_t)l], c.step[l]);
  }
  put32(&m[m.size() - 4], crc32c(m.data(), m.size() - 4));
  const std::string tmp = s.dir + "/manifest.tdgm.tmp";
  write_at(tmp, 0, m.data(), m.size(), true);
  std::error_code ec;
  std::filesystem::rename(tmp, s.dir + "/manifest.tdgm", ec);
}

// R27 (b): CPU-cache access of an S+ block.  Hit:
// touch.  Miss: take a new entry while fewer than H blocks are cached, else
// evict the least recently used entry whose block is in neither R_t nor
// R_{t+1} (the blocks the GPU holds are pinned); a dirty victim is appended to
// the patch log first.  Then the newest version is
// read through Index[k] ("Reads consult Index to materialize the
// newest version of each block").
CacheEntry& cache_access(Ctx& c, uint32_t l, const std::vector<uint32_t>& Rt,
                         const std::vector<uint32_t>& Rn) {
  Store& s = c.sto;
  auto it = s.cache.find(l);
  if (it != s.cache.end()) {
    s.hits += 1;
    it->second.stamp = ++s.clock;
    return it->second;
  }
  s.misses += 1;
  if (s.cache.size() >= s.H) {
    auto victim = s.cache.end();
    for (auto v = s.cache.begin(); v != s.cache.end(); ++v) {
      if (contains(Rt, v->first) || contains(Rn, v->first)) continue;
      if (victim == s.cache.end() || v->second.stamp < victim->second.stamp) victim = v;
    }
    // a victim exists: pinned entries <= |R_t u R_{t+1}| - 1 < 2C <= H
    s.evictions += 1;
    if (victim->second.dirty) {
      s.dirty_evictions += 1;
      append_version(c, victim->first, victim->second);
    }
    s.cache.erase(victim);
  }
  CacheEntry& e = s.cache[l];
  const IndexEntry& ix = s.index[l];
  if (s.data) {
    e.payload.assign((size_t)c.n_arr() * c.rec_floats(), 0.0f);
    read_at(seg_path(s, ix.file_id), ix.offset, e.payload.data(), s.payload);
  }
  s.read_bytes += s.S;
  e.dirty = false;
  e.stamp = ++s.clock;
  return e;
}

}  // namespace

struct or_ctx {
  Ctx c;
};

extern "C" {

int or_create(const or_config* cfg, const float* bounds_global, or_fill_fn fill, void* fill_user,
              int track_all, or_ctx** out) {
  if (!cfg || !out || !bounds_global) return OR_EINVAL;
  const or_config& g = *cfg;
  if (g.dim != D || g.block_size < 4 || g.block_size % 4 != 0 || g.capacity == 0 ||
      g.n_gaussians == 0)
    return OR_EINVAL;
  if (!(g.lambda >= 0.0 && g.lambda <= 1.0) || !(g.gamma > 0.0 && g.gamma < 1.0)) return OR_EINVAL;
  if (g.quota_den == 0 || g.quota_num > g.quota_den) return OR_EINVAL;
  if (g.world_size < 1 || g.rank < 0 || g.rank >= g.world_size) return OR_EINVAL;
  if (g.moments != OR_PERSIST && g.moments != OR_COLD_RESTART) return OR_EINVAL;
  if (g.refresh_bounds && !track_all) return OR_EINVAL;  // needs every block's rows
  uint32_t P = g.pool_slots ? g.pool_slots : 2u * g.capacity;
  if (P < g.capacity) return OR_EINVAL;
  or_ctx* o = new or_ctx();
  Ctx& c = o->c;
  c.cfg = g;
  c.P = P;
  c.K = (g.n_gaussians + g.block_size - 1) / g.block_size;
  c.Kloc = (uint32_t)((c.K > (uint64_t)g.rank) ? (c.K - g.rank + g.world_size - 1) / g.world_size : 0);
  c.bounds.resize((size_t)c.Kloc * 4);
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    const float* b = bounds_global + 4 * c.gid_block(l);
    for (int i = 0; i < 4; ++i) {
      if (!std::isfinite(b[i])) { delete o; return OR_EINVAL; }
      c.bounds[4 * l + i] = b[i];
    }
    if (b[3] < 0.0f) { delete o; return OR_EINVAL; }
  }
  c.fill = fill;
  c.fill_user = fill_user;
  c.track_all = track_all != 0;
  c.tracked.assign(c.Kloc, 0);
  c.last_access.assign(c.Kloc, -1);
  c.step.assign(c.Kloc, 0);
  c.slot_of.assign(c.Kloc, -1);
  c.ever_resident.assign(c.Kloc, 0);
  c.evicted_once.assign(c.Kloc, 0);
  c.admit_iter.assign(c.Kloc, 0);
  c.block_of.assign(P, -1);
  c.dirty.assign(P, 0);
  *out = o;
  return OR_OK;
}

void or_destroy(or_ctx* o) { delete o; }

int or_track_block(or_ctx* o, uint64_t kg) {
  Ctx& c = o->c;
  if (kg % c.cfg.world_size != (uint64_t)c.cfg.rank) return OR_EINVAL;
  uint64_t l = kg / c.cfg.world_size;
  if (l >= c.Kloc) return OR_EINVAL;
  if (c.slot_of[l] >= 0 && !c.tracked[l] && !c.track_all) return OR_ESTATE;  // track before admission
  if (c.sto.on && !c.sto.data) return OR_ESTATE;  // metadata-only store keeps no data
  c.tracked[l] = 1;
  return OR_OK;
}

using Clock = std::chrono::steady_clock;
static uint64_t ns_since(Clock::time_point a) {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - a).count();
}

int or_activate(or_ctx* o, const float* planes, uint32_t J) {
  Ctx& c = o->c;
  auto t0 = Clock::now();
  const or_config& g = c.cfg;
  if (J > g.max_cameras || (J > 0 && !planes)) return OR_EINVAL;
  for (uint32_t i = 0; i < J * 24; ++i)
    if (!std::isfinite(planes[i])) return OR_EINVAL;

  // ---- Alg. 1 l.1 / Eq. Kt_def: K^{(j)} and K = U_j K^{(j)}
  // R25: the refresh of the step two batches back enters the Level-1 test now
  if (g.refresh_bounds) {
    std::vector<float>& pd = c.pend[c.t & 1];
    for (uint32_t l = 0; l < c.Kloc && !pd.empty(); ++l)
      if (fbits(pd[l]) > fbits(c.bounds[4 * l + 3])) c.bounds[4 * l + 3] = pd[l];
    pd.assign(pd.size(), 0.0f);
  }
  c.planes.assign(planes, planes + (size_t)J * 24);
  c.percam.assign(J, {});
  for (uint32_t j = 0; j < J; ++j)
    for (uint32_t l = 0; l < c.Kloc; ++l)
      if (sphere_visible(&c.bounds[4 * l], planes + 24 * j)) c.percam[j].push_back(l);
  std::vector<uint32_t> Kn;
  for (uint32_t j = 0; j < J; ++j) Kn = set_union(Kn, c.percam[j]);
  c.phase_ns[0] += ns_since(t0);
  t0 = Clock::now();
  // locality of consecutive batches (the Jaccard of K_t and K_{t+1})
  c.st.k_inter_sum += set_inter(c.Kset, Kn).size();
  c.st.k_union_sum += set_union(c.Kset, Kn).size();

  // ---- Alg. 1 l.2: update Recency from R_t n K_t, the blocks
  //      accessed by the previous iteration (R12): stamp last access = t-1.
  if (c.t > 0)
    for (uint32_t l : c.A_prev) c.last_access[l] = c.t - 1;

  // ---- Alg. 1 l.3: candidate pool C_t = R_t u K_{t+1}
  //      (Tide off, PAPER.md:570-573 / SPEC.md:666: selection from K_{t+1} only)
  std::vector<uint32_t> cand = g.tide ? set_union(c.R, Kn) : Kn;

  // ---- Alg. 1 l.4-5: s(k) = lam*1[k in K_{t+1}] + (1-lam)*Recency(k)
  //      Recency(k) = gamma^age, reset on access and aged otherwise;
  //      R4: age = (t-1) - last_access, saturating at A_max; never accessed -> 0.
  auto score = [&](uint32_t l) -> double {
    double rec = 0.0;
    if (c.last_access[l] >= 0) {
      int64_t age = (c.t - 1) - c.last_access[l];
      if (age > (int64_t)g.max_age) age = g.max_age;
      rec = 1.0;
      for (int64_t i = 0; i < age; ++i) rec *= g.gamma;
    }
    double m = contains(Kn, l) ? 1.0 : 0.0;
    return g.lambda * m + (1.0 - g.lambda) * rec;
  };
  // R11 tie-break: higher score, then already resident (zero traffic), then lower id
  auto better = [&](uint32_t a, uint32_t b) {
    double sa = score(a), sb = score(b);
    if (sa != sb) return sa > sb;
    bool ra = contains(c.R, a), rb = contains(c.R, b);
    if (ra != rb) return ra;
    return a < b;
  };

  // ---- Alg. 1 l.6: R_{t+1} = CameraBalancedTopC({K^{(j)}}, C_t, s, C)
  //      (quota reading R10: q_j = min(|K^{(j)}|, floor(beta C / J)),
  //      union of per-camera top-q_j, then global fill by s over C_t).
  std::vector<uint32_t> Rn;
  const uint64_t C = g.capacity;
  if (cand.size() <= C) {
    Rn = cand;  // nothing to select
  } else {
    std::vector<uint32_t> Q;
    if (J > 0) {
      uint64_t q = (C * g.quota_num) / ((uint64_t)g.quota_den * J);
      for (uint32_t j = 0; j < J; ++j) {
        std::vector<uint32_t> kj = c.percam[j];
        std::sort(kj.begin(), kj.end(), better);
        uint64_t qj = std::min<uint64_t>(kj.size(), q);
        std::vector<uint32_t> top(kj.begin(), kj.begin() + qj);
        std::sort(top.begin(), top.end());
        Q = set_union(Q, top);
      }
    }
    std::vector<uint32_t> rest = set_minus(cand, Q);
    std::sort(rest.begin(), rest.end(), better);
    uint64_t fill_n = C - Q.size();
    std::vector<uint32_t> F(rest.begin(), rest.begin() + std::min<uint64_t>(fill_n, rest.size()));
    std::sort(F.begin(), F.end());
    Rn = set_union(Q, F);
  }

  // ---- Alg. 1 l.7-8: Omega, S+, S-
  std::vector<uint32_t> Om, Sp, Sm;
  if (g.tide) {
    Om = set_inter(c.R, Rn);
    Sp = set_minus(Rn, c.R);
    Sm = set_minus(c.R, Rn);
  } else {  // restage everything
    Sp = Rn;
    Sm = c.R;
  }

  // ---- slots (R13): S+ ascending -> lowest slots not holding R_t, then (if
  //      short) the slots S- releases, ascending.
  std::vector<int32_t> freelist;
  for (uint32_t s = 0; s < c.P; ++s)
    if (c.block_of[s] < 0) freelist.push_back((int32_t)s);
  if (freelist.size() < Sp.size()) {
    std::vector<int32_t> rel;
    for (uint32_t l : Sm) rel.push_back(c.slot_of[l]);
    std::sort(rel.begin(), rel.end());
    freelist.insert(freelist.end(), rel.begin(), rel.end());
  }

  c.phase_ns[1] += ns_since(t0);
  t0 = Clock::now();
  // ---- stage 4: evict S-, writing back dirty blocks
  const uint64_t rb = c.rec_bytes() * c.n_arr();
  c.evicted_dirty.clear();
  for (uint32_t l : Sm) {
    int32_t s = c.slot_of[l];
    if (c.dirty[s]) {
      if (c.sto.on) {
        // R27 (a): D2H into the block's CPU-cache entry, inserted dirty (PAPER.md:
        // 247-248); the entry exists (inclusion: every GPU-resident block is cached)
        CacheEntry& e = c.sto.cache.at(l);
        if (c.sto.data)
          std::memcpy(e.payload.data(), c.slot_data[s].data(),
                      sizeof(float) * c.n_arr() * c.rec_floats());
        e.dirty = true;
      } else if (c.is_tracked(l)) {
        std::vector<float>& h = c.host_rec(l);
        std::vector<float>& d = c.slot_data[s];
        std::memcpy(h.data(), d.data(), sizeof(float) * c.n_arr() * c.rec_floats());
      }
      c.st.d2h_bytes += rb;
      c.st.n_evict_dirty += 1;
      c.evicted_dirty.push_back(l);
      c.dirty[s] = 0;
    }
    // optimizer state is discarded with the slot in cold mode
    c.slot_data.erase(s);
    c.block_of[s] = -1;
    c.slot_of[l] = -1;
    c.evicted_once[l] = 1;
    c.st.resident_streak_sum += (uint64_t)(c.t - c.admit_iter[l]);
    c.st.streak_count += 1;
  }

  // ---- stage 2: materialise S+ (PAPER.md:150, 259); cold restart
  for (size_t i = 0; i < Sp.size(); ++i) {
    uint32_t l = Sp[i];
    int32_t s = freelist[i];
    c.slot_of[l] = s;
    c.block_of[s] = l;
    c.dirty[s] = 0;
    if (c.ever_resident[l]) c.st.readmissions += 1;
    c.ever_resident[l] = 1;
    c.admit_iter[l] = c.t;
    if (g.moments == OR_COLD_RESTART) c.step[l] = 0;
    if (c.sto.on) {
      // R27 (b): H2D from the block's CPU-cache entry, loaded from SSD on a miss
      CacheEntry& e = cache_access(c, l, c.R, Rn);
      if (c.sto.data) {
        std::vector<float> d(3 * c.rec_floats(), 0.0f);
        std::memcpy(d.data(), e.payload.data(), sizeof(float) * c.n_arr() * c.rec_floats());
        c.slot_data[s] = std::move(d);
      }
    } else if (c.is_tracked(l)) {
      std::vector<float>& h = c.host_rec(l);
      std::vector<float> d(3 * c.rec_floats(), 0.0f);
      std::memcpy(d.data(), h.data(), sizeof(float) * c.n_arr() * c.rec_floats());
      c.slot_data[s] = std::move(d);
    }
  }
  c.st.h2d_bytes += (uint64_t)Sp.size() * rb;
  // R27 (c): the blocks that left the GPU are accesses of the CPU cache too
  // ("The LRU policy is updated on each access"): touched in
  // ascending id after the S+ accesses; clean ones move no bytes (their entry
  // already holds the version the GPU had).
  if (c.sto.on)
    for (uint32_t l : Sm) c.sto.cache.at(l).stamp = ++c.sto.clock;

  // ---- bookkeeping
  c.Kset = Kn;
  c.Rnew = Rn;
  c.Splus = Sp;
  c.Sminus = Sm;
  c.Omega = Om;
  c.R = Rn;
  c.A = set_inter(Rn, Kn);
  c.A_prev = c.A;
  c.phase_ns[2] += ns_since(t0);
  c.st.iter += 1;
  c.st.n_visible += Kn.size();
  c.st.n_resident += Rn.size();
  c.st.n_active_blocks += c.A.size();
  c.st.n_stage_in += Sp.size();
  c.st.n_evict += Sm.size();
  c.t += 1;
  c.can_step = true;
  return OR_OK;
}

int or_step_adam(or_ctx* o, const float* lr, float beta1, float beta2, float eps,
                 or_grad_fn grad, void* grad_user, or_mask_fn mask, void* mask_user) {
  Ctx& c = o->c;
  const or_config& g = c.cfg;
  if (!c.can_step) return OR_ESTATE;
  if (!lr) return OR_EINVAL;
  c.can_step = false;
  struct PhaseTimer {  // Adam's share of the step (every return path)
    uint64_t& acc;
    Clock::time_point a = Clock::now();
    ~PhaseTimer() { acc += ns_since(a); }
  } timer{c.phase_ns[3]};
  const uint32_t B = g.block_size;
  const uint32_t nw = (B + 31) / 32;
  const uint64_t it = (uint64_t)(c.t - 1);  // iteration index of this batch
  const float omb1 = 1.0f - beta1, omb2 = 1.0f - beta2;
  std::vector<uint32_t> words(nw);
  std::vector<float> G((size_t)B * D);
  for (uint32_t l : c.A) {  // blocks in R n K, ascending
    const int32_t s = c.slot_of[l];
    const uint32_t nrows = c.rows(l);
    const uint64_t kg = c.gid_block(l);
    if (mask)
      mask(mask_user, kg, it, words.data());
    else
      std::fill(words.begin(), words.end(), 0xFFFFFFFFu);
    std::vector<char> active(B, 0);
    uint32_t n_act = 0;
    for (uint32_t r = 0; r < nrows; ++r)
      if ((words[r / 32] >> (r % 32)) & 1u) active[r] = 1, ++n_act;
    if (n_act == 0) continue;  // no row of I_t in this block: untouched, not dirty
    const uint32_t before = c.step[l];
    c.step[l] = before + 1;    // R7: per-block step counter
    c.dirty[s] = 1;            // PAPER.md:293 "marked dirty"
    c.st.total_updates += 1;
    c.st.n_active_rows += n_act;
    if (g.moments == OR_COLD_RESTART && before == 0 && c.evicted_once[l])
      c.st.cold_restart_updates += 1;
    if (!c.is_tracked(l)) continue;
    grad(grad_user, kg, it, G.data());
    // bias corrections 1 - beta^s, evaluated in double and rounded (R9)
    const double sd = (double)c.step[l];
    const float bc1 = (float)(1.0 - std::pow((double)beta1, sd));
    const float bc2 = (float)(1.0 - std::pow((double)beta2, sd));
    const float ibs = 1.0f / std::sqrt(bc2);
    std::vector<float>& d = c.slot_data[s];
    float* th = d.data();
    float* m = th + c.rec_floats();
    float* v = m + c.rec_floats();
    for (uint32_t r = 0; r < nrows; ++r) {
      if (!active[r]) continue;  // Eq. masked_update: theta unchanged off I_t
      bool finite = true;
      for (uint32_t a = 0; a < D; ++a)
        if (!std::isfinite(G[(size_t)r * D + a])) {
          uint64_t idx = (kg * B + r) * D + a;
          if (idx < c.nonfinite) c.nonfinite = idx;
          finite = false;
        }
      if (!finite) continue;  // R20: the row is skipped and reported
      for (uint32_t a = 0; a < D; ++a) {
        const size_t e = (size_t)r * D + a;
        const float gr = G[e];
        // Adam (Eq. masked_update u_t with first/second moments)
        float mt = beta1 * m[e];
        mt = mt + omb1 * gr;
        float g2 = gr * gr;
        float vt = beta2 * v[e];
        vt = vt + omb2 * g2;
        m[e] = mt;
        v[e] = vt;
        float den = std::sqrt(vt) * ibs;
        den = den + eps;
        float ss = lr[a] / bc1;
        float upd = mt / den;
        th[e] = th[e] - ss * upd;
      }
    }
    if (g.refresh_bounds) {  // R25: radius holding every row after the update
      std::vector<float>& pd = c.pend[it & 1];
      if (pd.empty()) pd.assign(c.Kloc, 0.0f);
      const float* bd = &c.bounds[4 * l];
      for (uint32_t r = 0; r < nrows; ++r) {
        const float rad = refresh_radius(th + (size_t)r * D, bd);
        if (fbits(rad) > fbits(pd[l])) pd[l] = rad;  // max on the bit pattern (R25)
      }
    }
  }
  return c.nonfinite != std::numeric_limits<uint64_t>::max() ? OR_ENONFINITE : OR_OK;
}

int or_flush(or_ctx* o) {
  Ctx& c = o->c;
  const uint64_t rb = c.rec_bytes() * c.n_arr();
  for (uint32_t l : c.R) {  // consistency barrier: write back dirty residents
    int32_t s = c.slot_of[l];
    if (!c.dirty[s]) continue;
    if (c.sto.on) {
      CacheEntry& e = c.sto.cache.at(l);
      if (c.sto.data)
        std::memcpy(e.payload.data(), c.slot_data[s].data(),
                    sizeof(float) * c.n_arr() * c.rec_floats());
      e.dirty = true;
    } else if (c.is_tracked(l)) {
      std::vector<float>& h = c.host_rec(l);
      std::memcpy(h.data(), c.slot_data[s].data(), sizeof(float) * c.n_arr() * c.rec_floats());
    }
    c.dirty[s] = 0;
    c.st.flush_bytes += rb;
    c.st.n_flush_blocks += 1;
  }
  // f3: "Dirty blocks are flushed to SSD patch segments ... at explicit
  // consistency barriers such as checkpointing and shutdown":
  // every dirty CPU-cache entry is appended, ascending id, and becomes clean;
  // the cache keeps its contents and LRU order.
  if (c.sto.on) {
    for (auto& kv : c.sto.cache)
      if (kv.second.dirty) {
        append_version(c, kv.first, kv.second);
        kv.second.dirty = false;
        c.sto.flush_appends += 1;
      }
    if (c.sto.data) write_manifest(c);  // R30: the durable end of the log
  }
  c.can_step = false;
  return OR_OK;
}

uint32_t or_get_list(or_ctx* o, int which, uint32_t* blocks, int32_t* slots, uint32_t cap) {
  Ctx& c = o->c;
  const std::vector<uint32_t>* v = nullptr;
  switch (which) {
    case 0: v = &c.Kset; break;
    case 1: v = &c.Rnew; break;
    case 2: v = &c.Splus; break;
    case 3: v = &c.Sminus; break;
    case 4: v = &c.Omega; break;
    case 5: v = &c.A; break;
    default: return 0;
  }
  uint32_t n = (uint32_t)v->size();
  for (uint32_t i = 0; i < n && i < cap; ++i) {
    uint32_t l = (*v)[i];
    if (blocks) blocks[i] = (uint32_t)c.gid_block(l);
    if (slots) slots[i] = (which == 3) ? -1 : c.slot_of[l];
  }
  return n;
}

uint32_t or_get_percam(or_ctx* o, uint32_t j, uint32_t* blocks, uint32_t cap) {
  Ctx& c = o->c;
  if (j >= c.percam.size()) return 0;
  uint32_t n = (uint32_t)c.percam[j].size();
  for (uint32_t i = 0; i < n && i < cap; ++i) blocks[i] = (uint32_t)c.gid_block(c.percam[j][i]);
  return n;
}

uint32_t or_get_evicted_dirty(or_ctx* o, uint32_t* blocks, uint32_t cap) {
  Ctx& c = o->c;
  uint32_t n = (uint32_t)c.evicted_dirty.size();
  for (uint32_t i = 0; i < n && i < cap; ++i) blocks[i] = (uint32_t)c.gid_block(c.evicted_dirty[i]);
  return n;
}

void or_get_slot_map(or_ctx* o, int64_t* out) {
  Ctx& c = o->c;
  for (uint32_t s = 0; s < c.P; ++s)
    out[s] = c.block_of[s] < 0 ? -1 : (int64_t)c.gid_block((uint32_t)c.block_of[s]);
}

void or_get_stats(or_ctx* o, or_stats* s) { *s = o->c.st; }
uint64_t or_nonfinite_index(or_ctx* o) { return o->c.nonfinite; }
uint32_t or_num_local_blocks(or_ctx* o) { return o->c.Kloc; }

float or_exp_det(float x) { return exp_det(x); }

// ---- NEXT f2b: Morton sort + blocking ("we Morton-sort
// Gaussians by the codes of their centers before blocking", 375-376; SPEC.md:
// 81-145, readings R26).  Step by step:
//  1. quantisation box = AABB of all centres; per axis q = min(2^21-1,
//     floor(((double)p - lo) * (2^21-1) / (hi - lo))) (0 if hi == lo)
//  2. code = bit-interleave of q, x lowest (bit 3i = x_i, 3i+1 = y_i, 3i+2 = z_i)
//  3. stable sort by code (ties keep the original index order)
//  4. block k = sorted positions [kB, min(N, (k+1)B))
//  5. c_k = centroid of its centres, summed in double in sorted order, rounded
//     to fp32; r_k = max_i (|mu_i - c_k| in double + 3 * exp_det(max log-scale_i))
//     rounded up to fp32 (conservative)
uint64_t or_morton3(uint32_t x, uint32_t y, uint32_t z) {
  uint64_t c = 0;
  for (int b = 0; b < 21; ++b) {
    c |= (uint64_t)((x >> b) & 1u) << (3 * b);
    c |= (uint64_t)((y >> b) & 1u) << (3 * b + 1);
    c |= (uint64_t)((z >> b) & 1u) << (3 * b + 2);
  }
  return c;
}

int or_build_layout(const float* cs /* n x 4 */, uint64_t n, uint32_t B, uint64_t* perm,
                    float* bounds /* ceil(n/B) x 4 */) {
  if (!cs || n == 0 || B == 0 || !perm || !bounds) return OR_EINVAL;
  float lo[3], hi[3];
  for (int a = 0; a < 3; ++a) lo[a] = hi[a] = cs[a];
  for (uint64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const float v = cs[4 * i + a];
      if (!std::isfinite(v)) return OR_EINVAL;
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  const double qmax = 2097151.0;  // 2^21 - 1
  double inv[3];
  for (int a = 0; a < 3; ++a)
    inv[a] = hi[a] > lo[a] ? qmax / ((double)hi[a] - (double)lo[a]) : 0.0;
  std::vector<std::pair<uint64_t, uint64_t>> key(n);
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
      double t = std::floor(((double)cs[4 * i + a] - (double)lo[a]) * inv[a]);
      if (t > qmax) t = qmax;
      if (t < 0.0) t = 0.0;
      q[a] = (uint32_t)t;
    }
    key[i] = {or_morton3(q[0], q[1], q[2]), i};
  }
  std::stable_sort(key.begin(), key.end(),
                   [](const std::pair<uint64_t, uint64_t>& a,
                      const std::pair<uint64_t, uint64_t>& b) { return a.first < b.first; });
  for (uint64_t i = 0; i < n; ++i) perm[i] = key[i].second;
  const uint64_t K = (n + B - 1) / B;
  for (uint64_t k = 0; k < K; ++k) {
    const uint64_t a0 = k * B, a1 = std::min<uint64_t>(n, a0 + B);
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (uint64_t p = a0; p < a1; ++p) {
      const float* r = cs + 4 * perm[p];
      sx += (double)r[0];
      sy += (double)r[1];
      sz += (double)r[2];
    }
    const double cnt = (double)(a1 - a0);
    const float cx = (float)(sx / cnt), cy = (float)(sy / cnt), cz = (float)(sz / cnt);
    double rad = 0.0;
    for (uint64_t p = a0; p < a1; ++p) {
      const float* r = cs + 4 * perm[p];
      const double dx = (double)r[0] - (double)cx, dy = (double)r[1] - (double)cy,
                   dz = (double)r[2] - (double)cz;
      const double dist = std::sqrt(dx * dx + dy * dy + dz * dz);
      const double e = dist + (double)(3.0f * exp_det(r[3]));
      if (e > rad) rad = e;
    }
    float rf = (float)rad;
    if ((double)rf < rad) rf = std::nextafterf(rf, INFINITY);
    bounds[4 * k] = cx;
    bounds[4 * k + 1] = cy;
    bounds[4 * k + 2] = cz;
    bounds[4 * k + 3] = rf;
  }
  return OR_OK;
}

int or_get_bound(or_ctx* o, uint64_t kg, float* out4) {
  Ctx& c = o->c;
  if (kg % c.cfg.world_size != (uint64_t)c.cfg.rank) return OR_EINVAL;
  const uint64_t l = kg / c.cfg.world_size;
  if (l >= c.Kloc) return OR_EINVAL;
  for (int i = 0; i < 4; ++i) out4[i] = c.bounds[4 * l + i];
  return OR_OK;
}

int or_fine_filter(or_ctx* o, uint64_t kg, uint32_t* words) {
  Ctx& c = o->c;
  if (kg % c.cfg.world_size != (uint64_t)c.cfg.rank) return OR_EINVAL;
  const uint64_t l = kg / c.cfg.world_size;
  const uint32_t nw = (c.cfg.block_size + 31) / 32;
  std::fill(words, words + nw, 0u);
  if (l >= c.Kloc || !contains(c.A, (uint32_t)l)) return OR_OK;  // I_t lies inside R n K
  if (!c.is_tracked((uint32_t)l)) return OR_EINVAL;
  const float* th = c.slot_data[c.slot_of[l]].data();
  const uint32_t nrows = c.rows((uint32_t)l);
  std::vector<uint32_t> cams;  // cameras whose K^(j) holds block l
  for (uint32_t j = 0; j < c.percam.size(); ++j)
    if (contains(c.percam[j], (uint32_t)l)) cams.push_back(j);
  for (uint32_t r = 0; r < nrows; ++r)
    if (gaussian_visible(th + (size_t)r * D, c.planes, cams)) words[r / 32] |= 1u << (r % 32);
  return OR_OK;
}

void or_fine_filter_cb(void* ctx, uint64_t kg, uint64_t /*t*/, uint32_t* words) {
  or_fine_filter((or_ctx*)ctx, kg, words);
}

uint32_t or_step_count(or_ctx* o, uint64_t kg) {
  Ctx& c = o->c;
  uint64_t l = kg / c.cfg.world_size;
  return l < c.Kloc ? c.step[l] : 0;
}

int or_read_block(or_ctx* o, uint64_t kg, float* theta, float* m, float* v) {
  Ctx& c = o->c;
  if (kg % c.cfg.world_size != (uint64_t)c.cfg.rank) return OR_EINVAL;
  uint64_t l = kg / c.cfg.world_size;
  if (l >= c.Kloc || !c.is_tracked((uint32_t)l)) return OR_EINVAL;
  const size_t n = c.rec_floats();
  const float* src;
  std::vector<float> zeros, stored;
  if (c.slot_of[l] >= 0) {
    src = c.slot_data[c.slot_of[l]].data();
  } else {
    if (c.sto.on) {  // f3: CPU-cache entry, else the newest version through Index[k]
      auto it = c.sto.cache.find((uint32_t)l);
      if (it != c.sto.cache.end()) {
        stored = it->second.payload;
      } else {
        const IndexEntry& ix = c.sto.index[l];
        stored.assign((size_t)c.n_arr() * n, 0.0f);
        read_at(seg_path(c.sto, ix.file_id), ix.offset, stored.data(), c.sto.payload);
      }
    }
    std::vector<float>& h = c.sto.on ? stored : c.host_rec((uint32_t)l);
    if (c.n_arr() == 3) {
      src = h.data();
    } else {  // cold restart: moments do not exist off-GPU
      zeros.assign(3 * n, 0.0f);
      std::memcpy(zeros.data(), h.data(), sizeof(float) * n);
      src = zeros.data();
    }
  }
  if (theta) std::memcpy(theta, src, sizeof(float) * n);
  if (m) std::memcpy(m, src + n, sizeof(float) * n);
  if (v) std::memcpy(v, src + 2 * n, sizeof(float) * n);
  return OR_OK;
}


// ---- NEXT f3: store tier (R27, R28)
int or_store_open(or_ctx* o, const char* dir, uint32_t cache_blocks, uint64_t segment_bytes) {
  Ctx& c = o->c;
  Store& s = c.sto;
  if (c.t != 0 || s.on) return OR_ESTATE;
  if (cache_blocks < 2ull * c.cfg.capacity) return OR_EINVAL;  // pinned entries < 2C (R27)
  bool any_tracked = c.track_all;
  for (char x : c.tracked) any_tracked = any_tracked || x;
  if ((dir != nullptr) != c.track_all) return OR_EINVAL;  // data mode <=> every block tracked
  if (!dir && any_tracked) return OR_EINVAL;
  s.payload = (uint64_t)c.n_arr() * c.rec_bytes();
  s.S = pad_page(s.payload);
  s.seg_budget = segment_bytes ? segment_bytes : (1ull << 30);
  if (s.seg_budget < 2 * kPage + s.S) return OR_EINVAL;
  s.on = true;
  s.data = dir != nullptr;
  s.H = cache_blocks;
  if (dir) {
    s.dir = dir;
    std::error_code ec;
    std::filesystem::create_directories(s.dir, ec);
  }
  // "The initial model is written once as an immutable base segment"
  // (PAPER.md:228): header page, then record l at 4096 + l * S, Index[l] =
  // (0, offset, size, 0).
  s.index.assign(c.Kloc, IndexEntry{});
  for (uint32_t l = 0; l < c.Kloc; ++l) s.index[l] = {0, kPage + (uint64_t)l * s.S, s.payload, 0};
  s.base_version.assign(c.Kloc, 0);
  if (s.data) {
    const std::string base = seg_path(s, 0);
    std::vector<unsigned char> h = segment_header(c, 0);
    write_at(base, 0, h.data(), kPage, true);
    std::vector<unsigned char> r(s.S, 0);
    std::vector<float> v((size_t)c.n_arr() * c.rec_floats());
    for (uint32_t l = 0; l < c.Kloc; ++l) {
      std::fill(v.begin(), v.end(), 0.0f);  // m = v = 0 (persist)
      if (c.fill) c.fill(c.fill_user, c.gid_block(l), v.data());
      std::memcpy(r.data(), v.data(), s.payload);
      write_at(base, kPage + (uint64_t)l * s.S, r.data(), s.S, false);
    }
    write_manifest(c);  // epoch 1: the base alone
  }
  return OR_OK;
}


// Checkpoint/resume of the store tier (reading R30): a new session over the
// files a barrier left.  SPEC.md log_store recover_index: scan the segments
// in file_id order, later records win; a truncated trailing record of the
// newest patch is dropped (the segment is cut back to the last whole record).
// Everything else starts afresh: an empty CPU cache, no resident block, step
// counters and recency at zero.
static uint64_t get64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
static uint32_t get32(const unsigned char* p) {
  uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

int or_store_reopen(or_ctx* o, const char* dir, uint32_t cache_blocks, uint64_t segment_bytes) {
  Ctx& c = o->c;
  Store& s = c.sto;
  if (c.t != 0 || s.on) return OR_ESTATE;
  if (!dir || !c.track_all || cache_blocks < 2ull * c.cfg.capacity) return OR_EINVAL;
  s.payload = (uint64_t)c.n_arr() * c.rec_bytes();
  s.S = pad_page(s.payload);
  s.seg_budget = segment_bytes ? segment_bytes : (1ull << 30);
  if (s.seg_budget < 2 * kPage + s.S) return OR_EINVAL;
  s.dir = dir;
  // the manifest of the last barrier: the durable end of the log, base
  // versions and step counters (R30); it must describe this shard and be intact
  const std::string mpath = s.dir + "/manifest.tdgm";
  std::error_code ec;
  const uint64_t msize = std::filesystem::file_size(mpath, ec);
  const uint64_t mwant = 64 + 12 * (uint64_t)c.Kloc + 4;
  if (ec || msize != mwant) return OR_EINVAL;
  std::vector<unsigned char> m(msize, 0);
  read_at(mpath, 0, m.data(), msize);
  if (std::memcmp(&m[0], "TDGM", 4) != 0 || get32(&m[4]) != 1 ||
      get32(&m[msize - 4]) != crc32c(m.data(), msize - 4) || get32(&m[32]) != c.n_arr() ||
      get64(&m[40]) != c.cfg.n_gaussians || get32(&m[48]) != c.cfg.block_size ||
      get32(&m[52]) != (uint32_t)c.cfg.world_size || get32(&m[56]) != (uint32_t)c.cfg.rank ||
      get32(&m[60]) != c.Kloc)
    return OR_EINVAL;
  const uint32_t last = get32(&m[16]);
  const uint64_t end = get64(&m[24]);
  // the base header must describe this shard
  std::vector<unsigned char> want = segment_header(c, 0), got(kPage, 0);
  read_at(seg_path(s, 0), 0, got.data(), kPage);
  if (got != want) return OR_EINVAL;
  s.index.assign(c.Kloc, IndexEntry{});
  s.base_version.assign(c.Kloc, 0);
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    s.base_version[l] = get64(&m[64 + 8 * (size_t)l]);
    s.index[l] = {0, kPage + (uint64_t)l * s.S, s.payload, s.base_version[l]};
  }
  // patch segments 1..last up to the durable end; every record there was made
  // durable at the barrier, so a bad one is corruption, not a torn tail
  const uint64_t rec = kPage + s.S;
  std::vector<unsigned char> payload(s.payload);
  for (uint32_t fid = 1; fid <= last; ++fid) {
    const std::string path = seg_path(s, fid);
    const uint64_t size = std::filesystem::file_size(path, ec);
    if (ec) return OR_EINVAL;
    std::vector<unsigned char> h(kPage, 0);
    read_at(path, 0, h.data(), kPage);
    if (h != segment_header(c, fid)) return OR_EINVAL;
    const uint64_t limit = fid == last ? end : size;
    if (limit > size || limit < kPage || (limit - kPage) % rec != 0) return OR_EINVAL;
    for (uint64_t off = kPage; off < limit; off += rec) {
      std::vector<unsigned char> r(kPage, 0);
      read_at(path, off, r.data(), kPage);
      const uint64_t gid = get64(&r[8]);
      if (std::memcmp(r.data(), "TREC", 4) != 0 || get32(&r[4]) != 2 ||
          get64(&r[24]) != s.payload || gid % c.cfg.world_size != (uint64_t)c.cfg.rank ||
          gid / c.cfg.world_size >= c.Kloc || get32(&r[36]) != crc32c(r.data(), 36))
        return OR_EINVAL;
      read_at(path, off + kPage, payload.data(), s.payload);
      if (get32(&r[32]) != crc32c(payload.data(), s.payload)) return OR_EINVAL;
      s.index[gid / c.cfg.world_size] = {fid, off + kPage, s.payload, get64(&r[16])};
    }
  }
  // appends after the barrier are not part of its state: cut and removed
  if (last) std::filesystem::resize_file(seg_path(s, last), end, ec);
  if (ec) return OR_EINVAL;
  for (uint32_t fid = last + 1; std::filesystem::exists(seg_path(s, fid), ec); ++fid)
    std::filesystem::remove(seg_path(s, fid), ec);
  for (uint32_t l = 0; l < c.Kloc; ++l) c.step[l] = get32(&m[64 + 8 * (size_t)c.Kloc + 4 * (size_t)l]);
  s.epoch = get64(&m[8]);
  s.cur_file = last;
  s.cur_size = last ? end : 0;
  s.segments = 0;
  s.on = true;
  s.data = true;
  s.H = cache_blocks;
  return OR_OK;
}


// Compaction ("Optional compaction can merge patch segments into
// a new base segment, but this is outside the training critical path";
// SPEC.md log_store compact; reading R31): at a barrier (the caller flushes
// first), a new base segment holds every block's newest version at the base
// offsets; it replaces the old base, the patch segments are removed, Index[k]
// becomes (0, base offset, size, version) -- versions keep counting -- and the
// next append opens patch segment 1 again.
int or_store_compact(or_ctx* o) {
  Ctx& c = o->c;
  Store& s = c.sto;
  if (!s.on || !s.data) return OR_EINVAL;
  for (const auto& kv : s.cache)
    if (kv.second.dirty) return OR_ESTATE;  // barrier first
  for (uint32_t l : c.R)
    if (c.dirty[c.slot_of[l]]) return OR_ESTATE;
  const std::string tmp = s.dir + "/base.tdgs.tmp";
  std::vector<unsigned char> h = segment_header(c, 0);
  write_at(tmp, 0, h.data(), kPage, true);
  std::vector<unsigned char> r(s.S, 0);
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    std::fill(r.begin(), r.end(), 0);
    const IndexEntry& ix = s.index[l];
    read_at(seg_path(s, ix.file_id), ix.offset, r.data(), s.payload);
    write_at(tmp, kPage + (uint64_t)l * s.S, r.data(), s.S, false);
  }
  std::error_code ec;
  std::filesystem::rename(tmp, seg_path(s, 0), ec);
  if (ec) return OR_EINVAL;
  const uint32_t old_last = s.cur_file;
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    s.index[l].file_id = 0;
    s.index[l].offset = kPage + (uint64_t)l * s.S;
    s.base_version[l] = s.index[l].version;
  }
  s.cur_file = 0;
  s.cur_size = 0;
  write_manifest(c);  // the base alone, with the versions it now holds
  for (uint32_t fid = 1; fid <= old_last; ++fid) std::filesystem::remove(seg_path(s, fid), ec);
  return OR_OK;
}

int or_store_index(or_ctx* o, uint64_t kg, uint64_t* out4) {
  Ctx& c = o->c;
  if (!c.sto.on || kg % c.cfg.world_size != (uint64_t)c.cfg.rank) return OR_EINVAL;
  const uint64_t l = kg / c.cfg.world_size;
  if (l >= c.Kloc) return OR_EINVAL;
  const IndexEntry& ix = c.sto.index[l];
  out4[0] = ix.file_id;
  out4[1] = ix.offset;
  out4[2] = ix.size;
  out4[3] = ix.version;
  return OR_OK;
}

/* hits, misses, evictions, dirty_evictions, flush_appends, read_bytes,
 * write_bytes, segments, cached blocks, dirty cached blocks */
int or_store_stats(or_ctx* o, uint64_t* out10) {
  const Store& s = o->c.sto;
  if (!s.on) return OR_EINVAL;
  uint64_t nd = 0;
  for (const auto& kv : s.cache) nd += kv.second.dirty ? 1 : 0;
  const uint64_t v[10] = {s.hits, s.misses, s.evictions, s.dirty_evictions, s.flush_appends,
                          s.read_bytes, s.write_bytes, s.segments, (uint64_t)s.cache.size(), nd};
  std::memcpy(out10, v, sizeof v);
  return OR_OK;
}

/* cached local->global ids in LRU order (least recent first) with dirty flags */
uint32_t or_store_lru(or_ctx* o, uint32_t* blocks, uint8_t* dirty, uint32_t cap) {
  const Store& s = o->c.sto;
  std::vector<std::pair<uint64_t, uint32_t>> v;
  for (const auto& kv : s.cache) v.push_back({kv.second.stamp, kv.first});
  std::sort(v.begin(), v.end());
  for (uint32_t i = 0; i < v.size() && i < cap; ++i) {
    if (blocks) blocks[i] = (uint32_t)o->c.gid_block(v[i].second);
    if (dirty) dirty[i] = s.cache.at(v[i].second).dirty ? 1 : 0;
  }
  return (uint32_t)v.size();
}


// ---- NEXT f4: clustered-TSP view ordering ("We use a clustered
// TSP-ordered (no-shuffle) camera sequence", 709-712 "applying a clustered
// traveling-salesperson (TSP) ordering over camera poses"
// order_views).  Reading R29, step by step (all arithmetic in double, no FMA):
//  d2(a, b) = sum over the D feature coordinates, in order, of (a_i - b_i)^2
//  1. k = ceil(sqrt(M)) (smallest k with k*k >= M)
//  2. maximin initialisation: centre 0 = the lexicographically smallest view
//     (features compared in order, then index); centre j = the view maximising
//     the min d2 to the centres so far (ties: lowest index)
//  3. Lloyd iterations (at most 100): assign every view to the nearest centre
//     (ties: lowest centre); stop when no assignment changed; otherwise every
//     non-empty cluster's centre becomes the mean of its members (summed in
//     ascending view index, then divided by the count)
//  4. cluster tour: nearest-neighbour over the non-empty clusters' centres,
//     starting at the cluster of the lexicographically smallest view (ties:
//     lowest cluster)
//  5. tour inside each cluster: nearest-neighbour over its members, starting
//     at the lexicographically smallest view (first cluster) or at the member
//     nearest to the preceding cluster's centre (ties: lowest index)
//  6. pi = the concatenation, cluster by cluster in tour order
static double d2(const double* a, const double* b, uint32_t D) {
  double s = 0.0;
  for (uint32_t i = 0; i < D; ++i) {
    const double t = a[i] - b[i];
    s = s + t * t;
  }
  return s;
}

static bool lex_less(const double* f, uint32_t D, uint32_t a, uint32_t b) {
  for (uint32_t i = 0; i < D; ++i) {
    if (f[(size_t)a * D + i] < f[(size_t)b * D + i]) return true;
    if (f[(size_t)a * D + i] > f[(size_t)b * D + i]) return false;
  }
  return a < b;
}

int or_order_views(const double* feat, uint32_t M, uint32_t D, uint32_t* perm,
                   uint32_t* cluster_out, uint32_t* k_out, uint32_t* iters_out) {
  if (!feat || !perm || M == 0 || D == 0 || D > 8) return OR_EINVAL;
  for (size_t i = 0; i < (size_t)M * D; ++i)
    if (!std::isfinite(feat[i])) return OR_EINVAL;
  uint32_t k = 1;
  while ((uint64_t)k * k < M) ++k;  // step 1
  uint32_t v0 = 0;
  for (uint32_t i = 1; i < M; ++i)
    if (lex_less(feat, D, i, v0)) v0 = i;
  // step 2
  std::vector<double> cen((size_t)k * D);
  std::vector<double> mind(M);
  for (uint32_t i = 0; i < D; ++i) cen[i] = feat[(size_t)v0 * D + i];
  for (uint32_t v = 0; v < M; ++v) mind[v] = d2(feat + (size_t)v * D, cen.data(), D);
  for (uint32_t j = 1; j < k; ++j) {
    uint32_t best = 0;
    for (uint32_t v = 1; v < M; ++v)
      if (mind[v] > mind[best]) best = v;
    for (uint32_t i = 0; i < D; ++i) cen[(size_t)j * D + i] = feat[(size_t)best * D + i];
    for (uint32_t v = 0; v < M; ++v) {
      const double e = d2(feat + (size_t)v * D, cen.data() + (size_t)j * D, D);
      if (e < mind[v]) mind[v] = e;
    }
  }
  // step 3
  std::vector<uint32_t> asg(M, UINT32_MAX);
  uint32_t it = 0;
  for (; it < 100; ++it) {
    bool changed = false;
    for (uint32_t v = 0; v < M; ++v) {
      uint32_t bj = 0;
      double bd = d2(feat + (size_t)v * D, cen.data(), D);
      for (uint32_t j = 1; j < k; ++j) {
        const double e = d2(feat + (size_t)v * D, cen.data() + (size_t)j * D, D);
        if (e < bd) bd = e, bj = j;
      }
      if (asg[v] != bj) changed = true;
      asg[v] = bj;
    }
    if (!changed) break;
    std::vector<double> sum((size_t)k * D, 0.0);
    std::vector<uint32_t> cnt(k, 0);
    for (uint32_t v = 0; v < M; ++v) {
      for (uint32_t i = 0; i < D; ++i) sum[(size_t)asg[v] * D + i] += feat[(size_t)v * D + i];
      cnt[asg[v]] += 1;
    }
    for (uint32_t j = 0; j < k; ++j)
      if (cnt[j])
        for (uint32_t i = 0; i < D; ++i) cen[(size_t)j * D + i] = sum[(size_t)j * D + i] / (double)cnt[j];
  }
  // step 4
  std::vector<std::vector<uint32_t>> mem(k);
  for (uint32_t v = 0; v < M; ++v) mem[asg[v]].push_back(v);
  std::vector<char> done(k, 0);
  for (uint32_t j = 0; j < k; ++j) done[j] = mem[j].empty();
  std::vector<uint32_t> tour{asg[v0]};
  done[asg[v0]] = 1;
  for (;;) {
    const uint32_t cur = tour.back();
    uint32_t best = UINT32_MAX;
    double bd = 0.0;
    for (uint32_t j = 0; j < k; ++j) {
      if (done[j]) continue;
      const double e = d2(cen.data() + (size_t)cur * D, cen.data() + (size_t)j * D, D);
      if (best == UINT32_MAX || e < bd) bd = e, best = j;
    }
    if (best == UINT32_MAX) break;
    done[best] = 1;
    tour.push_back(best);
  }
  // steps 5-6
  uint32_t n = 0;
  for (size_t ci = 0; ci < tour.size(); ++ci) {
    const std::vector<uint32_t>& ms = mem[tour[ci]];
    std::vector<char> used(ms.size(), 0);
    size_t cur = 0;
    if (ci == 0) {
      while (ms[cur] != v0) ++cur;
    } else {
      const double* pc = cen.data() + (size_t)tour[ci - 1] * D;
      double bd = d2(feat + (size_t)ms[0] * D, pc, D);
      for (size_t m = 1; m < ms.size(); ++m) {
        const double e = d2(feat + (size_t)ms[m] * D, pc, D);
        if (e < bd) bd = e, cur = m;
      }
    }
    for (size_t step = 0; step < ms.size(); ++step) {
      used[cur] = 1;
      perm[n++] = ms[cur];
      size_t nb = SIZE_MAX;
      double bd = 0.0;
      for (size_t m = 0; m < ms.size(); ++m) {
        if (used[m]) continue;
        const double e = d2(feat + (size_t)ms[m] * D, feat + (size_t)ms[cur] * D, D);
        if (nb == SIZE_MAX || e < bd) bd = e, nb = m;
      }
      if (nb == SIZE_MAX) break;
      cur = nb;
    }
  }
  if (cluster_out)
    for (uint32_t v = 0; v < M; ++v) cluster_out[v] = asg[v];
  if (k_out) *k_out = k;
  if (iters_out) *iters_out = it;
  return OR_OK;
}

}  // extern "C"

extern "C" void or_phase_ns(or_ctx* o, uint64_t* out4) {
  for (int i = 0; i < 4; ++i) out4[i] = o->c.phase_ns[i];
}

// Timing aid for bench.py's cpu_baseline (never used by a parity check): from
// now on every block is tracked.  Resident blocks that were not tracked get
// their slot record from the host tier's initial rows (their updates so far
// were not computed), so the contents are not the method's; the work per step
// is.  Not allowed on a store tier.
extern "C" int or_track_all_from_now(or_ctx* o) {
  Ctx& c = o->c;
  if (c.sto.on) return OR_ESTATE;
  for (uint32_t l = 0; l < c.Kloc; ++l) {
    const int32_t s = c.slot_of[l];
    if (s < 0 || c.is_tracked(l)) continue;
    std::vector<float>& h = c.host_rec(l);
    std::vector<float> d(3 * c.rec_floats(), 0.0f);
    std::memcpy(d.data(), h.data(), sizeof(float) * c.n_arr() * c.rec_floats());
    c.slot_data[s] = std::move(d);
  }
  c.track_all = true;
  return OR_OK;
}

extern "C" uint32_t or_crc32c(const void* data, uint64_t n) { return crc32c(data, n); }
