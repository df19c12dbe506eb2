// Native device-cache table (cache.py:42-109 + the gather loop of
// trainer.py:329-345 / cli._gather cli.py:111-136).
//
// Host-side decision logic identical to the reference (ratio band, LRU,
// byte budget counted as prefix_len·92, replacement returns the old dirty
// block, flush every flush_interval iterations) over cache blocks that live
// in HBM.  Blocks are packed f64 attribute blocks allocated stream-ordered
// (from a private pool) and released stream-ordered after their write-back, so
// a whole step's cache work is one C call: decisions, then one batch of
// zero-copy store transfers (loads on the main stream, write-backs on a
// side stream).
#include <stdint.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <list>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "../../include/glod_b200.h"
#include "common.cuh"

namespace glod {

cudaError_t launch_store_xfer(const glod_store_view& sv, const glod_prefix_item* items, int n_items,
                              long long total, int load, cudaStream_t st);
long long transfer_chunks(long long rows);
cudaError_t launch_materialize(const glod_mat_item* items, int n_items, long long total, const double* master,
                               long long cap, long long mstride, const int* rec_node, cudaStream_t st);
cudaError_t launch_load_blocks(const glod_store_view& sv, const glod_prefix_item* items, const int2* bmap,
                               long long nblocks, const glod_master_ref& mref, cudaStream_t st);
cudaError_t launch_pack_blocks(const glod_prefix_item* items, const int2* bmap, long long nblocks, float* out,
                               int interleaved, const glod_master_ref& mref, cudaStream_t st);

namespace {

constexpr int kFloats = 23;
constexpr int kSecOffH[7] = {0, 3, 6, 10, 11, 14, 23};

struct Entry {
  int32_t spt_id;
  double cached_distance;
  int64_t prefix_len;
  double* block;
  int64_t nbytes;
  bool dirty;
};

// A device region sub-allocated on the host (best fit, coalescing free
// list).  Frees take effect at host time, which is safe because every
// device user of an arena is ordered on one stream (blocks: the main
// stream; prefetch buffers: see CacheTable) — it replaces hundreds of
// cudaMallocFromPoolAsync/cudaFreeAsync driver calls per step that sat on
// the step's critical path while the GPU waited for the cache decisions.
class Arena {
 public:
  ~Arena() {
    if (base_) cudaFree(base_);
  }
  cudaError_t init(size_t bytes) {
    bytes = (bytes + kAlign - 1) / kAlign * kAlign;
    cudaError_t e = cudaMalloc(&base_, bytes);
    if (e != cudaSuccess) {
      base_ = nullptr;
      return e;
    }
    cap_ = bytes;
    put(0, bytes);
    return cudaSuccess;
  }
  bool ready() const { return base_ != nullptr; }
  void* alloc(size_t bytes) {
    if (!base_) return nullptr;
    bytes = bytes ? (bytes + kAlign - 1) / kAlign * kAlign : kAlign;
    auto it = by_size_.lower_bound({bytes, 0});
    if (it == by_size_.end()) return nullptr;
    const size_t off = it->second, sz = it->first;
    take(off, sz);
    if (sz > bytes) put(off + bytes, sz - bytes);
    live_[off] = bytes;
    return base_ + off;
  }
  bool release(void* p) {
    char* c = static_cast<char*>(p);
    if (!base_ || c < base_ || c >= base_ + cap_) return false;
    const size_t off = size_t(c - base_);
    auto lv = live_.find(off);
    if (lv == live_.end()) return false;
    size_t o = off, sz = lv->second;
    live_.erase(lv);
    auto nx = free_.lower_bound(o);
    if (nx != free_.end() && nx->first == o + sz) {
      sz += nx->second;
      take(nx->first, nx->second);
    }
    auto pv = free_.lower_bound(o);
    if (pv != free_.begin()) {
      --pv;
      if (pv->first + pv->second == o) {
        o = pv->first;
        sz += pv->second;
        take(pv->first, pv->second);
      }
    }
    put(o, sz);
    return true;
  }

 private:
  static constexpr size_t kAlign = 256;
  void put(size_t off, size_t sz) {
    free_[off] = sz;
    by_size_.insert({sz, off});
  }
  void take(size_t off, size_t sz) {
    free_.erase(off);
    by_size_.erase({sz, off});
  }
  char* base_ = nullptr;
  size_t cap_ = 0;
  std::map<size_t, size_t> free_;                 // offset -> size
  std::set<std::pair<size_t, size_t>> by_size_;   // (size, offset)
  std::unordered_map<size_t, size_t> live_;       // offset -> size
};

}  // namespace

struct CacheTable {
  // implicit refresh (glod_cache_set_master): the master rows and each
  // SPT's record node ids, to materialise touched rows before write-back
  const double* m_master = nullptr;
  int64_t m_cap = 0, m_stride = 0;
  const int32_t* m_rec_node = nullptr;
  std::vector<int64_t> m_rec_off;         // per spt_id
  std::vector<glod_mat_item> m_items;
  int64_t budget;
  double d_min, d_max;
  int64_t flush_interval;
  int32_t bytes_per_row;
  std::vector<int64_t> slot_start;        // per spt_id
  std::list<Entry> lru;                   // front = least recently used
  std::unordered_map<int32_t, std::list<Entry>::iterator> map;
  int64_t resident = 0, hits = 0, misses = 0, loaded_rows = 0;
  // transfer staging: one pinned host item table, rewritten once its last
  // H2D copy (event items_done) has run
  glod_prefix_item* h_items = nullptr;   // items, then the int2 block map
  size_t items_cap = 0;                   // bytes
  cudaEvent_t items_done = nullptr;
  std::vector<int32_t> step_ids;          // SPTs rendered this step (dirty at end)
  std::vector<double*> to_free;           // blocks dropped this step
  int device = 0;
  bool ready = false;

  // Memory.  Blocks and item tables: `blocks` arena (every user on the main
  // stream), falling back to a private stream-ordered pool when full.
  // Prefetch buffers: `pfmem` arena; their users are the prefetch stream
  // (DMA in) and one load kernel on the main stream, after which ev_pf_free
  // is recorded and the next prefetch DMA waits for it.
  Arena blocks, pfmem;
  cudaMemPool_t pool = nullptr;

  // Write-back: the blocks are packed to f32 on the main stream inside the
  // step (so a replaced dirty entry is written back after its stale reload,
  // and every written-back block is read before this step's ADAM refresh
  // rewrites it — the reference writes back at eviction); the copy engines
  // then move the f32 rows into the pinned store on the side stream (one
  // cudaMemcpyAsync per block for an interleaved store: the staging copy is
  // in row order).  The copies are issued at end_step, when the step's
  // kernels are queued and the host is idle.  Two persistent
  // f32 staging buffers used alternately; the main stream reuses one only
  // after the side stream's copies out of it (ev_stage).  The main stream
  // waits for write-backs only when a load reads store rows a not yet
  // finished write-back of an earlier step writes (wb_prev); a block
  // evicted and re-requested within one step is reloaded from the evicted
  // block itself (overlay).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_wb = nullptr;
  std::unordered_map<int32_t, int> wb_prev;   // SPT ids with write-backs in flight
  float* stage[2] = {nullptr, nullptr};
  size_t stage_cap[2] = {0, 0};
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_packed[2] = {nullptr, nullptr};
  int stage_next = 0;
  struct PendingWb {
    int sb = -1;
    std::vector<void*> dst, src;
    std::vector<size_t> size;
    std::vector<int32_t> sids;
  };
  std::vector<PendingWb> pending;
  float* dsec[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool interleaved = false;

  // Disk mode (the reference's FileBacking, store.py:
  // 84-112): the store stays in the .glod file.  Reads of SPT prefixes are
  // pread()s of the 6 section ranges into pinned bounce buffers followed by
  // one H2D copy (cold misses: on the main stream before the load kernel;
  // prefetches: on the prefetch stream, issued while the GPU computes the
  // current step); write-backs are D2H copies into a pinned bounce buffer
  // and pwrite()s, completed before the next read of the file, so every
  // read sees every earlier write-back exactly as the reference's
  // synchronous write_back.
  struct DiskPiece {
    int64_t file_off;
    size_t buf_off, bytes;
  };
  struct DiskIO {
    int fd = -1;
    int64_t off[6] = {0, 0, 0, 0, 0, 0};      // byte offset of section k in the file
    float* rd = nullptr;                       // pinned: cold-miss reads
    size_t rd_cap = 0;
    float* pfb = nullptr;                      // pinned: prefetch reads
    size_t pfb_cap = 0;
    char* wbb = nullptr;                       // pinned: write-back bytes awaiting pwrite
    size_t wbb_cap = 0, wbb_used = 0;
    float* dtmp = nullptr;                     // device f32 copies of cold misses
    size_t dtmp_cap = 0;
    cudaEvent_t rd_done = nullptr, pf_done = nullptr, wb_done = nullptr;
    std::vector<DiskPiece> writes;
    int64_t bytes_read = 0, bytes_written = 0;
  } disk;
  bool disk_mode() const { return disk.fd >= 0; }

  // Prefetch (glod_cache_prefetch): the predicted misses of the next view
  // are copied store → f32 HBM buffers by the copy engines on `pf_st`
  // while the current step computes; the next cache_step converts a
  // prefetched prefix from HBM instead of reading it over PCIe.  A prefetch
  // lives for one step and is used only when its prefix length matches and
  // no write-back of its store rows was ordered after it.
  struct Prefetch {
    int64_t rows;
    float* buf;
  };
  std::unordered_map<int32_t, Prefetch> pf;
  cudaStream_t pf_st = nullptr;
  cudaEvent_t ev_pf = nullptr, ev_pf_free = nullptr;
  int64_t pf_issued_rows = 0, pf_used_rows = 0;
  int64_t pool_allocs = 0, grow_events = 0;     // arena misses, staging re-allocations
  int64_t host_ns_step = 0, host_ns_prefetch = 0, pf_copies = 0;
  // host ns per cache_step phase: [0] checks + decisions, [1] disk reads,
  // [2] materialize, [3] loads (tables + kernels), [4] write-back staging,
  // [5] release of the step's prefetches (glod_cache_debug_profile)
  int64_t prof_ns[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  cudaError_t init(const glod_store_view& sv) {
    if (ready) return cudaSuccess;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaError_t e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    unsigned long long thr = ~0ull;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (e != cudaSuccess) return e;
    for (int k = 0; k < 2; ++k) {
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_stage[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_packed[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_wb, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&items_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pf_st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_pf, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_pf_free, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    if (disk_mode()) {
      for (cudaEvent_t* ev : {&disk.rd_done, &disk.pf_done, &disk.wb_done})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    // store addresses for the copy engines (UVA: the mapped pinned pages
    // or, for a device-resident store, HBM); interleaved: one row per slot
    interleaved = !disk_mode() && sv.row_stride != 0;
    for (int k = 0; k < 6 && !disk_mode(); ++k) dsec[k] = const_cast<float*>(sv.section[k]);
    // Arenas sized from the budget (counted in f32 store bytes): resident
    // f64 blocks ≤ 2·budget, blocks dropped within a step ≤ 2·budget more;
    // prefetch copies ≤ budget.  Capped by free HBM; a failed reservation
    // just leaves the pool path.
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t want_blocks = size_t(4) * size_t(budget) + (size_t(64) << 20);
    const size_t want_pf = size_t(budget) + (size_t(16) << 20);
    if (want_blocks + want_pf < fr / 2) {
      if (blocks.init(want_blocks) != cudaSuccess || pfmem.init(want_pf) != cudaSuccess) cudaGetLastError();
      // write-back staging: a batch is at most the resident set (budget
      // bytes of f32) plus the step's replacements; reserve it up front
      // (a re-allocation synchronises the device)
      for (int k = 0; k < 2; ++k) {
        const size_t want = size_t(budget) + size_t(budget) / 2;
        if (cudaMalloc(&stage[k], want) == cudaSuccess) stage_cap[k] = want;
        else { stage[k] = nullptr; cudaGetLastError(); }
      }
    }
    ready = true;
    return cudaSuccess;
  }

  cudaError_t dalloc(void** p, size_t bytes, cudaStream_t st) {
    *p = blocks.alloc(bytes);
    if (*p) return cudaSuccess;
    ++pool_allocs;
    return cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, st);
  }
  cudaError_t dfree(void* p, cudaStream_t st) {
    if (blocks.release(p)) return cudaSuccess;
    return cudaFreeAsync(p, st);
  }

  // Prefetch buffers go back to their arena once the main stream has
  // passed their last use (the caller recorded ev_pf_free on it).
  void release_prefetches(std::unordered_map<int32_t, Prefetch>& m) {
    for (auto& kv : m) pfmem.release(kv.second.buf);
    m.clear();
  }

  // Issue the queued write-back DMA (side stream).
  cudaError_t issue_pending() {
    if (disk_mode()) return issue_pending_disk();
    for (PendingWb& w : pending) {
      cudaError_t e = cudaStreamWaitEvent(side, ev_packed[w.sb], 0);
      if (e != cudaSuccess) return e;
      // one copy-engine transfer per range: a prefix of an interleaved
      // store is one range (6 for a section-major one)
      for (size_t i = 0; i < w.dst.size() && e == cudaSuccess; ++i)
        e = cudaMemcpyAsync(w.dst[i], w.src[i], w.size[i], cudaMemcpyDefault, side);
      if (e == cudaSuccess) e = cudaEventRecord(ev_stage[w.sb], side);
      if (e == cudaSuccess) e = cudaEventRecord(ev_wb, side);
      if (e != cudaSuccess) return e;
      for (int32_t sid : w.sids) wb_prev[sid] = 1;
    }
    pending.clear();
    return cudaSuccess;
  }

  // ---- disk mode helpers ----------------------------------------------
  static cudaError_t ensure_pinned(void** p, size_t* cap, size_t bytes) {
    if (bytes <= *cap) return cudaSuccess;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *cap = 0;
    const size_t want = bytes + bytes / 2 + (size_t(1) << 20);
    cudaError_t e = cudaMallocHost(p, want);
    if (e == cudaSuccess) *cap = want;
    return e;
  }
  // 6 preads of a prefix into dst (section-major, `rows` rows per section)
  bool read_prefix(int64_t slot, int64_t rows, float* dst) {
    for (int k = 0; k < 6; ++k) {
      const int cols = kSecOffH[k + 1] - kSecOffH[k];
      const size_t bytes = size_t(cols) * size_t(rows) * sizeof(float);
      char* d = reinterpret_cast<char*>(dst + (int64_t)kSecOffH[k] * rows);
      const int64_t at = disk.off[k] + slot * cols * int64_t(sizeof(float));
      size_t done = 0;
      while (done < bytes) {
        const ssize_t r = pread(disk.fd, d + done, bytes - done, at + int64_t(done));
        if (r <= 0) return false;
        done += size_t(r);
      }
      disk.bytes_read += int64_t(bytes);
    }
    return true;
  }
  // complete every write-back: wait for its D2H copy, then pwrite
  cudaError_t flush_disk_writes() {
    if (disk.writes.empty()) return cudaSuccess;
    cudaError_t e = cudaEventSynchronize(disk.wb_done);
    if (e != cudaSuccess) return e;
    for (const DiskPiece& p : disk.writes) {
      size_t done = 0;
      while (done < p.bytes) {
        const ssize_t r = pwrite(disk.fd, disk.wbb + p.buf_off + done, p.bytes - done, p.file_off + int64_t(done));
        if (r <= 0) return cudaErrorUnknown;
        done += size_t(r);
      }
      disk.bytes_written += int64_t(p.bytes);
    }
    disk.writes.clear();
    disk.wbb_used = 0;
    wb_prev.clear();
    return cudaSuccess;
  }
  cudaError_t issue_pending_disk() {
    for (PendingWb& w : pending) {
      size_t need = 0;
      for (size_t i = 0; i < w.size.size(); ++i) need += w.size[i];
      if (disk.wbb_used + need > disk.wbb_cap) {
        cudaError_t e = flush_disk_writes();       // drains the bounce buffer
        if (e == cudaSuccess) e = ensure_pinned(reinterpret_cast<void**>(&disk.wbb), &disk.wbb_cap, need);
        if (e != cudaSuccess) return e;
      }
      cudaError_t e = cudaStreamWaitEvent(side, ev_packed[w.sb], 0);
      if (e != cudaSuccess) return e;
      for (size_t i = 0; i < w.size.size(); ++i) {
        // w.dst holds the file offset of the piece in disk mode
        e = cudaMemcpyAsync(disk.wbb + disk.wbb_used, w.src[i], w.size[i], cudaMemcpyDeviceToHost, side);
        if (e != cudaSuccess) return e;
        disk.writes.push_back({int64_t(reinterpret_cast<intptr_t>(w.dst[i])), disk.wbb_used, w.size[i]});
        disk.wbb_used += w.size[i];
      }
      e = cudaEventRecord(ev_stage[w.sb], side);
      if (e == cudaSuccess) e = cudaEventRecord(ev_wb, side);
      if (e == cudaSuccess) e = cudaEventRecord(disk.wb_done, side);
      if (e != cudaSuccess) return e;
      for (int32_t sid : w.sids) wb_prev[sid] = 1;
    }
    pending.clear();
    return cudaSuccess;
  }

  ~CacheTable() {
    if (disk_mode()) flush_disk_writes();
    if (side) cudaStreamSynchronize(side);
    if (pf_st) cudaStreamSynchronize(pf_st);
    cudaDeviceSynchronize();
    for (auto& e : lru) dfree(e.block, 0);
    for (double* b : to_free) dfree(b, 0);
    cudaDeviceSynchronize();
    if (items_done) cudaEventDestroy(items_done);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_wb) cudaEventDestroy(ev_wb);
    if (ev_pf) cudaEventDestroy(ev_pf);
    if (ev_pf_free) cudaEventDestroy(ev_pf_free);
    if (side) cudaStreamDestroy(side);
    if (pf_st) cudaStreamDestroy(pf_st);
    if (h_items) cudaFreeHost(h_items);
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) cudaFree(stage[k]);
      if (ev_stage[k]) cudaEventDestroy(ev_stage[k]);
      if (ev_packed[k]) cudaEventDestroy(ev_packed[k]);
    }
    if (pool) cudaMemPoolDestroy(pool);
    if (disk.rd) cudaFreeHost(disk.rd);
    if (disk.pfb) cudaFreeHost(disk.pfb);
    if (disk.wbb) cudaFreeHost(disk.wbb);
    if (disk.dtmp) cudaFree(disk.dtmp);
    for (cudaEvent_t ev : {disk.rd_done, disk.pf_done, disk.wb_done})
      if (ev) cudaEventDestroy(ev);
  }

  // pinned item table of at least `bytes`, safe to rewrite
  cudaError_t ensure_items(size_t bytes) {
    cudaEventSynchronize(items_done);
    if (bytes <= items_cap) return cudaSuccess;
    if (h_items) cudaFreeHost(h_items);
    const size_t want = bytes * 2 + 4096;
    cudaError_t e = cudaMallocHost(&h_items, want);
    if (e != cudaSuccess) return e;
    items_cap = want;
    return cudaSuccess;
  }
};

namespace {

// A cache block: 23·P f64 values (section-major) + one touched bit per row.
size_t block_bytes(int64_t P) {
  const int64_t rows = P > 0 ? P : 1;
  return size_t(kFloats * rows + (rows + 63) / 64) * sizeof(double);
}

struct Xfer {
  int32_t spt_id;
  int64_t slot, rows;
  double* block;
  const double* overlay;       // loads: rows [0, overlay_rows) come from here
  int64_t overlay_rows;
  const float* src = nullptr;  // loads: prefetched f32 copy of the prefix (HBM)
};

// Touched rows of the blocks about to be written back (or overlaid) take
// their master values first (the refresh trainer.py:363 made implicit).
// The item table goes through `host` (pinned, stream-ordered reuse) when
// given, else through a pageable copy (tests / explicit calls).
cudaError_t materialize(CacheTable* c, const std::vector<Xfer>& v, cudaStream_t st, void* host = nullptr) {
  if (!c->m_master || v.empty()) return cudaSuccess;
  c->m_items.clear();
  long long acc = 0;
  for (const Xfer& x : v) {
    glod_mat_item it;
    it.block = x.block;
    it.rows = x.rows;
    it.elem_start = acc;
    it.rec_offset = c->m_rec_off[x.spt_id];
    c->m_items.push_back(it);
    acc += kFloats * x.rows;
  }
  const size_t bytes = c->m_items.size() * sizeof(glod_mat_item);
  const void* src = c->m_items.data();
  if (host) {
    memcpy(host, src, bytes);
    src = host;
  }
  void* d = nullptr;
  cudaError_t e = c->dalloc(&d, bytes, st);
  if (e == cudaSuccess)
    e = host ? launch_upload(d, src, bytes, st) : cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = launch_materialize(static_cast<glod_mat_item*>(d), int(c->m_items.size()), acc, c->m_master, c->m_cap,
                           c->m_stride, c->m_rec_node, st);
  if (e == cudaSuccess) e = c->dfree(d, st);
  return e;
}

size_t mat_bytes(const std::vector<Xfer>& v) { return (v.size() * sizeof(glod_mat_item) + 15) / 16 * 16; }

// Host bytes of one batch's table: items + int2 block map.
size_t table_bytes(const std::vector<Xfer>& v) {
  long long nb = 0;
  for (const Xfer& x : v) nb += transfer_chunks(x.rows);
  return (v.size() * sizeof(glod_prefix_item) + 15) / 16 * 16 + (size_t(nb) * sizeof(int2) + 15) / 16 * 16 +
         v.size() * sizeof(long long);
}

// Writes `v` and its block map into the pinned table at byte offset `off`
// and uploads both (main-stream ordered; the caller frees the device copy
// after its kernel).  Returns the device items, block map and block count.
cudaError_t stage_items(CacheTable* c, const std::vector<Xfer>& v, size_t off, cudaStream_t st,
                        glod_prefix_item** d_items, const int2** d_bmap, long long* nblocks,
                        const long long** d_rec_off) {
  char* base = reinterpret_cast<char*>(c->h_items) + off;
  glod_prefix_item* h = reinterpret_cast<glod_prefix_item*>(base);
  const size_t items_bytes = (v.size() * sizeof(glod_prefix_item) + 15) / 16 * 16;
  int2* bm = reinterpret_cast<int2*>(base + items_bytes);
  long long acc = 0, nb = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    h[i].slot_start = v[i].slot;
    h[i].rows = v[i].rows;
    h[i].elem_start = acc;
    h[i].block = v[i].block;
    h[i].overlay = v[i].overlay;
    h[i].overlay_rows = v[i].overlay_rows;
    h[i].src = v[i].src;
    acc += kFloats * v[i].rows;
    const long long nc = transfer_chunks(v[i].rows);
    for (long long k = 0; k < nc; ++k) bm[nb++] = make_int2(int(i), int(k));
  }
  // each item's first SPT record (its rows' master rows: touched bits)
  const size_t bmap_bytes = (size_t(nb) * sizeof(int2) + 15) / 16 * 16;
  long long* ro = reinterpret_cast<long long*>(base + items_bytes + bmap_bytes);
  for (size_t i = 0; i < v.size(); ++i) ro[i] = c->m_master ? c->m_rec_off[v[i].spt_id] : 0;
  const size_t bytes = items_bytes + bmap_bytes + v.size() * sizeof(long long);
  void* d = nullptr;
  cudaError_t e = c->dalloc(&d, bytes, st);
  if (e != cudaSuccess) return e;
  e = launch_upload(d, base, bytes, st);        // pinned table, off the copy engines
  if (e != cudaSuccess) return e;
  *d_items = static_cast<glod_prefix_item*>(d);
  *d_bmap = reinterpret_cast<const int2*>(static_cast<char*>(d) + items_bytes);
  *d_rec_off = reinterpret_cast<const long long*>(static_cast<char*>(d) + items_bytes + bmap_bytes);
  *nblocks = nb;
  return cudaSuccess;
}

// One batch of transfers.  Loads: one kernel on the main stream (zero-copy
// PCIe reads of the pinned store, or HBM reads of prefetched copies).
// Write-backs: packed to f32 staging on the main stream; the DMA into the
// store is queued (CacheTable::pending) and issued at end_step.
cudaError_t run_batch(CacheTable* c, const std::vector<Xfer>& loads, const std::vector<Xfer>& wbs,
                      bool join, bool wait_pf, const glod_store_view& sv, cudaStream_t st) {
  const size_t load_bytes = table_bytes(loads), wb_bytes = table_bytes(wbs);
  cudaError_t e = c->ensure_items(load_bytes + wb_bytes + mat_bytes(wbs) + 96);
  if (e != cudaSuccess) return e;
  if (join) {
    e = cudaStreamWaitEvent(st, c->ev_wb, 0);
    if (e != cudaSuccess) return e;
    c->wb_prev.clear();
  }
  if (wait_pf) {
    e = cudaStreamWaitEvent(st, c->ev_pf, 0);
    if (e != cudaSuccess) return e;
  }
  // touched rows of written-back / overlaid blocks are taken from the
  // master by the pack / load kernels themselves (no materialise pass)
  auto tq = std::chrono::steady_clock::now();
  auto lap = [&](int k) {
    const auto now = std::chrono::steady_clock::now();
    c->prof_ns[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(now - tq).count();
    tq = now;
  };
  glod_master_ref mref = {c->m_master, c->m_cap, c->m_stride, c->m_rec_node, nullptr};
  lap(2);
  if (!loads.empty()) {
    glod_prefix_item* d = nullptr;
    const int2* bm = nullptr;
    long long nb = 0;
    e = stage_items(c, loads, 0, st, &d, &bm, &nb, &mref.item_rec_off);
    if (e == cudaSuccess) e = launch_load_blocks(sv, d, bm, nb, mref, st);
    if (e == cudaSuccess) e = c->dfree(d, st);
    if (e != cudaSuccess) return e;
  }
  lap(3);
  if (!wbs.empty()) {
    glod_prefix_item* d = nullptr;
    const int2* bm = nullptr;
    long long nb = 0, total = 0;
    for (const Xfer& x : wbs) total += kFloats * x.rows;
    e = stage_items(c, wbs, (load_bytes + 15) / 16 * 16, st, &d, &bm, &nb, &mref.item_rec_off);
    if (e != cudaSuccess) return e;
    const int sb = c->stage_next;
    c->stage_next ^= 1;
    for (const auto& w : c->pending)          // staging buffer still queued: issue first
      if (w.sb == sb) {
        e = c->issue_pending();
        if (e != cudaSuccess) return e;
        break;
      }
    const size_t need = size_t(total) * sizeof(float);
    if (need > c->stage_cap[sb]) {
      e = cudaEventSynchronize(c->ev_stage[sb]);          // copies out of the old buffer
      if (c->stage[sb]) cudaFree(c->stage[sb]);
      c->stage[sb] = nullptr;
      c->stage_cap[sb] = 0;
      const size_t want = std::max(need + need / 2, 2 * c->stage_cap[sb]);
      if (e == cudaSuccess) e = cudaMalloc(&c->stage[sb], want);
      if (e != cudaSuccess) return e;
      c->stage_cap[sb] = want;
      ++c->grow_events;
    }
    float* staging = c->stage[sb];
    e = cudaStreamWaitEvent(st, c->ev_stage[sb], 0);
    if (e == cudaSuccess) e = launch_pack_blocks(d, bm, nb, staging, c->interleaved, mref, st);
    if (e == cudaSuccess) e = c->dfree(d, st);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_packed[sb], st);
    if (e != cudaSuccess) return e;
    CacheTable::PendingWb w;
    w.sb = sb;
    w.dst.reserve(6 * wbs.size()); w.src.reserve(6 * wbs.size()); w.size.reserve(6 * wbs.size());
    long long acc = 0;
    for (const Xfer& x : wbs) {
      if (c->interleaved) {
        w.dst.push_back(static_cast<void*>(c->dsec[0] + x.slot * kFloats));
        w.src.push_back(staging + acc);
        w.size.push_back(size_t(kFloats) * size_t(x.rows) * sizeof(float));
        acc += kFloats * x.rows;
        w.sids.push_back(x.spt_id);
        continue;
      }
      for (int k = 0; k < 6; ++k) {
        const int cols = kSecOffH[k + 1] - kSecOffH[k];
        w.dst.push_back(c->disk_mode()
                            ? reinterpret_cast<void*>(intptr_t(c->disk.off[k] + x.slot * cols * int64_t(sizeof(float))))
                            : static_cast<void*>(c->dsec[k] + x.slot * cols));
        w.src.push_back(staging + acc + (long long)kSecOffH[k] * x.rows);
        w.size.push_back(size_t(cols) * size_t(x.rows) * sizeof(float));
      }
      acc += kFloats * x.rows;
      w.sids.push_back(x.spt_id);
    }
    c->pending.push_back(std::move(w));
  }
  lap(4);
  return cudaEventRecord(c->items_done, st);
}

}  // namespace

cudaError_t cache_step(CacheTable* c, const glod_store_view& sv, int32_t n, const int32_t* spt_ids,
                       const double* d_root, const int32_t* prefix_len, double* dist_out,
                       uint64_t* block_out, int64_t* rows_out, int64_t* loaded_rows,
                       int64_t* hits, cudaStream_t st) {
  cudaError_t e = c->init(sv);
  if (e == cudaSuccess) e = c->issue_pending();       // end_step was skipped
  if (e != cudaSuccess) return e;
  // OverBudgetError before any state changes (the reference raises from
  // insert; an entry larger than the budget can never be resident, so a
  // prefix over budget that is not a hit now would be inserted)
  for (int32_t j = 0; j < n; ++j) {
    if (int64_t(prefix_len[j]) * c->bytes_per_row <= c->budget) continue;
    auto it = c->map.find(spt_ids[j]);
    bool hit = false;
    if (it != c->map.end()) {
      const double cd = it->second->cached_distance, d = d_root[j];
      hit = cd == 0.0 ? d == 0.0 : (c->d_min <= d / cd && d / cd <= c->d_max);
    }
    if (!hit) return cudaErrorNotPermitted;
  }
  // disk mode: every earlier write-back reaches the file before it is read
  if (c->disk_mode()) {
    e = c->flush_disk_writes();
    if (e != cudaSuccess) return e;
  }
  // write-backs of earlier steps already finished: nothing to wait for
  if (!c->wb_prev.empty() && cudaEventQuery(c->ev_wb) == cudaSuccess) c->wb_prev.clear();
  const auto tp0 = std::chrono::steady_clock::now();
  std::vector<Xfer> loads, wbs;
  std::unordered_map<int32_t, std::pair<const double*, int64_t>> evicted;   // dirty, this step
  bool join = false, wait_pf = false;
  std::unordered_map<int32_t, CacheTable::Prefetch> avail;   // issued last step
  avail.swap(c->pf);
  const int64_t hits0 = c->hits, loaded0 = c->loaded_rows;
  c->step_ids.assign(spt_ids, spt_ids + n);
  auto drop = [&](const Entry& v) {
    c->resident -= v.nbytes;
    if (v.dirty) {
      wbs.push_back({v.spt_id, c->slot_start[v.spt_id], v.prefix_len, v.block, nullptr, 0});
      evicted[v.spt_id] = {v.block, v.prefix_len};
    }
    c->to_free.push_back(v.block);
  };
  for (int32_t j = 0; j < n; ++j) {
    const int32_t sid = spt_ids[j];
    const double d = d_root[j];
    auto it = c->map.find(sid);
    bool hit = false;
    if (it != c->map.end()) {
      const double cd = it->second->cached_distance;
      if (cd == 0.0) hit = d == 0.0;
      else {
        const double ratio = d / cd;
        hit = c->d_min <= ratio && ratio <= c->d_max;
      }
    }
    if (hit) {
      ++c->hits;
      c->lru.splice(c->lru.end(), c->lru, it->second);   // move_to_end
    } else {
      ++c->misses;
      const int64_t P = prefix_len[j];
      const int64_t nbytes = P * c->bytes_per_row;
      if (nbytes > c->budget) return cudaErrorNotPermitted;   // OverBudgetError
      void* blk = nullptr;
      e = c->dalloc(&blk, block_bytes(P), st);
      if (e != cudaSuccess) return e;
      Xfer ld{sid, c->slot_start[sid], P, static_cast<double*>(blk), nullptr, 0};
      auto ev = evicted.find(sid);
      auto pv = avail.find(sid);
      if (pv != avail.end() && pv->second.rows == P && ev == evicted.end()) {
        // prefetched after every write-back of these rows so far: the store
        // contents the reference would read now
        ld.src = pv->second.buf;
        c->pf_used_rows += P;
        wait_pf = true;
      } else if (ev != evicted.end()) {
        // evicted (dirty) earlier in this step: the reference writes it back
        // and then reads the store, i.e. rows below the old prefix are the
        // f32 rounding of the evicted block, the rest the untouched store
        ld.overlay = ev->second.first;
        ld.overlay_rows = ev->second.second;      // its row count = its section stride
        // rows past the overlay come from the store: wait for a write-back
        // of an earlier step still writing them
        if (ld.overlay_rows < P && c->wb_prev.count(sid)) join = true;
      } else if (c->wb_prev.count(sid)) {
        join = true;                 // store rows still being written back
      }
      loads.push_back(ld);
      c->loaded_rows += P;
      // insert: replace (old dirty block written back after the load),
      // append, evict from the LRU front
      if (it != c->map.end()) {
        Entry old = *it->second;
        c->lru.erase(it->second);
        c->map.erase(sid);
        drop(old);
        evicted.erase(sid);          // never requested again this step
      }
      c->lru.push_back({sid, d, P, static_cast<double*>(blk), nbytes, false});
      c->map[sid] = std::prev(c->lru.end());
      c->resident += nbytes;
      while (c->resident > c->budget) {
        Entry v = c->lru.front();
        c->lru.pop_front();
        c->map.erase(v.spt_id);
        drop(v);
      }
    }
    const Entry& en = *c->map.find(sid)->second;
    dist_out[j] = en.cached_distance;
    block_out[j] = reinterpret_cast<uint64_t>(en.block);
    rows_out[j] = en.prefix_len;
  }
  if (c->disk_mode()) {
    // misses without a prefetch: pread into the pinned bounce, one H2D copy
    // on this stream, then the load kernel converts from HBM (overlaid
    // rows of a block evicted this step still come from that block)
    size_t rows = 0;
    for (const Xfer& x : loads)
      if (!x.src) rows += size_t(x.rows);
    if (rows > 0) {
      const size_t bytes = rows * kFloats * sizeof(float);
      e = cudaEventSynchronize(c->disk.rd_done);
      if (e == cudaSuccess)
        e = CacheTable::ensure_pinned(reinterpret_cast<void**>(&c->disk.rd), &c->disk.rd_cap, bytes);
      if (e == cudaSuccess && bytes > c->disk.dtmp_cap) {
        if (c->disk.dtmp) cudaFree(c->disk.dtmp);
        c->disk.dtmp = nullptr;
        c->disk.dtmp_cap = 0;
        const size_t want = bytes + bytes / 2;
        e = cudaMalloc(&c->disk.dtmp, want);
        if (e == cudaSuccess) c->disk.dtmp_cap = want;
      }
      if (e != cudaSuccess) return e;
      size_t at = 0;
      for (Xfer& x : loads) {
        if (x.src) continue;
        if (!c->read_prefix(x.slot, x.rows, c->disk.rd + at)) return cudaErrorUnknown;
        x.src = c->disk.dtmp + at;
        at += size_t(x.rows) * kFloats;
      }
      e = cudaMemcpyAsync(c->disk.dtmp, c->disk.rd, bytes, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = cudaEventRecord(c->disk.rd_done, st);
      if (e != cudaSuccess) return e;
    }
  }
  const auto tp1 = std::chrono::steady_clock::now();
  c->prof_ns[0] += std::chrono::duration_cast<std::chrono::nanoseconds>(tp1 - tp0).count();
  e = run_batch(c, loads, wbs, join, wait_pf, sv, st);
  if (e != cudaSuccess) return e;
  // every prefetch of the last step is done with once the load kernel ran
  if (!avail.empty()) {
    e = cudaEventRecord(c->ev_pf_free, st);
    if (e != cudaSuccess) return e;
    c->release_prefetches(avail);
  }
  *loaded_rows = c->loaded_rows - loaded0;
  *hits = c->hits - hits0;
  return cudaSuccess;
}

// Blocks dropped this step are still read by this step's kernels (the
// reference keeps its `entry` references alive): release them in
// main-stream order once the step is enqueued (their write-backs read the
// f32 staging copy, not the block).
cudaError_t cache_release(CacheTable* c, cudaStream_t st) {
  for (double* b : c->to_free) {
    cudaError_t e = c->dfree(b, st);
    if (e != cudaSuccess) return e;
  }
  c->to_free.clear();
  return cudaSuccess;
}

cudaError_t cache_end_step(CacheTable* c, const glod_store_view& sv, int64_t iteration,
                           int mark_dirty, cudaStream_t st) {
  cudaError_t e = c->init(sv);
  if (e != cudaSuccess) return e;
  if (mark_dirty)
    for (int32_t sid : c->step_ids) {
      auto it = c->map.find(sid);
      if (it != c->map.end()) it->second->dirty = true;
    }
  c->step_ids.clear();
  if (iteration >= 0 && iteration % c->flush_interval == 0) {
    std::vector<Xfer> none, wbs;
    for (auto& en : c->lru) {
      if (en.dirty) wbs.push_back({en.spt_id, c->slot_start[en.spt_id], en.prefix_len, en.block, nullptr, 0});
      c->to_free.push_back(en.block);
    }
    c->lru.clear();
    c->map.clear();
    c->resident = 0;
    // prefetched store rows may be rewritten now: drop them (no main-stream
    // user, so the arena takes them back at once)
    c->release_prefetches(c->pf);
    e = run_batch(c, none, wbs, false, false, sv, st);
    if (e != cudaSuccess) return e;
  }
  e = c->issue_pending();
  if (e != cudaSuccess) return e;
  return cache_release(c, st);
}

// Prefetch of a predicted view (the scheduler's next draw): every selected
// SPT the table would miss now is copied store → f32 HBM buffer on the
// prefetch stream by the copy engines (one cudaMemcpyAsync per prefix of an
// interleaved store, 6 section ranges otherwise), ordered after every
// write-back issued so far.
// Read-only on the table; correctness never depends on the prediction
// (cache_step checks the prefix length and same-step evictions before
// using one, and a flush drops them).
cudaError_t cache_prefetch(CacheTable* c, const glod_store_view& sv, int32_t n, const int32_t* spt_ids,
                           const double* d_root, const int32_t* prefix_len, int64_t max_rows,
                           int64_t* rows_out, cudaStream_t st) {
  (void)st;
  cudaError_t e = c->init(sv);
  if (e == cudaSuccess) e = c->issue_pending();
  if (e != cudaSuccess) return e;
  *rows_out = 0;
  if (!c->pfmem.ready()) return cudaSuccess;
  if (c->disk_mode()) {                       // the file holds every write-back so far
    e = c->flush_disk_writes();
    if (e != cudaSuccess) return e;
  }
  if (!c->wb_prev.empty() && cudaEventQuery(c->ev_wb) == cudaSuccess) c->wb_prev.clear();
  struct Want {
    int32_t sid;
    int64_t rows;
    float* buf;
  };
  std::vector<Want> now, after_wb;
  int64_t total = 0;
  for (int32_t j = 0; j < n; ++j) {
    const int32_t sid = spt_ids[j];
    const int64_t P = prefix_len[j];
    if (P <= 0 || c->pf.count(sid)) continue;
    auto it = c->map.find(sid);
    if (it != c->map.end()) {
      const double cd = it->second->cached_distance, d = d_root[j];
      bool hit;
      if (cd == 0.0) hit = d == 0.0;
      else {
        const double ratio = d / cd;
        hit = c->d_min <= ratio && ratio <= c->d_max;
      }
      if (hit) continue;
    }
    if (P * c->bytes_per_row > c->budget) continue;
    if (max_rows >= 0 && total + P > max_rows) break;
    float* buf = static_cast<float*>(c->pfmem.alloc(size_t(kFloats) * size_t(P) * sizeof(float)));
    if (!buf) break;                                  // prefetch memory full
    c->pf[sid] = {P, buf};
    (c->wb_prev.count(sid) ? after_wb : now).push_back({sid, P, buf});
    total += P;
  }
  if (now.empty() && after_wb.empty()) return cudaSuccess;
  // the buffers' previous users: the last load kernel on the main stream
  e = cudaStreamWaitEvent(c->pf_st, c->ev_pf_free, 0);
  if (e != cudaSuccess) return e;
  auto issue = [&](const std::vector<Want>& v) -> cudaError_t {
    if (v.empty()) return cudaSuccess;
    if (c->disk_mode()) {
      // pread on the host now (the GPU is busy with this step), then the
      // copy engines move the bounce buffer's prefixes to their HBM buffers
      size_t bytes = 0;
      for (const Want& w : v) bytes += size_t(w.rows) * kFloats * sizeof(float);
      cudaError_t er = cudaEventSynchronize(c->disk.pf_done);
      if (er == cudaSuccess)
        er = CacheTable::ensure_pinned(reinterpret_cast<void**>(&c->disk.pfb), &c->disk.pfb_cap, bytes);
      if (er != cudaSuccess) return er;
      size_t at = 0;
      for (const Want& w : v) {
        if (!c->read_prefix(c->slot_start[w.sid], w.rows, c->disk.pfb + at)) return cudaErrorUnknown;
        er = cudaMemcpyAsync(w.buf, c->disk.pfb + at, size_t(w.rows) * kFloats * sizeof(float),
                             cudaMemcpyHostToDevice, c->pf_st);
        if (er != cudaSuccess) return er;
        at += size_t(w.rows) * kFloats;
      }
      return cudaEventRecord(c->disk.pf_done, c->pf_st);
    }
    for (const Want& w : v) {
      const int64_t slot = c->slot_start[w.sid];
      ++c->pf_copies;
      if (c->interleaved) {
        cudaError_t er = cudaMemcpyAsync(w.buf, c->dsec[0] + slot * kFloats, size_t(w.rows) * kFloats * sizeof(float),
                                         cudaMemcpyDefault, c->pf_st);
        if (er != cudaSuccess) return er;
        continue;
      }
      for (int k = 0; k < 6; ++k) {
        const int cols = kSecOffH[k + 1] - kSecOffH[k];
        cudaError_t er = cudaMemcpyAsync(w.buf + (int64_t)kSecOffH[k] * w.rows, c->dsec[k] + slot * cols,
                                         size_t(cols) * size_t(w.rows) * sizeof(float), cudaMemcpyDefault, c->pf_st);
        if (er != cudaSuccess) return er;
      }
    }
    return cudaSuccess;
  };
  e = issue(now);
  if (e == cudaSuccess && !after_wb.empty()) {
    // store rows with a write-back in flight: copy them after it lands
    e = cudaStreamWaitEvent(c->pf_st, c->ev_wb, 0);
    if (e == cudaSuccess) e = issue(after_wb);
  }
  if (e == cudaSuccess) e = cudaEventRecord(c->ev_pf, c->pf_st);
  if (e != cudaSuccess) return e;
  c->pf_issued_rows += total;
  *rows_out = total;
  return cudaSuccess;
}

}  // namespace glod

// ---------------------------------------------------------------------------
struct glod_cache {
  glod::CacheTable t;
};

extern "C" {

int glod_cache_create(int64_t budget_bytes, double d_min, double d_max, int64_t flush_interval,
                      int32_t bytes_per_row, const int64_t* slot_start, int32_t num_spts,
                      glod_cache** out) {
  if (!out || budget_bytes <= 0 || !(d_min > 0 && d_min <= 1 && 1 <= d_max) || flush_interval < 1 ||
      (num_spts > 0 && !slot_start))
    return GLOD_ERR_INVALID_ARGUMENT;
  glod_cache* c = new glod_cache();
  c->t.budget = budget_bytes;
  c->t.d_min = d_min;
  c->t.d_max = d_max;
  c->t.flush_interval = flush_interval;
  c->t.bytes_per_row = bytes_per_row;
  c->t.slot_start.assign(slot_start, slot_start + num_spts);
  cudaGetDevice(&c->t.device);
  glod::retain_pool_memory();
  *out = c;
  return GLOD_OK;
}

int glod_cache_set_file(glod_cache* c, int32_t fd, const int64_t* section_offset) {
  if (!c || fd < 0 || !section_offset) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (c->t.ready) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "set the file before the first step");
  c->t.disk.fd = fd;
  for (int k = 0; k < 6; ++k) c->t.disk.off[k] = section_offset[k];
  return GLOD_OK;
}

int glod_cache_flush_io(glod_cache* c, int64_t* bytes_read, int64_t* bytes_written) {
  if (!c) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = c->t.issue_pending();
  if (e == cudaSuccess && c->t.disk_mode()) e = c->t.flush_disk_writes();
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  if (bytes_read) *bytes_read = c->t.disk.bytes_read;
  if (bytes_written) *bytes_written = c->t.disk.bytes_written;
  return GLOD_OK;
}

int glod_cache_destroy(glod_cache* c) {
  cudaDeviceSynchronize();
  delete c;
  return GLOD_OK;
}

int glod_cache_step(glod_cache* c, const glod_store_view* store, int32_t n, const int32_t* spt_ids,
                    const double* d_root, const int32_t* prefix_len, double* dist_out,
                    uint64_t* block_out, int64_t* rows_out, int64_t* counters_out, void* stream) {
  if (!c || !store || (n > 0 && (!spt_ids || !d_root || !prefix_len || !dist_out || !block_out ||
                                 !rows_out)) || !counters_out)
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (store->row_stride != 0 && store->row_stride != 23)
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "store row_stride must be 0 or 23");
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = glod::cache_step(&c->t, *store, n, spt_ids, d_root, prefix_len, dist_out, block_out,
                                   rows_out, counters_out, counters_out + 1,
                                   static_cast<cudaStream_t>(stream));
  c->t.host_ns_step += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  if (e == cudaErrorNotPermitted)
    return glod::set_error(GLOD_ERR_OVER_BUDGET, "cache entry exceeds the byte budget");
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_end_step(glod_cache* c, const glod_store_view* store, int64_t iteration,
                        int32_t mark_dirty, void* stream) {
  if (!c || !store) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (store->row_stride != 0 && store->row_stride != 23)
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "store row_stride must be 0 or 23");
  cudaError_t e = glod::cache_end_step(&c->t, *store, iteration, mark_dirty,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_prefetch(glod_cache* c, const glod_store_view* store, int32_t n, const int32_t* spt_ids,
                        const double* d_root, const int32_t* prefix_len, int64_t max_rows,
                        int64_t* rows_out, void* stream) {
  if (!c || !store || !rows_out || (n > 0 && (!spt_ids || !d_root || !prefix_len)))
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (store->row_stride != 0 && store->row_stride != 23)
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "store row_stride must be 0 or 23");
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = glod::cache_prefetch(&c->t, *store, n, spt_ids, d_root, prefix_len, max_rows, rows_out,
                                       static_cast<cudaStream_t>(stream));
  c->t.host_ns_prefetch += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_set_master(glod_cache* c, const double* master, int64_t capacity, int64_t master_stride,
                          const int32_t* rec_node, const int64_t* rec_offset, int32_t num_spts) {
  if (!c || !master || !rec_node || (num_spts > 0 && !rec_offset))
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  c->t.m_master = master;
  c->t.m_cap = capacity;
  c->t.m_stride = master_stride;
  c->t.m_rec_node = rec_node;
  c->t.m_rec_off.assign(rec_offset, rec_offset + num_spts);
  return GLOD_OK;
}

int glod_cache_materialize(glod_cache* c, void* stream) {
  if (!c) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<glod::Xfer> all;
  for (const auto& e : c->t.lru) all.push_back({e.spt_id, 0, e.prefix_len, e.block, nullptr, 0});
  cudaError_t e = glod::materialize(&c->t, all, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GLOD_OK : glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
}

int glod_cache_resident(const glod_cache* c, uint64_t* block, int64_t* rows, int32_t num_spts) {
  if (!c || (num_spts > 0 && (!block || !rows))) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  for (int32_t s = 0; s < num_spts; ++s) {
    block[s] = 0;
    rows[s] = 0;
  }
  for (const auto& e : c->t.lru)
    if (e.spt_id >= 0 && e.spt_id < num_spts) {
      block[e.spt_id] = reinterpret_cast<uint64_t>(e.block);
      rows[e.spt_id] = e.prefix_len;
    }
  return GLOD_OK;
}

int glod_cache_mark_dirty(glod_cache* c, const int32_t* flags, int32_t num_spts) {
  if (!c || (num_spts > 0 && !flags)) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  for (auto& e : c->t.lru)
    if (e.spt_id >= 0 && e.spt_id < num_spts && flags[e.spt_id]) e.dirty = true;
  return GLOD_OK;
}

int glod_memcpy_d2h(void* dst, const void* src, int64_t bytes) {
  if (!dst || !src) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = cudaMemcpy(dst, src, size_t(bytes), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_debug_profile(const glod_cache* c, int64_t* ns_out8) {
  if (!c || !ns_out8) return GLOD_ERR_INVALID_ARGUMENT;
  for (int k = 0; k < 8; ++k) ns_out8[k] = c->t.prof_ns[k];
  return GLOD_OK;
}

int glod_cache_stats(const glod_cache* c, glod_cache_stats_t* out) {
  if (!c || !out) return GLOD_ERR_INVALID_ARGUMENT;
  out->entries = int64_t(c->t.lru.size());
  out->resident_bytes = c->t.resident;
  out->hits = c->t.hits;
  out->misses = c->t.misses;
  out->loaded_rows = c->t.loaded_rows;
  out->prefetched_rows = c->t.pf_issued_rows;
  out->prefetch_used_rows = c->t.pf_used_rows;
  out->pool_allocs = c->t.pool_allocs;
  out->grow_events = c->t.grow_events;
  out->host_ns_step = c->t.host_ns_step;
  out->host_ns_prefetch = c->t.host_ns_prefetch;
  out->pf_copies = c->t.pf_copies;
  return GLOD_OK;
}

int glod_cache_entries(const glod_cache* c, int32_t* spt_id, double* cached_distance,
                       int64_t* prefix_len, uint64_t* block, int32_t* dirty, int64_t capacity) {
  if (!c) return GLOD_ERR_INVALID_ARGUMENT;
  int64_t i = 0;
  for (const auto& e : c->t.lru) {
    if (i >= capacity) break;
    spt_id[i] = e.spt_id;
    cached_distance[i] = e.cached_distance;
    prefix_len[i] = e.prefix_len;
    block[i] = reinterpret_cast<uint64_t>(e.block);
    dirty[i] = e.dirty;
    ++i;
  }
  return GLOD_OK;
}

}  // extern "C"
