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

#include <list>
#include <unordered_map>
#include <vector>

#include "../../include/glod_b200.h"
#include "common.cuh"

namespace glod {

cudaError_t launch_store_xfer(const glod_store_view& sv, const glod_prefix_item* items, int n_items,
                              long long total, int load, cudaStream_t st);
cudaError_t launch_pack_f32(const glod_prefix_item* items, int n_items, long long total, float* out,
                            cudaStream_t st);

namespace {

constexpr int kFloats = 23;

struct Entry {
  int32_t spt_id;
  double cached_distance;
  int64_t prefix_len;
  double* block;
  int64_t nbytes;
  bool dirty;
};

}  // namespace

struct CacheTable {
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
  glod_prefix_item* h_items = nullptr;
  size_t items_cap = 0;
  cudaEvent_t items_done = nullptr;
  std::vector<int32_t> step_ids;          // SPTs rendered this step (dirty at end)
  std::vector<double*> to_free;           // blocks dropped this step
  int device = 0;
  // Write-back copies run on a side stream so the D2H PCIe direction
  // overlaps the rest of the step.  The main stream waits for them only
  // when a load reads store rows a not-yet-finished write-back of an
  // earlier step writes (wb_prev); a block evicted and re-requested within
  // one step is reloaded from the evicted block itself (overlay, below).
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_wb = nullptr;
  std::unordered_map<int32_t, int> wb_prev;   // SPT ids with write-backs in flight

  // Blocks and item tables: a private stream-ordered pool (all allocations
  // and frees on the main stream).  Write-back staging: two persistent f32
  // buffers used alternately; the main stream reuses one only after the
  // side stream's copies out of it (ev_stage) — two batches earlier.
  cudaMemPool_t pool = nullptr;
  float* stage[2] = {nullptr, nullptr};
  size_t stage_cap[2] = {0, 0};
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  int stage_next = 0;

  cudaError_t ensure_side() {
    if (side) return cudaSuccess;
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
      e = cudaEventCreateWithFlags(&ev_stage[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_wb, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&items_done, cudaEventDisableTiming);
    return e;
  }

  ~CacheTable() {
    if (side) cudaStreamSynchronize(side);
    cudaDeviceSynchronize();
    if (items_done) cudaEventDestroy(items_done);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_wb) cudaEventDestroy(ev_wb);
    if (side) cudaStreamDestroy(side);
    for (auto& e : lru) cudaFree(e.block);
    for (double* b : to_free) cudaFree(b);
    if (h_items) cudaFreeHost(h_items);
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) cudaFree(stage[k]);
      if (ev_stage[k]) cudaEventDestroy(ev_stage[k]);
    }
    if (pool) cudaMemPoolDestroy(pool);
  }

  // pinned item table of at least n entries, safe to rewrite
  cudaError_t ensure_items(size_t n) {
    cudaError_t e = ensure_side();
    if (e != cudaSuccess) return e;
    cudaEventSynchronize(items_done);
    if (n <= items_cap) return cudaSuccess;
    if (h_items) cudaFreeHost(h_items);
    const size_t want = n * 2 + 64;
    e = cudaMallocHost(&h_items, want * sizeof(glod_prefix_item));
    if (e != cudaSuccess) return e;
    items_cap = want;
    return cudaSuccess;
  }
};

namespace {

struct Xfer {
  int32_t spt_id;
  int64_t slot, rows;
  double* block;
  const double* overlay;       // loads: rows [0, overlay_rows) come from here
  int64_t overlay_rows;
};

// Copies `v` into the pinned table at `off` and then to a stream-ordered
// device table; returns the device table (freed by the caller's stream
// order) and the element total.
cudaError_t stage_items(CacheTable* c, const std::vector<Xfer>& v, size_t off, cudaStream_t st,
                        glod_prefix_item** d_out, long long* total) {
  glod_prefix_item* h = c->h_items + off;
  long long acc = 0;
  for (size_t i = 0; i < v.size(); ++i) {
    h[i].slot_start = v[i].slot;
    h[i].rows = v[i].rows;
    h[i].elem_start = acc;
    h[i].block = v[i].block;
    h[i].overlay = v[i].overlay;
    h[i].overlay_rows = v[i].overlay_rows;
    acc += kFloats * v[i].rows;
  }
  glod_prefix_item* d = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&d, v.size() * sizeof(glod_prefix_item), c->pool, st);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(d, h, v.size() * sizeof(glod_prefix_item), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  *d_out = d;
  *total = acc;
  return cudaSuccess;
}

// Host address of a store section (the view holds device-mapped
// addresses; the copy engines take the host side under UVA).
cudaError_t host_section(const glod_store_view& sv, int k, float** out) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, sv.section[k]);
  if (e != cudaSuccess) return e;
  *out = static_cast<float*>(at.hostPointer ? at.hostPointer : const_cast<float*>(sv.section[k]));
  return cudaSuccess;
}

// One step's transfers.  Loads: one zero-copy kernel on the main stream.
// Write-backs: the blocks are packed to f32 on the main stream right after
// the loads (so a replaced dirty entry is written back after its stale
// reload, and every written-back block is read before this step's ADAM
// refresh rewrites it — the reference writes back at eviction), then the
// copy engines move the f32 rows into the pinned store on the side stream
// (cudaMemcpyBatchAsync, 6 section ranges per block): no SM time, so the
// D2H direction overlaps the rest of the step without slowing its kernels.
cudaError_t run_batch(CacheTable* c, const glod_store_view& sv, const std::vector<Xfer>& loads,
                      const std::vector<Xfer>& wbs, bool join, cudaStream_t st) {
  cudaError_t e = c->ensure_items(loads.size() + wbs.size() + 1);
  if (e != cudaSuccess) return e;
  if (join) {
    e = cudaStreamWaitEvent(st, c->ev_wb, 0);
    if (e != cudaSuccess) return e;
    c->wb_prev.clear();
  }
  if (!loads.empty()) {
    glod_prefix_item* d = nullptr;
    long long total = 0;
    e = stage_items(c, loads, 0, st, &d, &total);
    if (e == cudaSuccess) e = launch_store_xfer(sv, d, int(loads.size()), total, 1, st);
    if (e == cudaSuccess) e = cudaFreeAsync(d, st);
    if (e != cudaSuccess) return e;
  }
  if (!wbs.empty()) {
    glod_prefix_item* d = nullptr;
    long long total = 0;
    e = stage_items(c, wbs, loads.size(), st, &d, &total);
    if (e != cudaSuccess) return e;
    const int sb = c->stage_next;
    c->stage_next ^= 1;
    const size_t need = size_t(total) * sizeof(float);
    if (need > c->stage_cap[sb]) {
      e = cudaEventSynchronize(c->ev_stage[sb]);          // copies out of the old buffer
      if (c->stage[sb]) cudaFree(c->stage[sb]);
      c->stage[sb] = nullptr;
      c->stage_cap[sb] = 0;
      if (e == cudaSuccess) e = cudaMalloc(&c->stage[sb], need + need / 2);
      if (e != cudaSuccess) return e;
      c->stage_cap[sb] = need + need / 2;
    }
    float* staging = c->stage[sb];
    e = cudaStreamWaitEvent(st, c->ev_stage[sb], 0);
    if (e == cudaSuccess) e = launch_pack_f32(d, int(wbs.size()), total, staging, st);
    if (e == cudaSuccess) e = cudaFreeAsync(d, st);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_main, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_main, 0);
    if (e != cudaSuccess) return e;
    float* hsec[6];
    for (int k = 0; k < 6; ++k) {
      e = host_section(sv, k, &hsec[k]);
      if (e != cudaSuccess) return e;
    }
    static const int off[7] = {0, 3, 6, 10, 11, 14, 23};
    std::vector<void*> dst, src;
    std::vector<size_t> size;
    dst.reserve(6 * wbs.size()); src.reserve(6 * wbs.size()); size.reserve(6 * wbs.size());
    long long acc = 0;
    for (const Xfer& x : wbs) {
      for (int k = 0; k < 6; ++k) {
        const int cols = off[k + 1] - off[k];
        dst.push_back(hsec[k] + x.slot * cols);
        src.push_back(staging + acc + (long long)off[k] * x.rows);
        size.push_back(size_t(cols) * size_t(x.rows) * sizeof(float));
      }
      acc += kFloats * x.rows;
    }
    cudaMemcpyAttributes attr = {};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
    size_t attr_idx = 0, fail = 0;
    e = cudaMemcpyBatchAsync(dst.data(), src.data(), size.data(), dst.size(), &attr, &attr_idx, 1, &fail,
                             c->side);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_stage[sb], c->side);
    if (e == cudaSuccess) e = cudaEventRecord(c->ev_wb, c->side);
    if (e != cudaSuccess) return e;
    for (const Xfer& x : wbs) c->wb_prev[x.spt_id] = 1;
  }
  return cudaEventRecord(c->items_done, st);
}

}  // namespace

cudaError_t cache_step(CacheTable* c, const glod_store_view& sv, int32_t n, const int32_t* spt_ids,
                       const double* d_root, const int32_t* prefix_len, double* dist_out,
                       uint64_t* block_out, int64_t* rows_out, int64_t* loaded_rows,
                       int64_t* hits, cudaStream_t st) {
  cudaError_t e = c->ensure_side();
  if (e != cudaSuccess) return e;
  // write-backs of earlier steps already finished: nothing to wait for
  if (!c->wb_prev.empty() && cudaEventQuery(c->ev_wb) == cudaSuccess) c->wb_prev.clear();
  std::vector<Xfer> loads, wbs;
  std::unordered_map<int32_t, std::pair<const double*, int64_t>> evicted;   // dirty, this step
  bool join = false;
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
      double* blk = nullptr;
      e = cudaMallocFromPoolAsync(&blk, size_t(kFloats) * size_t(P > 0 ? P : 1) * sizeof(double), c->pool, st);
      if (e != cudaSuccess) return e;
      Xfer ld{sid, c->slot_start[sid], P, blk, nullptr, 0};
      auto ev = evicted.find(sid);
      if (ev != evicted.end()) {
        // evicted (dirty) earlier in this step: the reference writes it back
        // and then reads the store, i.e. rows below the old prefix are the
        // f32 rounding of the evicted block, the rest the untouched store
        ld.overlay = ev->second.first;
        ld.overlay_rows = ev->second.second;      // its row count = its section stride
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
      c->lru.push_back({sid, d, P, blk, nbytes, false});
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
  e = run_batch(c, sv, loads, wbs, join, st);
  if (e != cudaSuccess) return e;
  *loaded_rows = c->loaded_rows - loaded0;
  *hits = c->hits - hits0;
  return cudaSuccess;
}

// Blocks dropped this step are still read by this step's kernels (the
// reference keeps its `entry` references alive): free them in main-stream
// order once the step is enqueued (their write-backs read the f32 staging
// copy, not the block).
cudaError_t cache_release(CacheTable* c, cudaStream_t st) {
  for (double* b : c->to_free) {
    cudaError_t e = cudaFreeAsync(b, st);
    if (e != cudaSuccess) return e;
  }
  c->to_free.clear();
  return cudaSuccess;
}

cudaError_t cache_end_step(CacheTable* c, const glod_store_view& sv, int64_t iteration,
                           int mark_dirty, cudaStream_t st) {
  if (mark_dirty)
    for (int32_t sid : c->step_ids) {
      auto it = c->map.find(sid);
      if (it != c->map.end()) it->second->dirty = true;
    }
  c->step_ids.clear();
  cudaError_t e = cudaSuccess;
  if (iteration >= 0 && iteration % c->flush_interval == 0) {
    std::vector<Xfer> none, wbs;
    for (auto& en : c->lru) {
      if (en.dirty) wbs.push_back({en.spt_id, c->slot_start[en.spt_id], en.prefix_len, en.block, nullptr, 0});
      c->to_free.push_back(en.block);
    }
    c->lru.clear();
    c->map.clear();
    c->resident = 0;
    e = run_batch(c, sv, none, wbs, false, st);
    if (e != cudaSuccess) return e;
  }
  return cache_release(c, st);
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
  cudaError_t e = glod::cache_step(&c->t, *store, n, spt_ids, d_root, prefix_len, dist_out, block_out,
                                   rows_out, counters_out, counters_out + 1,
                                   static_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotPermitted)
    return glod::set_error(GLOD_ERR_OVER_BUDGET, "cache entry exceeds the byte budget");
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_end_step(glod_cache* c, const glod_store_view* store, int64_t iteration,
                        int32_t mark_dirty, void* stream) {
  if (!c || !store) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = glod::cache_end_step(&c->t, *store, iteration, mark_dirty,
                                       static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_memcpy_d2h(void* dst, const void* src, int64_t bytes) {
  if (!dst || !src) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = cudaMemcpy(dst, src, size_t(bytes), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
  return GLOD_OK;
}

int glod_cache_stats(const glod_cache* c, glod_cache_stats_t* out) {
  if (!c || !out) return GLOD_ERR_INVALID_ARGUMENT;
  out->entries = int64_t(c->t.lru.size());
  out->resident_bytes = c->t.resident;
  out->hits = c->t.hits;
  out->misses = c->t.misses;
  out->loaded_rows = c->t.loaded_rows;
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
