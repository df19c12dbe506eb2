// Native device-cache table (cache.py:42-109 + the gather loop of
// trainer.py:329-345 / cli._gather cli.py:111-136).
//
// Host-side decision logic identical to the reference (ratio band, LRU,
// byte budget counted as prefix_len·92, replacement returns the old dirty
// block, flush every flush_interval iterations) over cache blocks that live
// in HBM.  Blocks are packed f64 attribute blocks allocated stream-ordered
// (cudaMallocAsync) and released stream-ordered after their write-back, so
// a whole step's cache work is one C call: decisions, then batched
// zero-copy store transfers (loads before write-backs, a batch closed
// whenever an SPT about to be loaded has a write-back pending).
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
  // transfer staging
  glod_prefix_item* h_items = nullptr;    // pinned
  glod_prefix_item* d_items = nullptr;
  size_t items_cap = 0;
  std::vector<int32_t> step_ids;          // SPTs rendered this step (dirty at end)
  std::vector<double*> to_free;           // blocks freed after their write-back
  int device = 0;
  cudaEvent_t items_done = nullptr;       // last H2D from the pinned item table
  // Write-backs run on a side stream so the D2H PCIe direction overlaps the
  // rest of the step; the main stream waits for them before anything that
  // could observe the store (the next loads) or reuse a written-back block.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_main = nullptr, ev_wb = nullptr;
  bool wb_pending = false;

  cudaError_t ensure_side() {
    if (side) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_wb, cudaEventDisableTiming);
    return e;
  }

  // main stream waits for outstanding write-backs
  cudaError_t join(cudaStream_t st) {
    if (!wb_pending) return cudaSuccess;
    wb_pending = false;
    return cudaStreamWaitEvent(st, ev_wb, 0);
  }

  ~CacheTable() {
    if (side) cudaStreamSynchronize(side);
    if (items_done) cudaEventDestroy(items_done);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_wb) cudaEventDestroy(ev_wb);
    if (side) cudaStreamDestroy(side);
    for (auto& e : lru) cudaFree(e.block);
    if (h_items) cudaFreeHost(h_items);
    if (d_items) cudaFree(d_items);
  }

  cudaError_t ensure_items(size_t n) {
    if (!items_done) {
      cudaError_t e = cudaEventCreateWithFlags(&items_done, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    // the pinned table is rewritten below: its previous copies must be done
    cudaEventSynchronize(items_done);
    if (n <= items_cap) return cudaSuccess;
    size_t want = n * 2 + 64;
    // outstanding copies from the old pinned table must finish first
    cudaDeviceSynchronize();
    if (h_items) cudaFreeHost(h_items);
    if (d_items) cudaFree(d_items);
    cudaError_t e = cudaMallocHost(&h_items, want * sizeof(glod_prefix_item));
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&d_items, want * sizeof(glod_prefix_item));
    if (e != cudaSuccess) return e;
    items_cap = want;
    return cudaSuccess;
  }
};

namespace {

struct Xfer {
  int64_t slot, rows;
  double* block;
};

// Runs one batch: all loads (main stream), then all write-backs (side
// stream, after the loads), from one pinned item table.
cudaError_t run_batch(CacheTable* c, const glod_store_view& sv, std::vector<Xfer>& loads,
                      std::vector<Xfer>& wbs, size_t& table_off, cudaStream_t st) {
  cudaError_t e = c->ensure_side();
  if (e != cudaSuccess) return e;
  // loads observe every earlier write-back, and the device item table is
  // not rewritten while a write-back kernel may still read it
  e = c->join(st);
  if (e != cudaSuccess) return e;
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<Xfer>& v = pass == 0 ? loads : wbs;
    if (v.empty()) continue;
    glod_prefix_item* h = c->h_items + table_off;
    int64_t off = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      h[i].slot_start = v[i].slot;
      h[i].rows = v[i].rows;
      h[i].elem_start = off;
      h[i].block = v[i].block;
      off += kFloats * v[i].rows;
    }
    glod_prefix_item* d = c->d_items + table_off;
    e = cudaMemcpyAsync(d, h, v.size() * sizeof(glod_prefix_item), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(c->items_done, st);
    if (e != cudaSuccess) return e;
    if (pass == 0) {
      e = launch_store_xfer(sv, d, int(v.size()), off, 1, st);
    } else {
      // side stream: after this batch's loads and the item-table copy
      e = cudaEventRecord(c->ev_main, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c->side, c->ev_main, 0);
      if (e == cudaSuccess) e = launch_store_xfer(sv, d, int(v.size()), off, 0, c->side);
      if (e == cudaSuccess) e = cudaEventRecord(c->ev_wb, c->side);
      c->wb_pending = true;
    }
    if (e != cudaSuccess) return e;
    table_off += v.size();
    v.clear();
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t cache_step(CacheTable* c, const glod_store_view& sv, int32_t n, const int32_t* spt_ids,
                       const double* d_root, const int32_t* prefix_len, double* dist_out,
                       uint64_t* block_out, int64_t* rows_out, int64_t* loaded_rows,
                       int64_t* hits, cudaStream_t st) {
  // worst case: one load + every resident entry written back per selected SPT
  cudaError_t e = c->ensure_items(2 * size_t(n) + c->lru.size() + 1);
  if (e != cudaSuccess) return e;
  std::vector<Xfer> loads, wbs;
  std::vector<int32_t> wb_ids;
  size_t table_off = 0;
  const int64_t hits0 = c->hits, loaded0 = c->loaded_rows;
  c->step_ids.assign(spt_ids, spt_ids + n);
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
      bool pending = false;
      for (int32_t w : wb_ids) pending |= (w == sid);
      if (pending) {
        e = run_batch(c, sv, loads, wbs, table_off, st);
        if (e != cudaSuccess) return e;
        wb_ids.clear();
      }
      double* blk = nullptr;
      e = cudaMallocAsync(&blk, size_t(kFloats) * size_t(P > 0 ? P : 1) * sizeof(double), st);
      if (e != cudaSuccess) return e;
      loads.push_back({c->slot_start[sid], P, blk});
      c->loaded_rows += P;
      // insert: replace (old dirty block written back), append, evict LRU front
      if (it != c->map.end()) {
        Entry old = *it->second;
        c->lru.erase(it->second);
        c->map.erase(sid);
        c->resident -= old.nbytes;
        if (old.dirty) {
          wbs.push_back({c->slot_start[old.spt_id], old.prefix_len, old.block});
          wb_ids.push_back(old.spt_id);
        }
        c->to_free.push_back(old.block);
      }
      c->lru.push_back({sid, d, P, blk, nbytes, false});
      c->map[sid] = std::prev(c->lru.end());
      c->resident += nbytes;
      while (c->resident > c->budget) {
        Entry v = c->lru.front();
        c->lru.pop_front();
        c->map.erase(v.spt_id);
        c->resident -= v.nbytes;
        if (v.dirty) {
          wbs.push_back({c->slot_start[v.spt_id], v.prefix_len, v.block});
          wb_ids.push_back(v.spt_id);
        }
        c->to_free.push_back(v.block);
      }
      it = c->map.find(sid);
    }
    const Entry& en = *c->map.find(sid)->second;
    dist_out[j] = en.cached_distance;
    block_out[j] = reinterpret_cast<uint64_t>(en.block);
    rows_out[j] = en.prefix_len;
  }
  e = run_batch(c, sv, loads, wbs, table_off, st);
  if (e != cudaSuccess) return e;
  *loaded_rows = c->loaded_rows - loaded0;
  *hits = c->hits - hits0;
  return cudaSuccess;
}

// Blocks evicted this step are still read by this step's render (the
// reference keeps its `entry` references alive) — release them only once
// the step's kernels are enqueued.
cudaError_t cache_release(CacheTable* c, cudaStream_t st) {
  if (c->to_free.empty()) return cudaSuccess;
  cudaError_t j = c->join(st);     // a freed block may still be being written back
  if (j != cudaSuccess) return j;
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
    e = c->ensure_items(c->lru.size() + 1);
    if (e != cudaSuccess) return e;
    std::vector<Xfer> none, wbs;
    for (auto& en : c->lru) {
      if (en.dirty) wbs.push_back({c->slot_start[en.spt_id], en.prefix_len, en.block});
      c->to_free.push_back(en.block);
    }
    c->lru.clear();
    c->map.clear();
    c->resident = 0;
    size_t off = 0;
    e = run_batch(c, sv, none, wbs, off, st);
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
