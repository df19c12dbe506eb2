// K4: render-set gather and cache-block maintenance (trainer.py:325-364,
// store.py:304-333 data movement).
//
//  gather_rows_t render rows = master[upper ∪ passthrough] then, per selected
//                SPT, cache-block rows at the cut positions (AttributeArrays
//                .take + concat, core.py:120-159) — one transposing kernel;
//                a block row whose touched bit is set is read from the master
//                (the implicit refresh of trainer.py:363, see block_bits);
//                the train/render step fuses it into the rasteriser's
//                preprocess instead (raster.cu preprocess_plan_kernel)
//  materialize   touched rows → block (glod_cache_materialize: host reads of
//                a block; write-back and overlay take them on the fly)
//  scatter_back  explicit block[pos] = master[node] (public C-ABI)
//  convert       f32 store prefix ↔ f64 cache block (store.py:334,330)
#include <string.h>

#include "common.cuh"
#include "gather.cuh"
#include "../../include/glod_b200.h"

namespace glod {
namespace {

__constant__ int kSecOff[7] = {0, 3, 6, 10, 11, 14, 23};   // column offsets per section
__constant__ int kSecCols[6] = {3, 3, 4, 1, 3, 9};

// Column col of node `node`'s master row.
GLOD_DEV double master_val(const glod_master_ref& m, long long node, int col) {
  if (m.stride) return m.master[node * m.stride + col];
  const int off = col < 3 ? 0 : col < 6 ? 3 : col < 10 ? 6 : col < 11 ? 10 : col < 14 ? 11 : 14;
  const int cols = col < 6 ? 3 : col < 10 ? 4 : col < 11 ? 1 : col < 14 ? 3 : 9;
  return m.master[off * m.cap + node * cols + (col - off)];
}

// Rows [r0, r0 + nr) of the tile whose bit is set in `blk` (rows `rows`)
// take the master row (the implicit ADAM refresh, materialised on the fly).
GLOD_DEV void touched_from_master(float* tile, const double* blk, long long rows, long long r0, int nr,
                                  const glod_master_ref& m, long long rec_off) {
  for (int t = threadIdx.x; t < nr * 23; t += blockDim.x) {
    const int r = t / 23, col = t - r * 23;
    if (row_touched(blk, rows, r0 + r)) tile[r * 23 + col] = float(master_val(m, m.rec_node[rec_off + r0 + r], col));
  }
}

// Transposing gather: one CTA per kTRows render rows.  Row sources are
// resolved once per row into shared memory; rows are read as contiguous
// 23-value runs (node records / untouched block rows read per section) into
// a shared tile, which is written out section-major (the rasteriser's
// layout) as contiguous per-section runs.
constexpr int kTRows = 64, kTThreads = 256;

__global__ void __launch_bounds__(kTThreads)
gather_rows_t_kernel(glod_gather_plan p, long long R, double* __restrict__ out, int* __restrict__ row_node) {
  __shared__ double tile[kTRows][24];
  __shared__ const double* s_base[kTRows];
  __shared__ long long s_rows[kTRows], s_idx[kTRows];
  const long long r0 = (long long)blockIdx.x * kTRows;
  const int nr = int(min((long long)kTRows, R - r0));
  if (threadIdx.x < nr) {
    int node;
    const Src s = row_source(p, r0 + threadIdx.x, node);
    s_base[threadIdx.x] = s.base;
    s_rows[threadIdx.x] = s.rows;
    s_idx[threadIdx.x] = s.idx;
    if (row_node) row_node[r0 + threadIdx.x] = node;
  }
  __syncthreads();
  // thread t reads column c = t mod 23 of rows t/23, t/23 + 11, ... (256 =
  // 11·23 + 3; three threads idle): the column's section, offset and width
  // are fixed per thread, so an element costs one address computation
  constexpr int kRowsPerPass = kTThreads / 23;                 // 11
  constexpr int kIter = (kTRows + kRowsPerPass - 1) / kRowsPerPass;
  const int c = int(threadIdx.x) % 23, r_0 = int(threadIdx.x) / 23;
  const bool active = threadIdx.x < kRowsPerPass * 23;
  const int off = c < 3 ? 0 : c < 6 ? 3 : c < 10 ? 6 : c < 11 ? 10 : c < 14 ? 11 : 14;
  const int cols = c < 6 ? 3 : c < 10 ? 4 : c < 11 ? 1 : c < 14 ? 3 : 9;
  double v[kIter];
#pragma unroll
  for (int k = 0; k < kIter; ++k) {                // every load in flight before the tile writes
    const int lw = r_0 + k * kRowsPerPass;
    if (active && lw < nr) {
      const double* base = s_base[lw];
      const long long rows = s_rows[lw], idx = s_idx[lw];
      v[k] = rows > 0 ? base[off * rows + idx * cols + (c - off)] : base[idx * (-rows) + c];
    }
  }
#pragma unroll
  for (int k = 0; k < kIter; ++k) {
    const int lw = r_0 + k * kRowsPerPass;
    if (active && lw < nr) tile[lw][c] = v[k];
  }
  __syncthreads();
  // section-major output: per section a contiguous run of nr·cols values
  // starting at off·R + r0·cols; walk the six runs with compile-time widths
#pragma unroll
  for (int sec = 0; sec < 6; ++sec) {
    constexpr int offs[7] = {0, 3, 6, 10, 11, 14, 23};
    const int off = offs[sec], cols = offs[sec + 1] - offs[sec];
    double* dst = out + off * R + r0 * cols;
    for (int l = threadIdx.x; l < nr * cols; l += kTThreads) {
      const int lw = l / cols;
      dst[l] = tile[lw][off + l - lw * cols];
    }
  }
}

__global__ void scatter_back_kernel(glod_gather_plan p, long long n_sel) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n_sel || lane >= 23) return;
  const int j = p.sel_seg[gw];
  double* blk = reinterpret_cast<double*>(p.seg_block[j]);
  const long long P = p.seg_rows[j], pos = p.sel_pos[gw], node = p.sel_node[gw];
  int sec = 0;
#pragma unroll
  for (int k = 1; k < 6; ++k) sec += lane >= kSecOff[k];
  const int col = lane - kSecOff[sec], cols = kSecCols[sec];
  const Src m = {p.master, master_rows(p), node};
  blk[kSecOff[sec] * P + pos * cols + col] = src_at(m, kSecOff[sec], cols, col);
}

__global__ void f32_to_f64_kernel(const float4* __restrict__ in, double4* __restrict__ out, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    out[i] = make_double4(v.x, v.y, v.z, v.w);
  }
}

__global__ void f64_to_f32_kernel(const double4* __restrict__ in, float4* __restrict__ out, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const double4 v = in[i];
    out[i] = make_float4(float(v.x), float(v.y), float(v.z), float(v.w));
  }
}

__global__ void tail_f32_to_f64(const float* in, double* out, long long from, long long n) {
  const long long i = from + threadIdx.x;
  if (i < n) out[i] = in[i];
}

__global__ void tail_f64_to_f32(const double* in, float* out, long long from, long long n) {
  const long long i = from + threadIdx.x;
  if (i < n) out[i] = float(in[i]);
}

// Zero-copy store transfers: the pinned host store is mapped into the
// device address space (UVA), so one kernel moves every missed prefix of a
// step across PCIe with coalesced 128-B requests and converts f32 → f64 on
// the way (and the reverse for write-back) — no staging buffer and no
// per-range cudaMemcpy calls (a prefix is 6 ranges; a step has hundreds).
struct ItemRange {
  int lo, hi;
};

GLOD_DEV int find_item(const glod_prefix_item* items, int lo, int hi, long long e) {
  // last item with elem_start <= e
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (items[mid].elem_start <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Element l of an item's flat 23·rows index space → (row, block index).
// Section-major stores (row_stride 0) take l in block order (section, row,
// column); interleaved stores (row_stride 23: one 92-B row per slot) take
// l in row order, so the store side of every transfer is one contiguous
// run and the block side (always section-major) is computed.

struct ElemMap {
  long long row;      // prefix row
  long long blk;      // index into the section-major f64 block
  long long within;   // row·cols + column (index within the section)
  int sec;
};

GLOD_DEV ElemMap map_elem(long long l, long long rows, bool interleaved) {
  ElemMap m;
  if (interleaved) {
    m.row = l < 0xffffffffLL ? (long long)(unsigned(l) / 23u) : l / 23;
    const int col = int(l - m.row * 23);
    m.sec = (col >= 3) + (col >= 6) + (col >= 10) + (col >= 11) + (col >= 14);
    m.within = m.row * kSecCols[m.sec] + (col - kSecOff[m.sec]);
    m.blk = kSecOff[m.sec] * rows + m.within;
  } else {
    int sec = 0;
#pragma unroll
    for (int k = 1; k < 6; ++k) sec += l >= kSecOff[k] * rows;
    m.sec = sec;
    m.within = l - kSecOff[sec] * rows;
    m.row = m.within / kSecCols[sec];
    m.blk = l;
  }
  return m;
}

// sv.section[sec] without a local-memory copy of the parameter array
GLOD_DEV const float* section_of(const glod_store_view& sv, int sec) {
  const float* p = sv.section[0];
#pragma unroll
  for (int k = 1; k < 6; ++k) p = sec == k ? sv.section[k] : p;
  return p;
}

// Store address of element l of a prefix starting at slot `slot`.
GLOD_DEV float* store_at(const glod_store_view& sv, long long slot, long long l, const ElemMap& m) {
  if (sv.row_stride) return const_cast<float*>(sv.section[0]) + slot * 23 + l;
  return const_cast<float*>(section_of(sv, m.sec)) + slot * kSecCols[m.sec] + m.within;
}

// Grid-stride over 256-element chunks: the write-back runs on a side stream
// beside the main step, so its grid is capped (a few CTAs keep the posted
// PCIe writes saturated) instead of flooding every SM with long-latency
// blocks that would starve the main stream's kernels.
template <bool kLoad>
__global__ void __launch_bounds__(256)
store_xfer_kernel(glod_store_view sv, const glod_prefix_item* __restrict__ items, int n_items,
                  long long total) {
  __shared__ int s_lo, s_hi;
  const bool il = sv.row_stride != 0;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < total;
       base += (long long)gridDim.x * blockDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long last = min(total, base + (long long)blockDim.x) - 1;
      s_lo = find_item(items, 0, n_items - 1, base);
      s_hi = find_item(items, s_lo, n_items - 1, last);
    }
    __syncthreads();
    const long long e = base + threadIdx.x;
    if (e >= total) continue;
    const int it = s_lo == s_hi ? s_lo : find_item(items, s_lo, s_hi, e);
    const glod_prefix_item I = items[it];
    const long long local = e - I.elem_start;
    const long long rows = I.rows;
    if (kLoad && local < (rows + 63) / 64) block_bits(I.block, rows)[local] = 0;
    const ElemMap m = map_elem(local, rows, il);
    if (kLoad && I.src) {
      I.block[m.blk] = double(I.src[local]);    // prefetched copy in HBM (the store's layout)
    } else if (kLoad) {
      // overlay: rows below overlay_rows are the f32 rounding of a block whose
      // write-back to these store rows is still in flight (cache_table.cu)
      I.block[m.blk] = m.row < I.overlay_rows
                           ? double(float(I.overlay[kSecOff[m.sec] * I.overlay_rows + m.within]))
                           : double(*store_at(sv, I.slot_start, local, m));
    } else {
      *store_at(sv, I.slot_start, local, m) = float(I.block[m.blk]);
    }
  }
}

// View-sharded training: after the replicated ADAM on the union U of every
// rank's touched nodes, each rank's resident cache blocks must hold the new
// master values of every row any rank updated (the single-view rule
// entry.block.attrs.put(pos, h.attrs.take(node_ids)), trainer.py:363,
// applied to the union).  One thread per (node, column); a touched SPT is
// flagged so the host marks its entry dirty.
__global__ void refresh_resident_kernel(const double* __restrict__ master, long long cap, long long mstride,
                                        const int* __restrict__ ids, long long n,
                                        const int* __restrict__ spt_of_node, const int* __restrict__ rec_of_node,
                                        const unsigned long long* __restrict__ res_block,
                                        const long long* __restrict__ res_rows, int* __restrict__ touched) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 23 * n) return;
  const long long w = e / 23;
  const int col = int(e - w * 23);
  const long long id = ids[w];
  const int s = spt_of_node[id];
  if (s < 0) return;
  const long long rows = res_rows[s];
  const long long pos = rec_of_node[id];
  if (pos >= rows) return;                 // not resident / outside the cached prefix
  int sec = 0;
#pragma unroll
  for (int k = 1; k < 6; ++k) sec += col >= kSecOff[k];
  const int c = col - kSecOff[sec], cols = kSecCols[sec];
  (void)master; (void)cap; (void)mstride; (void)c; (void)cols;
  if (col == 0) {
    const double* blk = reinterpret_cast<const double*>(res_block[s]);
    atomicOr(block_bits(blk, rows) + (pos >> 6), 1ull << (pos & 63));   // implicit refresh
    touched[s] = 1;
  }
}

// Cache-path transfers driven by a block map: block b moves rows
// [chunk·kChunkRows, (chunk+1)·kChunkRows) of item bmap[b].x (chunk =
// bmap[b].y), so no thread searches the item table.  Each CTA transposes its
// rows through a shared f32 tile ([row][23], row order): the store side
// (rows of an interleaved store / prefetch copy, or six section runs of a
// section-major one) and the block side (six section runs) are both read
// and written as contiguous runs.
constexpr int kChunkRows = 88;
constexpr int kTileLd = 23;

// Section runs of rows [r0, r0 + nr) of a section-major array of `rows`
// rows: calls f(tile index, array index) for every value, consecutive
// threads on consecutive array indices.
template <typename F>
GLOD_DEV void for_section_runs(long long rows, long long r0, int nr, F f) {
#pragma unroll
  for (int sec = 0; sec < 6; ++sec) {
    constexpr int offs[7] = {0, 3, 6, 10, 11, 14, 23};
    const int off = offs[sec], cols = offs[sec + 1] - offs[sec];
    const long long base = off * rows + r0 * cols;
    for (int i = threadIdx.x; i < nr * cols; i += blockDim.x) {
      const int r = i / cols;
      f(r * kTileLd + off + (i - r * cols), base + i);
    }
  }
}

__global__ void __launch_bounds__(256)
load_blocks_kernel(glod_store_view sv, const glod_prefix_item* __restrict__ items,
                   const int2* __restrict__ bmap, glod_master_ref mref) {
  __shared__ float tile[kChunkRows * kTileLd];
  const int2 bm = bmap[blockIdx.x];
  const glod_prefix_item I = items[bm.x];
  const long long r0 = (long long)bm.y * kChunkRows;
  const int nr = int(min((long long)kChunkRows, I.rows - r0));
  const bool il = sv.row_stride != 0;
  if (bm.y == 0)                                 // a freshly loaded block: no row touched
    for (long long w = threadIdx.x; w < (I.rows + 63) / 64; w += blockDim.x) block_bits(I.block, I.rows)[w] = 0;
  // 1. the prefix rows in f32, from the prefetch / disk copy in HBM or the
  //    mapped store, laid out like the store
  if (il) {
    const float* src = I.src ? I.src + r0 * 23 : sv.section[0] + (I.slot_start + r0) * 23;
    for (int i = threadIdx.x; i < nr * 23; i += blockDim.x) tile[i] = src[i];
  } else if (I.src) {
    for_section_runs(I.rows, r0, nr, [&](int t, long long k) { tile[t] = I.src[k]; });
  } else {
#pragma unroll
    for (int sec = 0; sec < 6; ++sec) {
      constexpr int offs[7] = {0, 3, 6, 10, 11, 14, 23};
      const int off = offs[sec], cols = offs[sec + 1] - offs[sec];
      const float* src = section_of(sv, sec) + (I.slot_start + r0) * cols;
      for (int i = threadIdx.x; i < nr * cols; i += blockDim.x) {
        const int r = i / cols;
        tile[r * kTileLd + off + (i - r * cols)] = src[i];
      }
    }
  }
  // 2. overlay: rows below overlay_rows are the f32 rounding of a block whose
  //    write-back to these store rows is still in flight (cache_table.cu)
  const int nov = int(max(0LL, min((long long)nr, I.overlay_rows - r0)));
  if (nov > 0) {
    __syncthreads();
    for_section_runs(I.overlay_rows, r0, nov, [&](int t, long long k) { tile[t] = float(I.overlay[k]); });
    if (mref.master) {                           // its touched rows hold the master values
      __syncthreads();
      touched_from_master(tile, I.overlay, I.overlay_rows, r0, nov, mref, mref.item_rec_off[bm.x]);
    }
  }
  __syncthreads();
  // 3. the f64 block, section-major
  for_section_runs(I.rows, r0, nr, [&](int t, long long k) { I.block[k] = double(tile[t]); });
}

// Write-back staging: the block as f32 in the store's layout (row order for
// an interleaved store, so one copy per prefix moves it).
__global__ void __launch_bounds__(256)
pack_blocks_kernel(const glod_prefix_item* __restrict__ items, const int2* __restrict__ bmap,
                   float* __restrict__ out, int interleaved, glod_master_ref mref) {
  __shared__ float tile[kChunkRows * kTileLd];
  const int2 bm = bmap[blockIdx.x];
  const glod_prefix_item I = items[bm.x];
  const long long r0 = (long long)bm.y * kChunkRows;
  const int nr = int(min((long long)kChunkRows, I.rows - r0));
  float* o = out + I.elem_start;
  if (!interleaved && !mref.master) {  // same layout as the block: a straight convert
    for_section_runs(I.rows, r0, nr, [&](int, long long k) { o[k] = float(I.block[k]); });
    return;
  }
  for_section_runs(I.rows, r0, nr, [&](int t, long long k) { tile[t] = float(I.block[k]); });
  if (mref.master) {                   // touched rows are written back with their master values
    __syncthreads();
    touched_from_master(tile, I.block, I.rows, r0, nr, mref, mref.item_rec_off[bm.x]);
  }
  __syncthreads();
  if (!interleaved) {
    for_section_runs(I.rows, r0, nr, [&](int t, long long k) { o[k] = tile[t]; });
    return;
  }
  float* dst = o + r0 * 23;
  for (int i = threadIdx.x; i < nr * 23; i += blockDim.x) dst[i] = tile[i];
}

// Materialise touched rows before a block is written back / overlaid: one
// thread per block row (items tile a flat row space; elem_start = 23 ·
// earlier rows); a touched row copies its 23 master values (one contiguous
// record run) into the block.  Bits stay set (the row now equals the
// master, so either source gives the same value).
__global__ void __launch_bounds__(256)
materialize_kernel(const glod_mat_item* __restrict__ items, int n_items, long long total_rows,
                   const double* __restrict__ master, long long cap, long long mstride,
                   const int* __restrict__ rec_node) {
  __shared__ int s_lo, s_hi;
  const long long base = (long long)blockIdx.x * blockDim.x;
  if (threadIdx.x == 0) {                           // items covering this CTA's rows
    const long long last = min(total_rows, base + (long long)blockDim.x) - 1;
    int lo = 0, hi = n_items - 1;
    while (lo < hi) { const int m = (lo + hi + 1) >> 1; if (items[m].elem_start / 23 <= base) lo = m; else hi = m - 1; }
    s_lo = lo;
    hi = n_items - 1;
    while (lo < hi) { const int m = (lo + hi + 1) >> 1; if (items[m].elem_start / 23 <= last) lo = m; else hi = m - 1; }
    s_hi = lo;
  }
  __syncthreads();
  const long long e = base + threadIdx.x;
  if (e >= total_rows) return;
  int lo = s_lo, hi = s_hi;
  while (lo < hi) { const int m = (lo + hi + 1) >> 1; if (items[m].elem_start / 23 <= e) lo = m; else hi = m - 1; }
  const glod_mat_item I = items[lo];
  const long long row = e - I.elem_start / 23;
  if (!row_touched(I.block, I.rows, row)) return;
  const long long node = rec_node[I.rec_offset + row];
  const Src m = {master, mstride ? -mstride : cap, node};
  double v[23];
#pragma unroll
  for (int col = 0; col < 23; ++col) {
    const int sec = col < 3 ? 0 : col < 6 ? 1 : col < 10 ? 2 : col < 11 ? 3 : col < 14 ? 4 : 5;
    constexpr int offs[6] = {0, 3, 6, 10, 11, 14};
    v[col] = src_at(m, offs[sec], (sec == 2 ? 4 : sec == 3 ? 1 : sec == 5 ? 9 : 3), col - offs[sec]);
  }
#pragma unroll
  for (int col = 0; col < 23; ++col) {
    const int sec = col < 3 ? 0 : col < 6 ? 1 : col < 10 ? 2 : col < 11 ? 3 : col < 14 ? 4 : 5;
    constexpr int offs[6] = {0, 3, 6, 10, 11, 14};
    const int cols = sec == 2 ? 4 : sec == 3 ? 1 : sec == 5 ? 9 : 3;
    I.block[offs[sec] * I.rows + row * cols + (col - offs[sec])] = v[col];
  }
}

// Small device→host read-backs written by a kernel straight into mapped
// pinned memory: no copy-engine queueing behind the cache's bulk D2H
// write-back DMA (which would delay the step's host synchronisations).
__global__ void readback_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                long long bytes) {
  const long long words = bytes >> 2;
  const unsigned* s4 = reinterpret_cast<const unsigned*>(src);
  unsigned* d4 = reinterpret_cast<unsigned*>(dst);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x)
    d4[i] = s4[i];
  if (blockIdx.x == 0 && threadIdx.x < (bytes & 3)) dst[(words << 2) + threadIdx.x] = src[(words << 2) + threadIdx.x];
}

// Wire payloads of ServeSession.handle_pose (protocol.py:40-49,80-92): for
// message k (rows [seg[k], seg[k+1]) of ids), the section-major f32 SoA of
// master rows ids[...] at out + 23·seg[k].  blockIdx.y = section; one thread
// per (row, column): consecutive threads write consecutive floats of one
// message section (the out buffer may be mapped pinned host memory).
template <int SEC>
GLOD_DEV void wire_sec(const double* __restrict__ master, long long cap, const int* __restrict__ ids,
                       const long long* __restrict__ seg, int n_msgs, long long N, float* __restrict__ out) {
  constexpr int OFFS[7] = {0, 3, 6, 10, 11, 14, 23};
  constexpr int COLS = OFFS[SEC + 1] - OFFS[SEC];
  const long long local = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= N * COLS) return;
  const long long r = local / COLS;
  const int col = int(local - r * COLS);
  int lo = 0, hi = n_msgs - 1;                      // last k with seg[k] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid] <= r) lo = mid; else hi = mid - 1;
  }
  const long long a = seg[lo], n = seg[lo + 1] - a;
  const long long node = ids[r];
  out[23 * a + OFFS[SEC] * n + (r - a) * COLS + col] =
      __double2float_rn(master[OFFS[SEC] * cap + node * COLS + col]);
}

__global__ void __launch_bounds__(256)
wire_pack_kernel(const double* __restrict__ master, long long cap, const int* __restrict__ ids,
                 const long long* __restrict__ seg, int n_msgs, long long N, float* __restrict__ out) {
  switch (blockIdx.y) {
    case 0: wire_sec<0>(master, cap, ids, seg, n_msgs, N, out); break;
    case 1: wire_sec<1>(master, cap, ids, seg, n_msgs, N, out); break;
    case 2: wire_sec<2>(master, cap, ids, seg, n_msgs, N, out); break;
    case 3: wire_sec<3>(master, cap, ids, seg, n_msgs, N, out); break;
    case 4: wire_sec<4>(master, cap, ids, seg, n_msgs, N, out); break;
    case 5: wire_sec<5>(master, cap, ids, seg, n_msgs, N, out); break;
  }
}

int grid_for(long long n, int tb) {
  long long g = (n + tb - 1) / tb;
  return int(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace

cudaError_t launch_gather(const glod_gather_plan& p, long long R, double* out, int* row_node,
                          cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  const int TB = 256;
  count_launch();
  gather_rows_t_kernel<<<unsigned((R + kTRows - 1) / kTRows), kTThreads, 0, st>>>(p, R, out, row_node);
  return cudaGetLastError();
}

cudaError_t launch_wire_pack(const double* master, long long cap, const int* ids, const long long* seg,
                             int n_msgs, long long N, float* out, cudaStream_t st) {
  if (N <= 0 || n_msgs <= 0) return cudaSuccess;
  count_launch();
  const dim3 grid(unsigned((9 * N + 255) / 256), 6);
  wire_pack_kernel<<<grid, 256, 0, st>>>(master, cap, ids, seg, n_msgs, N, out);
  return cudaGetLastError();
}

cudaError_t launch_materialize(const glod_mat_item* items, int n_items, long long total, const double* master,
                               long long cap, long long mstride, const int* rec_node, cudaStream_t st) {
  if (total <= 0 || n_items <= 0) return cudaSuccess;
  count_launch();
  const long long rows = total / 23;
  materialize_kernel<<<unsigned((rows + 255) / 256), 256, 0, st>>>(items, n_items, rows, master, cap, mstride,
                                                                   rec_node);
  return cudaGetLastError();
}

cudaError_t launch_scatter_back(const glod_gather_plan& p, cudaStream_t st) {
  if (p.n_sel <= 0) return cudaSuccess;
  const int TB = 256;
  count_launch();
  scatter_back_kernel<<<int((p.n_sel * 32 + TB - 1) / TB), TB, 0, st>>>(p, p.n_sel);
  return cudaGetLastError();
}

cudaError_t launch_convert(const void* in, void* out, long long n, int to_f64, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long n4 = n / 4;
  const int TB = 256;
  if (to_f64) {
    if (n4) { count_launch(); f32_to_f64_kernel<<<grid_for(n4, TB), TB, 0, st>>>((const float4*)in, (double4*)out, n4); }
    if (n % 4) { count_launch(); tail_f32_to_f64<<<1, 4, 0, st>>>((const float*)in, (double*)out, n4 * 4, n); }
  } else {
    if (n4) { count_launch(); f64_to_f32_kernel<<<grid_for(n4, TB), TB, 0, st>>>((const double4*)in, (float4*)out, n4); }
    if (n % 4) { count_launch(); tail_f64_to_f32<<<1, 4, 0, st>>>((const double*)in, (float*)out, n4 * 4, n); }
  }
  return cudaGetLastError();
}

cudaError_t launch_readback(void* host_pinned, const void* src, long long bytes, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  void* dst = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dst, host_pinned, 0);
  if (e != cudaSuccess) return e;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3) {
    return cudaMemcpyAsync(host_pinned, src, size_t(bytes), cudaMemcpyDeviceToHost, st);
  }
  const long long words = (bytes + 3) >> 2;
  const int grid = int(words > 256 * 64 ? 64 : (words + 255) / 256);
  count_launch();
  readback_kernel<<<grid, 256, 0, st>>>(static_cast<const unsigned char*>(src),
                                        static_cast<unsigned char*>(dst), bytes);
  return cudaGetLastError();
}

// Up to 8 read-backs in one launch (blockIdx.y = range): the select's four
// per-view tables cost one kernel instead of four.
namespace {
struct ReadbackList {
  const unsigned* src[8];
  unsigned* dst[8];
  long long words[8];
};
__global__ void readback_multi_kernel(ReadbackList L) {
  const int r = blockIdx.y;
  const unsigned* __restrict__ s = L.src[r];
  unsigned* __restrict__ d = L.dst[r];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < L.words[r];
       i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}
}  // namespace

cudaError_t launch_readback_multi(int n, void* const* host_pinned, const void* const* src, const long long* bytes,
                                  cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > 8) return cudaErrorInvalidValue;
  ReadbackList L = {};
  long long maxw = 0;
  for (int r = 0; r < n; ++r) {
    void* dst = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dst, host_pinned[r], 0);
    if (e != cudaSuccess) return e;
    if (((reinterpret_cast<uintptr_t>(src[r]) | reinterpret_cast<uintptr_t>(dst)) & 3) || (bytes[r] & 3))
      return cudaErrorInvalidValue;
    L.src[r] = static_cast<const unsigned*>(src[r]);
    L.dst[r] = static_cast<unsigned*>(dst);
    L.words[r] = bytes[r] > 0 ? bytes[r] >> 2 : 0;
    maxw = L.words[r] > maxw ? L.words[r] : maxw;
  }
  const int gx = int(maxw > 256 * 16 ? 16 : (maxw + 255) / 256 > 0 ? (maxw + 255) / 256 : 1);
  count_launch();
  readback_multi_kernel<<<dim3(gx, n), 256, 0, st>>>(L);
  return cudaGetLastError();
}

// Stream-ordered small host→device upload from page-locked memory, read by
// a kernel through the mapped address: the copy engines may be busy with
// the cache's bulk prefetch DMA, and a main-stream cudaMemcpyAsync would
// queue behind it.  Pageable sources fall back to cudaMemcpyAsync.
cudaError_t launch_upload(void* dst, const void* host_pinned, long long bytes, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  void* src = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&src, const_cast<void*>(host_pinned), 0);
  if (e != cudaSuccess || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3)) {
    cudaGetLastError();
    return cudaMemcpyAsync(dst, host_pinned, size_t(bytes), cudaMemcpyHostToDevice, st);
  }
  const long long words = (bytes + 3) >> 2;
  const int grid = int(words > 256 * 64 ? 64 : (words + 255) / 256);
  count_launch();
  readback_kernel<<<grid, 256, 0, st>>>(static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                        bytes);
  return cudaGetLastError();
}

namespace {
struct Bytes64 {
  unsigned long long w[8];
};
__global__ void set_bytes_kernel(unsigned long long* dst, Bytes64 v, int words) {
  if (int(threadIdx.x) < words) dst[threadIdx.x] = v.w[threadIdx.x];
}
}  // namespace

// Stream-ordered write of ≤ 64 host bytes (a multiple of 8; dst 8-aligned)
// carried in the kernel parameters — for initial values that would
// otherwise be a pageable cudaMemcpyAsync through the copy engine.
cudaError_t launch_set_bytes(void* dst, const void* src, int bytes, cudaStream_t st) {
  if (bytes <= 0 || bytes > 64 || (bytes & 7) || (reinterpret_cast<uintptr_t>(dst) & 7))
    return cudaErrorInvalidValue;
  Bytes64 v = {};
  memcpy(v.w, src, size_t(bytes));
  count_launch();
  set_bytes_kernel<<<1, 32, 0, st>>>(static_cast<unsigned long long*>(dst), v, bytes / 8);
  return cudaGetLastError();
}

cudaError_t launch_refresh_resident(const double* master, long long cap, long long mstride, const int* ids,
                                    long long n,
                                    const int* spt_of_node, const int* rec_of_node,
                                    const unsigned long long* res_block, const long long* res_rows, int* touched,
                                    cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  refresh_resident_kernel<<<unsigned((23 * n + 255) / 256), 256, 0, st>>>(master, cap, mstride, ids, n, spt_of_node,
                                                                           rec_of_node, res_block, res_rows, touched);
  return cudaGetLastError();
}

long long transfer_chunks(long long rows) { return (rows + kChunkRows - 1) / kChunkRows; }

cudaError_t launch_load_blocks(const glod_store_view& sv, const glod_prefix_item* items, const int2* bmap,
                               long long nblocks, const glod_master_ref& mref, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  count_launch();
  load_blocks_kernel<<<unsigned(nblocks), 256, 0, st>>>(sv, items, bmap, mref);
  return cudaGetLastError();
}

cudaError_t launch_pack_blocks(const glod_prefix_item* items, const int2* bmap, long long nblocks, float* out,
                               int interleaved, const glod_master_ref& mref, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  count_launch();
  pack_blocks_kernel<<<unsigned(nblocks), 256, 0, st>>>(items, bmap, out, interleaved, mref);
  return cudaGetLastError();
}

cudaError_t launch_store_xfer(const glod_store_view& sv, const glod_prefix_item* items, int n_items,
                              long long total, int load, cudaStream_t st) {
  if (n_items <= 0 || total <= 0) return cudaSuccess;
  const int TB = 256;
  const long long nb = (total + TB - 1) / TB;
  // loads: 8 CTAs/SM in flight hide the PCIe read latency; write-backs
  // (posted writes, side stream): one CTA per SM
  const long long cap = load ? 148 * 8 : 148;
  const unsigned grid = unsigned(nb < cap ? nb : cap);
  count_launch();
  if (load)
    store_xfer_kernel<true><<<grid, TB, 0, st>>>(sv, items, n_items, total);
  else
    store_xfer_kernel<false><<<grid, TB, 0, st>>>(sv, items, n_items, total);
  return cudaGetLastError();
}

}  // namespace glod
