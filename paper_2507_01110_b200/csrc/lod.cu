// LoD selection on the device.
//
// K2 `select_kernel` replaces cut_hspt stage 1 (hspt.py:122-144) together
// with the passthrough bfs_cut calls it makes (hierarchy.py:244-266) and the
// per-SPT root distance / prefix search of stage 2 (hspt.py:147-153,
// spt.py:70).  One cooperative launch walks every BFS (the upper tree and
// all passthrough subtrees at once) level-synchronously with a software
// grid barrier between levels, marks the selections in bitmaps, compacts
// the bitmaps into sorted id lists (the reference's np.sort), then computes
// d_root and prefix_len for every selected SPT.
//
// K1 `compact_kernel` replaces cut_spt's interval test (spt.py:71-75) for
// all selected SPTs at once: the selected prefixes are laid end to end in a
// virtual index space and compacted by a single order-preserving pass with
// decoupled look-back, so each key_self is read exactly once.
#include <climits>

#include "common.cuh"
#include "lod.cuh"

namespace glod {

namespace {

constexpr int kSelectThreads = 512;
constexpr int kAlign = 4;                         // records per group (16-B vector loads)
constexpr int kMaxLevels = 250;

constexpr uint32_t kPass = 1u << 31;   // entry belongs to a passthrough BFS
constexpr uint32_t kStart = 1u << 30;  // first frontier of its BFS (size 1 → gemv order)
constexpr uint32_t kIdMask = kStart - 1;

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct SelectScratch {
  unsigned int* bar;        // [2]
  unsigned int* lvl_count;  // [kMaxLevels+1]
  uint32_t* bm_upper;
  uint32_t* bm_pass;
  uint32_t* bm_spt;
  uint32_t* frontier[2];
  long long* block_cnt;     // [3*grid]
  size_t zero_bytes;        // bytes to clear from bar onwards
};

SelectScratch carve_select(void* base, int64_t cap, int32_t S, int grid) {
  SelectScratch s;
  char* p = static_cast<char*>(base);
  size_t w_nodes = (size_t(cap) + 31) / 32, w_spt = (size_t(S) + 31) / 32;
  s.bar = reinterpret_cast<unsigned int*>(p);
  s.lvl_count = s.bar + 2;
  size_t off = align_up(sizeof(unsigned int) * (kMaxLevels + 3));
  s.bm_upper = reinterpret_cast<uint32_t*>(p + off); off += 4 * w_nodes;
  s.bm_pass = reinterpret_cast<uint32_t*>(p + off); off += 4 * w_nodes;
  s.bm_spt = reinterpret_cast<uint32_t*>(p + off); off += 4 * w_spt;
  s.zero_bytes = off;
  off = align_up(off);
  s.frontier[0] = reinterpret_cast<uint32_t*>(p + off); off = align_up(off + 4 * size_t(cap) + 4);
  s.frontier[1] = reinterpret_cast<uint32_t*>(p + off); off = align_up(off + 4 * size_t(cap) + 4);
  s.block_cnt = reinterpret_cast<long long*>(p + off);
  return s;
}

GLOD_DEV bool sphere_in_frustum(const double* P, double x, double y, double z,
                                double r, bool gemv) {
  // sphere_intersects_frustum (core.py:364-372): signed = c @ P[:, :3].T + P[:, 3].
  // numpy's matmul goes to OpenBLAS: dgemm for a frontier of ≥2 rows,
  // dgemv for a single row; their FMA chains differ.
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double a = P[4 * k], b = P[4 * k + 1], c = P[4 * k + 2], d = P[4 * k + 3];
    double s = gemv ? fma_(z, c, fma_(x, a, mul(y, b))) : fma_(z, c, fma_(y, b, mul(x, a)));
    s = add(s, d);
    if (!(s <= r)) return false;
  }
  return true;
}

// #{kp[i] > d} over a descending run (np.searchsorted(-key_parent, -d,
// 'left')) by one warp: 32-ary ballot search, ⌈log32 n⌉ dependent loads
// instead of log2 n.  Every lane returns the count.
template <typename K>
GLOD_DEV int warp_count_gt(const K* kp, long long n, double d, int lane) {
  long long a = 0, b = n;
  while (b - a > 32) {
    const long long step = (b - a + 31) / 32;
    const long long probe = a + step * lane;
    const bool gt = probe < b && (probe == a || double(kp[probe]) > d);
    const unsigned m = __ballot_sync(0xffffffffu, gt);
    const int last = 31 - __clz(m);
    const long long na = a + step * last;
    b = min(b, na + step);
    a = na;
  }
  const long long probe = a + lane;
  const bool gt = probe < b && double(kp[probe]) > d;
  return int(a + __popc(__ballot_sync(0xffffffffu, gt)));
}

GLOD_DEV double key_self_at(const LodScene& sc, int64_t rec) {
  return sc.key_f64 ? static_cast<const double*>(sc.key_self)[rec]
                    : double(static_cast<const float*>(sc.key_self)[rec]);
}

// Contiguous [lo, hi) share of `n` items for block b of g.
GLOD_DEV void block_range(long long n, int b, int g, long long& lo, long long& hi) {
  lo = n * b / g;
  hi = n * (b + 1) / g;
}

GLOD_DEV long long block_sum(long long v, long long* sm) {
  block_excl_scan(v, sm);
  const int nw = (blockDim.x + 31) >> 5;
  long long t = sm[nw];
  __syncthreads();
  return t;
}

// Phase A of a grid-wide bitmap compaction: popcount of this block's words.
GLOD_DEV long long bitmap_block_count(const uint32_t* bm, long long nwords, long long* sm) {
  long long lo, hi;
  block_range(nwords, blockIdx.x, gridDim.x, lo, hi);
  long long c = 0;
  for (long long w = lo + threadIdx.x; w < hi; w += blockDim.x) c += __popc(ld_cg(bm + w));
  return block_sum(c, sm);
}

// Phase B: write the set bit positions of this block's words, in order.
GLOD_DEV void bitmap_block_write(const uint32_t* bm, long long nwords, long long nbits,
                                 long long base, int32_t* out, long long* sm) {
  long long lo, hi;
  block_range(nwords, blockIdx.x, gridDim.x, lo, hi);
  long long span = hi - lo;
  long long chunk = (span + blockDim.x - 1) / blockDim.x;
  long long w0 = lo + chunk * threadIdx.x, w1 = min(hi, w0 + chunk);
  long long c = 0;
  for (long long w = w0; w < w1; ++w) c += __popc(ld_cg(bm + w));
  long long o = base + block_excl_scan(c, sm);
  for (long long w = w0; w < w1; ++w) {
    uint32_t bits = ld_cg(bm + w);
    while (bits) {
      int b = __ffs(bits) - 1;
      bits &= bits - 1;
      long long id = w * 32 + b;
      if (id < nbits) out[o++] = int32_t(id);
    }
  }
}

GLOD_DEV long long sum_before(const long long* cnt, int b, long long* sm) {
  long long v = 0;
  for (int i = threadIdx.x; i < b; i += blockDim.x) v += ld_cg(cnt + i);
  return block_sum(v, sm);
}

// Phase timestamps of the last select launch (block 0; diagnostics only:
// glod_debug_select_phases).
__device__ unsigned long long g_sel_ts[8];
GLOD_DEV void sel_stamp(int k) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sel_ts[k] = t;
  }
}

__global__ void __launch_bounds__(kSelectThreads)
select_kernel(LodScene sc, LodView v, SelectOut out, SelectScratch ws) {
  sel_stamp(0);
  __shared__ long long sm[kSelectThreads / 32 + 1];
  __shared__ double planes[24];
  if (threadIdx.x < 24) planes[threadIdx.x] = v.planes[threadIdx.x];
  const int lane = threadIdx.x & 31;
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const long long gwarp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll;
  if (!sc.cand) {                        // the level-synchronous BFS starts at the root
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ws.frontier[0][0] = uint32_t(sc.root) | kStart;
      ws.lvl_count[0] = 1;
    }
    grid_sync(ws.bar);
  }

  int level = 0;
  if (sc.cand) {
    // ---- every candidate at once (no BFS levels) ----
    // A node is visited by the level-synchronous BFS iff every proper
    // ancestor up to the BFS start was kept by the cull and expanded (not
    // taken): phase 1 evaluates each candidate's own tests into a flag byte
    // (bit0 kept with the dgemm order, bit1 kept with the dgemv order used
    // for the first frontier of a BFS — the root and passthrough starts —,
    // bit2 taken: dist >= m_d, bit3 leaf); phase 2 walks each candidate's
    // ancestor chain over those bytes and applies the BFS's rules (bit4:
    // passthrough root, bit5: passthrough root expanded by its own bfs_cut).
    uint8_t* flags = reinterpret_cast<uint8_t*>(ws.frontier[0]);
    const long long as = sc.attr_stride ? sc.attr_stride : 3;
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long i = gtid; i < sc.num_cand; i += gthreads) {
      const int node = sc.cand[i];
      const double* mp = sc.means + as * node;
      const double* sp = sc.scales + as * node;
      const double mx = mp[0], my = mp[1], mz = mp[2];
      const double s0 = sp[0], s1 = sp[1], s2 = sp[2];
      unsigned f = 3;
      if (v.cull) {
        const double r = mul(3.0, max3(s0, s1, s2));
        f = (sphere_in_frustum(planes, mx, my, mz, r, false) ? 1u : 0u) |
            (sphere_in_frustum(planes, mx, my, mz, r, true) ? 2u : 0u);
      }
      const double dist = norm3_plain(sub(mx, v.position[0]), sub(my, v.position[1]), sub(mz, v.position[2]));
      const double md = min_distance(v.threshold, v.metric, s0, s1, s2);
      if (dist >= md) f |= 4u;
      if (sc.children[2 * node] == -1) f |= 8u;
      if (sc.kind[node] == -2) f |= 16u;
      flags[node] = uint8_t(f);
    }
    grid_sync(ws.bar);
    sel_stamp(1);
    // phase 2a: the upper-BFS candidates (upper nodes, SPT roots,
    // passthrough roots — cand[0, num_cand_upper)): walk to the root; a
    // visited passthrough root that its own bfs_cut expands gets bit 5
    for (long long i = gtid; i < sc.num_cand_upper; i += gthreads) {
      const int node = sc.cand[i];
      bool ok = true;
      for (int c = node; c != sc.root;) {
        const int a = sc.parent[c];
        const unsigned fa = ld_cg(flags + a);
        if (!((fa & (a == sc.root ? 2u : 1u)) && !(fa & 4u))) { ok = false; break; }
        c = a;
      }
      if (!ok) continue;
      const int kd = sc.kind[node];
      const unsigned f = ld_cg(flags + node);
      const bool kept_up = f & (node == sc.root ? 2u : 1u);
      const bool sel = f & 12u;                // taken or leaf
      if (kd == -2) {                          // its own bfs_cut starts here (dgemv order)
        if (kept_up && (f & 2u)) {
          if (sel) atomicOr(ws.bm_pass + (node >> 5), 1u << (node & 31));
          else flags[node] = uint8_t(f | 32u);  // expanded: its subtree is visited
        }
      } else if (kd >= 0) {
        if (kept_up) atomicOr(ws.bm_spt + (kd >> 5), 1u << (kd & 31));
      } else if (kept_up && sel) {
        atomicOr(ws.bm_upper + (node >> 5), 1u << (node & 31));
      }
    }
    grid_sync(ws.bar);
    sel_stamp(2);
    // phase 2b: passthrough-subtree members (cand[num_cand_upper, num_cand)):
    // walk up to their passthrough root, which must have been expanded
    for (long long i = sc.num_cand_upper + gtid; i < sc.num_cand; i += gthreads) {
      const int node = sc.cand[i];
      bool ok = true;
      for (int c = node;;) {
        const int a = sc.parent[c];
        const unsigned fa = ld_cg(flags + a);
        if (fa & 16u) { ok = fa & 32u; break; }   // the passthrough root
        if (!((fa & 1u) && !(fa & 4u))) { ok = false; break; }
        c = a;
      }
      if (!ok) continue;
      const unsigned f = ld_cg(flags + node);
      if ((f & 1u) && (f & 12u)) atomicOr(ws.bm_pass + (node >> 5), 1u << (node & 31));
    }
    grid_sync(ws.bar);
    sel_stamp(3);
    level = -1;
  } else
  // ---- level-synchronous BFS over the upper tree + passthrough subtrees ----
  for (; level < kMaxLevels; ++level) {
    const long long n = ld_cg(ws.lvl_count + level);
    if (n == 0) break;
    const uint32_t* cur = ws.frontier[level & 1];
    uint32_t* nxt = ws.frontier[(level + 1) & 1];
    unsigned int* nxt_count = ws.lvl_count + level + 1;
    for (long long base = gwarp0; base < n; base += gthreads) {
      const long long i = base + lane;
      uint32_t push[2];
      int npush = 0;
      if (i < n) {
        const uint32_t e = ld_cg(cur + i);
        const int node = int(e & kIdMask);
        const bool pass = e & kPass, start = e & kStart;
        const long long as = sc.attr_stride ? sc.attr_stride : 3;
        const double* mp = sc.means + as * node;
        const double* sp = sc.scales + as * node;
        const double mx = mp[0], my = mp[1], mz = mp[2];
        const double s0 = sp[0], s1 = sp[1], s2 = sp[2];
        bool keep = true;
        if (v.cull) keep = sphere_in_frustum(planes, mx, my, mz, mul(3.0, max3(s0, s1, s2)), start);
        if (keep) {
          const int kd = pass ? -1 : sc.kind[node];
          if (kd >= 0) {                       // SPT root: stage 2 takes over
            atomicOr(ws.bm_spt + (kd >> 5), 1u << (kd & 31));
          } else if (kd == -2) {               // passthrough root: its own bfs_cut
            push[npush++] = uint32_t(node) | kPass | kStart;
          } else {
            const double dist = norm3_plain(sub(mx, v.position[0]), sub(my, v.position[1]), sub(mz, v.position[2]));
            const double md = min_distance(v.threshold, v.metric, s0, s1, s2);
            const int c0 = sc.children[2 * node], c1 = sc.children[2 * node + 1];
            if (dist >= md || c0 == -1) {
              uint32_t* bm = pass ? ws.bm_pass : ws.bm_upper;
              atomicOr(bm + (node >> 5), 1u << (node & 31));
            } else {
              const uint32_t tag = pass ? kPass : 0u;
              push[npush++] = uint32_t(c0) | tag;
              push[npush++] = uint32_t(c1) | tag;
            }
          }
        }
      }
      // warp-aggregated append to the next frontier
      int incl = npush;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int wtot = __shfl_sync(0xffffffffu, incl, 31);
      unsigned int wbase = 0;
      if (lane == 31 && wtot) wbase = atomicAdd(nxt_count, unsigned(wtot));
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      const unsigned int o = wbase + incl - npush;
      for (int k = 0; k < npush; ++k) nxt[o + k] = push[k];
    }
    grid_sync(ws.bar);
  }

  // ---- bitmaps → sorted id lists (np.sort of the concatenated selections) ----
  const long long wn = (sc.capacity + 31) / 32, ws_ = (sc.num_spts + 31) / 32;
  long long c_up = bitmap_block_count(ws.bm_upper, wn, sm);
  long long c_pa = bitmap_block_count(ws.bm_pass, wn, sm);
  long long c_sp = bitmap_block_count(ws.bm_spt, ws_, sm);
  if (threadIdx.x == 0) {
    ws.block_cnt[blockIdx.x] = c_up;
    ws.block_cnt[gridDim.x + blockIdx.x] = c_pa;
    ws.block_cnt[2 * gridDim.x + blockIdx.x] = c_sp;
  }
  grid_sync(ws.bar);
  sel_stamp(4);
  const long long b_up = sum_before(ws.block_cnt, blockIdx.x, sm);
  const long long b_pa = sum_before(ws.block_cnt + gridDim.x, blockIdx.x, sm);
  const long long b_sp = sum_before(ws.block_cnt + 2 * gridDim.x, blockIdx.x, sm);
  bitmap_block_write(ws.bm_upper, wn, sc.capacity, b_up, out.upper_ids, sm);
  bitmap_block_write(ws.bm_pass, wn, sc.capacity, b_pa, out.pass_ids, sm);
  bitmap_block_write(ws.bm_spt, ws_, sc.num_spts, b_sp, out.spt_ids, sm);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    out.counts[0] = int32_t(b_up + c_up);
    out.counts[1] = int32_t(b_pa + c_pa);
    out.counts[2] = int32_t(b_sp + c_sp);
    out.counts[3] = level;
  }
  grid_sync(ws.bar);
  sel_stamp(5);

  // ---- stage 2 prologue: d_root (BLAS ddot norm, hspt.py:150) + prefix ----
  // one warp per selected SPT (32-ary prefix search)
  const int n_spt = ld_cg(out.counts + 2);
  for (long long j = gwarp0 >> 5; j < n_spt; j += gthreads >> 5) {
    const int s = ld_cg(out.spt_ids + j);
    const double d = norm3_ddot(sub(sc.spt_center[3 * s], v.position[0]),
                                sub(sc.spt_center[3 * s + 1], v.position[1]),
                                sub(sc.spt_center[3 * s + 2], v.position[2]));
    const int64_t off = sc.spt_offset[s];
    const int pl = sc.key_f64 ? warp_count_gt(static_cast<const double*>(sc.key_parent) + off, sc.spt_count[s], d, lane)
                              : warp_count_gt(static_cast<const float*>(sc.key_parent) + off, sc.spt_count[s], d, lane);
    if (lane == 0) {
      out.d_root[j] = d;
      out.prefix_len[j] = pl;
    }
  }
  sel_stamp(6);
}

// ---------------------------------------------------------------------------
// K1: order-preserving compaction of every selected prefix (spt.py:67-75,
// trainer._spt_positions :302-309); two launches (three when many prefixes
// must be searched), no grid barriers, no memset:
//   prefix_kernel   one warp per selected SPT: prefix length (the caller's,
//                   or a 32-ary ballot search of #{key_parent > d}), root
//                   rule, virtual segment length (padded to kAlign records)
//                   — run inside segscan_kernel when it is cheap
//   segscan_kernel  one CTA: exclusive scan of the segment lengths (the
//                   selected prefixes laid end to end in one virtual
//                   space); resets the tile ticket and the look-back words
//   compact_kernel  persistent CTAs take tiles in order (atomic ticket).
//                   Warp w of a tile owns a contiguous 128·G-record span;
//                   lane l's group g = records [g·128 + 4l, +4), so every
//                   key load is a coalesced 16-B vector load and all G are
//                   issued before any is used.  Ranks: warp scans per group
//                   (four counts packed per word), warp totals, the tile's
//                   offset by decoupled look-back; selections are written
//                   straight out (each group's run is contiguous).  Every
//                   key_self is read once.
// ---------------------------------------------------------------------------
constexpr int kCThreads = 128;
constexpr int kCWarps = kCThreads / 32;
constexpr int kCBlocksPerSM = 8;
template <typename K> struct CTile {
  static constexpr int G = sizeof(K) == 4 ? 4 : 2;            // groups per lane
  static constexpr int kWarpRecs = 32 * kAlign * G;           // 512 / 256
  static constexpr int kTile = kCWarps * kWarpRecs;           // 2048 / 1024
};
#ifndef GLOD_K1_ROUNDS
#define GLOD_K1_ROUNDS 1   // tiles per CTA the sub-tile count aims at (1 vs 2: 10M records 61 -> 51 us, C4 step 79 -> 70 us; 4 no better)
#endif
constexpr int kSubTiles = 8;                                // sub-tiles per look-back tile
constexpr int kMinTile = 1024;
constexpr int kSegCache = 128;                               // segments cached per tile
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

struct CompactScratch {
  unsigned int* ticket;         // [1] tile ticket (reset by segscan_kernel)
  unsigned long long* status;   // [max_tiles] look-back words (reset by segscan_kernel)
  long long max_tiles;
};

size_t max_tiles(int64_t num_records, int32_t S) {
  return size_t((num_records + int64_t(kAlign) * S + kMinTile - 1) / kMinTile) + 2;
}

CompactScratch carve_compact(void* base, int32_t S, int64_t R) {
  CompactScratch s;
  char* p = static_cast<char*>(base);
  s.ticket = reinterpret_cast<unsigned int*>(p);
  s.status = reinterpret_cast<unsigned long long*>(p + 256);
  s.max_tiles = (long long)max_tiles(R, S);
  return s;
}

// look-back words: one aligned 64-bit access (flag and value together)
GLOD_DEV unsigned long long ld_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
GLOD_DEV void st_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// kAlign consecutive keys, aligned by the record layout (device.pad_records)
GLOD_DEV void load4(const float* p, long long a, float (&v)[4]) {
  const float4 x = __ldcs(reinterpret_cast<const float4*>(p + a));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
GLOD_DEV void load4(const double* p, long long a, double (&v)[4]) {
  const double2 x = __ldcs(reinterpret_cast<const double2*>(p + a));
  const double2 y = __ldcs(reinterpret_cast<const double2*>(p + a + 2));
  v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
}

// prefix length / root rule / padded segment length of selected SPT j
template <typename K>
GLOD_DEV void spt_prefix(const LodScene& sc, const CompactIn& in, const CompactOut& out, long long j, int lane) {
  const K* key_self = static_cast<const K*>(sc.key_self);
  const int s = in.spt_ids[j];
  const double d = in.dist[j];
  int pl;
  if (in.known_prefix) {
    pl = in.known_prefix[j];
  } else {
    // np.searchsorted(-key_parent, -d, 'left') == #{key_parent > d}
    pl = warp_count_gt(static_cast<const K*>(sc.key_parent) + sc.spt_offset[s], sc.spt_count[s], d, lane);
  }
  // root rule (spt.py:72-73): d >= key_self[root] selects exactly [root]
  const int rr = d >= double(key_self[sc.spt_offset[s] + sc.spt_root_rec[s]]);
  if (lane == 0) {
    out.prefix_len[j] = pl;
    out.root_rule[j] = rr;
    out.seg_start[j] = ((rr ? 1 : pl) + kAlign - 1) / kAlign * kAlign;   // length for now
  }
}

template <typename K>
__global__ void __launch_bounds__(256) prefix_kernel(LodScene sc, CompactIn in, CompactOut out) {
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int n_spt = *in.n_spt;
  for (long long j = gw; j < n_spt; j += nw) spt_prefix<K>(sc, in, out, j, threadIdx.x & 31);
}

template <typename K>
__global__ void __launch_bounds__(1024)
segscan_kernel(LodScene sc, CompactIn in, CompactOut out, CompactScratch ws, int with_prefix) {
  __shared__ long long sm[1024 / 32 + 1];
  const int n_spt = *in.n_spt;
  // known prefix lengths (the select's): one thread per SPT, the length
  // computed in the scan loop itself; else a warp per SPT searches first
  const bool known = with_prefix && in.known_prefix;
  if (with_prefix && !known) {
    for (long long j = threadIdx.x >> 5; j < n_spt; j += blockDim.x >> 5) spt_prefix<K>(sc, in, out, j, threadIdx.x & 31);
    __syncthreads();
  }
  long long carry = 0;
  for (int base = 0; base < n_spt; base += blockDim.x) {
    const int j = base + threadIdx.x;
    long long len = 0;
    if (j < n_spt) {
      if (known) {
        const int s = in.spt_ids[j];
        const int pl = in.known_prefix[j];
        const int rr = in.dist[j] >= double(static_cast<const K*>(sc.key_self)[sc.spt_offset[s] + sc.spt_root_rec[s]]);
        out.prefix_len[j] = pl;
        out.root_rule[j] = rr;
        len = ((rr ? 1 : pl) + kAlign - 1) / kAlign * kAlign;
      } else {
        len = out.seg_start[j];
      }
    }
    const long long ex = block_excl_scan(len, sm);
    const long long tot = sm[(blockDim.x + 31) >> 5];
    __syncthreads();
    if (j < n_spt) out.seg_start[j] = carry + ex;
    carry += tot;
  }
  const long long ntiles = (carry + CTile<K>::kTile - 1) / CTile<K>::kTile;   // upper bound (1 sub-tile)
  for (long long t = threadIdx.x; t < ntiles && t < ws.max_tiles; t += blockDim.x) ws.status[t] = 0;
  if (threadIdx.x == 0) {
    out.total[1] = carry;     // virtual records
    out.total[0] = 0;         // selections (the last tile overwrites)
    *ws.ticket = 0;
  }
}

// key <= d, exactly: for f32 keys against the largest float <= d (no
// per-key f32 -> f64 conversion), for f64 keys directly
GLOD_DEV bool key_le(float k, double, float df) { return k <= df; }
GLOD_DEV bool key_le(double k, double d, float) { return k <= d; }

// The segments overlapping a tile, cached in shared memory.
struct SegCache {
  long long vstart[kSegCache + 1];
  long long off[kSegCache];
  double d[kSegCache];
  float df[kSegCache];
  int len[kSegCache], rr[kSegCache], rootrec[kSegCache];
};

// One sub-tile's kAlign-record groups of this lane: segment, position,
// key-vector address and selection mask (bit e: record e selected).
template <typename K, int G>
struct Groups {
  int seg[G], loc[G], len[G];
  long long addr[G];
  unsigned rrmask;
  unsigned mask[G];

  // segment, position and key address of each group (no key loads)
  GLOD_DEV void locate(const LodScene& sc, const CompactIn& in, const CompactOut& out, const SegCache& c,
                       int j0, int nseg, long long cache_end, int n_spt, long long w_lo, long long t_hi,
                       int lane) {
    rrmask = 0;
    int cur = -1;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const long long v = w_lo + g * (32 * kAlign) + lane * kAlign;
      seg[g] = -1;
      len[g] = 0;
      loc[g] = 0;
      addr[g] = 0;
      if (v < t_hi) {
        if (v < cache_end) {
          if (cur < 0) {
            int a = 0, b = nseg;                   // last cached segment starting <= v
            while (a < b) { const int m = (a + b) >> 1; if (c.vstart[m] <= v) a = m + 1; else b = m; }
            cur = a - 1;
          } else {
            while (cur + 1 < nseg && c.vstart[cur + 1] <= v) ++cur;
          }
          seg[g] = cur;                            // local index
          loc[g] = int(v - c.vstart[cur]);
          len[g] = c.len[cur];
          if (c.rr[cur]) rrmask |= 1u << g;
          addr[g] = c.off[cur] + (c.rr[cur] ? c.rootrec[cur] : loc[g]);
        } else {
          int a = j0 + nseg, b = n_spt;
          while (a < b) { const int m = (a + b) >> 1; if (out.seg_start[m] <= v) a = m + 1; else b = m; }
          const int j = a - 1;
          const int sp = in.spt_ids[j];
          seg[g] = kSegCache + j;                  // global index, tagged
          loc[g] = int(v - out.seg_start[j]);
          const int rr = out.root_rule[j];
          len[g] = rr ? 1 : out.prefix_len[j];
          if (rr) rrmask |= 1u << g;
          addr[g] = sc.spt_offset[sp] + (rr ? sc.spt_root_rec[sp] : loc[g]);
        }
      }
    }
  }

  // Fast path, warp-uniform: the warp's whole span lies inside the valid
  // records of one cached segment without the root rule (the common case
  // for prefixes longer than a span).  Returns that segment, else -1.
  static GLOD_DEV int span_segment(const SegCache& c, int nseg, long long w_lo, long long t_hi) {
    constexpr long long kSpan = 32 * kAlign * G;
    if (w_lo + kSpan > t_hi) return -1;
    int a = 0, b = nseg;                         // last cached segment starting <= w_lo
    while (a < b) { const int m = (a + b) >> 1; if (c.vstart[m] <= w_lo) a = m + 1; else b = m; }
    const int cur = a - 1;
    if (cur < 0 || c.rr[cur] || w_lo + kSpan > c.vstart[cur] + c.len[cur]) return -1;
    return cur;
  }
  GLOD_DEV void locate_span(const SegCache& c, int cur, long long w_lo, int lane) {
    rrmask = 0;
    const int loc0 = int(w_lo - c.vstart[cur]) + lane * kAlign;
    const long long off = c.off[cur];
    const int ln = c.len[cur];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      seg[g] = cur;
      loc[g] = loc0 + g * (32 * kAlign);
      len[g] = ln;
      addr[g] = off + loc[g];
    }
  }
  // every record of every group valid and in segment `cur`
  GLOD_DEV void evaluate_span(const LodScene& sc, const SegCache& c, int cur) {
    const K* key_self = static_cast<const K*>(sc.key_self);
    K kv[G][kAlign];
#pragma unroll
    for (int g = 0; g < G; ++g) load4(key_self, addr[g], kv[g]);
    const double d = c.d[cur];
    const float df = c.df[cur];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      unsigned m = 0;
#pragma unroll
      for (int e = 0; e < kAlign; ++e) m |= key_le(kv[g][e], d, df) ? (1u << e) : 0u;
      mask[g] = m;
    }
  }

  // the keys of every group (all loads issued first), then the masks
  GLOD_DEV void evaluate(const LodScene& sc, const CompactIn& in, const SegCache& c) {
    const K* key_self = static_cast<const K*>(sc.key_self);
    K kv[G][kAlign];
#pragma unroll
    for (int g = 0; g < G; ++g)
      load4(key_self, (seg[g] >= 0 && !((rrmask >> g) & 1u) && loc[g] < len[g]) ? addr[g] : 0, kv[g]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      mask[g] = 0;
      if (seg[g] >= 0) {
        if ((rrmask >> g) & 1u) {
          mask[g] = loc[g] == 0 ? 1u : 0u;         // [root]
        } else {
          const double d = seg[g] < kSegCache ? c.d[seg[g]] : in.dist[seg[g] - kSegCache];
          const float df = seg[g] < kSegCache ? c.df[seg[g]] : __double2float_rd(d);
#pragma unroll
          for (int e = 0; e < kAlign; ++e)
            if (loc[g] + e < len[g] && key_le(kv[g][e], d, df)) mask[g] |= 1u << e;
        }
      }
    }
  }
};

template <typename K>
__global__ void __launch_bounds__(kCThreads, kCBlocksPerSM)
compact_kernel(LodScene sc, CompactIn in, CompactOut out, CompactScratch ws) {
  constexpr int G = CTile<K>::G;
  constexpr int kWarpRecs = CTile<K>::kWarpRecs;
  constexpr int kSubTile = CTile<K>::kTile;
  __shared__ SegCache c;
  __shared__ long long sub_cnt[kSubTiles][kCWarps];
  __shared__ unsigned masks[kSubTiles][kCThreads];
  __shared__ int2 stage[kCWarps][kWarpRecs];        // pass B staging (span path)
  __shared__ unsigned int tile_sh;
  __shared__ int j0_sh;
  __shared__ long long excl_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_spt = *in.n_spt;
  const long long total = out.total[1];
  // sub-tiles per look-back tile: as many as keep every CTA busy (large
  // inputs amortise the look-back over more records, small ones keep
  // their parallelism)
  const long long nsub_ll = total / ((long long)GLOD_K1_ROUNDS * gridDim.x * kSubTile);
  const int nsub = int(nsub_ll < 1 ? 1 : (nsub_ll > kSubTiles ? kSubTiles : nsub_ll));
  const long long kTile = (long long)nsub * kSubTile;
  const long long ntiles = (total + kTile - 1) / kTile;

  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned t = atomicAdd(ws.ticket, 1u);
      tile_sh = t;
      if ((long long)t < ntiles) {   // last j with seg_start[j] <= tile start
        const long long lo = (long long)t * kTile;
        int a = 0, b = n_spt;
        while (a < b) { const int m = (a + b) >> 1; if (out.seg_start[m] <= lo) a = m + 1; else b = m; }
        j0_sh = a - 1;
      }
    }
    __syncthreads();
    const long long tile = tile_sh;
    if (tile >= ntiles) break;
    const long long t_lo = tile * kTile, t_hi = min(total, t_lo + kTile);
    const int j0 = j0_sh;
    // segments overlapping the tile -> shared cache (seg_start is sorted)
    int valid = 0;
    if (threadIdx.x < kSegCache) {
      const int j = j0 + threadIdx.x;
      if (j < n_spt && (threadIdx.x == 0 || out.seg_start[j] < t_hi)) {
        valid = 1;
        const int sp = in.spt_ids[j];
        const int rr = out.root_rule[j];
        c.vstart[threadIdx.x] = out.seg_start[j];
        c.off[threadIdx.x] = sc.spt_offset[sp];
        c.d[threadIdx.x] = in.dist[j];
        c.df[threadIdx.x] = __double2float_rd(in.dist[j]);
        c.rr[threadIdx.x] = rr;
        c.len[threadIdx.x] = rr ? 1 : out.prefix_len[j];
        c.rootrec[threadIdx.x] = sc.spt_root_rec[sp];
      }
    }
    const int nseg = __syncthreads_count(valid);
    // more than kSegCache segments in this tile: groups past the cached ones
    // find their segment with a global search
    const long long cache_end = (j0 + nseg < n_spt) ? out.seg_start[j0 + nseg] : total;

    // pass A: stream the keys once, keep each lane's selection masks
    // (kAlign bits per group) in shared memory, count per sub-tile
#pragma unroll 1
    for (int st = 0; st < nsub; ++st) {
      Groups<K, G> gr;
      const long long w_lo = t_lo + (long long)st * kSubTile + (long long)warp * kWarpRecs;
      const int span = Groups<K, G>::span_segment(c, nseg, w_lo, t_hi);
      if (span >= 0) {
        gr.locate_span(c, span, w_lo, lane);
        gr.evaluate_span(sc, c, span);
      } else {
        gr.locate(sc, in, out, c, j0, nseg, cache_end, n_spt, w_lo, t_hi, lane);
        gr.evaluate(sc, in, c);
      }
      int cnt = 0;
      unsigned packed_mask = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        cnt += __popc(gr.mask[g]);
        packed_mask |= gr.mask[g] << (kAlign * g);
      }
      masks[st][threadIdx.x] = packed_mask;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0) sub_cnt[st][warp] = cnt;
    }
    __syncthreads();
    long long agg = 0;
    for (int st = 0; st < nsub; ++st)
#pragma unroll
      for (int w = 0; w < kCWarps; ++w) agg += sub_cnt[st][w];
    // decoupled look-back over the big tiles (warp 0, 32 predecessors per step)
    if (warp == 0) {
      if (lane == 0) st_u64(ws.status + tile, (tile == 0 ? kFlagIncl : kFlagAgg) | (unsigned long long)agg);
      long long excl = 0;
      if (tile > 0) {
        for (long long pred = tile - 1;; pred -= 32) {
          const long long idx = pred - lane;
          unsigned long long sv = kFlagIncl;
          if (idx >= 0) {
            sv = ld_u64(ws.status + idx);
            while ((sv >> 62) == 0) sv = ld_u64(ws.status + idx);
          }
          const unsigned incl_m = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
          const int first = incl_m ? __ffs(incl_m) - 1 : 32;
          long long v = lane <= first ? (long long)(sv & kValMask) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += v;
          if (incl_m) break;
        }
        if (lane == 0) st_u64(ws.status + tile, kFlagIncl | (unsigned long long)(excl + agg));
      }
      if (lane == 0) {
        excl_sh = excl;
        if (tile == ntiles - 1) out.total[0] = excl + agg;
      }
    }
    __syncthreads();
    // pass B: rank inside each group run from the kept masks and write the
    // selections in order (no key is read twice)
    long long run = excl_sh;
#pragma unroll 1
    for (int st = 0; st < nsub; ++st) {
      long long w_off = 0, st_tot = 0;
#pragma unroll
      for (int w = 0; w < kCWarps; ++w) {
        w_off += w < warp ? sub_cnt[st][w] : 0;
        st_tot += sub_cnt[st][w];
      }
      Groups<K, G> gr;
      const long long w_lo = t_lo + (long long)st * kSubTile + (long long)warp * kWarpRecs;
      const int span = Groups<K, G>::span_segment(c, nseg, w_lo, t_hi);
      if (span >= 0) gr.locate_span(c, span, w_lo, lane);
      else gr.locate(sc, in, out, c, j0, nseg, cache_end, n_spt, w_lo, t_hi, lane);
      const unsigned packed_mask = masks[st][threadIdx.x];
#pragma unroll
      for (int g = 0; g < G; ++g) gr.mask[g] = (packed_mask >> (kAlign * g)) & ((1u << kAlign) - 1u);
      // warp-inclusive scans of the per-group counts, four packed per word
      unsigned packed[(G + 3) / 4], incl[(G + 3) / 4];
#pragma unroll
      for (int i = 0; i < (G + 3) / 4; ++i) packed[i] = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) packed[g >> 2] |= unsigned(__popc(gr.mask[g])) << (8 * (g & 3));
#pragma unroll
      for (int i = 0; i < (G + 3) / 4; ++i) {
        unsigned x = packed[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        incl[i] = x;
      }
      // node ids of every group with a selection, all loads issued first
      int4 nd[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        nd[g] = make_int4(0, 0, 0, 0);
        if (gr.mask[g]) {
          if ((gr.rrmask >> g) & 1u) nd[g].x = sc.rec_node[gr.addr[g]];
          else nd[g] = *reinterpret_cast<const int4*>(sc.rec_node + gr.addr[g]);
        }
      }
      const long long base = run + w_off;
      if (span >= 0) {
        // one segment: (pos, node) staged at their warp-local ranks, then
        // the warp's run written with consecutive lanes on consecutive
        // outputs (coalesced, one store per array per 32 selections)
        int2* sb = stage[warp];
        int gs = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const unsigned x = (incl[g >> 2] >> (8 * (g & 3))) & 0xffu;
          const unsigned cg = (packed[g >> 2] >> (8 * (g & 3))) & 0xffu;
          const int gt = int(__shfl_sync(0xffffffffu, x, 31));
          int o = gs + int(x - cg);
          const int n4[4] = {nd[g].x, nd[g].y, nd[g].z, nd[g].w};
#pragma unroll
          for (int e = 0; e < kAlign; ++e)
            if (gr.mask[g] & (1u << e)) sb[o++] = make_int2(gr.loc[g] + e, n4[e]);
          gs += gt;
        }
        __syncwarp();
        const int j = j0 + span;
        for (int k = lane; k < gs; k += 32) {
          const int2 v = sb[k];
          out.sel_seg[base + k] = j;
          out.sel_pos[base + k] = v.x;
          out.sel_node[base + k] = v.y;
        }
        __syncwarp();
        run += st_tot;
        continue;
      }
      long long gsum = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const unsigned x = (incl[g >> 2] >> (8 * (g & 3))) & 0xffu;
        const unsigned cg = (packed[g >> 2] >> (8 * (g & 3))) & 0xffu;
        const unsigned gt = __shfl_sync(0xffffffffu, x, 31);
        if (gr.mask[g]) {
          const int sg = gr.seg[g];
          const int j = sg < kSegCache ? j0 + sg : sg - kSegCache;
          long long o = base + gsum + x - cg;
          if ((gr.rrmask >> g) & 1u) {
            out.sel_seg[o] = j;
            out.sel_pos[o] = sg < kSegCache ? c.rootrec[sg] : sc.spt_root_rec[in.spt_ids[j]];
            out.sel_node[o] = nd[g].x;
          } else {
            const int n4[4] = {nd[g].x, nd[g].y, nd[g].z, nd[g].w};
#pragma unroll
            for (int e = 0; e < kAlign; ++e)
              if (gr.mask[g] & (1u << e)) {
                out.sel_seg[o] = j;
                out.sel_pos[o] = gr.loc[g] + e;
                out.sel_node[o] = n4[e];
                ++o;
              }
          }
        }
        gsum += gt;
      }
      run += st_tot;
    }
    __syncthreads();            // the segment cache and counts are rewritten next tile
  }
}

int coop_grid(const void* kernel, int threads) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace

size_t select_scratch_bytes(int64_t cap, int32_t S, int grid) {
  size_t w_nodes = (size_t(cap) + 31) / 32, w_spt = (size_t(S) + 31) / 32;
  size_t off = align_up(sizeof(unsigned int) * (kMaxLevels + 3));
  off += 8 * w_nodes + 4 * w_spt;
  off = align_up(off);
  off = align_up(off + 4 * size_t(cap) + 4);
  off = align_up(off + 4 * size_t(cap) + 4);
  off += 3 * 8 * size_t(grid) + 256;
  return off;
}

size_t compact_scratch_bytes(int32_t S, int64_t R, int grid) {
  (void)grid;
  return align_up(256 + 8 * max_tiles(R, S)) + 256;
}

cudaError_t select_phase_ns(long long* out7) {
  unsigned long long t[8];
  cudaError_t e = cudaMemcpyFromSymbol(t, g_sel_ts, sizeof(t));
  if (e != cudaSuccess) return e;
  for (int k = 0; k < 7; ++k) out7[k] = (long long)t[k];
  return cudaSuccess;
}

int select_grid() { return coop_grid((const void*)select_kernel, kSelectThreads); }
int compact_grid() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * kCBlocksPerSM;
}

cudaError_t launch_select(const LodScene& sc, const LodView& v, const SelectOut& out,
                          void* scratch, size_t scratch_bytes, cudaStream_t st) {
  const int grid = select_grid();
  if (scratch_bytes < select_scratch_bytes(sc.capacity, sc.num_spts, grid)) return cudaErrorInvalidValue;
  SelectScratch ws = carve_select(scratch, sc.capacity, sc.num_spts, grid);
  cudaError_t e = cudaMemsetAsync(scratch, 0, ws.zero_bytes, st);
  if (e != cudaSuccess) return e;
  LodScene a = sc; LodView b = v; SelectOut c = out; SelectScratch d = ws;
  void* args[] = {&a, &b, &c, &d};
  count_launch();
  return cudaLaunchCooperativeKernel((const void*)select_kernel, dim3(grid), dim3(kSelectThreads),
                                     args, 0, st);
}

template <typename K>
cudaError_t launch_compact_t(const LodScene& sc, const CompactIn& in, const CompactOut& out,
                             const CompactScratch& ws, cudaStream_t st) {
  // prefix searches run inside the scan CTA when they are cheap (known
  // prefix lengths, or few SPTs), else one warp per SPT over the grid
  const bool split = !in.known_prefix && sc.num_spts > 32;
  if (split) {
    prefix_kernel<K><<<unsigned((sc.num_spts + 7) / 8), 256, 0, st>>>(sc, in, out);
    count_launch();
  }
  segscan_kernel<K><<<1, 1024, 0, st>>>(sc, in, out, ws, split ? 0 : 1);
  compact_kernel<K><<<unsigned(compact_grid()), kCThreads, 0, st>>>(sc, in, out, ws);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_compact(const LodScene& sc, const CompactIn& in, const CompactOut& out,
                           void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (scratch_bytes < compact_scratch_bytes(sc.num_spts, sc.num_records, 0)) return cudaErrorInvalidValue;
  CompactScratch ws = carve_compact(scratch, sc.num_spts, sc.num_records);
  return sc.key_f64 ? launch_compact_t<double>(sc, in, out, ws, st) : launch_compact_t<float>(sc, in, out, ws, st);
}

}  // namespace glod
