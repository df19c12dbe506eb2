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
constexpr int kCompactThreads = 512;
constexpr int kRows = 8;                          // items per thread per tile
constexpr int kTile = kCompactThreads * kRows;    // 4096 virtual records
constexpr int kAlign = 4;                         // records per lane group (16-B vector loads)
constexpr int kGroups = 4;                        // groups per lane in flight (K1 phase C)
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

template <typename K>
GLOD_DEV int prefix_search(const K* kp, int n, double d) {
  // np.searchsorted(-key_parent, -d, 'left') == #{key_parent > d}
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (double(kp[mid]) > d) lo = mid + 1; else hi = mid;
  }
  return lo;
}

GLOD_DEV int prefix_len_of(const LodScene& sc, int s, double d) {
  const int64_t off = sc.spt_offset[s];
  const int n = sc.spt_count[s];
  return sc.key_f64 ? prefix_search(static_cast<const double*>(sc.key_parent) + off, n, d)
                    : prefix_search(static_cast<const float*>(sc.key_parent) + off, n, d);
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

__global__ void __launch_bounds__(kSelectThreads)
select_kernel(LodScene sc, LodView v, SelectOut out, SelectScratch ws) {
  __shared__ long long sm[kSelectThreads / 32 + 1];
  __shared__ double planes[24];
  if (threadIdx.x < 24) planes[threadIdx.x] = v.planes[threadIdx.x];
  const int lane = threadIdx.x & 31;
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const long long gwarp0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ws.frontier[0][0] = uint32_t(sc.root) | kStart;
    ws.lvl_count[0] = 1;
  }
  grid_sync(ws.bar);

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

  // ---- stage 2 prologue: d_root (BLAS ddot norm, hspt.py:150) + prefix ----
  const int n_spt = ld_cg(out.counts + 2);
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n_spt; j += gthreads) {
    const int s = ld_cg(out.spt_ids + j);
    const double d = norm3_ddot(sub(sc.spt_center[3 * s], v.position[0]),
                                sub(sc.spt_center[3 * s + 1], v.position[1]),
                                sub(sc.spt_center[3 * s + 2], v.position[2]));
    out.d_root[j] = d;
    out.prefix_len[j] = prefix_len_of(sc, s, d);
  }
}

// ---------------------------------------------------------------------------
// K1: order-preserving compaction of every selected prefix.
// ---------------------------------------------------------------------------
struct CompactScratch {
  unsigned int* bar;            // [2]
  unsigned long long* status;   // [max_tiles] decoupled look-back words
  long long* block_cnt;         // [grid]
  size_t zero_bytes;
};

size_t max_tiles(int64_t num_records, int32_t S) {
  return size_t((num_records + S + kTile - 1) / kTile) + 1;
}

CompactScratch carve_compact(void* base, int32_t S, int64_t R, int grid) {
  CompactScratch s;
  char* p = static_cast<char*>(base);
  s.bar = reinterpret_cast<unsigned int*>(p);
  size_t off = 256;
  s.status = reinterpret_cast<unsigned long long*>(p + off);
  off += 8 * max_tiles(R, S);
  s.zero_bytes = off;
  off = align_up(off);
  s.block_cnt = reinterpret_cast<long long*>(p + off);
  return s;
}

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// 4 consecutive keys, aligned by the record layout (device.pad_records)
GLOD_DEV void load4(const float* p, long long a, float (&v)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p + a);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
GLOD_DEV void load4(const double* p, long long a, double (&v)[4]) {
  const double2 x = *reinterpret_cast<const double2*>(p + a);
  const double2 y = *reinterpret_cast<const double2*>(p + a + 2);
  v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
}
GLOD_DEV int rootrec_of(const LodScene& sc, const CompactIn& in, int j) {
  return sc.spt_root_rec[in.spt_ids[j]];
}

template <typename K>
__global__ void __launch_bounds__(kCompactThreads, 2)
compact_kernel(LodScene sc, CompactIn in, CompactOut out, CompactScratch ws) {
  __shared__ long long sm[kCompactThreads / 32 + 1];
  __shared__ int cnt[kRows][kCompactThreads / 32];
  __shared__ long long tile_base_sh;
  __shared__ int seg_lo_sh, seg_hi_sh;
  __shared__ long long seg_start_sh, seg_off_sh;
  __shared__ double seg_d_sh;
  __shared__ int seg_rr_sh, seg_rootrec_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = kCompactThreads / 32;
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  const int n_spt = *in.n_spt;
  const K* key_self = static_cast<const K*>(sc.key_self);

  // phase A: prefix length and root rule per selected SPT (spt.py:70-73);
  // the prefix comes from the caller when known, else a warp-cooperative
  // 32-ary search over key_parent (one warp per SPT)
  {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = gthreads >> 5;
    for (long long j = gw; j < n_spt; j += nw) {
      const int s = in.spt_ids[j];
      const double d = in.dist[j];
      int pl;
      if (in.known_prefix) {
        pl = in.known_prefix[j];
      } else {
        const K* kp = static_cast<const K*>(sc.key_parent) + sc.spt_offset[s];
        long long a = 0, b = sc.spt_count[s];        // answer in [a, b]
        while (b - a > 32) {
          const long long step = (b - a + 31) / 32;
          const long long probe = a + step * lane;    // lane 0 probes a (known > d or start)
          const bool gt = probe < b && (probe == a || double(kp[probe]) > d);
          const unsigned m = __ballot_sync(0xffffffffu, gt);
          const int last = 31 - __clz(m);             // last probe with key_parent > d
          const long long na = a + step * last;
          b = min(b, na + step);
          a = na;
        }
        // finish linearly over ≤ 32 candidates
        const long long probe = a + lane;
        const bool gt = probe < b && double(kp[probe]) > d;
        const unsigned m = __ballot_sync(0xffffffffu, gt);
        pl = int(a + __popc(m));
      }
      const int rr = d >= double(key_self[sc.spt_offset[s] + sc.spt_root_rec[s]]);
      if (lane == 0) {
        out.prefix_len[j] = pl;
        out.root_rule[j] = rr;
        // virtual segment length, padded to the record alignment so every
        // segment (and every lane's 4-item group) starts 16-B aligned
        out.seg_start[j] = ((rr ? 1 : pl) + kAlign - 1) / kAlign * kAlign;
      }
    }
  }
  grid_sync(ws.bar);

  // phase B: exclusive scan of segment lengths (block partition + offsets)
  long long lo, hi;
  block_range(n_spt, blockIdx.x, gridDim.x, lo, hi);
  {
    long long c = 0;
    for (long long j = lo + threadIdx.x; j < hi; j += blockDim.x) c += ld_cg(out.seg_start + j);
    c = block_sum(c, sm);
    if (threadIdx.x == 0) ws.block_cnt[blockIdx.x] = c;
  }
  grid_sync(ws.bar);
  {
    long long base = sum_before(ws.block_cnt, blockIdx.x, sm);
    long long span = hi - lo, chunk = (span + blockDim.x - 1) / blockDim.x;
    long long j0 = lo + chunk * threadIdx.x, j1 = min(hi, j0 + chunk);
    long long c = 0;
    for (long long j = j0; j < j1; ++j) c += ld_cg(out.seg_start + j);
    long long o = base + block_excl_scan(c, sm);
    for (long long j = j0; j < j1; ++j) {
      long long len = ld_cg(out.seg_start + j);
      out.seg_start[j] = o;
      o += len;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) out.total[1] = o;
  }
  grid_sync(ws.bar);

  // phase C: every warp owns a contiguous range of the virtual record space
  // (the selected prefixes laid end to end).  C1 counts each warp range's
  // selections; after a grid barrier each warp's output offset is the sum
  // of all earlier ranges; C2 re-streams its range and writes the
  // selections in order.  Inside a range everything is warp-synchronous:
  // striped coalesced key loads (kUnroll×32 keys in flight per warp),
  // ballot + popc for the in-order ranks, no block barriers.
  const long long total = ld_cg(out.total + 1);
  const long long nwarps_g = (long long)gridDim.x * nwarps;
  const long long gwarp = (long long)blockIdx.x * nwarps + warp;
  __shared__ long long wcount[kCompactThreads / 32];
  // per-warp staging of one lane-group step's selections (≤ 32·kAlign)
  __shared__ int st_seg[kCompactThreads / 32][32 * kAlign];
  __shared__ int st_pos[kCompactThreads / 32][32 * kAlign];
  __shared__ int st_node[kCompactThreads / 32][32 * kAlign];
  // waves small enough that the second pass re-reads the keys from L2
  const long long wave = sc.key_f64 ? (8ll << 20) : (16ll << 20);
  long long wave_base = 0;                      // selections before this wave
  for (long long w_lo = 0; w_lo < total || (total == 0 && w_lo == 0); w_lo += wave) {
  const long long w_len = min(wave, total - w_lo);
  // warp ranges in whole kAlign groups (virtual segments are padded to kAlign)
  const long long g_len = w_len / kAlign;
  const long long r_lo = w_lo + kAlign * (g_len * gwarp / nwarps_g);
  const long long r_hi = w_lo + kAlign * (g_len * (gwarp + 1) / nwarps_g);
  long long run = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // offset of this warp range = earlier waves + earlier blocks + earlier warps of this block
      const long long blk = sum_before(ws.block_cnt, blockIdx.x, sm);
      const long long all = sum_before(ws.block_cnt, gridDim.x, sm);
      long long w_before = 0;
      for (int w = 0; w < warp; ++w) w_before += wcount[w];
      run = wave_base + blk + w_before;
      if (threadIdx.x == 0 && blockIdx.x == 0 && w_lo + w_len >= total) out.total[0] = wave_base + all;
      wave_base += all;
    }
    // per-lane segment cursor
    int j = -1;
    long long s_start = 0, s_end = -1, off = 0;
    double d = 0.0;
    int rr = 0, rootrec = 0, seglen = 0;
    long long count = 0;
    for (long long base = r_lo; base < r_hi; base += 32LL * kAlign * kGroups) {
      // lane-owned groups of kAlign consecutive virtual records; a group
      // never straddles a segment (segments are padded to kAlign)
      int segk[kGroups], loc[kGroups], len[kGroups];
      long long addr[kGroups];
      bool isrr[kGroups];
#pragma unroll
      for (int k = 0; k < kGroups; ++k) {
        const long long vg = base + ((long long)k * 32 + lane) * kAlign;
        segk[k] = -1;
        loc[k] = 0;
        len[k] = 0;
        addr[k] = 0;
        isrr[k] = false;
        if (vg < r_hi) {
          if (vg >= s_end) {                         // move the cursor (usually 0-1 steps)
            if (j < 0 || vg >= s_end + 64 * kAlign) {
              int a = (j < 0 ? 0 : j), bb = n_spt;
              while (a < bb) { int m = (a + bb) >> 1; if (ld_cg(out.seg_start + m) <= vg) a = m + 1; else bb = m; }
              j = a - 1;
            } else {
              while (j + 1 < n_spt && ld_cg(out.seg_start + j + 1) <= vg) ++j;
            }
            s_start = ld_cg(out.seg_start + j);
            s_end = j + 1 < n_spt ? ld_cg(out.seg_start + j + 1) : total;
            const int sp = in.spt_ids[j];
            off = sc.spt_offset[sp];
            d = in.dist[j];
            rr = ld_cg(out.root_rule + j);
            rootrec = sc.spt_root_rec[sp];
            seglen = rr ? 1 : ld_cg(out.prefix_len + j);
          }
          segk[k] = j;
          loc[k] = int(vg - s_start);
          len[k] = seglen;
          isrr[k] = rr;
          addr[k] = off + (rr ? rootrec : loc[k]);
        }
      }
      // every group's key vector is requested before any is used
      K kv[kGroups][kAlign];
#pragma unroll
      for (int k = 0; k < kGroups; ++k) load4(key_self, (segk[k] >= 0 && !isrr[k]) ? addr[k] : 0, kv[k]);
      unsigned mask[kGroups];
#pragma unroll
      for (int k = 0; k < kGroups; ++k) {
        mask[k] = 0;
        if (segk[k] >= 0) {
          if (isrr[k]) {
            mask[k] = 1u;                            // [root] (spt.py:72-73)
          } else {
            const double d_k = segk[k] == j ? d : in.dist[segk[k]];
#pragma unroll
            for (int e = 0; e < kAlign; ++e)
              if (loc[k] + e < len[k] && double(kv[k][e]) <= d_k) mask[k] |= 1u << e;
          }
        }
      }
      if (pass == 0) {
#pragma unroll
        for (int k = 0; k < kGroups; ++k) count += __popc(mask[k]);
        continue;
      }
      int4 node[kGroups];
#pragma unroll
      for (int k = 0; k < kGroups; ++k) {
        node[k] = make_int4(0, 0, 0, 0);
        if (mask[k]) {
          if (isrr[k]) node[k].x = sc.rec_node[addr[k]];
          else node[k] = *reinterpret_cast<const int4*>(sc.rec_node + addr[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < kGroups; ++k) {
        const int c = __popc(mask[k]);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        // stage the group's selections in order in shared memory, then the
        // warp writes them out as coalesced runs of the three arrays
        int o = incl - c;
        const int nd[4] = {node[k].x, node[k].y, node[k].z, node[k].w};
#pragma unroll
        for (int e = 0; e < kAlign; ++e) {
          if (mask[k] & (1u << e)) {
            st_seg[warp][o] = segk[k];
            st_pos[warp][o] = isrr[k] ? rootrec_of(sc, in, segk[k]) : loc[k] + e;
            st_node[warp][o] = nd[e];
            ++o;
          }
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        for (int i = lane; i < tot; i += 32) {
          out.sel_seg[run + i] = st_seg[warp][i];
          out.sel_pos[run + i] = st_pos[warp][i];
          out.sel_node[run + i] = st_node[warp][i];
        }
        __syncwarp();
        run += tot;
      }
    }
    if (pass == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
      if (lane == 0) wcount[warp] = count;
      __syncthreads();
      long long c = 0;
      if (threadIdx.x < nwarps) c = wcount[threadIdx.x];
      c = block_sum(c, sm);
      if (threadIdx.x == 0) ws.block_cnt[blockIdx.x] = c;
      grid_sync(ws.bar);
    }
  }
  grid_sync(ws.bar);            // block_cnt is rewritten by the next wave
  if (total == 0) break;
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
  return align_up(256 + 8 * max_tiles(R, S)) + 8 * size_t(grid) + 256;
}

int select_grid() { return coop_grid((const void*)select_kernel, kSelectThreads); }
int compact_grid() { return coop_grid((const void*)compact_kernel<float>, kCompactThreads); }

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

cudaError_t launch_compact(const LodScene& sc, const CompactIn& in, const CompactOut& out,
                           void* scratch, size_t scratch_bytes, cudaStream_t st) {
  const int grid = compact_grid();
  if (scratch_bytes < compact_scratch_bytes(sc.num_spts, sc.num_records, grid)) return cudaErrorInvalidValue;
  CompactScratch ws = carve_compact(scratch, sc.num_spts, sc.num_records, grid);
  cudaError_t e = cudaMemsetAsync(scratch, 0, ws.zero_bytes, st);
  if (e != cudaSuccess) return e;
  LodScene a = sc; CompactIn b = in; CompactOut c = out; CompactScratch d = ws;
  void* args[] = {&a, &b, &c, &d};
  count_launch();
  const void* fn = sc.key_f64 ? (const void*)compact_kernel<double> : (const void*)compact_kernel<float>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kCompactThreads), args, 0, st);
}

}  // namespace glod
