// K12: HSPT / SPT build on the device.
//
// Replaces hspt.build_hspt (hspt.py:64-93) with build_spt (spt.py:45-64)
// for every SPT root at once, bit-exact:
//
//   small      vol = np.prod(scales, axis=1) = (s0·s1)·s2 < size_threshold
//   walk       per node, up the parent chain to the root: the volume BFS
//              of hspt.py:78-87 stops at the first small node on every
//              root path, so a node is "upper" iff no node on its path is
//              small, and otherwise belongs to the cut subtree of the
//              TOPMOST small node on the path (its cut root).  Nodes whose
//              chain does not reach the root through consistent
//              parent/child links (free slots) are unreachable.
//   counts     subtree_node_counts()[cut root] = #nodes labelled with it
//   lists      upper, cut roots split by count >= min_subtree into SPT
//              roots and passthrough roots — each ascending (np.sort)
//   keys       key_self = m_d(scales) + ‖μ − μ_root‖ (numpy axis-1 norm:
//              plain (x²+y²)+z²), key_parent = key_self[parent], +inf at
//              the root (spt.py:52-61)
//   order      np.lexsort((sub, -key_parent)) per SPT: members enumerated
//              in ascending node id, then two stable LSD radix sorts — by
//              key_parent descending (64-bit order-preserving transform of
//              the fp64 bits), then by SPT id.
//
// Everything is HBM-streaming integer/fp64 work; the walk is dependent
// loads of parent/children/small (L2-resident at C4: 20M nodes × 13 B).
#include <stdint.h>

#include "common.cuh"
#include "../../include/glod_b200.h"

namespace glod {

size_t radix_scratch_bytes(long long n);
size_t scan_scratch_bytes(long long n);
template <typename K>
cudaError_t radix_sort_pairs(K* keys, K* keys_alt, int* vals, int* vals_alt, long long n, int begin_bit,
                             int end_bit, void* scratch, size_t scratch_bytes, bool range_bits,
                             int* result_in_alt, cudaStream_t st);
cudaError_t exclusive_scan_i32(const int* in, long long* out, long long n, void* scratch, size_t bytes,
                               cudaStream_t st);

namespace {

constexpr int kThreads = 256;
constexpr int kUnreachable = -3;
constexpr int kUpper = -1;

int grid_for(long long n) {
  long long b = (n + kThreads - 1) / kThreads;
  return int(b < 1 ? 1 : b);
}

__global__ void small_kernel(const double* __restrict__ scales, long long cap, double thr,
                             unsigned char* __restrict__ small) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  const double v = mul(mul(scales[3 * i], scales[3 * i + 1]), scales[3 * i + 2]);
  small[i] = v < thr;
}

// label[i]: kUnreachable, kUpper, or the cut root holding i; counts[root]
// += 1 per labelled node (warp-aggregated: consecutive ids mostly share a
// cut root).
__global__ void walk_kernel(const int* __restrict__ parent, const int* __restrict__ children,
                            const unsigned char* __restrict__ small, long long cap, int root,
                            int* __restrict__ label, int* __restrict__ counts) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int lab = kUnreachable;
  if (i < cap) {
    int c = int(i), top = -1;
    bool ok = true;
    for (long long steps = 0; steps <= cap; ++steps) {
      if (small[c]) top = c;
      if (c == root) break;
      const int p = parent[c];
      if (p < 0 || p >= cap || (children[2 * p] != c && children[2 * p + 1] != c)) {
        ok = false;
        break;
      }
      c = p;
    }
    if (c != root) ok = false;
    lab = ok ? (top >= 0 ? top : kUpper) : kUnreachable;
    label[i] = lab;
  }
  const unsigned act = __ballot_sync(0xffffffffu, lab >= 0);
  if (lab >= 0) {
    const unsigned peers = __match_any_sync(act, lab);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + lab, __popc(peers));
  }
}

// One flag array per output list (upper, passthrough roots, SPT roots, SPT
// members), concatenated: flags[k * cap + i].
__global__ void flags_kernel(const int* __restrict__ label, const int* __restrict__ counts, long long cap,
                             int min_subtree, int* __restrict__ flags) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  const int lab = label[i];
  const bool big = lab >= 0 && counts[lab] >= min_subtree;
  flags[i] = lab == kUpper;
  flags[cap + i] = lab == int(i) && !big;
  flags[2 * cap + i] = lab == int(i) && big;
  flags[3 * cap + i] = big;
}

__global__ void scatter_kernel(const int* __restrict__ flags, const long long* __restrict__ pos, long long cap,
                               int* __restrict__ out, long long* __restrict__ total) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  if (flags[i]) out[pos[i]] = int(i);
  if (i == cap - 1) *total = pos[i] + flags[i];
}

__global__ void spt_id_kernel(const int* __restrict__ roots, const int* __restrict__ counts, long long n,
                              int* __restrict__ sid, int* __restrict__ spt_count) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  sid[roots[s]] = int(s);
  spt_count[s] = counts[roots[s]];
}

__global__ void key_self_kernel(const int* __restrict__ members, long long m, const int* __restrict__ label,
                                const int* __restrict__ sid, const double* __restrict__ means,
                                const double* __restrict__ scales, double T, int metric, int corrected,
                                double* __restrict__ key_of, unsigned* __restrict__ spt_of) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int node = members[j], r = label[node];
  double k = min_distance(T, metric, scales[3LL * node], scales[3LL * node + 1], scales[3LL * node + 2]);
  if (corrected)
    k = add(k, norm3_plain(sub(means[3LL * node], means[3LL * r]), sub(means[3LL * node + 1], means[3LL * r + 1]),
                           sub(means[3LL * node + 2], means[3LL * r + 2])));
  key_of[node] = k;
  spt_of[j] = unsigned(sid[r]);
}

// Order-preserving uint64 image of an fp64 value, inverted: ascending keys
// = descending key_parent (the -key_parent of the reference's lexsort).
GLOD_DEV unsigned long long desc_key(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const unsigned long long asc = (u >> 63) ? ~u : (u | (1ull << 63));
  return ~asc;
}

GLOD_DEV double key_parent_of(int node, const int* __restrict__ label, const int* __restrict__ parent,
                              const double* __restrict__ key_of) {
  return label[node] == node ? __longlong_as_double(0x7ff0000000000000ll) : key_of[parent[node]];
}

__global__ void parent_key_kernel(const int* __restrict__ members, long long m, const int* __restrict__ label,
                                  const int* __restrict__ parent, const double* __restrict__ key_of,
                                  unsigned long long* __restrict__ k64, int* __restrict__ val) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  k64[j] = desc_key(key_parent_of(members[j], label, parent, key_of));
  val[j] = int(j);
}

__global__ void spt_key_kernel(const int* __restrict__ order, const unsigned* __restrict__ spt_of, long long m,
                               unsigned* __restrict__ k32, int* __restrict__ val) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int j = order[r];
  k32[r] = spt_of[j];
  val[r] = j;
}

__global__ void records_kernel(const int* __restrict__ order, const int* __restrict__ members, long long m,
                               const int* __restrict__ label, const int* __restrict__ parent,
                               const double* __restrict__ key_of, int* __restrict__ rec_node,
                               double* __restrict__ key_self, double* __restrict__ key_parent) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const int node = members[order[r]];
  rec_node[r] = node;
  key_self[r] = key_of[node];
  key_parent[r] = key_parent_of(node, label, parent, key_of);
}

struct Scratch {
  unsigned char* small;
  int *label, *counts, *flags, *sid, *members, *v0, *v1;
  long long *pos, *totals;
  double* key_of;
  unsigned long long *k0, *k1;
  unsigned *s0, *s1, *spt_of;
  void* tmp;
  size_t tmp_bytes;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t tmp_bytes_for(long long cap) {
  const size_t a = radix_scratch_bytes(cap), b = scan_scratch_bytes(cap);
  return a > b ? a : b;
}

size_t carve(void* base, long long cap, Scratch* s) {
  char* p = static_cast<char*>(base);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += align_up(bytes);
    return q;
  };
  const size_t n = size_t(cap > 0 ? cap : 1);
  s->small = reinterpret_cast<unsigned char*>(take(n));
  s->label = reinterpret_cast<int*>(take(4 * n));
  s->counts = reinterpret_cast<int*>(take(4 * n));
  s->flags = reinterpret_cast<int*>(take(16 * n));
  s->sid = reinterpret_cast<int*>(take(4 * n));
  s->members = reinterpret_cast<int*>(take(4 * n));
  s->v0 = reinterpret_cast<int*>(take(4 * n));
  s->v1 = reinterpret_cast<int*>(take(4 * n));
  s->pos = reinterpret_cast<long long*>(take(8 * n));
  s->totals = reinterpret_cast<long long*>(take(8 * 8));
  s->key_of = reinterpret_cast<double*>(take(8 * n));
  s->k0 = reinterpret_cast<unsigned long long*>(take(8 * n));
  s->k1 = reinterpret_cast<unsigned long long*>(take(8 * n));
  s->s0 = reinterpret_cast<unsigned*>(take(4 * n));
  s->s1 = reinterpret_cast<unsigned*>(take(4 * n));
  s->spt_of = reinterpret_cast<unsigned*>(take(4 * n));
  s->tmp_bytes = tmp_bytes_for(cap);
  s->tmp = take(s->tmp_bytes);
  return off;
}

#define BK(x)                                   \
  do {                                          \
    cudaError_t e_ = (x);                       \
    if (e_ != cudaSuccess) return e_;           \
  } while (0)

cudaError_t hspt_build(const glod_hspt_build_in& in, const glod_hspt_build_out& out, void* scratch,
                       size_t scratch_bytes, int64_t* sizes, cudaStream_t st) {
  const long long cap = in.capacity;
  Scratch s;
  if (carve(nullptr, cap, &s) > scratch_bytes) return cudaErrorInvalidValue;
  carve(scratch, cap, &s);
  const int g = grid_for(cap);
  BK(cudaMemsetAsync(s.counts, 0, 4 * size_t(cap), st));
  BK(cudaMemsetAsync(s.sid, 0xff, 4 * size_t(cap), st));
  count_launch();
  small_kernel<<<g, kThreads, 0, st>>>(in.scales, cap, in.size_threshold, s.small);
  count_launch();
  walk_kernel<<<g, kThreads, 0, st>>>(in.parent, in.children, s.small, cap, in.root, s.label, s.counts);
  count_launch();
  flags_kernel<<<g, kThreads, 0, st>>>(s.label, s.counts, cap, in.min_subtree, s.flags);
  int* lists[4] = {out.upper_ids, out.pass_ids, out.spt_roots, s.members};
  for (int k = 0; k < 4; ++k) {
    BK(exclusive_scan_i32(s.flags + k * cap, s.pos, cap, s.tmp, s.tmp_bytes, st));
    count_launch();
    scatter_kernel<<<g, kThreads, 0, st>>>(s.flags + k * cap, s.pos, cap, lists[k], s.totals + k);
  }
  long long tot[4];
  BK(cudaMemcpyAsync(tot, s.totals, sizeof(tot), cudaMemcpyDeviceToHost, st));
  BK(cudaStreamSynchronize(st));
  const long long S = tot[2], M = tot[3];
  for (int k = 0; k < 4; ++k) sizes[k] = tot[k];
  if (S > 0) {
    count_launch();
    spt_id_kernel<<<grid_for(S), kThreads, 0, st>>>(out.spt_roots, s.counts, S, s.sid, out.spt_count);
    BK(exclusive_scan_i32(out.spt_count, reinterpret_cast<long long*>(out.spt_offset), S, s.tmp, s.tmp_bytes, st));
  }
  if (M == 0) return cudaGetLastError();
  const int gm = grid_for(M);
  count_launch();
  key_self_kernel<<<gm, kThreads, 0, st>>>(s.members, M, s.label, s.sid, in.means, in.scales, in.lod_threshold,
                                           in.metric, in.corrected, s.key_of, s.spt_of);
  count_launch();
  parent_key_kernel<<<gm, kThreads, 0, st>>>(s.members, M, s.label, in.parent, s.key_of, s.k0, s.v0);
  int alt = 0;
  BK(radix_sort_pairs<unsigned long long>(s.k0, s.k1, s.v0, s.v1, M, 0, 64, s.tmp, s.tmp_bytes, true, &alt, st));
  const int* order1 = alt ? s.v1 : s.v0;
  int* v2 = alt ? s.v0 : s.v1;
  count_launch();
  spt_key_kernel<<<gm, kThreads, 0, st>>>(order1, s.spt_of, M, s.s0, v2);
  int bits = 1;
  while ((1ll << bits) < S) ++bits;
  int* v3 = alt ? s.v1 : s.v0;       // the buffer order1 lived in is free again
  int alt2 = 0;
  BK(radix_sort_pairs<unsigned>(s.s0, s.s1, v2, v3, M, 0, bits, s.tmp, s.tmp_bytes, false, &alt2, st));
  const int* order = alt2 ? v3 : v2;
  count_launch();
  records_kernel<<<gm, kThreads, 0, st>>>(order, s.members, M, s.label, in.parent, s.key_of, out.rec_node,
                                          out.key_self, out.key_parent);
  return cudaGetLastError();
}

}  // namespace
}  // namespace glod

extern "C" {

int64_t glod_hspt_build_scratch_bytes(int64_t capacity) {
  glod::Scratch s;
  return int64_t(glod::carve(nullptr, capacity, &s));
}

int glod_hspt_build(const glod_hspt_build_in* in, const glod_hspt_build_out* out, void* scratch,
                    int64_t scratch_bytes, int64_t* sizes, void* stream) {
  if (!in || !out || !sizes || in->capacity <= 0 || in->root < 0 || in->root >= in->capacity)
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "glod_hspt_build: bad arguments");
  if (!(in->size_threshold > 0))
    return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "size_threshold must be > 0");
  if (in->min_subtree < 1) return glod::set_error(GLOD_ERR_INVALID_ARGUMENT, "min_subtree must be >= 1");
  cudaError_t e = glod::hspt_build(*in, *out, scratch, size_t(scratch_bytes), sizes,
                                   static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GLOD_OK : glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
