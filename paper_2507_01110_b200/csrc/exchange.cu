// K11-exchange: the sparse gradient exchange of view-sharded training
// (no single-view counterpart in the reference — the contract is
// "reduced gradient of node i = Σ over ranks of the single-view gradients").
//
// One process per GPU renders its own view.  Each step:
//   1. all-gather of the ranks' render-row node ids (4 B/id; rows are unique
//      within a view);
//   2. on-device union U: the ids are OR-ed into a node bitmap; node words
//      are owned round-robin, owner(id) = (id >> 5) mod N, and a scan over
//      the owner-major word order lays U out as N owner chunks, each sorted
//      by id (the same U on every rank, no sort);
//   3. every rank buckets its per-row gradients by owner (row = position in
//      the owner chunk + 23 f64) and the buckets travel point to point
//      (grouped ncclSend/ncclRecv — a sparse reduce-scatter: a rank ships
//      its R rows, not a dense |U| buffer);
//   4. the owner sums the received rows source by source (rank order: a
//      deterministic sum) into a section-major gradient block of its chunk;
//      the caller runs ADAM on it (glod_adam_step_records) — owner-sharded
//      ADAM, O(|U|/N) per rank, moments and step counts live on the owner;
//   5. the owners broadcast their updated attribute rows (23 f64) and every
//      rank writes all of U into its replicated node records.
// The kernels are usable without NCCL (glod_xchg_* phases, the transport
// supplied by the caller); glod_grad_exchange / glod_param_allgather compose
// them with NCCL over NVLink / NVSwitch.
#include <cub/cub.cuh>
#include <nccl.h>

#include <stdint.h>
#include <string.h>
#include <vector>

#include "../../include/glod_b200.h"
#include "common.cuh"

namespace glod {
namespace {

constexpr int F = 23;           // attribute values per node
constexpr int ROW = F + 1;      // wire row: owner-local position + 23 gradients
__constant__ int kOff[6] = {0, 3, 6, 10, 11, 14};
__constant__ int kCols[6] = {3, 3, 4, 1, 3, 9};

__global__ void mark_kernel(const int32_t* __restrict__ ids, long long n, uint32_t* __restrict__ bm,
                            long long cap) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int id = ids[i];
    if (id >= 0 && id < cap) atomicOr(bm + (id >> 5), 1u << (id & 31));
  }
}

// Virtual index v = o * Wmax + k  <->  word w = o + k * N (owner-major order).
__global__ void word_count_kernel(const uint32_t* __restrict__ bm, long long W, int N, long long Wmax,
                                  uint32_t* __restrict__ cnt) {
  const long long total = (long long)N * Wmax;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v <= total;
       v += (long long)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    if (v < total) {
      const long long w = v % Wmax * N + v / Wmax;
      c = w < W ? __popc(bm[w]) : 0u;
    }
    cnt[v] = c;
  }
}

__global__ void compact_kernel(const uint32_t* __restrict__ bm, long long W, int N, long long Wmax,
                               const uint32_t* __restrict__ base, int32_t* __restrict__ U) {
  const long long total = (long long)N * Wmax;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < total;
       v += (long long)gridDim.x * blockDim.x) {
    const long long w = v % Wmax * N + v / Wmax;
    if (w >= W) continue;
    uint32_t b = bm[w];
    uint32_t o = base[v];
    while (b) {
      const int bit = __ffs(b) - 1;
      U[o++] = int32_t(w * 32 + bit);
      b &= b - 1;
    }
  }
}

GLOD_DEV long long owner_pos(const uint32_t* bm, const uint32_t* base, int id, int N, long long Wmax,
                             int& owner) {
  const long long w = id >> 5;
  owner = int(w % N);
  const long long v = (long long)owner * Wmax + w / N;
  const uint32_t below = (1u << (id & 31)) - 1u;
  return (long long)base[v] + __popc(bm[w] & below) - (long long)base[(long long)owner * Wmax];
}

__global__ void bucket_count_kernel(const int32_t* __restrict__ row_node, long long R, int N,
                                    unsigned long long* __restrict__ cnt) {
  __shared__ unsigned long long s[32];
  if (threadIdx.x < 32) s[threadIdx.x] = 0;
  __syncthreads();
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < R; r += (long long)gridDim.x * blockDim.x)
    atomicAdd(&s[(row_node[r] >> 5) % N], 1ull);
  __syncthreads();
  if (threadIdx.x < N && s[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], s[threadIdx.x]);
}

// cnt[0..N) -> exclusive offsets in slot[0..N) (cursor) and off[0..N]
__global__ void bucket_scan_kernel(const unsigned long long* __restrict__ cnt, int N,
                                   unsigned long long* __restrict__ cursor, long long* __restrict__ counts_out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long a = 0;
    for (int o = 0; o < N; ++o) {
      cursor[o] = a;
      counts_out[o] = (long long)cnt[o];
      a += cnt[o];
    }
  }
}

// One warp per render row: owner position, then the 23 gradients (section-
// major, R rows) as one 24-value wire row.
__global__ void pack_rows_kernel(const int32_t* __restrict__ row_node, const double* __restrict__ G, long long R,
                                 const uint32_t* __restrict__ bm, const uint32_t* __restrict__ base, int N,
                                 long long Wmax, unsigned long long* __restrict__ cursor,
                                 double* __restrict__ send) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    const int id = row_node[r];
    int owner = 0;
    long long pos = 0;
    unsigned long long slot = 0;
    if (lane == 0) {
      pos = owner_pos(bm, base, id, N, Wmax, owner);
      slot = atomicAdd(&cursor[owner], 1ull);
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    double* out = send + slot * ROW;
    if (lane == 0) out[0] = double(pos);
    if (lane < F) {
      int sec = 0;
#pragma unroll
      for (int k = 1; k < 6; ++k) sec += lane >= kOff[k];
      const int col = lane - kOff[sec];
      out[1 + lane] = G[kOff[sec] * R + r * kCols[sec] + col];
    }
  }
}

// acc (section-major, n rows) += the rows of one source, in that source's
// order; the positions within one source are distinct, so no atomics.
__global__ void accumulate_kernel(const double* __restrict__ rows, long long m, double* __restrict__ acc,
                                  long long n) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long i = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
    const double* in = rows + i * ROW;
    const long long pos = (long long)in[0];
    if (lane < F && pos >= 0 && pos < n) {
      int sec = 0;
#pragma unroll
      for (int k = 1; k < 6; ++k) sec += lane >= kOff[k];
      const int col = lane - kOff[sec];
      double* a = acc + kOff[sec] * n + pos * kCols[sec] + col;
      *a = *a + in[1 + lane];
    }
  }
}

// params_all[j] (23 f64, row-major) <- record of U[j], for j in [lo, hi)
__global__ void pack_params_kernel(const double* __restrict__ rec, long long stride, const int32_t* __restrict__ U,
                                   long long lo, long long hi, double* __restrict__ out) {
  const long long n = (hi - lo) * F;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long j = lo + e / F;
    out[j * F + e % F] = rec[(long long)U[j] * stride + e % F];
  }
}

__global__ void scatter_params_kernel(const double* __restrict__ in, const int32_t* __restrict__ U, long long n,
                                      double* __restrict__ rec, long long stride) {
  const long long total = n * F;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / F;
    rec[(long long)U[j] * stride + e % F] = in[e];
  }
}

unsigned grid_for(long long n, int tb = 256) {
  long long g = (n + tb - 1) / tb;
  return unsigned(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

template <typename T>
cudaError_t ensure(T*& p, size_t& cap, size_t n) {
  if (n <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  size_t want = n + n / 4 + 64;
  cudaError_t e = cudaMalloc(&p, want * sizeof(T));
  if (e == cudaSuccess) cap = want;
  return e;
}

}  // namespace
}  // namespace glod

using namespace glod;

struct glod_xchg {
  int N = 1, rank = 0;
  long long cap = 0, W = 0, Wmax = 0;
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  uint32_t* bm = nullptr;
  uint32_t* cnt = nullptr;
  uint32_t* base = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int32_t* U = nullptr;
  size_t U_cap = 0;
  long long nU = 0;
  std::vector<long long> off;             // host: owner chunk offsets [N+1]
  uint32_t* h_off = nullptr;              // pinned staging for the N+1 offsets
  // step buffers
  int32_t* ids_send = nullptr;
  size_t ids_send_cap = 0;
  int32_t* ids_all = nullptr;
  size_t ids_all_cap = 0;
  long long* d_count = nullptr;           // [N] this rank's R (all-gathered) / bucket counts
  long long* d_counts_all = nullptr;      // [N*N]
  long long* h_counts = nullptr;          // pinned [N*N]
  unsigned long long* d_bucket = nullptr; // [2N]: counts | cursors
  double* send = nullptr;
  size_t send_cap = 0;
  double* recv = nullptr;
  size_t recv_cap = 0;
  double* acc = nullptr;
  size_t acc_cap = 0;
  double* params = nullptr;
  size_t params_cap = 0;
  std::vector<long long> send_cnt, recv_cnt;
  long long bytes_sent = 0, bytes_recv = 0;
};

namespace {
int xfail(int code, const char* what) { return glod::set_error(code, what); }
int cuda_fail(cudaError_t e) { return glod::set_error(GLOD_ERR_CUDA, cudaGetErrorString(e)); }
int nccl_fail(ncclResult_t r) { return glod::set_error(GLOD_ERR_CUDA, ncclGetErrorString(r)); }
#define XCUDA(x)                              \
  do {                                        \
    cudaError_t e_ = (x);                     \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)
#define XNCCL(x)                              \
  do {                                        \
    ncclResult_t r_ = (x);                    \
    if (r_ != ncclSuccess) return nccl_fail(r_); \
  } while (0)

int read_offsets(glod_xchg* x, cudaStream_t st) {
  // off[o] = base[o * Wmax], off[N] = base[N * Wmax] (= |U|)
  // kernel read-backs: the D2H copy engine may be busy with write-backs
  for (int o = 0; o <= x->N; ++o)
    XCUDA(launch_readback(x->h_off + o, x->base + (long long)o * x->Wmax, sizeof(uint32_t), st));
  XCUDA(cudaStreamSynchronize(st));
  x->off.assign(x->N + 1, 0);
  for (int o = 0; o <= x->N; ++o) x->off[o] = x->h_off[o];
  x->nU = x->off[x->N];
  return 0;
}
}  // namespace

extern "C" {

int glod_nccl_unique_id(void* out128) {
  if (!out128) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  ncclUniqueId id;
  XNCCL(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int glod_xchg_create(int32_t nranks, int32_t rank, int64_t capacity, const void* nccl_id128, glod_xchg** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || capacity < 1)
    return xfail(GLOD_ERR_INVALID_ARGUMENT, "invalid exchange arguments");
  glod_xchg* x = new glod_xchg();
  x->N = nranks;
  x->rank = rank;
  x->cap = capacity;
  x->W = (capacity + 31) / 32;
  x->Wmax = (x->W + nranks - 1) / nranks;
  const long long nv = (long long)nranks * x->Wmax + 1;
  cudaError_t e = cudaMalloc(&x->bm, x->W * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&x->cnt, nv * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&x->base, nv * sizeof(uint32_t));
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, x->cub_bytes, x->cnt, x->base, nv);
  if (e == cudaSuccess) e = cudaMalloc(&x->cub_tmp, x->cub_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&x->d_count, nranks * sizeof(long long));
  if (e == cudaSuccess) e = cudaMalloc(&x->d_counts_all, (size_t)nranks * nranks * sizeof(long long));
  if (e == cudaSuccess) e = cudaMalloc(&x->d_bucket, 2 * nranks * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMallocHost(&x->h_counts, (size_t)nranks * nranks * sizeof(long long));
  if (e == cudaSuccess) e = cudaMallocHost(&x->h_off, (nranks + 1) * sizeof(uint32_t));
  if (e != cudaSuccess) {
    delete x;
    return cuda_fail(e);
  }
  if (nccl_id128) {
    ncclUniqueId id;
    memcpy(&id, nccl_id128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&x->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete x;
      return nccl_fail(r);
    }
    x->own_comm = true;
  }
  *out = x;
  return 0;
}

int glod_xchg_destroy(glod_xchg* x) {
  if (!x) return 0;
  if (x->comm && x->own_comm) ncclCommDestroy(x->comm);
  void* dev[] = {x->bm, x->cnt, x->base, x->cub_tmp, x->U, x->ids_send, x->ids_all, x->d_count,
                 x->d_counts_all, x->d_bucket, x->send, x->recv, x->acc, x->params};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (x->h_counts) cudaFreeHost(x->h_counts);
  if (x->h_off) cudaFreeHost(x->h_off);
  delete x;
  return 0;
}

// Phase 2: union of the gathered ids (n entries, -1 = padding) -> owner-major
// U; returns the N+1 owner offsets on the host (one sync).
int glod_xchg_union(glod_xchg* x, const int32_t* ids_all, int64_t n, int64_t* owner_off, void* stream) {
  if (!x || (n > 0 && !ids_all)) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long nv = (long long)x->N * x->Wmax + 1;
  XCUDA(cudaMemsetAsync(x->bm, 0, x->W * sizeof(uint32_t), st));
  if (n > 0) {
    mark_kernel<<<grid_for(n), 256, 0, st>>>(ids_all, n, x->bm, x->cap);
    count_launch();
  }
  word_count_kernel<<<grid_for(nv), 256, 0, st>>>(x->bm, x->W, x->N, x->Wmax, x->cnt);
  count_launch();
  XCUDA(cub::DeviceScan::ExclusiveSum(x->cub_tmp, x->cub_bytes, x->cnt, x->base, nv, st));
  count_launch();
  if (int rc = read_offsets(x, st)) return rc;
  XCUDA(ensure(x->U, x->U_cap, size_t(x->nU > 0 ? x->nU : 1)));
  compact_kernel<<<grid_for(nv - 1), 256, 0, st>>>(x->bm, x->W, x->N, x->Wmax, x->base, x->U);
  count_launch();
  XCUDA(cudaGetLastError());
  if (owner_off)
    for (int o = 0; o <= x->N; ++o) owner_off[o] = x->off[o];
  return 0;
}

// The owner-major union (device pointer, |U| entries) of the last union call.
int glod_xchg_union_ids(glod_xchg* x, const int32_t** ids, int64_t* n) {
  if (!x || !ids || !n) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  *ids = x->U;
  *n = x->nU;
  return 0;
}

// Phase 3a: bucket this rank's R rows (node ids + section-major gradients)
// by owner into the send buffer; counts[o] (host) = rows for owner o, the
// bucket for o starts at row sum(counts[:o]).  One sync.
int glod_xchg_pack(glod_xchg* x, const int32_t* row_node, const double* grads, int64_t R, int64_t* counts,
                   const double** send_out, void* stream) {
  if (!x || (R > 0 && (!row_node || !grads))) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  XCUDA(ensure(x->send, x->send_cap, size_t(R > 0 ? R : 1) * ROW));
  XCUDA(cudaMemsetAsync(x->d_bucket, 0, 2 * x->N * sizeof(unsigned long long), st));
  if (R > 0) {
    bucket_count_kernel<<<grid_for(R), 256, 0, st>>>(row_node, R, x->N, x->d_bucket);
    count_launch();
  }
  bucket_scan_kernel<<<1, 32, 0, st>>>(x->d_bucket, x->N, x->d_bucket + x->N, x->d_count);
  count_launch();
  if (R > 0) {
    pack_rows_kernel<<<grid_for(R * 32), 256, 0, st>>>(row_node, grads, R, x->bm, x->base, x->N, x->Wmax,
                                                      x->d_bucket + x->N, x->send);
    count_launch();
  }
  XCUDA(cudaGetLastError());
  XCUDA(launch_readback(x->h_counts, x->d_count, x->N * sizeof(long long), st));
  XCUDA(cudaStreamSynchronize(st));
  x->send_cnt.assign(x->h_counts, x->h_counts + x->N);
  if (counts)
    for (int o = 0; o < x->N; ++o) counts[o] = x->send_cnt[o];
  if (send_out) *send_out = x->send;
  return 0;
}

// Phase 3b: the owner's accumulator (section-major, |U_rank| rows), zeroed.
int glod_xchg_begin_accumulate(glod_xchg* x, double** acc, int64_t* n_owned, void* stream) {
  if (!x) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long n = x->off[x->rank + 1] - x->off[x->rank];
  XCUDA(ensure(x->acc, x->acc_cap, size_t(n > 0 ? n : 1) * F));
  XCUDA(cudaMemsetAsync(x->acc, 0, size_t(n > 0 ? n : 1) * F * sizeof(double), st));
  if (acc) *acc = x->acc;
  if (n_owned) *n_owned = n;
  return 0;
}

// Phase 3c: add `m` received wire rows of one source (call in rank order).
int glod_xchg_accumulate(glod_xchg* x, const double* rows, int64_t m, void* stream) {
  if (!x || (m > 0 && !rows)) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  const long long n = x->off[x->rank + 1] - x->off[x->rank];
  if (m > 0) {
    accumulate_kernel<<<grid_for(m * 32), 256, 0, static_cast<cudaStream_t>(stream)>>>(rows, m, x->acc, n);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e);
}

// Owned ids (device pointer into U) and the accumulated gradients.
int glod_xchg_owned(glod_xchg* x, const int32_t** ids, const double** grads, int64_t* n) {
  if (!x) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (ids) *ids = x->U + x->off[x->rank];
  if (grads) *grads = x->acc;
  if (n) *n = x->off[x->rank + 1] - x->off[x->rank];
  return 0;
}

// Phase 5a: this rank's updated attribute rows -> its chunk of the |U| x 23
// row-major params buffer (returned, for the caller's transport).
int glod_xchg_pack_params(glod_xchg* x, const double* records, int64_t stride, double** params, void* stream) {
  if (!x || !records) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  XCUDA(ensure(x->params, x->params_cap, size_t(x->nU > 0 ? x->nU : 1) * F));
  const long long lo = x->off[x->rank], hi = x->off[x->rank + 1];
  if (hi > lo) {
    pack_params_kernel<<<grid_for((hi - lo) * F), 256, 0, st>>>(records, stride, x->U, lo, hi, x->params);
    count_launch();
  }
  if (params) *params = x->params;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e);
}

// Phase 5b: every row of U from the params buffer into the node records.
int glod_xchg_scatter_params(glod_xchg* x, double* records, int64_t stride, void* stream) {
  if (!x || !records) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (x->nU > 0) {
    scatter_params_kernel<<<grid_for(x->nU * F), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x->params, x->U, x->nU, records, stride);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : cuda_fail(e);
}

int glod_xchg_stats(glod_xchg* x, int64_t* out4) {
  if (!x || !out4) return xfail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  out4[0] = x->nU;
  out4[1] = x->off.empty() ? 0 : x->off[x->rank + 1] - x->off[x->rank];
  out4[2] = x->bytes_sent;
  out4[3] = x->bytes_recv;
  return 0;
}

// ---- the NCCL composition ---------------------------------------------------
// Phases 1-4: ids all-gather, union, bucketed gradients sent to their
// owners, owner-side sums.  On return the owned ids / gradients are ready
// for ADAM (glod_xchg_owned).
int glod_grad_exchange(glod_xchg* x, const int32_t* row_node, const double* grads, int64_t R, int64_t* n_owned,
                       void* stream) {
  if (!x || !x->comm) return xfail(GLOD_ERR_INVALID_ARGUMENT, "exchange has no communicator");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int N = x->N;
  // 1. row counts, then the padded id lists
  long long myR = R;
  XCUDA(launch_set_bytes(x->d_count, &myR, sizeof(long long), st));
  XNCCL(ncclAllGather(x->d_count, x->d_counts_all, 1, ncclInt64, x->comm, st));
  XCUDA(launch_readback(x->h_counts, x->d_counts_all, N * sizeof(long long), st));
  XCUDA(cudaStreamSynchronize(st));
  long long Rmax = 1;
  for (int s = 0; s < N; ++s) Rmax = x->h_counts[s] > Rmax ? x->h_counts[s] : Rmax;
  XCUDA(ensure(x->ids_send, x->ids_send_cap, size_t(Rmax)));
  XCUDA(ensure(x->ids_all, x->ids_all_cap, size_t(Rmax) * N));
  XCUDA(cudaMemsetAsync(x->ids_send, 0xff, Rmax * sizeof(int32_t), st));
  if (R > 0) XCUDA(cudaMemcpyAsync(x->ids_send, row_node, R * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  XNCCL(ncclAllGather(x->ids_send, x->ids_all, Rmax, ncclInt32, x->comm, st));
  // 2. union
  if (int rc = glod_xchg_union(x, x->ids_all, Rmax * N, nullptr, stream)) return rc;
  // 3. bucket by owner; the count matrix tells every rank what it receives
  if (int rc = glod_xchg_pack(x, row_node, grads, R, nullptr, nullptr, stream)) return rc;
  XNCCL(ncclAllGather(x->d_count, x->d_counts_all, N, ncclInt64, x->comm, st));
  XCUDA(launch_readback(x->h_counts, x->d_counts_all, (size_t)N * N * sizeof(long long), st));
  XCUDA(cudaStreamSynchronize(st));
  x->recv_cnt.assign(N, 0);
  long long total_recv = 0;
  for (int s = 0; s < N; ++s) total_recv += (x->recv_cnt[s] = x->h_counts[(size_t)s * N + x->rank]);
  XCUDA(ensure(x->recv, x->recv_cap, size_t(total_recv > 0 ? total_recv : 1) * ROW));
  XNCCL(ncclGroupStart());
  long long so = 0, ro = 0;
  for (int p = 0; p < N; ++p) {
    if (x->send_cnt[p] > 0) XNCCL(ncclSend(x->send + so * ROW, x->send_cnt[p] * ROW, ncclFloat64, p, x->comm, st));
    if (x->recv_cnt[p] > 0) XNCCL(ncclRecv(x->recv + ro * ROW, x->recv_cnt[p] * ROW, ncclFloat64, p, x->comm, st));
    so += x->send_cnt[p];
    ro += x->recv_cnt[p];
  }
  XNCCL(ncclGroupEnd());
  x->bytes_sent = (so - x->send_cnt[x->rank]) * ROW * 8 + Rmax * 4 * (N - 1);
  x->bytes_recv = (ro - x->recv_cnt[x->rank]) * ROW * 8 + Rmax * 4 * (N - 1);
  // 4. owner sums, source by source
  if (int rc = glod_xchg_begin_accumulate(x, nullptr, n_owned, stream)) return rc;
  ro = 0;
  for (int s = 0; s < N; ++s) {
    if (int rc = glod_xchg_accumulate(x, x->recv + ro * ROW, x->recv_cnt[s], stream)) return rc;
    ro += x->recv_cnt[s];
  }
  return 0;
}

// Phase 5: owners broadcast their updated rows; every rank writes all of U
// into its node records.
int glod_param_allgather(glod_xchg* x, double* records, int64_t stride, void* stream) {
  if (!x || !x->comm) return xfail(GLOD_ERR_INVALID_ARGUMENT, "exchange has no communicator");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = glod_xchg_pack_params(x, records, stride, nullptr, stream)) return rc;
  XNCCL(ncclGroupStart());
  for (int o = 0; o < x->N; ++o) {
    const long long n = x->off[o + 1] - x->off[o];
    if (n > 0) {
      double* p = x->params + x->off[o] * F;
      XNCCL(ncclBroadcast(p, p, n * F, ncclFloat64, o, x->comm, st));
    }
  }
  XNCCL(ncclGroupEnd());
  x->bytes_recv += (x->nU - (x->off[x->rank + 1] - x->off[x->rank])) * F * 8;
  return glod_xchg_scatter_params(x, records, stride, stream);
}

}  // extern "C"
