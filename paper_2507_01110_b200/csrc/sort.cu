// K6: hand-written stable LSD radix sort (key, value) for the rasteriser.
//
// Two uses: the global depth order (fp64 depth bits, ties by render-set
// index — renderer.py:127's lexsort((idx, depth))) and the per-tile binning
// (13-bit tile ids over instances emitted in depth-rank order).  8-bit
// digits; per pass three kernels:
//   hist     per-block digit histograms of a contiguous chunk
//   scan     digit-major exclusive scan of the block histograms
//   scatter  each block re-reads its chunk in input order, ranks every
//            element stably within its warp (match_any per item slot,
//            warp-private running counters) and across warps (per-digit
//            prefix over the 8 warps), reorders each 2048-element round by
//            digit in shared memory and writes it out as contiguous
//            per-digit runs (coalesced stores)
// Only the bit range where keys differ is sorted (min/max reduction first),
// so positive fp64 depths cost ~6-7 passes, tile ids 2.
#include <stdint.h>

#include "common.cuh"
#include "../../include/glod_b200.h"

namespace glod {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItems = 8;                                   // per thread per round
constexpr int kRound = kSortThreads * kItems;               // 2048 elements
constexpr int kBins = 256;
static_assert(kSortThreads == kBins, "scatter_kernel: one thread per digit");

template <typename K> GLOD_DEV unsigned digit_of(K k, int shift) { return unsigned(k >> shift) & 0xffu; }

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
hist_kernel(const K* __restrict__ keys, long long n, long long chunk, int shift,
            unsigned* __restrict__ bh, int nblocks) {
  __shared__ unsigned h[kBins];
  for (int i = threadIdx.x; i < kBins; i += kSortThreads) h[i] = 0;
  __syncthreads();
  const long long lo = (long long)blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (long long i = lo + threadIdx.x; i < hi; i += kSortThreads) atomicAdd(&h[digit_of(keys[i], shift)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < kBins; d += kSortThreads) bh[(long long)d * nblocks + blockIdx.x] = h[d];
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads)
scatter_kernel(const K* __restrict__ kin, K* __restrict__ kout, const int* __restrict__ vin,
               int* __restrict__ vout, long long n, long long chunk, int shift,
               const unsigned* __restrict__ bh, int nblocks) {
  __shared__ unsigned base[kBins];                 // global slot of this block's next element per digit
  __shared__ unsigned wcnt[kSortWarps][kBins];     // per-warp counts → per-warp offsets within the round
  __shared__ unsigned dstart[kBins];               // round-local start of each digit's run
  __shared__ long long scan_sm[kSortThreads / 32 + 1];
  __shared__ K skey[kRound];                       // the round in (digit, input) order
  __shared__ int sval[kRound];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kBins; d += kSortThreads) base[d] = bh[(long long)d * nblocks + blockIdx.x];
  const long long lo = (long long)blockIdx.x * chunk, hi = min(n, lo + chunk);
  for (long long r0 = lo; r0 < hi; r0 += kRound) {
    for (int i = threadIdx.x; i < kSortWarps * kBins; i += kSortThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    // warp w owns elements [r0 + w*256, r0 + (w+1)*256): slot k, lane l → +k*32+l
    K kv[kItems];
    int vv[kItems];
    unsigned pos[kItems];
    unsigned dg[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const long long i = r0 + warp * (kItems * 32) + k * 32 + lane;
      const bool ok = i < hi;
      kv[k] = ok ? kin[i] : K(0);
      vv[k] = ok ? vin[i] : 0;
      const unsigned d = digit_of(kv[k], shift);
      dg[k] = ok ? d : 0xffffffffu;
      const unsigned peers = __match_any_sync(0xffffffffu, dg[k]);
      unsigned p = 0;
      if (ok) p = wcnt[warp][d] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (ok && (peers & lanemask_lt()) == 0) wcnt[warp][d] += __popc(peers);   // leader
      __syncwarp();
      pos[k] = p;
    }
    __syncthreads();
    // per digit (thread d): exclusive prefix over warps, round total → scan
    // over digits gives each digit's run start inside the round
    unsigned tot = 0;
    {
      const int d = threadIdx.x;                   // kSortThreads == kBins
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const unsigned c = wcnt[w][d];
        wcnt[w][d] = tot;
        tot += c;
      }
    }
    const unsigned ds = unsigned(block_excl_scan((long long)tot, scan_sm));
    dstart[threadIdx.x] = ds;
    __syncthreads();
    // scatter into shared memory in (digit, input) order — stable
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      if (dg[k] != 0xffffffffu) {
        const unsigned lp = dstart[dg[k]] + wcnt[warp][dg[k]] + pos[k];
        skey[lp] = kv[k];
        sval[lp] = vv[k];
      }
    }
    __syncthreads();
    // write out: consecutive threads → consecutive slots of one digit's run
    const int cnt = int(min((long long)kRound, hi - r0));
    for (int i = threadIdx.x; i < cnt; i += kSortThreads) {
      const K key = skey[i];
      const unsigned d = digit_of(key, shift);
      const unsigned g = base[d] + (unsigned(i) - dstart[d]);
      kout[g] = key;
      vout[g] = sval[i];
    }
    __syncthreads();
    base[threadIdx.x] += tot;
  }
}

// min/max over keys != ~0 (the "invalid" marker: invisible Gaussians, which
// the rasteriser skips wherever they land — only the valid keys' relative
// order matters)
template <typename K>
__global__ void minmax_kernel(const K* __restrict__ keys, long long n, K* __restrict__ out) {
  __shared__ K smin[kSortThreads], smax[kSortThreads];
  K mn = ~K(0), mx = K(0);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const K k = keys[i];
    if (k == ~K(0)) continue;
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int s = kSortThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = smin[threadIdx.x + s] < smin[threadIdx.x] ? smin[threadIdx.x + s] : smin[threadIdx.x];
      smax[threadIdx.x] = smax[threadIdx.x + s] > smax[threadIdx.x] ? smax[threadIdx.x + s] : smax[threadIdx.x];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicMin(reinterpret_cast<unsigned long long*>(out), (unsigned long long)smin[0]);
    atomicMax(reinterpret_cast<unsigned long long*>(out) + 1, (unsigned long long)smax[0]);
  }
}

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;

template <typename In>
__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const In* __restrict__ in, long long n, long long* __restrict__ bsum) {
  __shared__ long long sm[kScanThreads / 32 + 1];
  const long long base = (long long)blockIdx.x * kScanThreads * kScanItems;
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long i = base + (long long)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  block_excl_scan(s, sm);
  if (threadIdx.x == 0) bsum[blockIdx.x] = sm[kScanThreads / 32];
}

__global__ void __launch_bounds__(kScanThreads)
scan_blocks_kernel(long long* __restrict__ bsum, int nb) {
  __shared__ long long sm[kScanThreads / 32 + 1];
  const int per = (nb + kScanThreads - 1) / kScanThreads;
  const int a = per * threadIdx.x, b = min(nb, a + per);
  long long s = 0;
  for (int i = a; i < b; ++i) s += bsum[i];
  long long o = block_excl_scan(s, sm);
  for (int i = a; i < b; ++i) {
    const long long v = bsum[i];
    bsum[i] = o;
    o += v;
  }
}

// blocked arrangement per thread (kScanItems consecutive) for the final scan
template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads)
scan_final_kernel(const In* __restrict__ in, long long n, const long long* __restrict__ bsum,
                  Out* __restrict__ out) {
  __shared__ long long sm[kScanThreads / 32 + 1];
  const long long base = (long long)blockIdx.x * kScanThreads * kScanItems + (long long)threadIdx.x * kScanItems;
  long long v[kScanItems];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? (long long)in[base + k] : 0;
    s += v[k];
  }
  long long o = bsum[blockIdx.x] + block_excl_scan(s, sm);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = Out(o);
    o += v[k];
  }
}

}  // namespace

size_t scan_scratch_bytes(long long n) {
  const long long nb = (n + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems);
  return size_t(nb > 0 ? nb : 1) * 8 + 64;
}

// out[i] = sum(in[0..i)) for i in [0, n): reduce / scan block sums / final
template <typename In, typename Out>
cudaError_t exclusive_scan(const In* in, Out* out, long long n, void* scratch, size_t bytes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (bytes < scan_scratch_bytes(n)) return cudaErrorInvalidValue;
  const int nb = int((n + kScanThreads * kScanItems - 1) / (kScanThreads * kScanItems));
  long long* bsum = static_cast<long long*>(scratch);
  count_launch();
  scan_reduce_kernel<In><<<nb, kScanThreads, 0, st>>>(in, n, bsum);
  count_launch();
  scan_blocks_kernel<<<1, kScanThreads, 0, st>>>(bsum, nb);
  count_launch();
  scan_final_kernel<In, Out><<<nb, kScanThreads, 0, st>>>(in, n, bsum, out);
  return cudaGetLastError();
}

cudaError_t exclusive_scan_i32(const int* in, long long* out, long long n, void* scratch, size_t bytes,
                               cudaStream_t st) {
  return exclusive_scan<int, long long>(in, out, n, scratch, bytes, st);
}

size_t scan_scratch_bytes(long long n);
template <typename In, typename Out>
cudaError_t exclusive_scan(const In* in, Out* out, long long n, void* scratch, size_t bytes, cudaStream_t st);

// Each block sorts a chunk of whole rounds; ~4 blocks per SM keeps the
// digit-major histogram scan short.
long long chunk_for(long long n) {
  long long rounds = (n + kRound - 1) / kRound;
  long long per = (rounds + 148 * 4 - 1) / (148 * 4);
  return (per < 1 ? 1 : per) * kRound;
}

// Scratch: histograms (256 × nblocks u32), their exclusive scan (u32),
// 2 × u64 min/max, scan block sums.
// Sized for the block count bound min(rounds, 148·4) rather than the exact
// count, so the size is monotone in n (a buffer sized for n fits every
// shorter sort).
size_t radix_scratch_bytes(long long n) {
  const long long rounds = (n + kRound - 1) / kRound;
  const long long nb = rounds < 148 * 4 ? rounds : 148 * 4;
  const size_t m = size_t(kBins) * size_t(nb > 0 ? nb : 1);
  return 2 * m * 4 + 64 + scan_scratch_bytes((long long)m) + 256;
}

// Sorts (keys, vals) of length n stably by key bits [begin_bit, end_bit).
// Ping-pongs between the in/alt buffers; returns 0 if the result is in the
// original buffers, 1 if in the alternates.  `range_bits`: narrow the bit
// range to where min and max keys differ (needs one host sync).
template <typename K>
cudaError_t radix_sort_pairs(K* keys, K* keys_alt, int* vals, int* vals_alt, long long n, int begin_bit,
                             int end_bit, void* scratch, size_t scratch_bytes, bool range_bits,
                             int* result_in_alt, cudaStream_t st) {
  *result_in_alt = 0;
  if (n <= 1) return cudaSuccess;
  if (scratch_bytes < radix_scratch_bytes(n)) return cudaErrorInvalidValue;
  const long long chunk = chunk_for(n);
  const int nblocks = int((n + chunk - 1) / chunk);
  const size_t m = size_t(kBins) * nblocks;
  unsigned* bh = static_cast<unsigned*>(scratch);
  unsigned* bo = bh + m;
  char* tail = static_cast<char*>(scratch) + 2 * m * 4;
  unsigned long long* mm = reinterpret_cast<unsigned long long*>(tail);
  void* scan_tmp = tail + 64;
  const size_t scan_bytes = scratch_bytes - (2 * m * 4 + 64);
  if (range_bits) {
    unsigned long long init[2] = {~0ull, 0ull};
    cudaError_t e = launch_set_bytes(mm, init, sizeof(init), st);
    if (e != cudaSuccess) return e;
    count_launch();
    minmax_kernel<K><<<148 * 4, kSortThreads, 0, st>>>(keys, n, reinterpret_cast<K*>(mm));
    // read back through a kernel into pinned memory (the D2H copy engine may
    // be busy with the cache's write-back DMA)
    static thread_local unsigned long long* hp = nullptr;
    if (!hp && (e = cudaMallocHost(&hp, 16)) != cudaSuccess) return e;
    e = launch_readback(hp, mm, 16, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const unsigned long long h[2] = {hp[0], hp[1]};
    if (h[0] > h[1]) return cudaSuccess;               // no valid keys
    const unsigned long long diff = (h[0] ^ h[1]) >> begin_bit << begin_bit;
    if (diff == 0) return cudaSuccess;                 // all valid keys equal: order kept
    const int top = 64 - __builtin_clzll(diff);
    end_bit = top < end_bit ? top : end_bit;
  }
  K* kin = keys; K* kout = keys_alt;
  int* vin = vals; int* vout = vals_alt;
  int flips = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    count_launch();
    hist_kernel<K><<<nblocks, kSortThreads, 0, st>>>(kin, n, chunk, shift, bh, nblocks);
    cudaError_t e = exclusive_scan<unsigned, unsigned>(bh, bo, (long long)m, scan_tmp, scan_bytes, st);
    if (e != cudaSuccess) return e;
    count_launch();
    scatter_kernel<K><<<nblocks, kSortThreads, 0, st>>>(kin, kout, vin, vout, n, chunk, shift, bo, nblocks);
    K* tk = kin; kin = kout; kout = tk;
    int* tv = vin; vin = vout; vout = tv;
    ++flips;
  }
  *result_in_alt = flips & 1;
  return cudaGetLastError();
}

template cudaError_t radix_sort_pairs<unsigned long long>(unsigned long long*, unsigned long long*, int*, int*,
                                                          long long, int, int, void*, size_t, bool, int*,
                                                          cudaStream_t);
template cudaError_t radix_sort_pairs<unsigned>(unsigned*, unsigned*, int*, int*, long long, int, int, void*,
                                                size_t, bool, int*, cudaStream_t);

}  // namespace glod

extern "C" {

int64_t glod_sort_scratch_bytes(int64_t n) { return int64_t(glod::radix_scratch_bytes(n)); }

int glod_sort_pairs_u64(uint64_t* keys, uint64_t* keys_alt, int32_t* vals, int32_t* vals_alt, int64_t n,
                        int32_t begin_bit, int32_t end_bit, void* scratch, int64_t scratch_bytes,
                        int32_t* result_in_alt, void* stream) {
  int alt = 0;
  cudaError_t e = glod::radix_sort_pairs<unsigned long long>(
      reinterpret_cast<unsigned long long*>(keys), reinterpret_cast<unsigned long long*>(keys_alt), vals,
      vals_alt, n, begin_bit, end_bit, scratch, size_t(scratch_bytes), false, &alt,
      static_cast<cudaStream_t>(stream));
  if (result_in_alt) *result_in_alt = alt;
  return e == cudaSuccess ? 0 : glod::set_error(2, cudaGetErrorString(e));
}

int glod_sort_pairs_u32(uint32_t* keys, uint32_t* keys_alt, int32_t* vals, int32_t* vals_alt, int64_t n,
                        int32_t begin_bit, int32_t end_bit, void* scratch, int64_t scratch_bytes,
                        int32_t* result_in_alt, void* stream) {
  int alt = 0;
  cudaError_t e = glod::radix_sort_pairs<unsigned>(keys, keys_alt, vals, vals_alt, n, begin_bit, end_bit,
                                                   scratch, size_t(scratch_bytes), false, &alt,
                                                   static_cast<cudaStream_t>(stream));
  if (result_in_alt) *result_in_alt = alt;
  return e == cudaSuccess ? 0 : glod::set_error(2, cudaGetErrorString(e));
}

}  // extern "C"
