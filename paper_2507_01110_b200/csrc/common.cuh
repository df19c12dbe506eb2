// Shared device helpers for the glod_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GLOD_DEV __device__ __forceinline__

namespace glod {

// One block to materialise (cache_table.cu → gather.cu materialize_kernel).
struct glod_mat_item {
  double* block;
  long long rows;
  long long elem_start;    // 23 · rows of all earlier items
  long long rec_offset;    // first record of the block's SPT in rec_node
};

// Small stream-ordered transfers that stay off the copy engines (gather.cu):
// kernel reads of mapped pinned memory / kernel writes of ≤ 64 bytes.
cudaError_t launch_upload(void* dst, const void* host_pinned, long long bytes, cudaStream_t st);
cudaError_t launch_readback(void* host_pinned, const void* src, long long bytes, cudaStream_t st);
cudaError_t launch_set_bytes(void* dst, const void* src, int bytes, cudaStream_t st);

// The master rows behind a cache block's touched bits (cache_table.cu →
// gather.cu load/pack kernels): node records of `stride` doubles (or packed
// section-major rows of `cap`), the LoD scene's record → node map, and the
// first record of each transfer item's SPT.  master == nullptr: no block
// row is ever touched.
struct glod_master_ref {
  const double* master;
  long long cap, stride;
  const int* rec_node;
  const long long* item_rec_off;
};

// Host-side count of kernel launches issued by this library (reported by
// bench.py as gpu_launches; defined in capi.cu).
void count_launch(unsigned long long n = 1);
// Sets the thread-local message returned by glod_last_error(); returns code.
int set_error(int code, const char* what);
// Keep the default stream-ordered pool's reservations (capi.cu).
void retain_pool_memory();

// ---------------------------------------------------------------------------
// Exact-rounding fp64 arithmetic.  The LoD decisions must reproduce the
// reference's numpy/OpenBLAS float paths bit for bit, so every
// product/sum on that path is spelled out with an explicit rounding
// intrinsic: nvcc can never contract or reassociate them.
// ---------------------------------------------------------------------------
GLOD_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
GLOD_DEV double add(double a, double b) { return __dadd_rn(a, b); }
GLOD_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
GLOD_DEV double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
GLOD_DEV double div(double a, double b) { return __ddiv_rn(a, b); }
GLOD_DEV double sqrt_(double a) { return __dsqrt_rn(a); }

// np.linalg.norm(v, axis=1) on an (n,3) array: add.reduce → ((x²+y²)+z²).
GLOD_DEV double norm3_plain(double x, double y, double z) {
  return sqrt_(add(add(mul(x, x), mul(y, y)), mul(z, z)));
}
// np.linalg.norm(v) on a 1-D array goes through BLAS ddot: FMA chain.
GLOD_DEV double norm3_ddot(double x, double y, double z) {
  return sqrt_(fma_(z, z, fma_(y, y, mul(x, x))));
}

// LoD metric m_d (core.py:356-361).
GLOD_DEV double min_distance(double T, int metric, double s0, double s1, double s2) {
  if (metric == 0) {
    double m = s0;
    // np.max propagates NaN; fmax would drop it.
    m = (s1 > m || s1 != s1) ? s1 : m;
    m = (s2 > m || s2 != s2) ? s2 : m;
    if (s0 != s0) m = s0;
    return div(T, m);
  }
  return div(T, sqrt_(add(add(mul(s0, s1), mul(s0, s2)), mul(s1, s2))));
}

GLOD_DEV double max3(double a, double b, double c) {
  double m = a;
  m = (b > m || b != b) ? b : m;
  m = (c > m || c != c) ? c : m;
  if (a != a) m = a;
  return m;
}

// ---------------------------------------------------------------------------
// Software grid barrier for cooperative (co-resident) launches.
// bar[0] = arrivals, bar[1] = generation.  Zeroed by the launcher.
// ---------------------------------------------------------------------------
GLOD_DEV void grid_sync(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = bar + 1;
    unsigned int gen = *vgen;
    __threadfence();
    unsigned int prev = atomicAdd(bar, 1u);
    if (prev == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Loads of data produced by other CTAs earlier in the same launch bypass L1.
template <typename T> GLOD_DEV T ld_cg(const T* p) { return __ldcg(p); }

GLOD_DEV unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one int64 per thread (blockDim ≤ 1024).
// `sm` needs blockDim/32 + 1 slots.  Returns the exclusive prefix; the block
// total is left in sm[nwarps].
GLOD_DEV long long block_excl_scan(long long v, long long* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < nw ? sm[lane] : 0;
    long long s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sm[lane] = s - w;
    if (lane == nw - 1) sm[nw] = s;
  }
  __syncthreads();
  long long r = sm[warp] + x - v;
  __syncthreads();
  return r;
}

}  // namespace glod
