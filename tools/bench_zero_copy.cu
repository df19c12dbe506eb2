// Micro-benchmark: a zero-copy range-copy kernel (pinned host -> HBM) on a
// side stream, alone and beside HBM-streaming / fp64-atomic kernels on the
// main stream: copy bandwidth vs the main kernels' slowdown.
// Build: nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bench_zero_copy tools/bench_zero_copy.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int U, typename T>
__global__ void __launch_bounds__(256) zcopy(const T* __restrict__ src, T* __restrict__ dst, long long n) {
  const long long step = (long long)gridDim.x * 256 * U;
  for (long long base = (long long)blockIdx.x * 256 * U; base < n; base += step) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = base + u * 256 + threadIdx.x;
      if (e < n) v[u] = __ldcv(src + e);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = base + u * 256 + threadIdx.x;
      if (e < n) dst[e] = v[u];
    }
  }
}

__global__ void triad(const double4* a, const double4* b, double4* c, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double4 x = a[i], y = b[i];
    c[i] = make_double4(x.x + 2 * y.x, x.y + 2 * y.y, x.z + 2 * y.z, x.w + 2 * y.w);
  }
}

__global__ void atom(double* acc, long long n, int m) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned h = unsigned(i * 2654435761u);
  for (int k = 0; k < 64; ++k) {
    h = h * 1664525u + 1013904223u;
    atomicAdd(acc + (h % unsigned(m)) * 9 + (k % 9), 1.0);
  }
}

int main() {
  const long long nf = 64ll << 20;            // 64M floats = 256 MB host
  float* h;
  CK(cudaMallocHost(&h, nf * 4));
  for (long long i = 0; i < nf; i += 1024) h[i] = 1.f;
  float* d;
  CK(cudaMalloc(&d, nf * 4));
  const long long tn = 64ll << 20;            // doubles per triad array (512 MB)
  double *a, *b, *c, *acc;
  CK(cudaMalloc(&a, tn * 8));
  CK(cudaMalloc(&b, tn * 8));
  CK(cudaMalloc(&c, tn * 8));
  const int m = 1 << 22;
  CK(cudaMalloc(&acc, (long long)m * 9 * 8));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a0, a1, b0, b1;
  for (cudaEvent_t* e : {&a0, &a1, &b0, &b1}) CK(cudaEventCreate(e));
  const long long copy_n = 18ll << 20;        // 72 MB of floats
  auto main_kernel = [&](int which) {
    if (which == 1) for (int r = 0; r < 8; ++r) triad<<<148 * 8, 256, 0, s1>>>((double4*)a, (double4*)b, (double4*)c, tn / 4);
    if (which == 2) for (int r = 0; r < 4; ++r) atom<<<(1 << 20) / 256 * 4, 256, 0, s1>>>(acc, 1 << 22, m);
  };
  for (int which = 1; which <= 2; ++which) {
    float alone;
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a0, s1));
    main_kernel(which);
    CK(cudaEventRecord(a1, s1));
    CK(cudaEventSynchronize(a1));
    CK(cudaEventElapsedTime(&alone, a0, a1));
    printf("%s alone: %.3f ms\n", which == 1 ? "triad x8" : "atomics x4", alone);
    for (int grid : {8, 16, 32, 64, 148}) {
      for (int vec : {0, 1}) {
        float ms_main, ms_copy, ms_copy_alone;
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(b0, s2));
        if (vec) zcopy<2, float4><<<grid, 256, 0, s2>>>((const float4*)h, (float4*)d, copy_n / 4);
        else zcopy<8, float><<<grid, 256, 0, s2>>>(h, d, copy_n);
        CK(cudaEventRecord(b1, s2));
        CK(cudaEventSynchronize(b1));
        CK(cudaEventElapsedTime(&ms_copy_alone, b0, b1));
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(b0, s2));
        if (vec) zcopy<2, float4><<<grid, 256, 0, s2>>>((const float4*)h, (float4*)d, copy_n / 4);
        else zcopy<8, float><<<grid, 256, 0, s2>>>(h, d, copy_n);
        CK(cudaEventRecord(b1, s2));
        CK(cudaEventRecord(a0, s1));
        main_kernel(which);
        CK(cudaEventRecord(a1, s1));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms_main, a0, a1));
        CK(cudaEventElapsedTime(&ms_copy, b0, b1));
        printf("  copy grid=%3d %s: alone %.3f ms (%.1f GB/s); concurrent copy %.3f ms, main %.3f ms (x%.2f)\n",
               grid, vec ? "float4x2" : "floatx8 ", ms_copy_alone, copy_n * 4 / 1e6 / ms_copy_alone, ms_copy,
               ms_main, ms_main / alone);
      }
    }
  }
  return 0;
}
