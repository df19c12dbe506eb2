// Micro-benchmark: copy-engine transfers of SPT prefix section ranges
// (pinned host store <-> HBM) issued as one cudaMemcpyAsync per range.
// Reports host issue time per call and the DMA completion bandwidth, with
// and without a concurrent compute kernel on another stream.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/bmr tools/bench_memcpy_ranges.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <chrono>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));        \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void busy(double* x, long long n, int iters) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  for (int k = 0; k < iters; ++k) v = v * 1.0000001 + 1e-9;
  x[i] = v;
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const long long N = 20000000;                 // slots
  const int cols[6] = {3, 3, 4, 1, 3, 9};
  float* sec[6];
  for (int k = 0; k < 6; ++k) {
    CK(cudaMallocHost(&sec[k], N * cols[k] * sizeof(float)));
    for (long long i = 0; i < N * cols[k]; i += 1024) sec[k][i] = 1.f;
  }
  float* dev;
  const size_t dev_bytes = size_t(256) << 20;
  CK(cudaMalloc(&dev, dev_bytes));
  double* work;
  const long long wn = 1 << 24;
  CK(cudaMalloc(&work, wn * sizeof(double)));
  cudaStream_t s1, s2, cst[8];
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  for (int i = 0; i < 8; ++i) CK(cudaStreamCreateWithFlags(&cst[i], cudaStreamNonBlocking));
  cudaEvent_t a, b, done[8];
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int i = 0; i < 8; ++i) CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
  std::mt19937 rng(1);
  struct Case { int items; int rows; };
  for (Case cs : {Case{100, 7500}, Case{300, 2500}, Case{600, 1200}, Case{30, 25000}}) {
    for (int dir = 0; dir < 2; ++dir) {
      for (int nst : {1, 2, 4, 8}) {
        const int concurrent = 0;
        std::vector<long long> slot(cs.items);
        for (int i = 0; i < cs.items; ++i) slot[i] = (long long)(rng() % (N - cs.rows));
        double best_issue = 1e9, best_ms = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaDeviceSynchronize());
          if (concurrent) busy<<<(wn + 255) / 256, 256, 0, s2>>>(work, wn, 4000);
          CK(cudaEventRecord(a, s1));
          const double t0 = now();
          size_t at = 0;
          for (int i = 0; i < cs.items; ++i)
            for (int k = 0; k < 6; ++k) {
              const size_t bytes = size_t(cs.rows) * cols[k] * sizeof(float);
              float* h = sec[k] + slot[i] * cols[k];
              char* d = reinterpret_cast<char*>(dev) + (at % (dev_bytes - bytes));
              cudaStream_t q = cst[(i * 6 + k) % nst];
              if (i * 6 + k < nst) CK(cudaStreamWaitEvent(q, a, 0));
              if (dir == 0) CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, q));
              else CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, q));
              at += bytes;
            }
          const double t1 = now();
          for (int q = 0; q < nst; ++q) {
            CK(cudaEventRecord(done[q], cst[q]));
            CK(cudaStreamWaitEvent(s1, done[q], 0));
          }
          CK(cudaEventRecord(b, s1));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          CK(cudaDeviceSynchronize());
          if (rep) {
            best_issue = std::min(best_issue, (t1 - t0) * 1e6 / (6.0 * cs.items));
            best_ms = std::min(best_ms, double(ms));
          }
        }
        const double mb = 92.0 * cs.items * cs.rows / 1e6;
        printf("%s items=%4d rows=%6d (%6.1f MB, %4d ranges) streams=%d: issue %.2f us/call, %.3f ms = %.1f GB/s\n",
               dir ? "D2H" : "H2D", cs.items, cs.rows, mb, 6 * cs.items, nst, best_issue, best_ms,
               mb / best_ms);
      }
    }
  }
  // one big copy for reference
  for (int dir = 0; dir < 2; ++dir) {
    const size_t bytes = size_t(200) << 20;
    CK(cudaEventRecord(a, s1));
    if (dir == 0) CK(cudaMemcpyAsync(dev, sec[5], bytes, cudaMemcpyHostToDevice, s1));
    else CK(cudaMemcpyAsync(sec[5], dev, bytes, cudaMemcpyDeviceToHost, s1));
    CK(cudaEventRecord(b, s1));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%s one 200 MiB copy: %.1f GB/s\n", dir ? "D2H" : "H2D", bytes / 1e6 / ms);
  }
  return 0;
}
