// 3DGS tile rasteriser with the reference's exact compositing semantics
// (renderer.py:75-304), fp64 per-Gaussian setup, fp32 per-pixel alpha,
// fp64 transmittance.
//
//   K5 preprocess_kernel   _projection + footprint  (renderer.py:75-114,132-148)
//   K6 depth sort + tile binning: global stable (depth, index) order
//      (renderer.py:127 lexsort) → instances emitted in rank order → stable
//      sort by tile id, so every tile list is in the global order.
//   K7 blend_fwd_kernel    compositing loop          (renderer.py:131-165)
//   K8 blend_bwd_kernel    reverse loop, 2D partials (renderer.py:219-261)
//   K9 preprocess_bwd_kernel 2D→3D chain rule        (renderer.py:262-303)
#include <stdio.h>
#include <algorithm>
#include <string>

#include "common.cuh"
#include "gather.cuh"
#include "raster.cuh"

#ifndef GLOD_PRE_MINB
#define GLOD_PRE_MINB 4     // ≤ 64 registers: more warps to hide the fp64 latency (3 → 4: fused gather + preprocess 0.327 → 0.316 ms; 2: 0.41)
#endif
#ifndef GLOD_PBWD_MINB
#define GLOD_PBWD_MINB 4
#endif
// resident CTAs per SM blend_bwd is compiled for (10: 48 registers, more
// warps, but 1.74 -> 1.79 ms; the forward likewise got slower at 8)
#ifndef GLOD_BWD_MINB
#define GLOD_BWD_MINB 8
#endif
#ifndef GLOD_DIRECT_LANES
#define GLOD_DIRECT_LANES 2
#endif

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

constexpr double kLowpass = 0.3;
constexpr double kShC1 = 0.4886025119029199;
constexpr float kAlphaMax = 0.99f;
constexpr double kTEps = 1e-4;
constexpr float kQMax = 32.0f;   // 2 * (3 + 1)^2
constexpr int kPruneMaxTiles = 64;   // splats spanning more tiles keep their full bbox

struct CamD {
  double p[3], W[9], fx, fy, cx, cy, near_;
  int w, h, tw, th;
};

CamD make_cam(const glod_camera& c) {
  CamD k;
  for (int i = 0; i < 3; ++i) k.p[i] = c.position[i];
  for (int i = 0; i < 9; ++i) k.W[i] = c.w2c[i];
  k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy; k.near_ = c.near_plane;
  k.w = c.width; k.h = c.height;
  k.tw = (c.width + kTileW - 1) / kTileW;
  k.th = (c.height + kTileH - 1) / kTileH;
  return k;
}

// Where the rasteriser reads render row i: a packed section-major block of
// n rows (glod_render_forward), or straight through the K4 gather plan
// (glod_render_forward_plan): the same source row the gather kernel would
// copy (row_source, gather.cuh), so the values are identical and the
// gathered copy is never materialised.  In plan mode the preprocess also
// writes each row's node id (the gather's row_node output).
struct AttrSrc {
  const double* attrs;
  long long n;
  glod_gather_plan plan;
  int* row_node;
};

// Everything the forward and backward passes derive from one Gaussian.
struct Proj {
  double t[3];       // camera-space position
  double m2[2];      // pixel mean
  double R[9];       // rotation (normalised quaternion)
  double qn[4];      // normalised quaternion
  double qnorm;
  double M[9];       // W Σ Wᵀ
  double J[6];       // 2x3 Jacobian
  double c00, c01, c11;   // cov2d
  double v[3];       // view direction
  double rng;        // ‖μ − p‖
  double col[3];
};

GLOD_DEV void project(const RowView& s, const CamD& c, Proj& P) {
  const double m0 = s.mean[0], m1 = s.mean[1], m2 = s.mean[2];
  const double d0 = sub(m0, c.p[0]), d1 = sub(m1, c.p[1]), d2 = sub(m2, c.p[2]);
  // t = (μ − p) @ Wᵀ through dgemm: fma(c2,w2,fma(c1,w1,c0*w0))
#pragma unroll
  for (int k = 0; k < 3; ++k)
    P.t[k] = fma_(d2, c.W[3 * k + 2], fma_(d1, c.W[3 * k + 1], mul(d0, c.W[3 * k])));
  const double tz = P.t[2];
  P.m2[0] = add(div(mul(c.fx, P.t[0]), tz), c.cx);
  P.m2[1] = add(div(mul(c.fy, P.t[1]), tz), c.cy);
  double q0 = s.rot[0], q1 = s.rot[1], q2 = s.rot[2], q3 = s.rot[3];
  P.qnorm = sqrt_(add(add(add(mul(q0, q0), mul(q1, q1)), mul(q2, q2)), mul(q3, q3)));
  const double w = q0 / P.qnorm, x = q1 / P.qnorm, y = q2 / P.qnorm, z = q3 / P.qnorm;
  P.qn[0] = w; P.qn[1] = x; P.qn[2] = y; P.qn[3] = z;
  double* R = P.R;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
  const double s0 = s.scale[0], s1 = s.scale[1], s2 = s.scale[2];
  const double ss[3] = {s0 * s0, s1 * s1, s2 * s2};
  double Sg[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      Sg[3 * a + b] = R[3 * a] * ss[0] * R[3 * b] + R[3 * a + 1] * ss[1] * R[3 * b + 1] +
                      R[3 * a + 2] * ss[2] * R[3 * b + 2];
  double WS[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      WS[3 * a + b] = c.W[3 * a] * Sg[b] + c.W[3 * a + 1] * Sg[3 + b] + c.W[3 * a + 2] * Sg[6 + b];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      P.M[3 * a + b] = WS[3 * a] * c.W[3 * b] + WS[3 * a + 1] * c.W[3 * b + 1] + WS[3 * a + 2] * c.W[3 * b + 2];
  P.J[0] = c.fx / tz; P.J[1] = 0.0; P.J[2] = -c.fx * P.t[0] / (tz * tz);
  P.J[3] = 0.0; P.J[4] = c.fy / tz; P.J[5] = -c.fy * P.t[1] / (tz * tz);
  double JM[6];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      JM[3 * a + b] = P.J[3 * a] * P.M[b] + P.J[3 * a + 1] * P.M[3 + b] + P.J[3 * a + 2] * P.M[6 + b];
  P.c00 = JM[0] * P.J[0] + JM[1] * P.J[1] + JM[2] * P.J[2] + kLowpass;
  P.c01 = JM[0] * P.J[3] + JM[1] * P.J[4] + JM[2] * P.J[5];
  P.c11 = JM[3] * P.J[3] + JM[4] * P.J[4] + JM[5] * P.J[5] + kLowpass;
  P.rng = norm3_plain(d0, d1, d2);
  const double inv = P.rng > 0 ? P.rng : 1.0;
  P.v[0] = d0 / inv; P.v[1] = d1 / inv; P.v[2] = d2 / inv;
  const double* f = s.sh;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    P.col[k] = s.base[k] + kShC1 * (-P.v[1] * f[k] + P.v[2] * f[3 + k] - P.v[0] * f[6 + k]);
}

GLOD_DEV bool finite(double x) { return isfinite(x); }

// Does any pixel of tile (tx, ty) ∩ bbox lie in the q ≤ 32 ellipse?  Exact
// minimum of the positive-definite quadratic over the continuous rectangle
// (a superset of the integer pixels), with a small margin — conservative, so
// dropping a tile never changes a pixel (its q > 32 pixels have α = 0).
// Used identically when counting and when emitting instances.
GLOD_DEV float edge_min(float a, float b, float c, float fixed, float lo, float hi) {
  // min over t∈[lo,hi] of a·f² + 2b·f·t + c·t²
  float t = fminf(fmaxf(__fdiv_rn(-__fmul_rn(b, fixed), c), lo), hi);
  return __fadd_rn(__fadd_rn(__fmul_rn(a, __fmul_rn(fixed, fixed)),
                             __fmul_rn(__fmul_rn(2.f, b), __fmul_rn(fixed, t))),
                   __fmul_rn(c, __fmul_rn(t, t)));
}

// Does any integer pixel of [xa, xb] × [ya, yb] (inclusive, already
// clipped to the bbox) lie in the q ≤ 32 ellipse?  Conservative (see above).
GLOD_DEV bool rect_hit(const Splat& g, int xa, int xb, int ya, int yb) {
  const float dxa = __fsub_rn(float(xa - g.x0), g.mx), dxb = __fsub_rn(float(xb - g.x0), g.mx);
  const float dya = __fsub_rn(float(ya - g.y0), g.my), dyb = __fsub_rn(float(yb - g.y0), g.my);
  if (dxa <= 0.f && dxb >= 0.f && dya <= 0.f && dyb >= 0.f) return true;
  float m = edge_min(g.ca, g.cb, g.cc, dxa, dya, dyb);
  m = fminf(m, edge_min(g.ca, g.cb, g.cc, dxb, dya, dyb));
  m = fminf(m, edge_min(g.cc, g.cb, g.ca, dya, dxa, dxb));
  m = fminf(m, edge_min(g.cc, g.cb, g.ca, dyb, dxa, dxb));
  return m <= 32.01f;
}

GLOD_DEV bool tile_hit(const Splat& g, int tx, int ty) {
  const int xa = max(tx * kTileW, int(g.x0)), xb = min(tx * kTileW + kTileW - 1, int(g.x1) - 1);
  const int ya = max(ty * kTileH, int(g.y0)), yb = min(ty * kTileH + kTileH - 1, int(g.y1) - 1);
  return rect_hit(g, xa, xb, ya, yb);
}

// Blend kernel layout: a 16x16 tile per block of kBlendWarps warps; warp w
// owns the 8x8 pixel block at (8(w&1), 8(w>>1)) and lane l the two pixels
// (l&7, l>>3) and (l&7, (l>>3)+4) of it.  Two pixels per lane halve the
// per-pixel share of every per-splat cost (the splat read from shared
// memory, the loop, and in the backward the warp reduction and the fp64
// atomics).  Each warp iterates only over the splats that can reach its
// block (bbox overlap and the conservative ellipse test, block_hit) —
// skipping one changes none of its pixels.
constexpr int kBlendWarps = 4;
constexpr int kBlendTB = 32 * kBlendWarps;
// backward: up to this many hitting lanes issue their own fp64 atomics
// instead of a warp reduction
constexpr int kDirectLanes = GLOD_DIRECT_LANES;
// The forward keeps one pixel per lane (8 warps, 8x4 blocks): its per-pixel
// state is a sequential fp64 chain, so it wants more warps in flight more
// than it wants the shared per-splat cost halved.
constexpr int kFwdWarps = 8;
constexpr int kFwdTB = 32 * kFwdWarps;

// One Gaussian; returns its tile count (0 = contributes nothing) and sets
// its depth key.
GLOD_DEV int preprocess_one(const RowView& s, long long i, const CamD& cam,
                            Splat* __restrict__ splats, unsigned long long* __restrict__ keys,
                            int* __restrict__ vals, int* __restrict__ tiles, int* __restrict__ bad) {
  // _check_finite (renderer.py:67-72): first section, then first row
  auto check = [&](const double* v, int cols, int k) {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < cols; ++c) ok &= finite(v[c]);
    if (!ok) atomicMin(bad + k, int(i));
  };
  check(s.mean, 3, 0); check(s.scale, 3, 1); check(s.rot, 4, 2);
  check(s.opac, 1, 3); check(s.base, 3, 4); check(s.sh, 9, 5);
  vals[i] = int(i);
  keys[i] = ~0ull;
  tiles[i] = 0;
  Proj P;
  project(s, cam, P);
  const double depth = P.t[2];
  if (!(depth > cam.near_)) return 0;            // ok = depth > near
  const double det = P.c00 * P.c11 - P.c01 * P.c01;
  if (!(det > 0)) return 0;                      // `if det <= 0: continue`
  const double half = (P.c00 + P.c11) / 2;
  const double lmax = half + sqrt(fmax(half * half - det, 0.0));
  const double rad = 3.0 * sqrt(lmax);
  // int(np.floor(.)) never overflows in Python; clamp in fp64 first
  const double big = 1e9;
  double fx0 = fmin(fmax(floor(P.m2[0] - rad), -big), big);
  double fx1 = fmin(fmax(ceil(P.m2[0] + rad) + 1, -big), big);
  double fy0 = fmin(fmax(floor(P.m2[1] - rad), -big), big);
  double fy1 = fmin(fmax(ceil(P.m2[1] + rad) + 1, -big), big);
  const int x0 = max(int(fx0), 0), x1 = min(int(fx1), cam.w);
  const int y0 = max(int(fy0), 0), y1 = min(int(fy1), cam.h);
  if (x0 >= x1 || y0 >= y1) return 0;
  Splat sp;
  sp.mx = float(P.m2[0] - x0);
  sp.my = float(P.m2[1] - y0);
  sp.ca = float(P.c11 / det);
  sp.cb = float(-P.c01 / det);
  sp.cc = float(P.c00 / det);
  sp.opac = float(s.opac[0]);
  sp.x0 = int16_t(x0); sp.y0 = int16_t(y0); sp.x1 = int16_t(x1); sp.y1 = int16_t(y1);
  sp.r = float(P.col[0]); sp.g = float(P.col[1]); sp.b = float(P.col[2]);
  sp.idx = int(i);
  const int tx0 = x0 / kTileW, tx1 = (x1 - 1) / kTileW;
  const int ty0 = y0 / kTileH, ty1 = (y1 - 1) / kTileH;
  const int nbox = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
  int nt = nbox;
  if (nbox <= kPruneMaxTiles) {                // exact ellipse test for normal splats
    nt = 0;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) nt += tile_hit(sp, tx, ty);
  }
  if (nt == 0) return 0;                       // every bbox pixel has q > 32: α = 0
  splats[i] = sp;
  keys[i] = __double_as_longlong(depth);       // positive doubles order as uint64
  tiles[i] = nt;
  return nt;
}

// K5 over all Gaussians.  Also reduces, for the one host read-back of the
// forward pass, stats = {Σ tile instances, min key, max key} over the
// contributing splats (the depth sort only needs the bits where they differ).
// Block reduction of the forward's read-back stats (Σ tile instances, min/max key).
GLOD_DEV void reduce_stats(int nt, long long i, const unsigned long long* __restrict__ keys,
                           unsigned long long* __restrict__ stats) {
  __shared__ unsigned long long red[3][8];
  unsigned long long cnt = (unsigned long long)nt;
  unsigned long long kmn = ~0ull, kmx = 0;
  if (nt) kmn = kmx = keys[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmn, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmx, o);
    kmn = a < kmn ? a : kmn;
    kmx = b > kmx ? b : kmx;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][w] = cnt;
    red[1][w] = kmn;
    red[2][w] = kmx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      cnt += red[0][k];
      kmn = red[1][k] < kmn ? red[1][k] : kmn;
      kmx = red[2][k] > kmx ? red[2][k] : kmx;
    }
    if (cnt) {
      atomicAdd(stats, cnt);
      atomicMin(stats + 1, kmn);
      atomicMax(stats + 2, kmx);
    }
  }
}

__global__ void __launch_bounds__(256, GLOD_PRE_MINB)
preprocess_kernel(const double* __restrict__ attrs, long long n, CamD cam, Splat* __restrict__ splats,
                  unsigned long long* __restrict__ keys, int* __restrict__ vals, int* __restrict__ tiles,
                  int* __restrict__ bad, unsigned long long* __restrict__ stats) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int nt = 0;
  if (i < n) nt = preprocess_one(row_view(Src{attrs, n, i}), i, cam, splats, keys, vals, tiles, bad);
  reduce_stats(nt, i, keys, stats);
}

// K4 + K5 fused (glod_render_forward_plan): a CTA resolves the sources of
// its 256 render rows (row_source, exactly the gather kernel's), reads them
// into a shared tile the way gather_rows_t_kernel does — thread t owns
// column t mod 23, so each row is fetched as contiguous runs and every
// thread has several independent loads in flight — and preprocesses row t
// from the tile.  The gathered copy never goes through HBM.
template <int kThreads>
GLOD_DEV void stage_rows(double* __restrict__ tile, const double* const* s_base, const long long* s_rows,
                         const long long* s_idx, int nr) {
  // thread t reads column c = t mod 23 of rows t/23 + k·(kThreads/23):
  // the column's section, offset and width are fixed per thread
  constexpr int kRowsPerPass = kThreads / 23;
  constexpr int kBatch = 8;
  const int c = int(threadIdx.x) % 23, rt = int(threadIdx.x) / 23;
  const bool active = threadIdx.x < kRowsPerPass * 23;
  const int off = c < 3 ? 0 : c < 6 ? 3 : c < 10 ? 6 : c < 11 ? 10 : c < 14 ? 11 : 14;
  const int cols = c < 6 ? 3 : c < 10 ? 4 : c < 11 ? 1 : c < 14 ? 3 : 9;
  for (int b = 0; b * kBatch * kRowsPerPass < nr; ++b) {
    double v[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {          // the batch's loads in flight before its tile writes
      const int lw = rt + (b * kBatch + k) * kRowsPerPass;
      if (active && lw < nr) {
        const double* base = s_base[lw];
        const long long rows = s_rows[lw], idx = s_idx[lw];
        v[k] = rows > 0 ? base[off * rows + idx * cols + (c - off)] : base[idx * (-rows) + c];
      }
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const int lw = rt + (b * kBatch + k) * kRowsPerPass;
      if (active && lw < nr) tile[lw * 23 + c] = v[k];
    }
  }
}

// A render row's resolved source (row_source), kept by the plan forward
// for the backward: 16 B per row, so the backward reaches the row's values
// in one dependent load instead of the plan's three (segment → block →
// touched bit).  The sources cannot change in between: cache decisions
// precede the forward, and ADAM (which sets touched bits) follows the
// backward.
struct __align__(16) RowSrc {
  const double* base;
  int rows;       // Src::rows (block rows, or -GLOD_NODE_RECORD)
  int idx;        // Src::idx (block position, or node id)
};

constexpr int kPlanRows = 256;
constexpr size_t kPlanSmem = sizeof(double) * kPlanRows * 23 + (sizeof(void*) + 16) * kPlanRows;

__global__ void __launch_bounds__(kPlanRows, GLOD_PRE_MINB)
preprocess_plan_kernel(const glod_gather_plan p, long long n, int* __restrict__ row_node, CamD cam,
                       Splat* __restrict__ splats, unsigned long long* __restrict__ keys,
                       int* __restrict__ vals, int* __restrict__ tiles, int* __restrict__ bad,
                       unsigned long long* __restrict__ stats, RowSrc* __restrict__ rsrc) {
  extern __shared__ __align__(16) double plan_smem[];
  double* tile = plan_smem;                                           // [kPlanRows][23]
  const double** s_base = reinterpret_cast<const double**>(tile + kPlanRows * 23);
  long long* s_rows = reinterpret_cast<long long*>(s_base + kPlanRows);
  long long* s_idx = s_rows + kPlanRows;
  const long long r0 = (long long)blockIdx.x * kPlanRows;
  const int nr = int(min((long long)kPlanRows, n - r0));
  if (threadIdx.x < nr) {
    int node;
    const Src s = row_source(p, r0 + threadIdx.x, node);
    s_base[threadIdx.x] = s.base;
    s_rows[threadIdx.x] = s.rows;
    s_idx[threadIdx.x] = s.idx;
    row_node[r0 + threadIdx.x] = node;
    rsrc[r0 + threadIdx.x] = RowSrc{s.base, int(s.rows), int(s.idx)};
  }
  __syncthreads();
  stage_rows<kPlanRows>(tile, s_base, s_rows, s_idx, nr);
  __syncthreads();
  const long long i = r0 + threadIdx.x;
  int nt = 0;
  if (i < n) nt = preprocess_one(row_view(Src{tile + threadIdx.x * 23, -23, 0}), i, cam, splats, keys, vals,
                                 tiles, bad);
  reduce_stats(nt, i, keys, stats);
}

// Top-bits depth sort fix-up: within each run of keys whose bits
// [begin_bit, end_bit) tie, the radix passes kept index order; the run's head
// thread insertion-sorts it by the full 64-bit key (stable, so equal depths
// stay in index order).  Runs are short (mostly 2).  A run longer than
// kMaxFixRun (near-equal depths spanning many splats, e.g. a fronto-parallel
// facade in a scene whose depth range is large) is left alone and flagged:
// the host then finishes the order with full-width radix passes over the
// top-sorted keys (stable, so the result is the same exact order) — never
// the O(run²) worst case.
constexpr int kDepthBits = 32;
constexpr long long kMaxFixRun = 64;

__global__ void fixup_runs_kernel(unsigned long long* __restrict__ keys, int* __restrict__ vals, long long n,
                                  int begin_bit, int end_bit, unsigned long long* __restrict__ long_run) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long m = ((end_bit - begin_bit) >= 64 ? ~0ull : ((1ull << (end_bit - begin_bit)) - 1)) << begin_bit;
  if (keys[i] == ~0ull) return;            // non-contributing splats (no instances): order irrelevant
  const unsigned long long top = keys[i] & m;
  if (i > 0 && (keys[i - 1] & m) == top) return;          // not a run head
  long long j = i + 1;
  while (j < n && j - i <= kMaxFixRun && (keys[j] & m) == top) ++j;
  if (j - i > kMaxFixRun) {
    atomicMax(long_run, 1ull);
    return;
  }
  for (long long a = i + 1; a < j; ++a) {
    const unsigned long long k = keys[a];
    const int v = vals[a];
    long long b = a - 1;
    while (b >= i && keys[b] > k) {
      keys[b + 1] = keys[b];
      vals[b + 1] = vals[b];
      --b;
    }
    keys[b + 1] = k;
    vals[b + 1] = v;
  }
}

__global__ void gather_kernel(const int* __restrict__ order, const Splat* __restrict__ splats,
                              const int* __restrict__ tiles, Splat* __restrict__ sorted,
                              int* __restrict__ tiles_sorted, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int g = order[r];
  const int c = tiles[g];
  tiles_sorted[r] = c;
  if (c) sorted[r] = splats[g];
}

__global__ void emit_kernel(const Splat* __restrict__ sorted, const int* __restrict__ tiles_sorted,
                            const long long* __restrict__ offs, int tw,
                            unsigned* __restrict__ ikey, int* __restrict__ ival, long long n) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || tiles_sorted[r] == 0) return;
  const Splat sp = sorted[r];
  const int tx0 = sp.x0 / kTileW, tx1 = (sp.x1 - 1) / kTileW;
  const int ty0 = sp.y0 / kTileH, ty1 = (sp.y1 - 1) / kTileH;
  long long o = offs[r];
  const bool prune = (tx1 - tx0 + 1) * (ty1 - ty0 + 1) <= kPruneMaxTiles;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      if (prune && !tile_hit(sp, tx, ty)) continue;
      ikey[o] = unsigned(ty * tw + tx);
      ival[o] = int(r);
      ++o;
    }
}

__global__ void ranges_kernel(const unsigned* __restrict__ ikey, long long n, int2* __restrict__ range) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned k = ikey[i];
  if (i == 0 || ikey[i - 1] != k) range[k].x = int(i);
  if (i == n - 1 || ikey[i + 1] != k) range[k].y = int(i + 1);
}

// Per-pixel alpha with an explicit rounding sequence so the forward and the
// backward kernels produce bit-identical values (no contraction variance).
// The x-dependent factors of q are per (splat, column) — `SplatRow` holds
// them so a lane's two pixels of one column share them.
//   q = a dx² + c dy² + 2 b dy dx   (renderer.py:151-152)
//     = fma(a·dx, dx, fma(c·dy, dy, ((2b)·dx)·dy))
struct SplatCol {
  float dx, adx, bdx;   // dx, a·dx, (2b)·dx
};
GLOD_DEV SplatCol splat_col(const Splat& g, int xi) {
  SplatCol c;
  c.dx = __fsub_rn(float(xi), g.mx);
  c.adx = __fmul_rn(g.ca, c.dx);
  c.bdx = __fmul_rn(__fmul_rn(2.0f, g.cb), c.dx);
  return c;
}
// α of the pixel at bbox-relative row yi (the caller tested the bbox).
// `a` is the unclamped opac·G (its < 0.99 test selects the live branch).
GLOD_DEV bool col_alpha(const Splat& g, const SplatCol& c, int yi, float& dy, float& gauss, float& a,
                        float& alpha) {
  dy = __fsub_rn(float(yi), g.my);
  const float q = __fmaf_rn(c.adx, c.dx, __fmaf_rn(__fmul_rn(g.cc, dy), dy, __fmul_rn(c.bdx, dy)));
  if (!(q <= kQMax)) return false;
  // exp(-q/2) = 2^(q · (-log2(e)/2)): one multiply + MUFU.EX2
  // (q ≤ 32: the argument is ≥ -23.1, far from the denormal range)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gauss) : "f"(__fmul_rn(q, -0.72134752044448170368f)));
  a = __fmul_rn(g.opac, gauss);
  alpha = fminf(a, kAlphaMax);
  return alpha > 0.0f;
}

// Front-to-back compositing of one pixel with one splat (renderer.py:149-164).
// The α part is branch-free (every lane evaluates it; the warp runs the
// union of its lanes' paths anyway), the fp64 blend only where α > 0.
GLOD_DEV void fwd_pixel(const Splat& g, int px, int py, int inst, double& T, float& cr, float& cg, float& cb,
                        int& last, bool& done) {
  const int xi = px - g.x0, yi = py - g.y0;
  const bool act = !done && unsigned(xi) < unsigned(g.x1 - g.x0) && unsigned(yi) < unsigned(g.y1 - g.y0);
  const SplatCol c = splat_col(g, xi);
  const float dy = __fsub_rn(float(yi), g.my);
  const float q = __fmaf_rn(c.adx, c.dx, __fmaf_rn(__fmul_rn(g.cc, dy), dy, __fmul_rn(c.bdx, dy)));
  float gs;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gs) : "f"(__fmul_rn(q, -0.72134752044448170368f)));
  const float al = fminf(__fmul_rn(g.opac, gs), kAlphaMax);
  if (!(act && q <= kQMax && al > 0.0f)) return;
  const double w = double(al) * T;
  cr += float(w) * g.r;
  cg += float(w) * g.g;
  cb += float(w) * g.b;
  T = T * (1.0 - double(al));
  last = inst;
  if (T <= kTEps) done = true;           // later alphas are gated to 0
}

// Can splat g reach a pixel of the W x H block at (xa, ya)?  Bbox overlap
// and the conservative ellipse test (rect_hit): skipping a splat that fails
// it changes none of the block's pixels.
template <int W, int H>
GLOD_DEV bool block_hit(const Splat& g, int xa, int ya) {
  if (g.x1 <= xa || g.x0 >= xa + W || g.y1 <= ya || g.y0 >= ya + H) return false;
  return rect_hit(g, max(xa, int(g.x0)), min(xa + W - 1, int(g.x1) - 1), max(ya, int(g.y0)),
                  min(ya + H - 1, int(g.y1) - 1));
}

// Warp-streamed blending: every warp walks its tile's instance list on its
// own, 32 splats per step (one coalesced 48-B record per lane, staged in a
// warp-private shared slice), keeps the ones that can reach its pixel block
// (ballot) and composites them in order.  No block barriers: a warp never
// waits for a slower warp of the same tile, and a warp whose pixels are all
// saturated leaves at once.  The other warps of the tile read the same
// records, so the repeats are L1 hits.
GLOD_DEV void load_splat(const Splat* __restrict__ sorted, int si, float4 (&dst)[3], Splat& g) {
  const float4* src = reinterpret_cast<const float4*>(sorted) + 3LL * si;
  float4* gv = reinterpret_cast<float4*>(&g);
  gv[0] = __ldg(src);
  gv[1] = __ldg(src + 1);
  gv[2] = __ldg(src + 2);
  dst[0] = gv[0];
  dst[1] = gv[1];
  dst[2] = gv[2];
}

GLOD_DEV void read_splat(const float4 (&src)[3], Splat& g) {
  float4* gv = reinterpret_cast<float4*>(&g);
  gv[0] = src[0];
  gv[1] = src[1];
  gv[2] = src[2];
}

__global__ void __launch_bounds__(kFwdTB)
blend_fwd_kernel(const Splat* __restrict__ sorted, const int* __restrict__ ival,
                 const int2* __restrict__ range, CamD cam, float* __restrict__ image,
                 double* __restrict__ t_final, int* __restrict__ last_out) {
  __shared__ float4 sm[kFwdWarps][32][3];
  const int tile = blockIdx.x;
  const int tx = tile % cam.tw, ty = tile / cam.tw;
  // warp w owns the 8x4 pixel block at (8(w&1), 4(w>>1))
  const int wid = int(threadIdx.x >> 5), ln = int(threadIdx.x & 31);
  const int bx = tx * kTileW + (wid & 1) * 8, by = ty * kTileH + (wid >> 1) * 4;
  const int px = bx + (ln & 7), py = by + (ln >> 3);
  const bool inside = px < cam.w && py < cam.h;
  const int2 rg = range[tile];
  double T = 1.0;
  float cr = 0.f, cg = 0.f, cb = 0.f;
  int last = -1;
  bool done = !inside;
  for (int base = rg.x; base < rg.y; base += 32) {
    if (__all_sync(0xffffffffu, done)) break;
    const int k = base + ln;
    bool mine = false;
    if (k < rg.y) {
      Splat g;
      load_splat(sorted, ival[k], sm[wid][ln], g);
      mine = block_hit<8, 4>(g, bx, by);
    }
    __syncwarp();
    unsigned bits = __ballot_sync(0xffffffffu, mine);
    while (bits) {
      const int j = __ffs(bits) - 1;
      bits &= bits - 1;
      Splat g;
      read_splat(sm[wid][j], g);
      fwd_pixel(g, px, py, base + j, T, cr, cg, cb, last, done);
    }
    __syncwarp();
  }
  if (inside) {
    const long long pix = (long long)py * cam.w + px;
    image[3 * pix] = cr;
    image[3 * pix + 1] = cg;
    image[3 * pix + 2] = cb;
    t_final[pix] = T;
    last_out[pix] = last;
  }
}

// Transposed warp reduction of 8 values (9 shuffles instead of 8x5): after
// it, lane l holds the warp total of value ((l >> 2) & 7).
GLOD_DEV float warp_reduce8(const float (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b4 ? v[i] : v[i + 4];
    const float keep = b4 ? v[i + 4] : v[i];
    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float x[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b3 ? w[i] : w[i + 2];
    const float keep = b3 ? w[i + 2] : w[i];
    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float y = (b2 ? x[1] : x[0]) + __shfl_xor_sync(0xffffffffu, b2 ? x[0] : x[1], 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  return y;
}

GLOD_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Back-to-front per pixel with the reference's rear accumulator
// (renderer.py:219-261).  Per-pixel math is fp32 (T recovered as
// T_front = T_after / (1 − α) from the fp64 final transmittance); a lane's
// two pixels add into one set of nine partials.
struct BwdPix {
  float T, gr, gg, gb, rr, rg, rb;
  int last;
  bool inside;
};

// One pixel of a lane's column, branch-free: `active` carries the bbox and
// last-contributor tests; a pixel that does not composite this splat (not
// active, q > 32 or α = 0) runs the same instructions with α = 0, which
// leaves its state unchanged and adds exact zeros (no divergent paths and
// no re-zeroed accumulators per exit).  The dl/dq terms use the shared
// column factors (2a·dx, 2b·dx).
GLOD_DEV bool bwd_pixel(const Splat& g, const SplatCol& c, int yi, bool active, BwdPix& s, float (&cv)[9],
                        float a2dx, float b2dx, float nhop) {
  const float dy = __fsub_rn(float(yi), g.my);
  const float q = __fmaf_rn(c.adx, c.dx, __fmaf_rn(__fmul_rn(g.cc, dy), dy, __fmul_rn(c.bdx, dy)));
  float gs;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(gs) : "f"(__fmul_rn(q, -0.72134752044448170368f)));
  const float a = __fmul_rn(g.opac, gs);
  const float alr = fminf(a, kAlphaMax);
  const bool ok = active && q <= kQMax && alr > 0.0f;
  const float al = ok ? alr : 0.0f;
  float inv;                                           // 1/(1-α), 1-α ≥ 0.01: approx rcp
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(1.f - al));
  const float Tf = ok ? s.T * inv : s.T;               // T before this splat
  const float w = al * Tf;
  cv[0] += w * s.gr; cv[1] += w * s.gg; cv[2] += w * s.gb;   // dl_dcolor
  const float gc = s.gr * g.r + s.gg * g.g + s.gb * g.b;
  const float grear = s.gr * s.rr + s.gg * s.rg + s.gb * s.rb;
  const float dla = gc * Tf - grear * inv;
  s.rr += w * g.r; s.rg += w * g.g; s.rb += w * g.b;
  s.T = Tf;
  const float gd = (ok && a < kAlphaMax) ? gs * dla : 0.0f;   // live: unclamped
  cv[3] += gd;
  const float dq = nhop * gd;                          // -0.5·opac·G·dl/dα
  cv[4] += -dq * (a2dx + 2.f * g.cb * dy);
  cv[5] += -dq * (b2dx + 2.f * g.cc * dy);
  const float dqdx = dq * c.dx;
  cv[6] += dqdx * c.dx;
  cv[7] += dqdx * dy;
  cv[8] += dq * dy * dy;
  return ok;
}

GLOD_DEV BwdPix bwd_init(const CamD& cam, int px, int py, const float* __restrict__ dimg,
                         const double* __restrict__ t_final, const int* __restrict__ last_in) {
  BwdPix s{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, -1, px < cam.w && py < cam.h};
  if (s.inside) {
    const long long pix = (long long)py * cam.w + px;
    s.T = float(t_final[pix]);
    s.last = last_in[pix];
    s.gr = dimg[3 * pix]; s.gg = dimg[3 * pix + 1]; s.gb = dimg[3 * pix + 2];
  }
  return s;
}

// Warp-streamed like the forward: each warp walks its tile's list back to
// front from its own last contributor, 32 splats per step.  For each
// (splat, warp) with at least one hit the nine per-Gaussian partials are
// warp-reduced (transposed reduction) and nine lanes issue one fp64
// reduction each (or, with one or two hitting lanes, those lanes issue
// theirs directly).
__global__ void __launch_bounds__(kBlendTB, GLOD_BWD_MINB)
blend_bwd_kernel(const Splat* __restrict__ sorted, const int* __restrict__ ival,
                 const int2* __restrict__ range, CamD cam, const float* __restrict__ dimg,
                 const double* __restrict__ t_final, const int* __restrict__ last_in,
                 double* __restrict__ g2) {
  __shared__ float4 sm[kBlendWarps][32][3];
  const int tile = blockIdx.x;
  const int tx = tile % cam.tw, ty = tile / cam.tw;
  const int wid = int(threadIdx.x >> 5), ln = int(threadIdx.x & 31);
  const int bx = tx * kTileW + (wid & 1) * 8, by = ty * kTileH + (wid >> 1) * 8;
  const int px = bx + (ln & 7);
  const int py0 = by + (ln >> 3), py1 = py0 + 4;
  const int2 rg = range[tile];
  BwdPix s0 = bwd_init(cam, px, py0, dimg, t_final, last_in);
  BwdPix s1 = bwd_init(cam, px, py1, dimg, t_final, last_in);
  int wlast = max(s0.last, s1.last);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, o));
  // nothing beyond this warp's last contributor matters
  for (int top = min(wlast + 1, rg.y); top > rg.x; top -= 32) {
    const int lo = max(rg.x, top - 32);
    const int k = top - 1 - ln;                  // slot ln holds instance top-1-ln
    bool mine = false;
    if (k >= lo) {
      Splat g;
      load_splat(sorted, ival[k], sm[wid][ln], g);
      mine = block_hit<8, 8>(g, bx, by);
    }
    __syncwarp();
    unsigned bits = __ballot_sync(0xffffffffu, mine);
    while (bits) {
      const int j = __ffs(bits) - 1;             // ascending slot = back to front
      bits &= bits - 1;
      const int inst = top - 1 - j;
      Splat g;
      read_splat(sm[wid][j], g);
      float cv[9];
#pragma unroll
      for (int u = 0; u < 9; ++u) cv[u] = 0.f;
      // bbox tests once per lane (both pixels share the column)
      const int xi = px - g.x0, yi0 = py0 - g.y0;
      const unsigned bh = unsigned(g.y1 - g.y0);
      const bool inx = unsigned(xi) < unsigned(g.x1 - g.x0);
      const bool p0 = inx && unsigned(yi0) < bh && inst <= s0.last;
      const bool p1 = inx && unsigned(yi0 + 4) < bh && inst <= s1.last;
      const SplatCol c = splat_col(g, xi);
      const float a2dx = 2.f * g.ca * c.dx, b2dx = 2.f * g.cb * c.dx, nhop = -0.5f * g.opac;
      const bool h0 = bwd_pixel(g, c, yi0, p0, s0, cv, a2dx, b2dx, nhop);
      const bool h1 = bwd_pixel(g, c, yi0 + 4, p1, s1, cv, a2dx, b2dx, nhop);
      const bool hit = h0 || h1;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (bal == 0) continue;
      double* dst = g2 + (long long)kG2 * g.idx;
      if (__popc(bal) <= kDirectLanes) {
        // a few hitting lanes: their partials go straight to the
        // fp64 accumulators (cheaper than a 32-lane reduction)
        if (hit) {
#pragma unroll
          for (int u = 0; u < 9; ++u)
            if (cv[u] != 0.f) atomicAdd(dst + u, double(cv[u]));
        }
        continue;
      }
      const float t8 = warp_reduce8(*reinterpret_cast<const float(*)[8]>(cv), ln);
      const float s8 = warp_sum(cv[8]);
      if ((ln & 3) == 0) {
        if (t8 != 0.f) atomicAdd(dst + (ln >> 2), double(t8));
      } else if (ln == 1) {
        if (s8 != 0.f) atomicAdd(dst + 8, double(s8));
      }
    }
    __syncwarp();
  }
}

// K9: 2D partials → gradients of the raw attributes (renderer.py:262-303).
// A row that contributed no tile instance has zero gradients.
GLOD_DEV void bwd_zero(long long i, long long n, double* __restrict__ grads) {
  for (int k = 0; k < 3; ++k) { grads[3 * i + k] = 0; grads[3 * n + 3 * i + k] = 0; grads[11 * n + 3 * i + k] = 0; }
  for (int k = 0; k < 4; ++k) grads[6 * n + 4 * i + k] = 0;
  for (int k = 0; k < 9; ++k) grads[14 * n + 9 * i + k] = 0;
  grads[10 * n + i] = 0;
}

GLOD_DEV void bwd_one(const RowView& s, long long i, long long n, const CamD& cam, const double* __restrict__ a2,
                      double* __restrict__ grads) {
  double* gm = grads;                 // means [3n]
  double* gsc = grads + 3 * n;        // scales
  double* grot = grads + 6 * n;       // rotations
  double* gop = grads + 10 * n;       // opacities
  double* gbase = grads + 11 * n;     // base colours
  double* gsh = grads + 14 * n;       // sh_rest
  Proj P;
  project(s, cam, P);
  // gradients only (the forward's projection and bbox decisions are
  // untouched): reciprocals once, products after — 4 fp64 divisions per
  // row instead of 16, each a long dependent DFMA chain
  const double det = P.c00 * P.c11 - P.c01 * P.c01;
  const double idet = 1.0 / det;
  const double ca = P.c11 * idet, cb = -P.c01 * idet, cc = P.c00 * idet;
  const double dcol[3] = {a2[0], a2[1], a2[2]};
  gop[i] = a2[3];
  const double dmx = a2[4], dmy = a2[5];
  const double daa = a2[6], dbb = a2[7], dcc = a2[8];
  // dl_dcov2d = -C dC C with C = [[a,b],[b,c]], dC = [[daa,dbb],[dbb,dcc]]
  const double t00 = ca * daa + cb * dbb, t01 = ca * dbb + cb * dcc;
  const double t10 = cb * daa + cc * dbb, t11 = cb * dbb + cc * dcc;
  const double D00 = -(t00 * ca + t01 * cb), D01 = -(t00 * cb + t01 * cc);
  const double D10 = -(t10 * ca + t11 * cb), D11 = -(t10 * cb + t11 * cc);
  const double Dc[4] = {D00, D01, D10, D11};
  // dl_dm = Jᵀ Dc J (3x3); dl_dsigma = Wᵀ dl_dm W
  double DJ[6];   // Dc @ J (2x3)
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) DJ[3 * a + b] = Dc[2 * a] * P.J[b] + Dc[2 * a + 1] * P.J[3 + b];
  double dM[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dM[3 * a + b] = P.J[a] * DJ[b] + P.J[3 + a] * DJ[3 + b];
  const double* W = cam.W;
  double tmp[9], dS[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) tmp[3 * a + b] = dM[3 * a] * W[b] + dM[3 * a + 1] * W[3 + b] + dM[3 * a + 2] * W[6 + b];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) dS[3 * a + b] = W[a] * tmp[b] + W[3 + a] * tmp[3 + b] + W[6 + a] * tmp[6 + b];
  // dl_dj = (Dc + Dcᵀ) J M  (2x3)
  const double S00 = 2 * D00, S01 = D01 + D10, S11 = 2 * D11;
  double JM[6];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      JM[3 * a + b] = P.J[3 * a] * P.M[b] + P.J[3 * a + 1] * P.M[3 + b] + P.J[3 * a + 2] * P.M[6 + b];
  double dJ[6];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    dJ[b] = S00 * JM[b] + S01 * JM[3 + b];
    dJ[3 + b] = S01 * JM[b] + S11 * JM[3 + b];
  }
  const double tx = P.t[0], ty = P.t[1], tz = P.t[2];
  const double fx = cam.fx, fy = cam.fy;
  const double itz = 1.0 / tz, itz2 = itz * itz, itz3 = itz2 * itz;
  double dt[3];
  dt[0] = dmx * fx * itz + dJ[2] * (-fx * itz2);
  dt[1] = dmy * fy * itz + dJ[5] * (-fy * itz2);
  dt[2] = dmx * (-fx * tx * itz2) + dmy * (-fy * ty * itz2) + dJ[0] * (-fx * itz2) +
          dJ[4] * (-fy * itz2) + dJ[2] * (2 * fx * tx * itz3) +
          dJ[5] * (2 * fy * ty * itz3);
  double dmean[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dmean[k] = W[k] * dt[0] + W[3 + k] * dt[1] + W[6 + k] * dt[2];
  // colour path (renderer.py:281-291)
  const double* f = s.sh;
  const double* v = P.v;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gbase[3 * i + k] = dcol[k];
    gsh[9 * i + k] = -kShC1 * v[1] * dcol[k];
    gsh[9 * i + 3 + k] = kShC1 * v[2] * dcol[k];
    gsh[9 * i + 6 + k] = -kShC1 * v[0] * dcol[k];
  }
  const double dv0 = kShC1 * -(f[6] * dcol[0] + f[7] * dcol[1] + f[8] * dcol[2]);
  const double dv1 = kShC1 * -(f[0] * dcol[0] + f[1] * dcol[1] + f[2] * dcol[2]);
  const double dv2 = kShC1 * (f[3] * dcol[0] + f[4] * dcol[1] + f[5] * dcol[2]);
  const double vd = v[0] * dv0 + v[1] * dv1 + v[2] * dv2;
  const double irng = 1.0 / P.rng;
  dmean[0] += (dv0 - v[0] * vd) * irng;
  dmean[1] += (dv1 - v[1] * vd) * irng;
  dmean[2] += (dv2 - v[2] * vd) * irng;
#pragma unroll
  for (int k = 0; k < 3; ++k) gm[3 * i + k] = dmean[k];
  // covariance → scale and normalised quaternion
  double sym[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) sym[3 * a + b] = 0.5 * (dS[3 * a + b] + dS[3 * b + a]);
  const double* R = P.R;
  const double sc[3] = {s.scale[0], s.scale[1], s.scale[2]};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double acc = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) acc += R[3 * a + k] * sym[3 * a + b] * R[3 * b + k];
    gsc[3 * i + k] = 2 * sc[k] * acc;
  }
  // dl_dr = 2 sym R diag(s²)
  double dR[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      dR[3 * a + b] = 2 * (sym[3 * a] * R[b] + sym[3 * a + 1] * R[3 + b] + sym[3 * a + 2] * R[6 + b]) *
                      (sc[b] * sc[b]);
  const double w = P.qn[0], x = P.qn[1], y = P.qn[2], z = P.qn[3];
  // dR/dq for each quaternion component (renderer.py:177-194)
  const double Dw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
  const double Dx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
  const double Dy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
  const double Dz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
  double dq[4] = {0, 0, 0, 0};
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    dq[0] += dR[e] * 2 * Dw[e];
    dq[1] += dR[e] * 2 * Dx[e];
    dq[2] += dR[e] * 2 * Dy[e];
    dq[3] += dR[e] * 2 * Dz[e];
  }
  const double qd = w * dq[0] + x * dq[1] + y * dq[2] + z * dq[3];
  const double iqn = 1.0 / P.qnorm;
  for (int k = 0; k < 4; ++k) grot[4 * i + k] = (dq[k] - P.qn[k] * qd) * iqn;
}

__global__ void __launch_bounds__(128, GLOD_PBWD_MINB)
preprocess_bwd_kernel(const double* __restrict__ attrs, long long n, CamD cam, const int* __restrict__ tiles_of,
                      const double* __restrict__ g2, double* __restrict__ grads) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (tiles_of[i] == 0) return bwd_zero(i, n, grads);
  bwd_one(row_view(Src{attrs, n, i}), i, n, cam, g2 + (long long)kG2 * i, grads);
}

// K9 after a plan forward: each contributing render row is read in place
// through the source the forward resolved for it (RowSrc), not staged: only
// part of the rows contributed, and a staged tile costs more in barriers
// and idle lanes than the indirection does.
__global__ void __launch_bounds__(128, GLOD_PBWD_MINB)
preprocess_bwd_src_kernel(const RowSrc* __restrict__ rsrc, long long n, CamD cam, const int* __restrict__ tiles_of,
                          const double* __restrict__ g2, double* __restrict__ grads) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (tiles_of[i] == 0) return bwd_zero(i, n, grads);
  const RowSrc r = rsrc[i];
  bwd_one(row_view(Src{r.base, r.rows, r.idx}), i, n, cam, g2 + (long long)kG2 * i, grads);
}

}  // namespace

// ---------------------------------------------------------------------------
// Workspace: device buffers grown stream-ordered (cudaMallocAsync).
// ---------------------------------------------------------------------------
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes, cudaStream_t st) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFreeAsync(p, st);
    // geometric growth: a view with a larger render set than any before
    // costs one re-allocation, not one per few-% increase
    size_t want = std::max(bytes + bytes / 4, 2 * cap) + 4096;
    cudaError_t e = cudaMallocAsync(&p, want, st);
    cap = e == cudaSuccess ? want : 0;
    return e;
  }
  void release(cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    cap = 0;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

constexpr int kTimed = 3;   // timed kernels: blend_fwd, blend_bwd, preprocess

struct RasterCtx {
  Buf splats, sorted, keys, keys2, vals, vals2, tiles, tiles_sorted, offs;
  Buf ikey, ikey2, ival, ival2, range, tfinal, last, g2, temp, bad, host_pin, rsrc;
  bool long_runs = false;       // last forward finished its depth order with full-width passes
  cudaEvent_t ev_runs = nullptr;  // the long-run flag's read-back landed
  CamD cam{};
  AttrSrc src{};
  bool plan_src = false;
  long long n = 0, n_inst = 0, n_visible = 0;
  int bad_section = -1, bad_index = -1;
  cudaStream_t stream = nullptr;
  bool have_forward = false;
  bool defer_blend = false, blend_pending = false;   // raster_set_defer_blend / raster_blend
  float* blend_image = nullptr;
  const unsigned* ikey_sorted = nullptr;
  const int* ival_sorted = nullptr;
  // optional CUDA-event timing of the two blend kernels and the preprocess
  // (bench.py roofline)
  bool timing = false;
  cudaEvent_t ev[2 * kTimed] = {};
  double blend_ms[kTimed] = {};
  long long blend_n[kTimed] = {};
  bool pending[kTimed] = {};
};

static void timing_begin(RasterCtx* R, int k, cudaStream_t st) {
  if (!R->timing) return;
  if (!R->ev[0])
    for (int i = 0; i < 2 * kTimed; ++i) cudaEventCreate(&R->ev[i]);
  cudaEventRecord(R->ev[2 * k], st);
}

static void timing_end(RasterCtx* R, int k, cudaStream_t st) {
  if (!R->timing) return;
  cudaEventRecord(R->ev[2 * k + 1], st);
  R->pending[k] = true;
}

// Accumulate the finished launches' durations (synchronises on the events).
void raster_timing_collect(RasterCtx* R, int enable, double* ms_out, long long* n, int nk) {
  for (int k = 0; k < kTimed; ++k)
    if (R->pending[k]) {
      float ms = 0.f;
      cudaEventSynchronize(R->ev[2 * k + 1]);
      if (cudaEventElapsedTime(&ms, R->ev[2 * k], R->ev[2 * k + 1]) == cudaSuccess) {
        R->blend_ms[k] += ms;
        R->blend_n[k] += 1;
      }
      R->pending[k] = false;
    }
  for (int k = 0; k < nk && k < kTimed; ++k) {
    if (ms_out) ms_out[k] = R->blend_ms[k];
    if (n) n[k] = R->blend_n[k];
  }
  if (enable >= 0) {
    R->timing = enable != 0;
    for (int k = 0; k < kTimed; ++k) {
      R->blend_ms[k] = 0.0;
      R->blend_n[k] = 0;
    }
  }
}

static int bits_for(long long v) {
  int b = 1;
  while ((1ll << b) < v) ++b;
  return b;
}

#define CK(x)                                   \
  do {                                          \
    cudaError_t _e = (x);                       \
    if (_e != cudaSuccess) return _e;           \
  } while (0)

// K7 of the last forward (its ranges, sorted splats and instance list).
static cudaError_t blend_forward(RasterCtx* R, float* image, cudaStream_t st) {
  const CamD& cam = R->cam;
  count_launch();
  timing_begin(R, 0, st);
  blend_fwd_kernel<<<cam.tw * cam.th, kFwdTB, 0, st>>>(R->n_inst > 0 ? R->sorted.as<Splat>() : nullptr,
                                                      R->n_inst > 0 ? R->ival_sorted : nullptr,
                                                      R->range.as<int2>(), cam, image, R->tfinal.as<double>(),
                                                      R->last.as<int>());
  timing_end(R, 0, st);
  return cudaGetLastError();
}

// With blend deferral on (raster_set_defer_blend), the forward stops before
// K7 and raster_blend enqueues it: a caller can put other work (the next
// frame's LoD select) between the tile sort and the blend.
static cudaError_t blend_or_defer(RasterCtx* R, float* image, cudaStream_t st) {
  if (R->defer_blend) {
    R->blend_image = image;
    R->blend_pending = true;
    return cudaSuccess;
  }
  R->blend_pending = false;
  return blend_forward(R, image, st);
}

void raster_set_defer_blend(RasterCtx* R, bool on) { R->defer_blend = on; }

cudaError_t raster_blend(RasterCtx* R, cudaStream_t st) {
  if (!R->blend_pending) return cudaErrorInvalidValue;
  R->blend_pending = false;
  return blend_forward(R, R->blend_image, st);
}

static cudaError_t raster_forward_src(RasterCtx* R, const AttrSrc& src, bool plan, const glod_camera& c,
                               float* image, cudaStream_t st) {
  const long long n = src.n;
  R->cam = make_cam(c);
  R->src = src;
  R->plan_src = plan;
  R->n = n;
  R->stream = st;
  R->have_forward = true;
  R->bad_section = -1;
  const CamD& cam = R->cam;
  const long long npix = (long long)cam.w * cam.h;
  const int ntiles = cam.tw * cam.th;
  CK(R->tfinal.ensure(8 * npix, st));
  CK(R->last.ensure(4 * npix, st));
  CK(R->range.ensure(8 * (size_t)ntiles, st));
  CK(cudaMemsetAsync(R->range.p, 0, 8 * (size_t)ntiles, st));
  if (n == 0) {
    CK(cudaMemsetAsync(image, 0, 12 * npix, st));
    CK(cudaMemsetAsync(R->tfinal.p, 0, 8 * npix, st));
    R->n_inst = 0;
    R->n_visible = 0;
    // T=1 everywhere, no contributors: the blend kernel writes exactly that
    return blend_or_defer(R, image, st);
  }
  CK(R->splats.ensure(sizeof(Splat) * n, st));
  CK(R->sorted.ensure(sizeof(Splat) * n, st));
  CK(R->keys.ensure(8 * n, st));
  CK(R->keys2.ensure(8 * n, st));
  CK(R->vals.ensure(4 * n, st));
  CK(R->vals2.ensure(4 * n, st));
  CK(R->tiles.ensure(4 * n, st));
  CK(R->tiles_sorted.ensure(4 * n + 4, st));
  CK(R->offs.ensure(8 * (n + 1), st));
  CK(R->bad.ensure(64, st));
  CK(R->host_pin.p ? cudaSuccess : cudaMallocHost(&R->host_pin.p, 256));
  R->host_pin.cap = 256;
  // bad[0..7]: first non-finite row per section; then u64 stats {Σ tile
  // instances, min key, max key} — one 56-B read-back, the forward's only
  // host synchronisation.
  unsigned char init[64];
  int* ib = reinterpret_cast<int*>(init);
  for (int k = 0; k < 8; ++k) ib[k] = 0x7fffffff;
  unsigned long long* is = reinterpret_cast<unsigned long long*>(init + 32);
  is[0] = 0; is[1] = ~0ull; is[2] = 0; is[3] = 0;
  CK(launch_set_bytes(R->bad.p, init, sizeof(init), st));
  unsigned long long* stats = reinterpret_cast<unsigned long long*>(static_cast<char*>(R->bad.p) + 32);
  const int TB = 256;
  const int nb = int((n + TB - 1) / TB);
  count_launch();
  timing_begin(R, 2, st);
  if (plan) CK(R->rsrc.ensure(sizeof(RowSrc) * n, st));
  if (plan) {
    static bool smem_set = false;
    if (!smem_set) {
      CK(cudaFuncSetAttribute(preprocess_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPlanSmem)));
      smem_set = true;
    }
    preprocess_plan_kernel<<<int((n + kPlanRows - 1) / kPlanRows), kPlanRows, kPlanSmem, st>>>(
        src.plan, n, src.row_node, cam, R->splats.as<Splat>(), R->keys.as<unsigned long long>(), R->vals.as<int>(),
        R->tiles.as<int>(), R->bad.as<int>(), stats, R->rsrc.as<RowSrc>());
  } else {
    preprocess_kernel<<<nb, TB, 0, st>>>(src.attrs, n, cam, R->splats.as<Splat>(), R->keys.as<unsigned long long>(),
                                         R->vals.as<int>(), R->tiles.as<int>(), R->bad.as<int>(), stats);
  }
  timing_end(R, 2, st);
  CK(cudaGetLastError());
  unsigned char* hp = static_cast<unsigned char*>(R->host_pin.p);
  CK(launch_readback(hp, R->bad.p, 64, st));
  CK(cudaStreamSynchronize(st));
  const int* badh = reinterpret_cast<const int*>(hp);
  for (int k = 0; k < 6; ++k)
    if (badh[k] != 0x7fffffff) {
      R->bad_section = k;
      R->bad_index = badh[k];
      return cudaErrorInvalidValue;
    }
  const unsigned long long* hs = reinterpret_cast<const unsigned long long*>(hp + 32);
  const long long n_inst = (long long)hs[0];
  R->n_inst = n_inst;
  if (n_inst > 0x7fffffffll) return cudaErrorMemoryAllocation;
  // global stable sort on fp64 depth bits (ties keep index order), K6, over
  // the bits where the contributing keys differ (non-contributing splats
  // emit no instances, so their relative order is irrelevant)
  int end_bit = 0;
  if (n_inst > 0 && hs[1] != hs[2]) end_bit = 64 - __builtin_clzll(hs[1] ^ hs[2]);
  CK(R->temp.ensure(std::max(radix_scratch_bytes(n), scan_scratch_bytes(n + 1)), st));
  // Radix passes only over the top kDepthBits of that range (4 passes instead
  // of ~7); keys whose top bits tie (depths within ~2^-kDepthBits of the
  // range — a few thousand pairs per view) are put in full (depth, index)
  // order by the run fix-up, so the result is the exact lexsort order.
  const int begin_bit = end_bit > kDepthBits ? end_bit - kDepthBits : 0;
  int alt = 0;
  if (end_bit > 0)
    CK(radix_sort_pairs<unsigned long long>(R->keys.as<unsigned long long>(), R->keys2.as<unsigned long long>(),
                                            R->vals.as<int>(), R->vals2.as<int>(), n, begin_bit, end_bit, R->temp.p,
                                            R->temp.cap, false, &alt, st));
  const int* order = alt ? R->vals2.as<int>() : R->vals.as<int>();
  R->long_runs = false;
  // the rest of the forward from a depth order: instances, tile sort, blend
  auto tail = [&](const int* ord) -> cudaError_t {
    count_launch();
    gather_kernel<<<nb, TB, 0, st>>>(ord, R->splats.as<Splat>(), R->tiles.as<int>(), R->sorted.as<Splat>(),
                                     R->tiles_sorted.as<int>(), n);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(R->tiles_sorted.as<int>() + n, 0, 4, st));
    CK(exclusive_scan_i32(R->tiles_sorted.as<int>(), R->offs.as<long long>(), n + 1, R->temp.p, R->temp.cap, st));
    CK(R->ikey.ensure(4 * n_inst + 4, st));
    CK(R->ikey2.ensure(4 * n_inst + 4, st));
    CK(R->ival.ensure(4 * n_inst + 4, st));
    CK(R->ival2.ensure(4 * n_inst + 4, st));
    count_launch();
    emit_kernel<<<nb, TB, 0, st>>>(R->sorted.as<Splat>(), R->tiles_sorted.as<int>(), R->offs.as<long long>(),
                                   cam.tw, R->ikey.as<unsigned>(), R->ival.as<int>(), n);
    CK(cudaGetLastError());
    if (n_inst > 0) {
      const int kb = bits_for(ntiles);
      CK(R->temp.ensure(radix_scratch_bytes(n_inst), st));
      int alt2 = 0;
      CK(radix_sort_pairs<unsigned>(R->ikey.as<unsigned>(), R->ikey2.as<unsigned>(), R->ival.as<int>(),
                                    R->ival2.as<int>(), n_inst, 0, kb, R->temp.p, R->temp.cap, false, &alt2, st));
      R->ikey_sorted = alt2 ? R->ikey2.as<unsigned>() : R->ikey.as<unsigned>();
      R->ival_sorted = alt2 ? R->ival2.as<int>() : R->ival.as<int>();
      count_launch();
      ranges_kernel<<<int((n_inst + TB - 1) / TB), TB, 0, st>>>(R->ikey_sorted, n_inst, R->range.as<int2>());
      CK(cudaGetLastError());
    }
    return blend_or_defer(R, image, st);
  };
  if (begin_bit == 0) return tail(order);
  count_launch();
  fixup_runs_kernel<<<nb, TB, 0, st>>>(alt ? R->keys2.as<unsigned long long>() : R->keys.as<unsigned long long>(),
                                       const_cast<int*>(order), n, begin_bit, end_bit, stats + 3);
  CK(cudaGetLastError());
  CK(launch_readback(hp + 64, stats + 3, 8, st));
  if (!R->ev_runs) CK(cudaEventCreateWithFlags(&R->ev_runs, cudaEventDisableTiming));
  CK(cudaEventRecord(R->ev_runs, st));
  // the rest is enqueued before the host looks at the long-run flag, so the
  // GPU never idles on this check; in the rare case of long tie runs the
  // order is finished by full-width stable radix passes over the top-sorted
  // keys and everything after the sort is enqueued again (stream order
  // makes the second pass overwrite the first)
  CK(tail(order));
  CK(cudaEventSynchronize(R->ev_runs));
  if (*reinterpret_cast<const unsigned long long*>(hp + 64)) {
    R->long_runs = true;
    int alt2 = 0;
    unsigned long long* k0 = alt ? R->keys2.as<unsigned long long>() : R->keys.as<unsigned long long>();
    unsigned long long* k1 = alt ? R->keys.as<unsigned long long>() : R->keys2.as<unsigned long long>();
    int* v0 = alt ? R->vals2.as<int>() : R->vals.as<int>();
    int* v1 = alt ? R->vals.as<int>() : R->vals2.as<int>();
    CK(radix_sort_pairs<unsigned long long>(k0, k1, v0, v1, n, 0, end_bit, R->temp.p, R->temp.cap, false,
                                            &alt2, st));
    CK(tail(alt2 ? v1 : v0));
  }
  return cudaSuccess;
}

cudaError_t raster_backward(RasterCtx* R, const float* dimg, double* grads, cudaStream_t st) {
  if (R->blend_pending) return cudaErrorInvalidValue;     // the deferred blend never ran
  const CamD& cam = R->cam;
  const long long n = R->n;
  if (n == 0) return cudaSuccess;
  const int ntiles = cam.tw * cam.th;
  CK(R->g2.ensure(8 * kG2 * (size_t)n, st));
  CK(cudaMemsetAsync(R->g2.p, 0, 8 * kG2 * (size_t)n, st));
  if (R->n_inst > 0) {
    count_launch();
    timing_begin(R, 1, st);
    blend_bwd_kernel<<<ntiles, kBlendTB, 0, st>>>(R->sorted.as<Splat>(), R->ival_sorted,
                                                         R->range.as<int2>(), cam, dimg,
                                                         R->tfinal.as<double>(), R->last.as<int>(),
                                                         R->g2.as<double>());
    timing_end(R, 1, st);
  }
  CK(cudaGetLastError());
  const int TB = 128;
  count_launch();
  if (R->plan_src) {
    preprocess_bwd_src_kernel<<<int((n + TB - 1) / TB), TB, 0, st>>>(R->rsrc.as<RowSrc>(), n, cam,
                                                                     R->tiles.as<int>(), R->g2.as<double>(), grads);
  } else {
    preprocess_bwd_kernel<<<int((n + TB - 1) / TB), TB, 0, st>>>(R->src.attrs, n, cam, R->tiles.as<int>(),
                                                                 R->g2.as<double>(), grads);
  }
  return cudaGetLastError();
}

cudaError_t raster_forward(RasterCtx* R, const double* attrs, long long n, const glod_camera& cam,
                           float* image, cudaStream_t st) {
  AttrSrc a{};
  a.attrs = attrs;
  a.n = n;
  return raster_forward_src(R, a, false, cam, image, st);
}

cudaError_t raster_forward_plan(RasterCtx* R, const glod_gather_plan& plan, int* row_node,
                                const glod_camera& cam, float* image, cudaStream_t st) {
  AttrSrc a{};
  a.n = (long long)plan.n_upper + plan.n_pass + plan.n_sel;
  a.plan = plan;
  a.row_node = row_node;
  return raster_forward_src(R, a, true, cam, image, st);
}

RasterCtx* raster_create() { return new RasterCtx(); }

void raster_stats(const RasterCtx* R, glod_render_stats* out) {
  out->n_gaussians = R->n;
  out->n_instances = R->n_inst;
  out->tiles_x = R->cam.tw;
  out->tiles_y = R->cam.th;
  out->depth_full_sort = R->long_runs ? 1 : 0;
  out->reserved = 0;
}

bool raster_bad_input(const RasterCtx* R, int* section, int* index) {
  if (R->bad_section < 0) return false;
  *section = R->bad_section;
  *index = R->bad_index;
  return true;
}

void raster_destroy(RasterCtx* R) {
  cudaStream_t st = R->stream;
  Buf* all[] = {&R->splats, &R->sorted, &R->keys, &R->keys2, &R->vals, &R->vals2, &R->tiles,
                &R->tiles_sorted, &R->offs, &R->ikey, &R->ikey2, &R->ival, &R->ival2, &R->range,
                &R->tfinal, &R->last, &R->g2, &R->temp, &R->bad};
  for (Buf* b : all) b->release(st);
  if (R->host_pin.p) cudaFreeHost(R->host_pin.p);
  for (int i = 0; i < 2 * kTimed; ++i)
    if (R->ev[i]) cudaEventDestroy(R->ev[i]);
  if (R->ev_runs) cudaEventDestroy(R->ev_runs);
  delete R;
}

}  // namespace glod
