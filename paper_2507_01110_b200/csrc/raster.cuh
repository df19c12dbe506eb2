// Tile rasteriser (K5-K9): internal declarations.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/glod_b200.h"

namespace glod {

constexpr int kTileW = 16;
constexpr int kTileH = 16;
constexpr int kBlendThreads = kTileW * kTileH;

// Compact per-Gaussian render record (48 B).  The pixel mean is stored
// relative to the integer bbox origin so fp32 pixel offsets are exact to
// ~1e-7 px regardless of the image size.
struct __align__(16) Splat {
  float mx, my;         // mean2d - (x0, y0)
  float ca, cb, cc;     // conic (inverse cov2d)
  float opac;
  int16_t x0, y0, x1, y1;
  float r, g, b;        // SH degree-1 colour
  int32_t idx;          // render-set row
};
static_assert(sizeof(Splat) == 48, "Splat layout");

// Per-Gaussian 2D gradient accumulators written by the backward blend.
constexpr int kG2 = 9;   // d_r, d_g, d_b, d_opac, d_mx, d_my, d_aa, d_bb, d_cc

struct RasterCtx;   // workspace + forward state kept for the backward pass

RasterCtx* raster_create();
void raster_destroy(RasterCtx* r);
cudaError_t raster_forward(RasterCtx* r, const double* attrs, long long n, const glod_camera& cam,
                           float* image, cudaStream_t st);
// The same forward reading render row r straight from its gather-plan
// source (gather.cuh row_source) and writing row_node[r]; the plan's device
// arrays must stay unchanged until the matching raster_backward.
cudaError_t raster_forward_plan(RasterCtx* r, const glod_gather_plan& plan, int* row_node,
                                const glod_camera& cam, float* image, cudaStream_t st);
// Blend deferral: while on, raster_forward(_plan) enqueues everything up to
// the blend; raster_blend enqueues the blend of the last forward.
void raster_set_defer_blend(RasterCtx* r, bool on);
cudaError_t raster_blend(RasterCtx* r, cudaStream_t st);
cudaError_t raster_backward(RasterCtx* r, const float* dimg, double* grads, cudaStream_t st);
cudaError_t launch_readback(void* host_pinned, const void* src, long long bytes, cudaStream_t st);
void raster_stats(const RasterCtx* r, glod_render_stats* out);
bool raster_bad_input(const RasterCtx* r, int* section, int* index);
void raster_timing_collect(RasterCtx* r, int enable, double* ms_out, long long* n, int nk);

}  // namespace glod
