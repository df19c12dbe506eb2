// extern "C" entry points (include/glod_b200.h).
#include <stdio.h>
#include <atomic>
#include <string>

#include "../../include/glod_b200.h"
#include "lod.cuh"
#include "raster.cuh"

namespace glod {
static std::atomic<unsigned long long> g_launches{0};
void count_launch(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int set_error(int code, const char* what);
void retain_pool_memory();
size_t loss_scratch_bytes(int W, int H);
cudaError_t launch_loss(const float* X, const float* Y, int W, int H, double lam, double* out,
                        float* grad, void* scratch, size_t bytes, cudaStream_t st);
cudaError_t launch_adam(double* params, double* mv, long long* step, long long cap,
                        const int* ids, const double* grads, const int* rows, long long grad_rows,
                        long long n, const double* lrs, const double* bias, long long bias_len,
                        const glod_gather_plan* plan, cudaStream_t st);
cudaError_t launch_adam_records(double* rec, const int* ids, const double* grads, const int* rows,
                                long long grad_rows, long long n, const double* lrs, const double* bias,
                                long long bias_len, const glod_gather_plan* plan, cudaStream_t st);
cudaError_t launch_gather(const glod_gather_plan& p, long long R, double* out, int* row_node,
                          cudaStream_t st);
cudaError_t launch_scatter_back(const glod_gather_plan& p, cudaStream_t st);
cudaError_t launch_wire_pack(const double* master, long long cap, const int* ids, const long long* seg,
                             int n_msgs, long long N, float* out, cudaStream_t st);
cudaError_t launch_refresh_resident(const double* master, long long cap, long long mstride, const int* ids,
                                    long long n,
                                    const int* spt_of_node, const int* rec_of_node,
                                    const unsigned long long* res_block, const long long* res_rows, int* touched,
                                    cudaStream_t st);
cudaError_t launch_convert(const void* in, void* out, long long n, int to_f64, cudaStream_t st);
cudaError_t launch_store_xfer(const glod_store_view& sv, const glod_prefix_item* items, int n_items,
                              long long total, int load, cudaStream_t st);
cudaError_t launch_upload(void* dst, const void* host_pinned, long long bytes, cudaStream_t st);
cudaError_t launch_readback_multi(int n, void* const* host_pinned, const void* const* src, const long long* bytes,
                                  cudaStream_t st);
cudaError_t select_phase_ns(long long* out7);
cudaError_t launch_readback(void* host_pinned, const void* src, long long bytes, cudaStream_t st);
}  // namespace glod

struct glod_raster {
  glod::RasterCtx* ctx;
};

namespace {
thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

}  // namespace

// Workspaces and cache blocks come from the device's default stream-ordered
// pool.  Its default release threshold (0) hands memory back to the driver
// at every synchronisation, so the next step's cudaMallocAsync re-maps
// pages; keep what was reserved instead (HBM is sized for it).
void glod::retain_pool_memory() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  unsigned long long thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

int glod::set_error(int code, const char* what) {
  g_err = what;
  return code;
}

namespace {
int check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return GLOD_OK;
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return GLOD_ERR_CUDA;
}
}  // namespace

extern "C" {

int glod_version(void) { return 1; }

uint64_t glod_launch_count(void) { return glod::g_launches.load(std::memory_order_relaxed); }

const char* glod_last_error(void) { return g_err.c_str(); }

int64_t glod_lod_select_scratch_bytes(int64_t capacity, int32_t num_spts) {
  return int64_t(glod::select_scratch_bytes(capacity, num_spts, glod::select_grid()));
}

int glod_lod_select(const glod_lod_scene* scene, const glod_lod_view* view,
                    const glod_lod_select_out* out, void* scratch, int64_t scratch_bytes,
                    void* stream) {
  if (!scene || !view || !out || !scratch) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (scene->capacity < 1 || scene->capacity >= (int64_t(1) << 30))
    return fail(GLOD_ERR_INVALID_ARGUMENT, "capacity out of range");
  if (scene->root < 0 || scene->root >= scene->capacity)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "root out of range");
  return check(glod::launch_select(*scene, *view, *out, scratch, size_t(scratch_bytes),
                                   static_cast<cudaStream_t>(stream)),
               "glod_lod_select");
}

int64_t glod_spt_compact_scratch_bytes(int32_t num_spts, int64_t num_records) {
  return int64_t(glod::compact_scratch_bytes(num_spts, num_records, glod::compact_grid()));
}

int glod_spt_compact(const glod_lod_scene* scene, const glod_spt_compact_in* in,
                     const glod_spt_compact_out* out, void* scratch, int64_t scratch_bytes,
                     void* stream) {
  if (!scene || !in || !out || !scratch) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_compact(*scene, *in, *out, scratch, size_t(scratch_bytes),
                                    static_cast<cudaStream_t>(stream)),
               "glod_spt_compact");
}

int glod_raster_create(glod_raster** out) {
  if (!out) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  glod::retain_pool_memory();
  *out = new glod_raster{glod::raster_create()};
  return GLOD_OK;
}

int glod_raster_destroy(glod_raster* r) {
  if (r) {
    glod::raster_destroy(r->ctx);
    delete r;
  }
  return GLOD_OK;
}

static int render_result(glod_raster* r, cudaError_t e, const char* what) {
  int sec, idx;
  if (glod::raster_bad_input(r->ctx, &sec, &idx)) {
    static const char* names[6] = {"means", "scales", "rotations", "opacities", "base_colors", "sh_rest"};
    char buf[128];
    snprintf(buf, sizeof(buf), "non-finite %s on Gaussian %d", names[sec], idx);
    return fail(GLOD_ERR_INVALID_INPUT, buf);
  }
  return check(e, what);
}

int glod_render_forward(glod_raster* r, const double* attrs, int64_t n, const glod_camera* cam,
                        float* image, void* stream) {
  if (!r || !cam || !image || (n > 0 && !attrs)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (cam->width < 1 || cam->height < 1 || cam->width > 32767 || cam->height > 32767)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "camera resolution out of range");
  if (n < 0 || n > 0x7fffffffll) return fail(GLOD_ERR_INVALID_ARGUMENT, "n out of range");
  cudaError_t e = glod::raster_forward(r->ctx, attrs, n, *cam, image, static_cast<cudaStream_t>(stream));
  return render_result(r, e, "glod_render_forward");
}

int glod_render_forward_plan(glod_raster* r, const glod_gather_plan* plan, int32_t* row_node,
                             const glod_camera* cam, float* image, void* stream) {
  if (!r || !plan || !cam || !image) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (cam->width < 1 || cam->height < 1 || cam->width > 32767 || cam->height > 32767)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "camera resolution out of range");
  const long long n = (long long)plan->n_upper + plan->n_pass + plan->n_sel;
  if (plan->n_upper < 0 || plan->n_pass < 0 || plan->n_sel < 0 || n > 0x7fffffffll)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "row counts out of range");
  if (n > 0 && (!row_node || !plan->master)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (plan->master_stride != 0 && plan->master_stride != GLOD_NODE_RECORD)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "master_stride must be 0 or GLOD_NODE_RECORD");
  cudaError_t e = glod::raster_forward_plan(r->ctx, *plan, row_node, *cam, image, static_cast<cudaStream_t>(stream));
  return render_result(r, e, "glod_render_forward_plan");
}

int glod_render_defer_blend(glod_raster* r, int32_t enable) {
  if (!r) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  glod::raster_set_defer_blend(r->ctx, enable != 0);
  return GLOD_OK;
}

int glod_render_blend(glod_raster* r, void* stream) {
  if (!r) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  cudaError_t e = glod::raster_blend(r->ctx, static_cast<cudaStream_t>(stream));
  if (e == cudaErrorInvalidValue) return fail(GLOD_ERR_INVALID_ARGUMENT, "no deferred blend pending");
  return check(e, "glod_render_blend");
}

int glod_render_backward(glod_raster* r, const float* dl_dimage, double* grads, void* stream) {
  if (!r || !dl_dimage || !grads) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::raster_backward(r->ctx, dl_dimage, grads, static_cast<cudaStream_t>(stream)),
               "glod_render_backward");
}

int glod_render_blend_timing(glod_raster* r, int32_t enable, double* ms_out, int64_t* launches_out) {
  if (!r) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  long long n[2] = {0, 0};
  glod::raster_timing_collect(r->ctx, enable, ms_out, n, 2);
  if (launches_out) {
    launches_out[0] = n[0];
    launches_out[1] = n[1];
  }
  return GLOD_OK;
}

int glod_render_kernel_timing(glod_raster* r, int32_t enable, double* ms_out, int64_t* launches_out) {
  if (!r) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  long long n[3] = {0, 0, 0};
  glod::raster_timing_collect(r->ctx, enable, ms_out, n, 3);
  if (launches_out)
    for (int k = 0; k < 3; ++k) launches_out[k] = n[k];
  return GLOD_OK;
}

int glod_render_stats_get(const glod_raster* r, glod_render_stats* out) {
  if (!r || !out) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  glod::raster_stats(r->ctx, out);
  return GLOD_OK;
}

int64_t glod_loss_scratch_bytes(int32_t width, int32_t height) {
  return int64_t(glod::loss_scratch_bytes(width, height));
}

int glod_loss_l1_ssim(const float* rendered, const float* target, int32_t width, int32_t height,
                      double lam, double* value, float* grad, void* scratch, int64_t scratch_bytes,
                      void* stream) {
  if (!rendered || !target || !value || !grad || !scratch)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (!(lam >= 0.0 && lam <= 1.0)) return fail(GLOD_ERR_INVALID_INPUT, "lambda must lie in [0, 1]");
  if (width < 1 || height < 1) return fail(GLOD_ERR_INVALID_INPUT, "image dimensions differ");
  return check(glod::launch_loss(rendered, target, width, height, lam, value, grad, scratch,
                                 size_t(scratch_bytes), static_cast<cudaStream_t>(stream)),
               "glod_loss_l1_ssim");
}

int glod_adam_step(double* params, double* mv, int64_t* step, int64_t capacity,
                   const int32_t* ids, const double* grads, const int32_t* rows, int64_t grad_rows,
                   int64_t n, const double* lrs, const double* bias_table, int64_t bias_len,
                   const glod_gather_plan* refresh, void* stream) {
  if (n > 0 && (!params || !mv || !step || !ids || !grads || !lrs))
    return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_adam(params, mv, reinterpret_cast<long long*>(step), capacity, ids,
                                 grads, rows, grad_rows, n, lrs, bias_table, bias_len, refresh,
                                 static_cast<cudaStream_t>(stream)),
               "glod_adam_step");
}

int glod_adam_step_records(double* records, int64_t capacity, const int32_t* ids, const double* grads,
                           const int32_t* rows, int64_t grad_rows, int64_t n, const double* lrs,
                           const double* bias_table, int64_t bias_len, const glod_gather_plan* refresh,
                           void* stream) {
  (void)capacity;
  if (n > 0 && (!records || !ids || !grads || !lrs)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_adam_records(records, ids, grads, rows, grad_rows, n, lrs, bias_table, bias_len,
                                         refresh, static_cast<cudaStream_t>(stream)),
               "glod_adam_step_records");
}

int glod_gather_render_rows(const glod_gather_plan* plan, double* out, int32_t* row_node,
                            void* stream) {
  if (!plan) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  const long long R = (long long)plan->n_upper + plan->n_pass + plan->n_sel;
  if (R > 0 && !out) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_gather(*plan, R, out, row_node, static_cast<cudaStream_t>(stream)),
               "glod_gather_render_rows");
}

int glod_wire_pack(const double* master, int64_t capacity, const int32_t* ids, const int64_t* seg_start,
                   int32_t n_msgs, int64_t n_rows, float* out, void* stream) {
  if (n_rows > 0 && (!master || !ids || !seg_start || !out || n_msgs <= 0))
    return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_wire_pack(master, capacity, ids, reinterpret_cast<const long long*>(seg_start),
                                      n_msgs, n_rows, out, static_cast<cudaStream_t>(stream)),
               "glod_wire_pack");
}

int glod_refresh_resident_blocks(const double* master, int64_t capacity, int64_t master_stride,
                                 const int32_t* ids, int64_t n,
                                 const int32_t* spt_of_node, const int32_t* rec_of_node,
                                 const uint64_t* res_block, const int64_t* res_rows, int32_t* touched,
                                 void* stream) {
  if (n > 0 && (!master || !ids || !spt_of_node || !rec_of_node || !res_block || !res_rows || !touched))
    return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_refresh_resident(master, capacity, master_stride, ids, n, spt_of_node, rec_of_node,
                                             reinterpret_cast<const unsigned long long*>(res_block),
                                             reinterpret_cast<const long long*>(res_rows), touched,
                                             static_cast<cudaStream_t>(stream)),
               "glod_refresh_resident_blocks");
}

int glod_scatter_to_blocks(const glod_gather_plan* plan, void* stream) {
  if (!plan) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_scatter_back(*plan, static_cast<cudaStream_t>(stream)),
               "glod_scatter_to_blocks");
}

int glod_convert(const void* in, void* out, int64_t n, int32_t to_f64, void* stream) {
  if (n > 0 && (!in || !out)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_convert(in, out, n, to_f64, static_cast<cudaStream_t>(stream)),
               "glod_convert");
}

int glod_debug_select_phases(int64_t* ns_out7) {
  if (!ns_out7) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  long long t[7];
  const int rc = check(glod::select_phase_ns(t), "glod_debug_select_phases");
  for (int k = 0; k < 7; ++k) ns_out7[k] = t[k];
  return rc;
}

int glod_upload(void* dst, const void* host_pinned, int64_t bytes, void* stream) {
  if ((!host_pinned || !dst) && bytes > 0) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_upload(dst, host_pinned, bytes, static_cast<cudaStream_t>(stream)), "glod_upload");
}

int glod_readback_multi(int32_t n, void* const* host_pinned, const void* const* src, const int64_t* bytes,
                        void* stream) {
  if (n < 0 || n > 8 || (n > 0 && (!host_pinned || !src || !bytes)))
    return fail(GLOD_ERR_INVALID_ARGUMENT, "n must be 0..8 with non-null arrays");
  long long b[8];
  for (int r = 0; r < n; ++r) b[r] = bytes[r];
  return check(glod::launch_readback_multi(n, host_pinned, src, b, static_cast<cudaStream_t>(stream)),
               "glod_readback_multi");
}

int glod_readback(void* host_pinned, const void* src, int64_t bytes, void* stream) {
  if ((!host_pinned || !src) && bytes > 0) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(glod::launch_readback(host_pinned, src, bytes, static_cast<cudaStream_t>(stream)),
               "glod_readback");
}

int glod_host_device_ptr(void* host, void** dev) {
  if (!host || !dev) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  return check(cudaHostGetDevicePointer(dev, host, 0), "glod_host_device_ptr");
}

int glod_store_load_prefixes(const glod_store_view* store, const glod_prefix_item* items,
                             int32_t n_items, int64_t total_elems, void* stream) {
  if (!store || (n_items > 0 && !items)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (store->row_stride != 0 && store->row_stride != 23)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "store row_stride must be 0 or 23");
  return check(glod::launch_store_xfer(*store, items, n_items, total_elems, 1,
                                       static_cast<cudaStream_t>(stream)),
               "glod_store_load_prefixes");
}

int glod_store_write_back(const glod_store_view* store, const glod_prefix_item* items,
                          int32_t n_items, int64_t total_elems, void* stream) {
  if (!store || (n_items > 0 && !items)) return fail(GLOD_ERR_INVALID_ARGUMENT, "null argument");
  if (store->row_stride != 0 && store->row_stride != 23)
    return fail(GLOD_ERR_INVALID_ARGUMENT, "store row_stride must be 0 or 23");
  return check(glod::launch_store_xfer(*store, items, n_items, total_elems, 0,
                                       static_cast<cudaStream_t>(stream)),
               "glod_store_write_back");
}

}  // extern "C"
