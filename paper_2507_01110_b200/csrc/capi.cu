// extern "C" entry points (include/glod_b200.h).
#include <stdio.h>
#include <string>

#include "../../include/glod_b200.h"
#include "lod.cuh"

namespace {
thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

int check(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return GLOD_OK;
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return GLOD_ERR_CUDA;
}
}  // namespace

extern "C" {

int glod_version(void) { return 1; }

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

}  // extern "C"
