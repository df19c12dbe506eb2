// LoD selection kernels: the hierarchical cut (K2) and the SPT prefix cut (K1).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include "../../include/glod_b200.h"

namespace glod {

using LodScene = glod_lod_scene;
using LodView = glod_lod_view;
using SelectOut = glod_lod_select_out;
using CompactIn = glod_spt_compact_in;
using CompactOut = glod_spt_compact_out;

size_t select_scratch_bytes(int64_t cap, int32_t num_spts, int grid);
size_t compact_scratch_bytes(int32_t num_spts, int64_t num_records, int grid);
int select_grid();
int compact_grid();

cudaError_t launch_select(const LodScene& sc, const LodView& v, const SelectOut& out,
                          void* scratch, size_t scratch_bytes, cudaStream_t st);
cudaError_t launch_compact(const LodScene& sc, const CompactIn& in, const CompactOut& out,
                           void* scratch, size_t scratch_bytes, cudaStream_t st);

}  // namespace glod
