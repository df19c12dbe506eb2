"""ctypes binding of include/glod_b200.h.

The product path has no fallback: if `libglod_b200.so` is missing or a CUDA
device is absent, `lib()` raises.  (`import paper_2507_01110_b200` works
without a GPU so the CPU test-suite can check the library's exports.)
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# GLOD_LIB: an alternative build of the same library (kernel variants for
# A/B timing runs); default: the in-tree build.
LIB_PATH = Path(os.environ.get("GLOD_LIB") or Path(__file__).resolve().parent / "libglod_b200.so")

GLOD_OK = 0
GLOD_ERR_INVALID_ARGUMENT = 1
GLOD_ERR_CUDA = 2
GLOD_ERR_INVALID_INPUT = 3
GLOD_ERR_OVER_BUDGET = 4

P = C.c_void_p


class LodScene(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("root", C.c_int32), ("attr_stride", C.c_int32),
                ("children", P), ("kind", P), ("means", P), ("scales", P),
                ("num_spts", C.c_int32), ("key_f64", C.c_int32), ("num_records", C.c_int64),
                ("spt_offset", P), ("spt_count", P), ("spt_root_rec", P), ("spt_center", P),
                ("key_self", P), ("key_parent", P), ("rec_node", P),
                ("parent", P), ("cand", P), ("num_cand", C.c_int64), ("num_cand_upper", C.c_int64)]


class HsptBuildIn(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("root", C.c_int32), ("min_subtree", C.c_int32),
                ("parent", P), ("children", P), ("means", P), ("scales", P),
                ("size_threshold", C.c_double), ("lod_threshold", C.c_double),
                ("metric", C.c_int32), ("corrected", C.c_int32)]


class HsptBuildOut(C.Structure):
    _fields_ = [("upper_ids", P), ("pass_ids", P), ("spt_roots", P), ("spt_count", P),
                ("spt_offset", P), ("rec_node", P), ("key_self", P), ("key_parent", P)]


class LodView(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("planes", C.c_double * 24),
                ("cull", C.c_int32), ("metric", C.c_int32), ("threshold", C.c_double)]


class SelectOut(C.Structure):
    _fields_ = [("upper_ids", P), ("pass_ids", P), ("spt_ids", P), ("d_root", P),
                ("prefix_len", P), ("counts", P)]


class CompactIn(C.Structure):
    _fields_ = [("n_spt", P), ("spt_ids", P), ("dist", P), ("known_prefix", P)]


class CompactOut(C.Structure):
    _fields_ = [("prefix_len", P), ("root_rule", P), ("seg_start", P), ("sel_seg", P),
                ("sel_pos", P), ("sel_node", P), ("total", P)]


class Camera(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("w2c", C.c_double * 9), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("near_plane", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class RenderStats(C.Structure):
    _fields_ = [("n_gaussians", C.c_int64), ("n_instances", C.c_int64),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("depth_full_sort", C.c_int32),
                ("reserved", C.c_int32)]


class GatherPlan(C.Structure):
    _fields_ = [("master", P), ("capacity", C.c_int64), ("upper_ids", P), ("pass_ids", P),
                ("n_upper", C.c_int32), ("n_pass", C.c_int32), ("sel_seg", P), ("sel_pos", P),
                ("sel_node", P), ("n_sel", C.c_int64), ("seg_block", P), ("seg_rows", P),
                ("master_stride", C.c_int64), ("spt_from_master", C.c_int32)]


class StoreView(C.Structure):
    _fields_ = [("section", P * 6), ("nslots", C.c_int64), ("row_stride", C.c_int64)]


class PrefixItem(C.Structure):
    _fields_ = [("slot_start", C.c_int64), ("rows", C.c_int64), ("elem_start", C.c_int64),
                ("block", P), ("overlay", P), ("overlay_rows", C.c_int64), ("src", P)]


class CacheStats(C.Structure):
    _fields_ = [("entries", C.c_int64), ("resident_bytes", C.c_int64), ("hits", C.c_int64),
                ("misses", C.c_int64), ("loaded_rows", C.c_int64), ("prefetched_rows", C.c_int64),
                ("prefetch_used_rows", C.c_int64), ("pool_allocs", C.c_int64), ("grow_events", C.c_int64),
                ("host_ns_step", C.c_int64), ("host_ns_prefetch", C.c_int64), ("pf_copies", C.c_int64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "glod_version": (C.c_int, []),
    "glod_last_error": (C.c_char_p, []),
    "glod_launch_count": (C.c_uint64, []),
    "glod_lod_select_scratch_bytes": (C.c_int64, [C.c_int64, C.c_int32]),
    "glod_lod_select": (C.c_int, [C.POINTER(LodScene), C.POINTER(LodView),
                                  C.POINTER(SelectOut), P, C.c_int64, P]),
    "glod_spt_compact_scratch_bytes": (C.c_int64, [C.c_int32, C.c_int64]),
    "glod_spt_compact": (C.c_int, [C.POINTER(LodScene), C.POINTER(CompactIn),
                                   C.POINTER(CompactOut), P, C.c_int64, P]),
    "glod_hspt_build_scratch_bytes": (C.c_int64, [C.c_int64]),
    "glod_hspt_build": (C.c_int, [C.POINTER(HsptBuildIn), C.POINTER(HsptBuildOut), P, C.c_int64,
                                  C.POINTER(C.c_int64), P]),
    "glod_raster_create": (C.c_int, [C.POINTER(P)]),
    "glod_raster_destroy": (C.c_int, [P]),
    "glod_render_forward": (C.c_int, [P, P, C.c_int64, C.POINTER(Camera), P, P]),
    "glod_render_backward": (C.c_int, [P, P, P, P]),
    "glod_render_stats_get": (C.c_int, [P, C.POINTER(RenderStats)]),
    "glod_render_blend_timing": (C.c_int, [P, C.c_int32, P, P]),
    "glod_render_kernel_timing": (C.c_int, [P, C.c_int32, P, P]),
    "glod_render_defer_blend": (C.c_int, [P, C.c_int32]),
    "glod_render_blend": (C.c_int, [P, P]),
    "glod_loss_scratch_bytes": (C.c_int64, [C.c_int32, C.c_int32]),
    "glod_loss_l1_ssim": (C.c_int, [P, P, C.c_int32, C.c_int32, C.c_double, P, P, P, C.c_int64, P]),
    "glod_adam_step": (C.c_int, [P, P, P, C.c_int64, P, P, P, C.c_int64, C.c_int64,
                                 C.POINTER(C.c_double), P, C.c_int64, P, P]),
    "glod_adam_step_records": (C.c_int, [P, C.c_int64, P, P, P, C.c_int64, C.c_int64,
                                         C.POINTER(C.c_double), P, C.c_int64, P, P]),
    "glod_gather_render_rows": (C.c_int, [C.POINTER(GatherPlan), P, P, P]),
    "glod_render_forward_plan": (C.c_int, [P, C.POINTER(GatherPlan), P, C.POINTER(Camera), P, P]),
    "glod_scatter_to_blocks": (C.c_int, [C.POINTER(GatherPlan), P]),
    "glod_wire_pack": (C.c_int, [P, C.c_int64, P, P, C.c_int32, C.c_int64, P, P]),
    "glod_refresh_resident_blocks": (C.c_int, [P, C.c_int64, C.c_int64, P, C.c_int64, P, P, P, P, P, P]),
    "glod_cache_resident": (C.c_int, [P, P, P, C.c_int32]),
    "glod_cache_mark_dirty": (C.c_int, [P, P, C.c_int32]),
    "glod_convert": (C.c_int, [P, P, C.c_int64, C.c_int32, P]),
    "glod_host_device_ptr": (C.c_int, [P, C.POINTER(P)]),
    "glod_store_load_prefixes": (C.c_int, [C.POINTER(StoreView), P, C.c_int32, C.c_int64, P]),
    "glod_store_write_back": (C.c_int, [C.POINTER(StoreView), P, C.c_int32, C.c_int64, P]),
    "glod_cache_create": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_int32, P,
                                    C.c_int32, C.POINTER(P)]),
    "glod_cache_destroy": (C.c_int, [P]),
    "glod_cache_set_file": (C.c_int, [P, C.c_int32, P]),
    "glod_cache_flush_io": (C.c_int, [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "glod_cache_step": (C.c_int, [P, C.POINTER(StoreView), C.c_int32, P, P, P, P, P, P, P, P]),
    "glod_cache_end_step": (C.c_int, [P, C.POINTER(StoreView), C.c_int64, C.c_int32, P]),
    "glod_cache_prefetch": (C.c_int, [P, C.POINTER(StoreView), C.c_int32, P, P, P, C.c_int64, P, P]),
    "glod_cache_debug_profile": (C.c_int, [P, P]),
    "glod_cache_stats": (C.c_int, [P, C.POINTER(CacheStats)]),
    "glod_cache_set_master": (C.c_int, [P, P, C.c_int64, C.c_int64, P, P, C.c_int32]),
    "glod_cache_materialize": (C.c_int, [P, P]),
    "glod_cache_entries": (C.c_int, [P, P, P, P, P, P, C.c_int64]),
    "glod_memcpy_d2h": (C.c_int, [P, P, C.c_int64]),
    "glod_nccl_unique_id": (C.c_int, [P]),
    "glod_xchg_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, P, C.POINTER(P)]),
    "glod_xchg_destroy": (C.c_int, [P]),
    "glod_grad_exchange": (C.c_int, [P, P, P, C.c_int64, C.POINTER(C.c_int64), P]),
    "glod_param_allgather": (C.c_int, [P, P, C.c_int64, P]),
    "glod_xchg_union": (C.c_int, [P, P, C.c_int64, C.POINTER(C.c_int64), P]),
    "glod_xchg_union_ids": (C.c_int, [P, C.POINTER(P), C.POINTER(C.c_int64)]),
    "glod_xchg_pack": (C.c_int, [P, P, P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(P), P]),
    "glod_xchg_begin_accumulate": (C.c_int, [P, C.POINTER(P), C.POINTER(C.c_int64), P]),
    "glod_xchg_accumulate": (C.c_int, [P, P, C.c_int64, P]),
    "glod_xchg_owned": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(C.c_int64)]),
    "glod_xchg_pack_params": (C.c_int, [P, P, C.c_int64, C.POINTER(P), P]),
    "glod_xchg_scatter_params": (C.c_int, [P, P, C.c_int64, P]),
    "glod_xchg_stats": (C.c_int, [P, P]),
    "glod_readback": (C.c_int, [P, P, C.c_int64, P]),
    "glod_readback_multi": (C.c_int, [C.c_int32, P, P, P, P]),
    "glod_upload": (C.c_int, [P, P, C.c_int64, P]),
    "glod_debug_select_phases": (C.c_int, [P]),
    "glod_sort_scratch_bytes": (C.c_int64, [C.c_int64]),
    "glod_sort_pairs_u64": (C.c_int, [P, P, P, P, C.c_int64, C.c_int32, C.c_int32, P, C.c_int64,
                                      C.POINTER(C.c_int32), P]),
    "glod_sort_pairs_u32": (C.c_int, [P, P, P, P, C.c_int64, C.c_int32, C.c_int32, P, C.c_int64,
                                      C.POINTER(C.c_int32), P]),
}

_LIB = None


class GlodError(RuntimeError):
    pass


def load(path: Path = LIB_PATH) -> C.CDLL:
    """dlopen the library and bind every declared symbol (no GPU needed)."""
    global _LIB
    if _LIB is None:
        if not path.exists():
            raise GlodError(f"{path} not built: run python -m paper_2507_01110_b200.build")
        lib = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def lib() -> C.CDLL:
    """The library, for device work: requires a CUDA device."""
    import torch
    if not torch.cuda.is_available():
        raise GlodError("glod_b200 needs a CUDA device (no CPU fallback)")
    return load()


def check(code: int):
    if code == GLOD_OK:
        return
    msg = load().glod_last_error().decode(errors="replace")
    if code == GLOD_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == GLOD_ERR_INVALID_INPUT:
        from .renderer import InvalidInputError
        raise InvalidInputError(msg)
    if code == GLOD_ERR_OVER_BUDGET:
        from .cache import OverBudgetError
        raise OverBudgetError(msg)
    raise GlodError(msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None → NULL)."""
    return 0 if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream`, or of the current torch stream (read with
    the raw getters: torch.cuda.current_stream() costs ~20 µs of Python,
    and the step passes a stream to ~20 calls)."""
    import torch
    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


class _DevArray:
    """__cuda_array_interface__ over a library-owned device buffer, so
    torch.as_tensor can view it without a copy."""

    def __init__(self, addr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(addr), False), "shape": tuple(int(x) for x in shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def device_view(addr: int, shape, dtype):
    """A torch tensor viewing `addr` (device memory owned by the library)."""
    import torch
    typestr = {torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8", torch.float32: "<f4"}[dtype]
    if int(np.prod(shape)) == 0 or not addr:
        return torch.empty(shape, dtype=dtype, device="cuda")
    return torch.as_tensor(_DevArray(addr, shape, typestr), device="cuda")


def upload(dst, host_pinned, nbytes: int | None = None, stream=None):
    """Stream-ordered small upload of a pinned host tensor into a device
    tensor (kernel-read through the mapped address; see glod_upload)."""
    n = host_pinned.numel() * host_pinned.element_size() if nbytes is None else nbytes
    check(lib().glod_upload(ptr(dst), ptr(host_pinned), int(n), stream_ptr(stream)))


def readback_multi(pairs, stream=None):
    """Several read-backs (host_pinned, src[, nbytes]) in one kernel launch
    (glod_readback_multi; ≤ 8)."""
    n = len(pairs)
    dst = (C.c_void_p * n)()
    src = (C.c_void_p * n)()
    nb = (C.c_int64 * n)()
    for i, p in enumerate(pairs):
        h, s = p[0], p[1]
        dst[i] = ptr(h)
        src[i] = ptr(s)
        nb[i] = p[2] if len(p) > 2 else s.numel() * s.element_size()
    check(lib().glod_readback_multi(n, dst, src, nb, stream_ptr(stream)))


def readback(host_pinned, src, nbytes: int | None = None, stream=None):
    """Stream-ordered read-back of a device tensor into a pinned host tensor
    (kernel-written through the mapped address; see glod_readback)."""
    n = src.numel() * src.element_size() if nbytes is None else nbytes
    check(lib().glod_readback(ptr(host_pinned), ptr(src), int(n), stream_ptr(stream)))

