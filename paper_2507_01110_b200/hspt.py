"""Hierarchical SPT container, host-side build, and the drop-in `cut_hspt`.

Mirrors hspt.py of the reference: `Hspt` (hspt.py:17-29), `SptSelection`
(:32-37), `RenderSet` (:40-61), `build_hspt` (:64-93),
`default_size_threshold` (:96-101).  `cut_hspt` (:104-158) and `bfs_cut`
(hierarchy.py:244-266) run on the device (csrc/lod.cu); this module only
packs arguments and unpacks the device result into the reference's types.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .core import Camera, Frustum, LodConfig
from .hierarchy import NONE, CutSet, Hierarchy
from .spt import Spt, build_spts

DEFAULT_MIN_SUBTREE = 32


@dataclass
class Hspt:
    upper_nodes: np.ndarray
    spts: list
    passthrough_roots: np.ndarray
    size_threshold: float
    min_subtree: int
    lod: LodConfig
    spt_id_of: dict = field(default_factory=dict)
    flat: dict | None = None     # concatenated records (set by build_hspt)

    @property
    def passthrough_leaves(self) -> np.ndarray:
        return self.passthrough_roots

    @staticmethod
    def from_any(hs) -> "Hspt":
        if isinstance(hs, Hspt):
            return hs
        lod = LodConfig(threshold=hs.lod.threshold, metric=hs.lod.metric)
        return Hspt(upper_nodes=np.asarray(hs.upper_nodes, dtype=np.int64),
                    spts=[Spt.from_any(s) for s in hs.spts],
                    passthrough_roots=np.asarray(hs.passthrough_roots, dtype=np.int64),
                    size_threshold=float(hs.size_threshold), min_subtree=int(hs.min_subtree),
                    lod=lod, spt_id_of=dict(hs.spt_id_of))

    def flat_records(self) -> dict:
        """Concatenated record arrays + per-SPT offsets (device layout)."""
        if self.flat is None:
            spts = self.spts
            counts = np.array([s.subtree_size for s in spts], dtype=np.int64)
            offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64) \
                if spts else np.zeros(0, dtype=np.int64)
            cat = (lambda k, dt: np.concatenate([getattr(s, k) for s in spts]).astype(dt)
                   if spts else np.zeros(0, dtype=dt))
            self.flat = {
                "nodes": cat("nodes", np.int64), "key_self": cat("key_self", np.float64),
                "key_parent": cat("key_parent", np.float64), "offset": offs, "count": counts,
                "centers": (np.stack([s.root_center for s in spts]) if spts
                            else np.zeros((0, 3))),
                "roots": np.array([s.root for s in spts], dtype=np.int64)}
        return self.flat


@dataclass
class SptSelection:
    spt_id: int
    d_root: float
    prefix_len: int
    selected: np.ndarray


@dataclass
class RenderSet:
    upper: np.ndarray
    passthrough: np.ndarray
    per_spt: list

    @property
    def spt_nodes(self) -> np.ndarray:
        parts = [s.selected for s in self.per_spt]
        return np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)

    @property
    def nodes(self) -> np.ndarray:
        return np.concatenate([self.upper, self.passthrough, self.spt_nodes])

    def source_tags(self) -> dict:
        return {"upper": self.upper, "passthrough": self.passthrough, "spt": self.spt_nodes}

    def __len__(self):
        return int(self.upper.size + self.passthrough.size + self.spt_nodes.size)


def build_hspt(h, size_threshold: float, min_subtree: int, cfg: LodConfig,
               corrected: bool = True) -> Hspt:
    """Drop-in for hspt.build_hspt (hspt.py:64-93) on the GPU (K12,
    csrc/build.cu): the volume-threshold partition and build_spt
    (spt.py:45-64) of every SPT in one pass — same upper / passthrough /
    SPT-root lists, record order and f64 keys, bit for bit.  Raises
    ValueError like the reference for size_threshold <= 0 or
    min_subtree < 1; needs a CUDA device (no CPU fallback)."""
    if size_threshold <= 0:
        raise ValueError("size_threshold must be > 0")
    if min_subtree < 1:
        raise ValueError("min_subtree must be >= 1")
    import torch

    from . import _lib
    hh = Hierarchy.from_any(h)
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    cap = hh.capacity
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt)
    parent = t(hh.parent, torch.int32)
    children = t(hh.children.reshape(-1), torch.int32)
    means = t(hh.attrs.means.reshape(-1), torch.float64)
    scales = t(hh.attrs.scales.reshape(-1), torch.float64)
    i32 = lambda: torch.empty(cap, dtype=torch.int32, device=dev)
    out_t = {"upper": i32(), "pass": i32(), "roots": i32(), "count": i32(),
             "offset": torch.empty(cap, dtype=torch.int64, device=dev), "nodes": i32(),
             "key_self": torch.empty(cap, dtype=torch.float64, device=dev),
             "key_parent": torch.empty(cap, dtype=torch.float64, device=dev)}
    scratch = torch.empty(int(L.glod_hspt_build_scratch_bytes(cap)), dtype=torch.uint8, device=dev)
    bi = _lib.HsptBuildIn(capacity=cap, root=int(hh.root), min_subtree=int(min_subtree),
                          parent=parent.data_ptr(), children=children.data_ptr(),
                          means=means.data_ptr(), scales=scales.data_ptr(),
                          size_threshold=float(size_threshold), lod_threshold=float(cfg.threshold),
                          metric=0 if cfg.metric == "max_scale" else 1, corrected=int(bool(corrected)))
    bo = _lib.HsptBuildOut(*[out_t[k].data_ptr() for k in ("upper", "pass", "roots", "count", "offset",
                                                           "nodes", "key_self", "key_parent")])
    sizes = (C.c_int64 * 4)()
    _lib.check(L.glod_hspt_build(C.byref(bi), C.byref(bo), scratch.data_ptr(), scratch.numel(),
                                 sizes, _lib.stream_ptr()))
    nu, npass, S, R = (int(x) for x in sizes)
    host = lambda k, n, dt: out_t[k][:n].cpu().numpy().astype(dt)
    roots = host("roots", S, np.int64)
    counts = host("count", S, np.int64)
    flat = {"nodes": host("nodes", R, np.int64), "key_self": host("key_self", R, np.float64),
            "key_parent": host("key_parent", R, np.float64), "offset": host("offset", S, np.int64),
            "count": counts, "centers": hh.attrs.means[roots].copy(), "roots": roots}
    spts = [Spt(root=int(r), root_center=flat["centers"][i], nodes=flat["nodes"][o:o + c],
                key_self=flat["key_self"][o:o + c], key_parent=flat["key_parent"][o:o + c])
            for i, (r, o, c) in enumerate(zip(roots, flat["offset"], counts))]
    return Hspt(upper_nodes=host("upper", nu, np.int64), spts=spts,
                passthrough_roots=host("pass", npass, np.int64),
                size_threshold=float(size_threshold), min_subtree=int(min_subtree), lod=cfg,
                spt_id_of={int(r): i for i, r in enumerate(roots)}, flat=flat)


def build_hspt_host(h: Hierarchy, size_threshold: float, min_subtree: int,
               cfg: LodConfig) -> Hspt:
    """Host (numpy) restatement of build_hspt (hspt.py:64-93) with vectorised
    SPT flattening — scene tooling for CPU-only contexts (scene generators
    in the CPU test-suite); the product build is `build_hspt` (device)."""
    if size_threshold <= 0:
        raise ValueError("size_threshold must be > 0")
    if min_subtree < 1:
        raise ValueError("min_subtree must be >= 1")
    counts = h.subtree_node_counts()
    upper, cut = [], []
    frontier = np.array([h.root], dtype=np.int64)
    while frontier.size:
        vol = np.prod(h.attrs.scales[frontier], axis=1)
        small = vol < size_threshold
        cut.append(frontier[small])
        stay = frontier[~small]
        upper.append(stay)
        ch = h.children[stay]
        frontier = ch[ch[:, 0] != NONE].ravel().astype(np.int64)
    upper = np.sort(np.concatenate(upper))
    cut = np.sort(np.concatenate(cut))
    big = counts[cut] >= min_subtree
    roots = cut[big]
    spts, flat = build_spts(h, roots, cfg)
    return Hspt(upper_nodes=upper, spts=spts, passthrough_roots=cut[~big],
                size_threshold=float(size_threshold), min_subtree=int(min_subtree),
                lod=cfg, spt_id_of={int(r): i for i, r in enumerate(roots)}, flat=flat)


def default_size_threshold(h: Hierarchy) -> float:
    leaves = h.leaf_ids
    span = h.attrs.means[leaves].max(axis=0) - h.attrs.means[leaves].min(axis=0)
    return max((float(np.linalg.norm(span)) / 64.0) ** 3, 1e-30)


def cut_hspt(hspt, h, cam, cfg: LodConfig, cull: bool = True) -> RenderSet:
    """Drop-in for hspt.cut_hspt (hspt.py:104-158) on the GPU.

    Bit-exact RenderSet: sorted upper ids, sorted passthrough ids, then per
    selected SPT (ascending spt_id) its d_root, prefix_len and selected
    nodes in record order.  Live means/scales are read from `h.attrs`.
    """
    from .device import lod_scene_for
    dev = lod_scene_for(Hspt.from_any(hspt), Hierarchy.from_any(h))
    return dev.cut(Camera.from_any(cam), cfg, cull)


def bfs_cut(h, cam, cfg: LodConfig, frustum: Frustum | None = None,
            start: int | None = None) -> CutSet:
    """Drop-in for hierarchy.bfs_cut (hierarchy.py:244-266) on the GPU: the
    same kernel with an empty HSPT (the whole tree, or the subtree at
    `start`, is one passthrough BFS)."""
    from .device import bfs_scene_for
    hh = Hierarchy.from_any(h)
    dev = bfs_scene_for(hh, start)
    return dev.bfs(Camera.from_any(cam), cfg, frustum)
