"""Sequential Point Tree records and the drop-in `cut_spt`.

Mirrors spt.py of the reference: a subtree flattened into records
(key_self, key_parent, node) sorted by key_parent descending, ties by node
id (spt.py:45-64).  `cut_spt` (spt.py:67-75) runs on the device through
`glod_spt_compact` — the same kernel the hierarchical cut uses for every
selected SPT at once.  `build_spts` is host tooling that flattens all SPTs
of an HSPT in one vectorised pass.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import LodConfig, min_distance_batch
from .hierarchy import NONE, Hierarchy

RECORD_DTYPE = np.dtype([("key_self", "<f4"), ("key_parent", "<f4"), ("node", "<u4")])
RECORD_BYTES = RECORD_DTYPE.itemsize   # 12


@dataclass
class Spt:
    root: int
    root_center: np.ndarray
    nodes: np.ndarray        # record order (key_parent descending)
    key_self: np.ndarray
    key_parent: np.ndarray

    @property
    def subtree_size(self) -> int:
        return int(self.nodes.size)

    def packed(self) -> np.ndarray:
        rec = np.empty(self.subtree_size, dtype=RECORD_DTYPE)
        rec["key_self"] = self.key_self.astype(np.float32)
        rec["key_parent"] = self.key_parent.astype(np.float32)
        rec["node"] = self.nodes.astype(np.uint32)
        return rec

    @staticmethod
    def from_packed(root: int, root_center, rec: np.ndarray) -> "Spt":
        return Spt(root=int(root), root_center=np.asarray(root_center, dtype=np.float64),
                   nodes=rec["node"].astype(np.int64),
                   key_self=rec["key_self"].astype(np.float64),
                   key_parent=rec["key_parent"].astype(np.float64))

    @staticmethod
    def from_any(s) -> "Spt":
        if isinstance(s, Spt):
            return s
        return Spt(root=int(s.root), root_center=np.asarray(s.root_center, dtype=np.float64),
                   nodes=np.asarray(s.nodes, dtype=np.int64),
                   key_self=np.asarray(s.key_self, dtype=np.float64),
                   key_parent=np.asarray(s.key_parent, dtype=np.float64))


def spt_labels(h: Hierarchy, roots: np.ndarray) -> np.ndarray:
    """label[node] = index of the SPT root whose subtree holds it, else -1."""
    label = np.full(h.capacity, -1, dtype=np.int64)
    label[roots] = np.arange(roots.size)
    for lvl in h.levels():
        lab = label[lvl]
        inner = (lab >= 0) & (h.children[lvl, 0] != NONE)
        if inner.any():
            p = lvl[inner]
            label[h.children[p, 0]] = lab[inner]
            label[h.children[p, 1]] = lab[inner]
    return label


def build_spts(h: Hierarchy, roots, cfg: LodConfig, corrected: bool = True):
    """Flatten every subtree in `roots` at once.

    Same keys as build_spt (spt.py:50-64): key_self = m_d + ‖μ − μ_root‖
    (numpy norm over axis 1, i.e. plain (x²+y²)+z²), key_parent = parent's
    key or +inf at the root, records ordered by (−key_parent, node).
    Returns (list of Spt, flat dict) where the flat dict holds the
    concatenated record arrays and per-SPT offsets.
    """
    roots = np.asarray(roots, dtype=np.int64)
    label = spt_labels(h, roots)
    member = np.nonzero(label >= 0)[0]
    lab = label[member]
    centers = h.attrs.means[roots].copy()
    md = min_distance_batch(h.attrs.scales[member], cfg)
    if corrected:
        key_self = md + np.linalg.norm(h.attrs.means[member] - centers[lab], axis=1)
    else:
        key_self = md
    key_of = np.full(h.capacity, np.nan)
    key_of[member] = key_self
    is_root = np.zeros(h.capacity, dtype=bool)
    is_root[roots] = True
    par = h.parent[member].astype(np.int64)
    key_parent = np.where(is_root[member], np.inf, key_of[np.maximum(par, 0)])
    order = np.lexsort((member, -key_parent, lab))
    nodes = member[order]
    ks = key_self[order]
    kp = key_parent[order]
    counts = np.bincount(lab, minlength=roots.size).astype(np.int64)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    spts = [Spt(root=int(r), root_center=centers[i], nodes=nodes[o:o + c],
                key_self=ks[o:o + c], key_parent=kp[o:o + c])
            for i, (r, o, c) in enumerate(zip(roots, offs, counts))]
    flat = {"nodes": nodes, "key_self": ks, "key_parent": kp, "offset": offs,
            "count": counts, "centers": centers, "roots": roots}
    return spts, flat


def build_spt(h: Hierarchy, subtree_root: int, cfg: LodConfig, corrected: bool = True) -> Spt:
    spts, _ = build_spts(h, [subtree_root], cfg, corrected)
    return spts[0]


def cut_spt(spt, d_root: float):
    """Drop-in for spt.cut_spt (spt.py:67-75), evaluated on the GPU.

    Returns (prefix_len, selected node ids int64) exactly as the reference:
    prefix_len = #{key_parent > d_root}; [root] when d_root ≥ key_self(root);
    otherwise the prefix records with key_self ≤ d_root in record order.
    """
    from .device import single_spt_cut
    return single_spt_cut(Spt.from_any(spt), float(d_root))
