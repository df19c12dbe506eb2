"""Device-resident LoD scene: packs a Hierarchy + Hspt into the flat buffers
of `glod_lod_scene` and runs the cut kernels through the C-ABI.

Layout in HBM (per HSPT version, uploaded once):
  children  int32 [cap, 2]      topology
  kind      int32 [cap]         spt_id / -2 passthrough root / -1
  means     f64   [cap, 3]      live (master params or an upload of h.attrs)
  scales    f64   [cap, 3]
  spt_*     per-SPT offset/count/root record/centre
  key_self, key_parent  f32 or f64 [R]  (f32 when every key is f32-exact,
                                          i.e. scenes read from .glod files)
  rec_node  int32 [R]
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import Camera, Frustum, LodConfig
from .hierarchy import CutSet, Hierarchy


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _t(a, dtype, device):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype)


RECORD_ALIGN = 4   # each SPT's records start on a 16-B boundary (K1 vector loads)


def pad_records(flat: dict) -> dict:
    """Device record layout: every SPT's records start at a multiple of
    RECORD_ALIGN (padding: key_self NaN, key_parent -inf, node -1), so the
    compaction kernel streams keys with aligned 16-B vector loads.  Only
    the offsets change; per-SPT record order and counts are untouched."""
    counts = np.asarray(flat["count"], dtype=np.int64)
    offs = np.asarray(flat["offset"], dtype=np.int64)
    S = counts.size
    padded = (counts + RECORD_ALIGN - 1) // RECORD_ALIGN * RECORD_ALIGN
    new_off = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64) if S else offs
    total = int(padded.sum()) if S else 0
    out = dict(flat)
    ks = np.full(max(total, 1), np.nan)
    kp = np.full(max(total, 1), -np.inf)
    nd = np.full(max(total, 1), -1, dtype=np.int64)
    if S and counts.sum():
        spt_of = np.repeat(np.arange(S), counts)
        src = np.concatenate([np.arange(o, o + c) for o, c in zip(offs, counts)]) if S < 64 else \
            (np.arange(int(counts.sum())) - np.repeat(np.cumsum(counts) - counts, counts)
             + np.repeat(offs, counts))
        dst = new_off[spt_of] + (np.arange(int(counts.sum())) - np.repeat(np.cumsum(counts) - counts, counts))
        ks[dst] = np.asarray(flat["key_self"])[src]
        kp[dst] = np.asarray(flat["key_parent"])[src]
        nd[dst] = np.asarray(flat["nodes"])[src]
    out.update(key_self=ks[:total] if total else ks[:0], key_parent=kp[:total] if total else kp[:0],
               nodes=nd[:total] if total else nd[:0], offset=new_off)
    return out


def keys_are_f32_exact(*arrs) -> bool:
    for a in arrs:
        fin = np.isfinite(a)
        if not np.array_equal(a[fin].astype(np.float32).astype(np.float64), a[fin]):
            return False
    return True


@dataclass
class SelectResult:
    upper: torch.Tensor
    passthrough: torch.Tensor
    spt_ids: torch.Tensor
    d_root: torch.Tensor
    prefix_len: torch.Tensor
    counts: torch.Tensor      # device int32[4]


@dataclass
class CompactResult:
    prefix_len: torch.Tensor
    root_rule: torch.Tensor
    seg_start: torch.Tensor
    sel_seg: torch.Tensor
    sel_pos: torch.Tensor
    sel_node: torch.Tensor
    total: torch.Tensor       # device int64[2]


class DeviceLodScene:
    """Static cut data on one device + preallocated outputs and scratch."""

    def __init__(self, h: Hierarchy, hspt=None, means: torch.Tensor | None = None,
                 scales: torch.Tensor | None = None, root: int | None = None,
                 force_f64_keys: bool = False, attr_stride: int = 0):
        dev = _dev()
        self.device = dev
        self.cap = h.capacity
        self.attr_stride = int(attr_stride)   # 0: dense [cap, 3]; else node records
        self.root = int(h.root if root is None else root)
        self.children = _t(h.children.reshape(-1), torch.int32, dev)
        kind = np.full(self.cap, -1, dtype=np.int32)
        if hspt is not None:
            flat = pad_records(hspt.flat_records())
            # Device SPT index k enumerates SPT roots in ascending node id
            # (cut_hspt visits sorted(selected_spts), hspt.py:147); spt_perm
            # maps k back to the caller's spt_id.
            perm = np.argsort(flat["roots"], kind="stable")
            for key in ("offset", "count", "centers", "roots"):
                flat[key] = flat[key][perm]
            self.spt_perm = perm.astype(np.int64)
            # first (padded) record of each caller spt_id
            self.rec_offset_by_sid = np.empty(perm.size, dtype=np.int64)
            self.rec_offset_by_sid[perm] = flat["offset"]
            kind[flat["roots"]] = np.arange(flat["roots"].size, dtype=np.int32)
            if hspt.passthrough_roots.size:
                kind[hspt.passthrough_roots] = -2
        else:
            flat = {"nodes": np.zeros(0, np.int64), "key_self": np.zeros(0), "key_parent": np.zeros(0),
                    "offset": np.zeros(0, np.int64), "count": np.zeros(0, np.int64),
                    "centers": np.zeros((0, 3)), "roots": np.zeros(0, np.int64)}
            self.spt_perm = np.zeros(0, np.int64)
        self.kind = _t(kind, torch.int32, dev)
        self.parent = _t(h.parent.reshape(-1), torch.int32, dev)
        self._kind_host = kind
        self.set_candidates(h.children, kind)
        self.S = int(flat["roots"].size)
        self.R = int(flat["nodes"].size)
        self.key_f64 = force_f64_keys or not keys_are_f32_exact(flat["key_self"], flat["key_parent"])
        kdt = torch.float64 if self.key_f64 else torch.float32
        self.key_self = _t(flat["key_self"], kdt, dev) if self.R else torch.zeros(1, dtype=kdt, device=dev)
        self.key_parent = _t(flat["key_parent"], kdt, dev) if self.R else torch.zeros(1, dtype=kdt, device=dev)
        self.rec_node = _t(flat["nodes"], torch.int32, dev) if self.R else torch.zeros(1, dtype=torch.int32, device=dev)
        self.spt_offset = _t(flat["offset"], torch.int64, dev)
        self.spt_count = _t(flat["count"], torch.int32, dev)
        root_rec = np.zeros(self.S, dtype=np.int32)
        for i in range(self.S):
            o, c = int(flat["offset"][i]), int(flat["count"][i])
            hit = np.nonzero(flat["nodes"][o:o + c] == flat["roots"][i])[0]
            root_rec[i] = int(hit[0]) if hit.size else 0
        self.root_rec_host = root_rec
        self.spt_root_rec = _t(root_rec, torch.int32, dev)
        self.spt_center = _t(flat["centers"].reshape(-1), torch.float64, dev)
        self.spt_roots_host = flat["roots"]
        self.means = means if means is not None else torch.empty(self.cap * 3, dtype=torch.float64, device=dev)
        self.scales = scales if scales is not None else torch.empty(self.cap * 3, dtype=torch.float64, device=dev)
        self._owns_attrs = means is None
        # outputs
        S1 = max(self.S, 1)
        self.o_upper = torch.empty(self.cap, dtype=torch.int32, device=dev)
        self.o_pass = torch.empty(self.cap, dtype=torch.int32, device=dev)
        self.o_spt = torch.empty(S1, dtype=torch.int32, device=dev)
        self.o_droot = torch.empty(S1, dtype=torch.float64, device=dev)
        self.o_prefix = torch.empty(S1, dtype=torch.int32, device=dev)
        self.o_counts = torch.zeros(4, dtype=torch.int32, device=dev)
        self.c_prefix = torch.empty(S1, dtype=torch.int32, device=dev)
        self.c_rootrule = torch.empty(S1, dtype=torch.int32, device=dev)
        self.c_segstart = torch.empty(S1, dtype=torch.int64, device=dev)
        R1 = max(self.R, 1)
        self.c_seg = torch.empty(R1, dtype=torch.int32, device=dev)
        self.c_pos = torch.empty(R1, dtype=torch.int32, device=dev)
        self.c_node = torch.empty(R1, dtype=torch.int32, device=dev)
        self.c_total = torch.zeros(2, dtype=torch.int64, device=dev)
        L = _lib.lib()
        self.sel_scratch = torch.empty(int(L.glod_lod_select_scratch_bytes(self.cap, self.S)),
                                       dtype=torch.uint8, device=dev)
        self.cmp_scratch = torch.empty(int(L.glod_spt_compact_scratch_bytes(self.S, self.R)),
                                       dtype=torch.uint8, device=dev)
        self._struct = self._make_struct()

    def set_candidates(self, children: np.ndarray, kind: np.ndarray):
        """Every node a cut can visit: reachable from root without entering
        an SPT subtree (upper nodes, SPT roots, passthrough subtrees)."""
        ch = np.asarray(children).reshape(-1, 2)
        up, pas = [], []
        frontier = np.array([self.root], dtype=np.int64)
        while frontier.size:                      # upper BFS region
            up.append(frontier)
            k = kind[frontier]
            pas_roots = frontier[(k == -2) & (ch[frontier, 0] != -1)]
            if pas_roots.size:
                pas.append(pas_roots)
            go = frontier[(k == -1) & (ch[frontier, 0] != -1)]
            frontier = ch[go].ravel().astype(np.int64)
        members = []
        frontier = ch[np.concatenate(pas)].ravel().astype(np.int64) if pas else np.zeros(0, np.int64)
        while frontier.size:                      # passthrough subtrees below their roots
            members.append(frontier)
            go = frontier[ch[frontier, 0] != -1]
            frontier = ch[go].ravel().astype(np.int64)
        cu = np.sort(np.concatenate(up))
        cm = np.sort(np.concatenate(members)) if members else np.zeros(0, np.int64)
        cand = np.concatenate([cu, cm]).astype(np.int32)
        self.cand = _t(cand, torch.int32, self.device) if cand.size else torch.zeros(1, dtype=torch.int32,
                                                                                      device=self.device)
        self.num_cand = int(cand.size)
        self.num_cand_upper = int(cu.size)
        if hasattr(self, "_struct"):
            self._struct = self._make_struct()

    def _make_struct(self) -> _lib.LodScene:
        p = _lib.ptr
        return _lib.LodScene(
            capacity=self.cap, root=self.root, attr_stride=self.attr_stride, children=p(self.children), kind=p(self.kind),
            means=p(self.means), scales=p(self.scales), num_spts=self.S, key_f64=int(self.key_f64),
            num_records=self.R, spt_offset=p(self.spt_offset), spt_count=p(self.spt_count),
            spt_root_rec=p(self.spt_root_rec), spt_center=p(self.spt_center),
            key_self=p(self.key_self), key_parent=p(self.key_parent), rec_node=p(self.rec_node),
            parent=p(self.parent), cand=p(self.cand), num_cand=self.num_cand,
            num_cand_upper=self.num_cand_upper)

    def upload_attrs(self, h: Hierarchy):
        """Refresh the live traversal attributes from a host hierarchy."""
        self.means.copy_(torch.from_numpy(np.ascontiguousarray(h.attrs.means, dtype=np.float64).reshape(-1)))
        self.scales.copy_(torch.from_numpy(np.ascontiguousarray(h.attrs.scales, dtype=np.float64).reshape(-1)))

    # ---- kernels ----------------------------------------------------------
    def _alt_outputs(self):
        """A second output set (speculative selects of a predicted view)."""
        if getattr(self, "_alt", None) is None:
            dev, S1 = self.device, max(self.S, 1)
            self._alt = (torch.empty(self.cap, dtype=torch.int32, device=dev),
                         torch.empty(self.cap, dtype=torch.int32, device=dev),
                         torch.empty(S1, dtype=torch.int32, device=dev),
                         torch.empty(S1, dtype=torch.float64, device=dev),
                         torch.empty(S1, dtype=torch.int32, device=dev),
                         torch.zeros(4, dtype=torch.int32, device=dev))
        return self._alt

    def select(self, cam: Camera, cfg: LodConfig, cull: bool = True,
               frustum: Frustum | None = None, stream=None, alt: bool = False) -> SelectResult:
        v = _lib.LodView()
        v.position[:] = [float(x) for x in cam.position]
        if cull:
            fr = frustum if frustum is not None else Frustum.from_camera(cam)
            v.planes[:] = [float(x) for x in np.asarray(fr.planes, dtype=np.float64).reshape(-1)]
        v.cull = int(bool(cull))
        v.metric = cfg.metric_code if hasattr(cfg, "metric_code") else (0 if cfg.metric == "max_scale" else 1)
        v.threshold = float(cfg.threshold)
        bufs = self._alt_outputs() if alt else (self.o_upper, self.o_pass, self.o_spt, self.o_droot,
                                                 self.o_prefix, self.o_counts)
        out = _lib.SelectOut(*[_lib.ptr(b) for b in bufs])
        _lib.check(_lib.lib().glod_lod_select(C.byref(self._struct), C.byref(v), C.byref(out),
                                              _lib.ptr(self.sel_scratch), self.sel_scratch.numel(),
                                              _lib.stream_ptr(stream)))
        return SelectResult(*bufs)

    def compact(self, n_spt: torch.Tensor, spt_ids: torch.Tensor, dist: torch.Tensor,
                known_prefix: torch.Tensor | None = None, stream=None) -> CompactResult:
        cin = _lib.CompactIn(n_spt=_lib.ptr(n_spt), spt_ids=_lib.ptr(spt_ids), dist=_lib.ptr(dist),
                             known_prefix=_lib.ptr(known_prefix))
        cout = _lib.CompactOut(prefix_len=_lib.ptr(self.c_prefix), root_rule=_lib.ptr(self.c_rootrule),
                               seg_start=_lib.ptr(self.c_segstart), sel_seg=_lib.ptr(self.c_seg),
                               sel_pos=_lib.ptr(self.c_pos), sel_node=_lib.ptr(self.c_node),
                               total=_lib.ptr(self.c_total))
        _lib.check(_lib.lib().glod_spt_compact(C.byref(self._struct), C.byref(cin), C.byref(cout),
                                               _lib.ptr(self.cmp_scratch), self.cmp_scratch.numel(),
                                               _lib.stream_ptr(stream)))
        return CompactResult(self.c_prefix, self.c_rootrule, self.c_segstart, self.c_seg,
                             self.c_pos, self.c_node, self.c_total)

    # ---- reference-typed results -----------------------------------------
    def cut(self, cam: Camera, cfg: LodConfig, cull: bool = True):
        from .hspt import RenderSet, SptSelection
        sel = self.select(cam, cfg, cull)
        cmp = self.compact(sel.counts[2:3], sel.spt_ids, sel.d_root, known_prefix=sel.prefix_len)
        counts = sel.counts.cpu().numpy()
        n_up, n_pa, n_sp = int(counts[0]), int(counts[1]), int(counts[2])
        total = int(cmp.total[0].item())
        upper = sel.upper[:n_up].cpu().numpy().astype(np.int64)
        passthrough = sel.passthrough[:n_pa].cpu().numpy().astype(np.int64)
        spt_ids = self.spt_perm[sel.spt_ids[:n_sp].cpu().numpy().astype(np.int64)]
        d_root = sel.d_root[:n_sp].cpu().numpy()
        prefix = sel.prefix_len[:n_sp].cpu().numpy().astype(np.int64)
        nodes = cmp.sel_node[:total].cpu().numpy().astype(np.int64)
        segs = cmp.sel_seg[:total].cpu().numpy()
        bounds = np.searchsorted(segs, np.arange(n_sp + 1))
        per = [SptSelection(spt_id=int(spt_ids[j]), d_root=float(d_root[j]),
                            prefix_len=int(prefix[j]), selected=nodes[bounds[j]:bounds[j + 1]])
               for j in range(n_sp)]
        return RenderSet(upper=upper, passthrough=passthrough, per_spt=per)

    def bfs(self, cam: Camera, cfg: LodConfig, frustum: Frustum | None) -> CutSet:
        sel = self.select(cam, cfg, cull=frustum is not None, frustum=frustum)
        n = int(sel.counts[0].item())
        return CutSet(node_ids=sel.upper[:n].cpu().numpy().astype(np.int64))


# ---- caches for the numpy drop-in path ------------------------------------
_CACHE: dict = {}


def lod_scene_for(hspt, h: Hierarchy) -> DeviceLodScene:
    key = ("hspt", id(hspt), h.capacity, h.root)
    dev = _CACHE.get(key)
    if dev is None or dev._hspt_ref is not hspt:
        _CACHE.clear()
        dev = DeviceLodScene(h, hspt)
        dev._hspt_ref = hspt
        _CACHE[key] = dev
    dev.upload_attrs(h)
    return dev


def bfs_scene_for(h: Hierarchy, start) -> DeviceLodScene:
    key = ("bfs", id(h.children), h.capacity, start)
    dev = _CACHE.get(key)
    if dev is None:
        dev = DeviceLodScene(h, None, root=h.root if start is None else int(start))
        _CACHE[key] = dev
    dev.children.copy_(torch.from_numpy(h.children.reshape(-1).astype(np.int32)))
    dev.parent.copy_(torch.from_numpy(h.parent.reshape(-1).astype(np.int32)))
    dev.set_candidates(h.children, dev._kind_host)
    dev.upload_attrs(h)
    return dev


def single_spt_cut(spt, d_root: float):
    """cut_spt for one Spt object: its records uploaded once (cached on the
    object) and cut by the batched compaction kernel with one segment."""
    dev = getattr(spt, "_glod_dev", None)
    if dev is None:
        dev = _SingleSpt(spt)
        try:
            spt._glod_dev = dev
        except Exception:
            pass
    return dev.cut(d_root)


class _SingleSpt:
    def __init__(self, spt):
        from .hspt import Hspt
        from .core import LodConfig as LC
        n = spt.subtree_size
        # a one-node stand-in hierarchy: only the SPT tables matter here
        hs = Hspt(upper_nodes=np.zeros(0, np.int64), spts=[spt],
                  passthrough_roots=np.zeros(0, np.int64), size_threshold=1.0,
                  min_subtree=1, lod=LC(1.0))
        stub = Hierarchy(attrs=None, parent=np.full(1, -1, np.int32),
                         children=np.full((1, 2), -1, np.int32), root=0)
        flat = hs.flat_records()
        flat["roots"] = np.array([spt.root], dtype=np.int64)
        self.scene = DeviceLodScene(stub, None)
        # graft the SPT tables onto the stub scene
        s = self.scene
        dev = s.device
        s.S, s.R = 1, n
        s.key_f64 = not keys_are_f32_exact(flat["key_self"], flat["key_parent"])
        kdt = torch.float64 if s.key_f64 else torch.float32
        s.key_self = _t(flat["key_self"], kdt, dev)
        s.key_parent = _t(flat["key_parent"], kdt, dev)
        s.rec_node = _t(flat["nodes"], torch.int32, dev)
        s.spt_offset = _t(flat["offset"], torch.int64, dev)
        s.spt_count = _t(flat["count"], torch.int32, dev)
        hit = np.nonzero(flat["nodes"] == spt.root)[0]
        s.spt_root_rec = _t(np.array([hit[0] if hit.size else 0]), torch.int32, dev)
        s.spt_center = _t(np.asarray(spt.root_center, dtype=np.float64), torch.float64, dev)
        s.c_seg = torch.empty(n, dtype=torch.int32, device=dev)
        s.c_pos = torch.empty(n, dtype=torch.int32, device=dev)
        s.c_node = torch.empty(n, dtype=torch.int32, device=dev)
        s.cmp_scratch = torch.empty(int(_lib.lib().glod_spt_compact_scratch_bytes(1, n)),
                                    dtype=torch.uint8, device=dev)
        s._struct = s._make_struct()
        self.n_spt = torch.ones(1, dtype=torch.int32, device=dev)
        self.ids = torch.zeros(1, dtype=torch.int32, device=dev)
        self.dist = torch.zeros(1, dtype=torch.float64, device=dev)
        self.root = spt.root

    def cut(self, d: float):
        self.dist.fill_(d)
        r = self.scene.compact(self.n_spt, self.ids, self.dist)
        total = int(r.total[0].item())
        prefix = int(r.prefix_len[0].item())
        nodes = r.sel_node[:total].cpu().numpy().astype(np.int64)
        return prefix, nodes
