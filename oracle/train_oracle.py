"""ORACLE — test infrastructure only (see oracle/glod_oracle.py header).

CPU restatement of the reference's training step with its out-of-core
store and device-cache semantics (trainer.py:302-378, cache.py:42-109,
store.py:143-333), built on the glod_oracle primitives.  Used by
tests/test_train_gpu.py as the step-level checker and by bench.py as the
CPU baseline of the train step.
"""
from __future__ import annotations

from collections import OrderedDict

import numpy as np

from . import glod_oracle as O

NAMES = ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest")
COLS = (3, 3, 4, 1, 3, 9)


def _take(P, idx):
    return {k: P[k][idx] for k in NAMES}


class OracleTrainer:
    """State: params P (f64, capacity rows), moments, per-node steps, the
    f32 slot-ordered store, the cache model, scheduler graph + RNG."""

    def __init__(self, params, children, root, kind, spt_tables, store_sections, slot_start,
                 views, lod_threshold, lod_metric, cache_budget, d_min=0.8, d_max=1.4,
                 flush_interval=1000, lam=0.2, lrs=None):
        self.P = {k: np.array(params[k], dtype=np.float64, copy=True) for k in NAMES}
        cap = self.P["means"].shape[0]
        self.M = {k: np.zeros_like(self.P[k]) for k in NAMES}
        self.V = {k: np.zeros_like(self.P[k]) for k in NAMES}
        self.step = np.zeros(cap, dtype=np.int64)
        self.children, self.root, self.kind = children, int(root), kind
        self.spt = spt_tables     # dict: offset, count, roots, centers, key_self, key_parent, nodes
        self.store = [np.array(s, dtype=np.float32, copy=True) for s in store_sections]
        self.slot_start = slot_start   # spt_id -> first slot
        self.views = views             # list of (Cam, target f64 image)
        self.T, self.metric = float(lod_threshold), int(lod_metric)
        self.budget, self.d_min, self.d_max = int(cache_budget), d_min, d_max
        self.flush_interval = int(flush_interval)
        self.lam = lam
        self.lrs = lrs
        self.cache = OrderedDict()     # spt_id -> [cached_distance, prefix_len, block, dirty]
        self.resident = 0
        self.hits = 0
        self.bytes_read = 0
        self.current_view = 0

    # store.py:304-333
    def _load(self, sid, P):
        s = self.slot_start[sid]
        self.bytes_read += P * 92
        return {k: self.store[i][s:s + P].astype(np.float64).reshape(P, c) if c > 1
                else self.store[i][s:s + P].astype(np.float64).reshape(P)
                for i, (k, c) in enumerate(zip(NAMES, COLS))}

    def _write_back(self, sid, blk):
        s = self.slot_start[sid]
        for i, (k, c) in enumerate(zip(NAMES, COLS)):
            v = np.asarray(blk[k], dtype=np.float32)
            n = v.shape[0]
            self.store[i][s:s + n] = v.reshape(self.store[i][s:s + n].shape)

    # cache.py:56-106
    def _lookup(self, sid, d):
        e = self.cache.get(sid)
        if e is not None:
            cd = e[0]
            hit = (d == 0.0) if cd == 0.0 else (self.d_min <= d / cd <= self.d_max)
            if hit:
                self.hits += 1
                self.cache.move_to_end(sid)
                return e
        return None

    def _insert(self, sid, e):
        out = []
        nbytes = e[1] * 92
        if nbytes > self.budget:
            raise ValueError("OverBudgetError")
        old = self.cache.pop(sid, None)
        if old is not None:
            self.resident -= old[1] * 92
            if old[3]:
                out.append((sid, old[2]))
        self.cache[sid] = e
        self.resident += nbytes
        while self.resident > self.budget:
            vs, victim = self.cache.popitem(last=False)
            self.resident -= victim[1] * 92
            if victim[3]:
                out.append((vs, victim[2]))
        return out

    def _positions(self, sid, d):
        """trainer._spt_positions (trainer.py:302-309)."""
        o, c = int(self.spt["offset"][sid]), int(self.spt["count"][sid])
        ks = self.spt["key_self"][o:o + c]
        kp = self.spt["key_parent"][o:o + c]
        nd = self.spt["nodes"][o:o + c]
        root = int(self.spt["roots"][sid])
        pl, sel = O.cut_spt(ks, kp, nd, root, d)
        if sel.size == 1 and sel[0] == root:
            pos = np.nonzero(nd[:pl] == root)[0]
        else:
            pos = np.nonzero(ks[:pl] <= d)[0]
        return pos, nd[pos]

    def cut(self, cam):
        planes = O.frustum_planes(cam.orientation, cam.position, cam.focal, cam.principal_point,
                                  cam.resolution, cam.far)
        return O.cut_hspt(self.root, self.children, self.kind, self.P["means"], self.P["scales"],
                          self.spt["offset"], self.spt["count"], self.spt["roots"], self.spt["centers"],
                          self.spt["key_self"], self.spt["key_parent"], self.spt["nodes"],
                          cam.position, self.T, self.metric, planes)

    def train_step(self, iteration, view, timing=None):
        """trainer.train_step (trainer.py:312-378) for the scheduled `view`
        (scheduler.next_view is host code shared by both sides); returns
        (counters, extras).  `timing` (a dict) receives per-stage seconds
        (the CPU baseline's breakdown)."""
        import time
        clock = [time.perf_counter()]

        def mark(name):
            if timing is not None:
                t = time.perf_counter()
                timing[name] = timing.get(name, 0.0) + t - clock[0]
                clock[0] = t

        self.current_view = view
        cam, target = self.views[self.current_view]
        rs = self.cut(cam)
        mark("cut")
        bytes_before, hits_before = self.bytes_read, self.hits
        loaded = 0
        mem = np.concatenate([rs["upper"], rs["passthrough"]]).astype(np.int64)
        parts = [_take(self.P, mem)]
        rows = []
        off = mem.size
        for j, sid in enumerate(rs["spt_id"]):
            sid = int(sid)
            d, P = float(rs["d_root"][j]), int(rs["prefix_len"][j])
            e = self._lookup(sid, d)
            if e is None:
                blk = self._load(sid, P)
                loaded += P
                e = [d, P, blk, False]
                for esid, eblk in self._insert(sid, e):
                    self._write_back(esid, eblk)
            pos, nodes = self._positions(sid, e[0])
            parts.append(_take(e[2], pos))
            rows.append((e, pos, nodes, off))
            off += pos.size
        A = {k: np.concatenate([p[k] for p in parts]) for k in NAMES}
        mark("gather")
        img, ctx = O.render_forward(A, cam)
        mark("forward")
        value, dimg = O.ssim_l1_loss(img, target, self.lam)
        mark("loss")
        G = O.backward(ctx, dimg)
        mark("backward")
        if timing is not None:
            timing["splats_backward"] = len(ctx["splats"])
        O.adam_update(self.P, self.M, self.V, self.step, mem, G, np.arange(mem.size), self.lrs)
        for e, pos, nodes, o in rows:
            O.adam_update(self.P, self.M, self.V, self.step, nodes, G, np.arange(o, o + pos.size),
                          self.lrs)
            for k in NAMES:
                e[2][k][pos] = self.P[k][nodes]
            e[3] = True
        mark("adam")
        if iteration % self.flush_interval == 0:
            for sid, e in list(self.cache.items()):
                if e[3]:
                    self._write_back(sid, e[2])
            self.cache.clear()
            self.resident = 0
        mark("flush")
        counters = {"iteration": iteration, "view": self.current_view, "loss": float(value),
                    "gaussians_rendered": int(A["means"].shape[0]),
                    "gaussians_loaded_from_store": int(loaded),
                    "cache_hits": int(self.hits - hits_before),
                    "bytes_streamed": int(self.bytes_read - bytes_before)}
        row_nodes = np.concatenate([mem] + [r[2] for r in rows]) if rows else mem
        return counters, {"grads": G, "row_nodes": row_nodes, "image": img}
