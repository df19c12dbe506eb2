"""Device-resident training step (mirrors trainer.train_step, trainer.py:312-378).

Layout in HBM (per scene):
  node records   f64 [capacity][72] (GLOD_NODE_RECORD): the authoritative
                 `h.attrs` values, the ADAM moments (OptimizerState,
                 trainer.py:93-124) and the per-node step count of a node in
                 one 576-B record
  LoD tables     DeviceLodScene (means/scales read at the record stride)
  cache blocks   one packed f64 block per resident SPT prefix (DeviceCache)
Host: the pinned f32 store (HostStore), cache metadata, scheduler RNG.

One step = scheduler draw → LoD select (K2) → cache decisions on the host
(one small D2H) → H2D of missed prefixes + f32→f64 upcast → SPT compaction
at the cached distances (K1) → render-row gather (K4) → rasterise (K5-K7)
→ L1+SSIM (K10) → backward (K8/K9) → ADAM on the touched nodes (K11) →
cache blocks refreshed from the master rows → periodic flush.  Every
counter the reference returns is reproduced exactly.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .cache import CacheConfig, NativeCache
from .core import BYTES_PER_GAUSSIAN_F32, FLOATS_PER_GAUSSIAN, SECTIONS, AttributeArrays, Camera, LodConfig
from .device import DeviceLodScene
from .renderer import Rasterizer
from .scheduler import DEFAULT_K, DEFAULT_RANDOM_EVERY, build_view_graph, next_view
from .hierarchy import Hierarchy
from .store import HostStore

DEFAULT_LEARNING_RATES = {
    "means": 1.6e-4,        # × scene extent
    "scales": 5e-3,
    "rotations": 1e-3,
    "opacities": 5e-2,
    "base_colors": 2.5e-3,
    "sh_rest": 2.5e-3 / 20.0,
}


class NonFiniteLossError(RuntimeError):
    pass


@dataclass
class TrainConfig:
    """Subset of trainer.TrainConfig (trainer.py:64-90) the step uses."""

    total_iterations: int = 1
    init_iterations: int = 2000
    loss_lambda: float = 0.2
    learning_rates: dict = field(default_factory=lambda: dict(DEFAULT_LEARNING_RATES))
    lod: LodConfig = field(default_factory=lambda: LodConfig(threshold=1.0))
    cache: CacheConfig = field(default_factory=lambda: CacheConfig(budget_bytes=64 << 20))
    scheduler_k: int = DEFAULT_K
    scheduler_exploration: float | None = None
    scheduler_random_every: int = DEFAULT_RANDOM_EVERY
    seed: int = 0
    # copy-engine prefetch of the scheduler's next view's cache misses
    # (not in the reference; decisions and counters are unchanged)
    prefetch: bool = True
    # where the f32 scene store lives: "host" (pinned DRAM, out-of-core) or
    # "device" (HBM, config C2 — fully device-resident)
    store_location: str = "host"
    # densification schedule (trainer.py:68-70)
    densify_interval: int = 500
    dead_opacity_threshold: float = 0.005
    spawns_per_densify: int | None = None   # None -> 0.5% of leaf count
    skybox_points: int = 0                  # initialize() only (host)
    size_threshold: float | None = None     # initialize() only (host)
    min_subtree: int = 32                   # hspt.DEFAULT_MIN_SUBTREE
    # the rasteriser reads the render rows in place through the gather plan
    # (glod_render_forward_plan) instead of a K4-gathered packed copy; the
    # values, image and gradients are the same (not in the reference)
    fuse_gather: bool = True
    # render_view(view, next_view): the next frame's LoD select is enqueued
    # between this frame's tile sort and its blend, so the next call's cache
    # decisions run on the host while this blend runs (not in the reference;
    # images and counters unchanged)
    pipeline_render: bool = True

    def __post_init__(self):
        for name, lr in self.learning_rates.items():
            if not lr > 0:
                raise ValueError(f"learning rate for {name} must be > 0")


def _packed(t: torch.Tensor, rows: int, name: str) -> torch.Tensor:
    off = 0
    for n, cols in SECTIONS:
        if n == name:
            return t[off * rows:(off + cols) * rows]
        off += cols
    raise KeyError(name)


NODE_RECORD, REC_MV, REC_STEP = 72, 24, 70     # glod_b200.h GLOD_NODE_RECORD layout


class DeviceScene:
    """Master params + ADAM state + LoD tables + host store for one HSPT.

    The master state is one 576-B node record per node (GLOD_NODE_RECORD,
    glod_b200.h): 23 attribute values, 23 (m, v) moment pairs and the step
    count, so ADAM moves whole records.  `params`, `mv` and `step` give the
    reference-shaped views (packed section-major params, [cap][23][m, v]
    moments, int64 steps)."""

    def __init__(self, h, hspt, device=None, store_location: str = "host", store: HostStore | None = None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.cap = h.capacity
        # records assembled on the device one section at a time (no host copy
        # of the 576-B/node table: 69 GB at C5)
        self.records = torch.zeros((self.cap, NODE_RECORD), dtype=torch.float64, device=dev)
        off = 0
        for name, cols in SECTIONS:
            a = np.ascontiguousarray(getattr(h.attrs, name), dtype=np.float64).reshape(self.cap, cols)
            self.records[:, off:off + cols] = torch.from_numpy(a).to(dev)
            off += cols
        self.lod = DeviceLodScene(h, hspt, means=self.records.view(-1), scales=self.records.view(-1)[3:],
                                  attr_stride=NODE_RECORD)
        # a prebuilt store (e.g. scenefile.Scene.host_store: sections read from
        # a .glod file straight into pinned memory) or one built from h.attrs
        self.store = store if store is not None else HostStore(h, hspt, location=store_location)
        self.hspt = hspt

    @property
    def params(self) -> torch.Tensor:
        """Packed section-major copy of the attribute values (h.attrs layout)."""
        parts, off = [], 0
        for _, cols in SECTIONS:
            parts.append(self.records[:, off:off + cols].reshape(-1))
            off += cols
        return torch.cat(parts)

    @property
    def mv(self) -> torch.Tensor:
        """ADAM moments [cap][23][m, v] (a copy)."""
        return self.records[:, REC_MV:REC_MV + 2 * FLOATS_PER_GAUSSIAN].reshape(-1)

    @property
    def step(self) -> torch.Tensor:
        return self.records.view(torch.int64)[:, REC_STEP].contiguous()

    def moments_packed(self):
        """(m, v) as packed section-major f64 blocks (the h.attrs layout)."""
        mv = self.records[:, REC_MV:REC_MV + 2 * FLOATS_PER_GAUSSIAN].reshape(self.cap, FLOATS_PER_GAUSSIAN, 2)
        out = []
        for k in range(2):
            x = mv[:, :, k]
            parts, off = [], 0
            for _, cols in SECTIONS:
                parts.append(x[:, off:off + cols].reshape(-1))
                off += cols
            out.append(torch.cat(parts))
        return out[0], out[1]

    def attrs_host(self) -> AttributeArrays:
        return AttributeArrays.from_packed(self.params.cpu().numpy(), self.cap)


class Trainer:
    """The per-GPU training engine.  `views` is a list of (Camera, target)
    with targets (h, w, 3) float images (numpy or pinned torch)."""

    def __init__(self, h, hspt, views, cfg: TrainConfig, extent: float, device_targets: bool = True,
                 group=None, store=None, graph=None, rng=None):
        import torch.distributed as dist
        self.cfg = cfg
        # view sharding: with an initialised process group of >1 ranks each
        # step's gradients are summed over ranks on the union of touched
        # nodes and ADAM runs owner-sharded (parallel.py, csrc/exchange.cu)
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized() and \
            dist.get_world_size(group) > 1
        self.hierarchy = Hierarchy.from_any(h)        # host topology (attrs live on the device)
        self.scene = DeviceScene(h, hspt, store_location=cfg.store_location, store=store)
        dev = self.scene.device
        self.cache = NativeCache(cfg.cache, self.scene.store)
        self._register_master()
        self.rast = Rasterizer()
        # SPT render rows from the master records instead of the cache
        # blocks: required when ranks share updates (the replicated records
        # are authoritative); selectable on one GPU for comparisons
        self.spt_from_master = self.distributed
        if self.distributed:
            from .parallel import make_exchange
            self.xchg = make_exchange(self.scene.cap, group)
        self.views = [(Camera.from_any(c), t) for c, t in views]
        pos = np.stack([c.position for c, _ in self.views])
        # the drop-in (train_step(state, it)) passes the reference state's own
        # view graph and RNG, so the draw sequence advances the caller's RNG
        self.graph = graph if graph is not None else build_view_graph(
            pos, k=cfg.scheduler_k, exploration=cfg.scheduler_exploration,
            random_every=cfg.scheduler_random_every)
        self.rng = rng if rng is not None else np.random.default_rng(cfg.seed)
        self.current_view = 0
        self.iteration = 0
        self.extent = float(extent)
        lrs = dict(cfg.learning_rates)
        lrs["means"] = lrs["means"] * self.extent
        self.lrs = (C.c_double * 6)(*[float(lrs[n]) for n, _ in SECTIONS])
        # targets: device-resident f32, or pinned host copied every step (e2e)
        self.device_targets = device_targets
        self.targets = []
        for _, t in self.views:
            tt = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
            tt = tt.to(torch.float32)
            self.targets.append(tt.to(dev) if device_targets else tt.pin_memory())
        self._scene_buffers()
        self._h_total = torch.empty(2, dtype=torch.int64).pin_memory()
        self._h_loss = torch.empty(3, dtype=torch.float64).pin_memory()
        self._rows = None
        self._row_node = None
        self._grads = None
        self._bias = None
        self._bias_len = 0
        self._target_dev = None
        self.last_stats = {}
        self._pf_rows_cap = cfg.cache.budget_bytes // BYTES_PER_GAUSSIAN_F32
        self.timing = None          # {stage: [ms, ...]} when profiling is on
        self.host_timing = None     # {stage: [host ms, ...]} (enable_host_timing)
        self._host_last = None
        self._ev = []

    def _register_master(self):
        """Implicit block refresh: the cache materialises touched rows from
        the node records before writing blocks back (glod_cache_set_master)."""
        sc = self.scene
        if sc.lod.S:
            self.cache.set_master(sc.records, sc.cap, NODE_RECORD, sc.lod.rec_node, sc.lod.rec_offset_by_sid)

    def _scene_buffers(self):
        """Per-HSPT host/device tables (rebuilt after densification)."""
        dev = self.scene.device
        S1 = max(self.scene.lod.S, 1)
        self._h_sel = torch.empty(4 + 4 * S1, dtype=torch.int32).pin_memory()   # counts | ids | prefix
        self._h_droot = torch.empty(S1, dtype=torch.float64).pin_memory()
        self._h_dist = torch.empty(S1, dtype=torch.float64).pin_memory()
        self._h_blk = torch.empty(2 * S1, dtype=torch.int64).pin_memory()       # ptr | rows
        self._d_dist = torch.empty(S1, dtype=torch.float64, device=dev)
        self._d_blk = torch.empty(2 * S1, dtype=torch.int64, device=dev)
        self._h_pref = torch.empty(S1, dtype=torch.int32).pin_memory()
        self._d_pref = torch.empty(S1, dtype=torch.int32, device=dev)
        # prefetch: last selection per view (host) and the predicted next view
        self._hist = {}
        self._next_view = None
        self._pred = None
        self._spec = None
        self._sel_ev = self._spec_ev = None
        self._h_sel2 = torch.empty(4 + 4 * S1, dtype=torch.int32).pin_memory()
        self._h_droot2 = torch.empty(S1, dtype=torch.float64).pin_memory()
        self._presel = None                  # (view, SelectResult) enqueued by render_view
        self._pipelined = False
        self._spt_of_node = None

    def train(self, metrics_out=None) -> list:
        """trainer.train (trainer.py:446-458): train_step for every iteration
        up to cfg.total_iterations, densify every densify_interval."""
        import json
        records = []
        for it in range(self.iteration + 1, self.cfg.total_iterations + 1):
            rec = self.train_step(it)
            if it % self.cfg.densify_interval == 0 and it < self.cfg.total_iterations:
                rec.update(self.densify(self.cfg.dead_opacity_threshold, self.cfg.spawns_per_densify))
            records.append(rec)
            if metrics_out is not None:
                metrics_out.write(json.dumps(rec) + "\n")
        return records

    # -- densification (trainer.densify, trainer.py:411-443) -------------------
    def densify(self, dead_opacity_threshold: float = 0.005, spawns_per_densify: int | None = None) -> dict:
        """Respawn dead leaves, spawn opacity-sampled leaves (host tree
        surgery, densify.py, on the scheduler RNG like the reference), zero
        the new nodes' moments, rebuild the HSPT on the device with the
        surface-area metric (hspt.py:161-165) and re-lay the store and the
        node records out for it (_sync_scene, trainer.py:395-408: the store
        is rewritten from the authoritative master values, the cache starts
        empty, byte counters survive)."""
        from .densify import Moments, densify_tree
        from .hspt import build_hspt
        if self.distributed:
            # the ranks' moments live with their owners and the tree surgery
            # draws on the scheduler RNG, which differs per rank: a sharded
            # densify would give every rank a different hierarchy
            raise NotImplementedError("densify in view-sharded training: gather the state on one rank "
                                      "(sync_state) and densify there")
        torch.cuda.synchronize()
        sc, h = self.scene, self.hierarchy
        rec = sc.records.cpu().numpy()
        F = FLOATS_PER_GAUSSIAN

        def unpack(cols_of_rec):
            parts, off = [], 0
            for _, c in SECTIONS:
                parts.append(cols_of_rec[:, off:off + c] if c > 1 else cols_of_rec[:, off].copy())
                off += c
            return AttributeArrays(*[np.ascontiguousarray(p) for p in parts])

        h.attrs = unpack(rec[:, :F])
        mv = rec[:, REC_MV:REC_MV + 2 * F].reshape(-1, F, 2)
        opt = Moments(unpack(mv[:, :, 0]), unpack(mv[:, :, 1]), rec.view(np.int64)[:, REC_STEP].copy())
        del rec, mv
        out = densify_tree(h, opt, self.rng, dead_opacity_threshold, spawns_per_densify)
        old = sc.hspt
        hs = build_hspt(h, old.size_threshold, old.min_subtree, LodConfig(old.lod.threshold, "surface_area"))
        consumed = sc.store.attribute_bytes_read
        location = sc.store.location
        self.cache = None
        self.scene = None
        sc = None
        torch.cuda.empty_cache()
        self.scene = DeviceScene(h, hs, store_location=location)
        self.scene.store.attribute_bytes_read = consumed
        recs = self.scene.records
        for k, blk in enumerate((opt.m, opt.v)):
            cols = np.concatenate([np.asarray(a, dtype=np.float64).reshape(h.capacity, -1) for _, a in blk.arrays()],
                                  axis=1)
            recs[:, REC_MV + k:REC_MV + 2 * F:2] = torch.from_numpy(cols).to(recs.device)
        recs.view(torch.int64)[:, REC_STEP] = torch.from_numpy(opt.step).to(recs.device)
        self.cache = NativeCache(self.cfg.cache, self.scene.store)
        self._register_master()
        self._scene_buffers()
        return out

    # -- optimizer state in / cache flush (drop-in train_step) ----------------
    def load_optimizer(self, opt) -> None:
        """ADAM moments and per-node steps from an OptimizerState
        (trainer.py:93-124; dict- or attribute-keyed) into the node records."""
        recs = self.scene.records
        for k, blk in enumerate((opt.m, opt.v)):
            c = np.concatenate([_moment(blk, n).reshape(self.scene.cap, -1) for n, _ in SECTIONS], axis=1)
            recs[:, REC_MV + k:REC_MV + 2 * FLOATS_PER_GAUSSIAN:2] = torch.from_numpy(c).to(recs.device)
        recs.view(torch.int64)[:, REC_STEP] = torch.from_numpy(
            np.ascontiguousarray(opt.step, dtype=np.int64)).to(recs.device)

    def flush_cache(self) -> None:
        """Write every dirty resident block back to the store and empty the
        cache (the reference's flush, cache.py:98-106)."""
        self.cache.end_step(0, mark_dirty=False)
        self.cache.flush_io()               # disk store: write-backs reach the file

    # -- optional per-stage CUDA-event timing (bench.py) ---------------------
    def enable_timing(self, on: bool = True):
        self.timing = {} if on else None

    def _mark(self, name):
        if self.timing is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self._ev.append((name, e))
        if self.host_timing is not None:
            import time
            t = time.perf_counter()
            if self._host_last is not None and name != "start":
                self.host_timing.setdefault(name, []).append((t - self._host_last) * 1e3)
            self._host_last = t

    def _collect(self):
        if self.timing is None or not self._ev:
            return
        torch.cuda.current_stream().synchronize()
        for (a, ea), (b, eb) in zip(self._ev[:-1], self._ev[1:]):
            self.timing.setdefault(b, []).append(ea.elapsed_time(eb))
        self._ev = []

    # ------------------------------------------------------------------
    def _bias_table(self, iteration: int):
        """1-β^t for every step count a node can have after this iteration,
        computed with numpy's power exactly like the reference
        (trainer.py:261-263); grown by doubling."""
        need = iteration + 2
        if self._bias is None or self._bias_len < need:
            n = max(1024, 2 * need)
            t = np.arange(n, dtype=np.float64)
            tab = np.concatenate([1.0 - 0.9 ** t, 1.0 - 0.999 ** t])
            self._bias = torch.from_numpy(tab).to(self.scene.device)
            self._bias_len = n
        return self._bias, self._bias_len

    def _ensure(self, name, numel, dtype):
        t = getattr(self, name)
        if t is None or t.numel() < numel:
            grow = 2 * t.numel() if t is not None else 0
            t = torch.empty(max(numel + numel // 4, grow, 1), dtype=dtype, device=self.scene.device)
            setattr(self, name, t)
        return t

    # ------------------------------------------------------------------
    def select(self, cam: Camera, spec_cam: Camera | None = None, pre=None):
        """LoD select + one D2H of the per-SPT table (the step's host sync).
        With `spec_cam`, a speculative select of that (predicted next) view
        is enqueued after the read-back the host waits for, so it runs on
        the GPU while the host makes this step's cache decisions; its
        per-SPT table is read later (`_spec_table`, before the prefetch)."""
        sc = self.scene
        S1 = max(sc.lod.S, 1)
        if pre is not None:
            # enqueued by the previous frame (_preselect): alternate buffers
            sel = pre
            self._spec_ev.synchronize()
            self._spec = None
            h, hd = self._h_sel2, self._h_droot2
        else:
            sel = sc.lod.select(cam, self.cfg.lod, cull=True, frustum=self._frustum(cam))
            self._read_select(sel, self._h_sel, self._h_droot)
            if self._sel_ev is None:
                self._sel_ev, self._spec_ev = torch.cuda.Event(), torch.cuda.Event()
            self._sel_ev.record()
            self._spec = None
            if spec_cam is not None:
                self._read_select(sc.lod.select(spec_cam, self.cfg.lod, cull=True, alt=True,
                                                frustum=self._frustum(spec_cam)), self._h_sel2, self._h_droot2)
                self._spec_ev.record()
                self._spec = "pending"
            self._sel_ev.synchronize()
            h, hd = self._h_sel, self._h_droot
        n_up, n_pa, n_sp = (int(x) for x in h[:3].tolist())
        dev_ids = h[4:4 + n_sp].numpy().astype(np.int64)
        return sel, n_up, n_pa, n_sp, dev_ids, h[4 + S1:4 + S1 + n_sp].numpy(), hd[:n_sp].numpy()

    def _read_select(self, sel, h, hd):
        """Kernel-written read-back of a select's per-SPT table (never queues
        behind the write-back DMA)."""
        S1 = max(self.scene.lod.S, 1)
        _lib.readback_multi([(h[:4], sel.counts[:4]), (h[4:4 + S1], sel.spt_ids[:S1]),
                             (h[4 + S1:4 + 2 * S1], sel.prefix_len[:S1]), (hd, sel.d_root[:S1])])

    def _preselect(self, view: int):
        """Enqueue the LoD select of the next frame's view into the alternate
        device/host buffers (read by that frame's `select` and, before it,
        by the prefetch through `_spec_table`)."""
        sc = self.scene
        cam = self.views[view][0]
        sel = sc.lod.select(cam, self.cfg.lod, cull=True, alt=True, frustum=self._frustum(cam))
        self._read_select(sel, self._h_sel2, self._h_droot2)
        if self._sel_ev is None:
            self._sel_ev, self._spec_ev = torch.cuda.Event(), torch.cuda.Event()
        self._spec_ev.record()
        self._spec = "pending"
        self._presel = (view, sel)

    def _frustum(self, cam: Camera):
        """Frustum.from_camera, memoised per camera (the host BLAS calls cost
        ~0.2 ms per select; a run's views repeat)."""
        cache = getattr(self, "_frusta", None)
        if cache is None:
            cache = self._frusta = {}
        # keyed on everything the planes depend on (Camera is mutable)
        key = (np.asarray(cam.position, dtype=np.float64).tobytes(),
               np.asarray(cam.orientation, dtype=np.float64).tobytes(), tuple(cam.focal),
               tuple(cam.principal_point), tuple(cam.resolution), float(cam.near), float(cam.far))
        fr = cache.get(key)
        if fr is None:
            from .core import Frustum
            fr = cache[key] = Frustum.from_camera(cam)
            if len(cache) > 4096:
                cache.pop(next(iter(cache)))
        return fr

    def _spec_table(self):
        """The speculative select's per-SPT table (spt ids, d_root,
        prefix), read back behind this step's select (select())."""
        if isinstance(self._spec, str):
            self._spec_ev.synchronize()
            S1 = max(self.scene.lod.S, 1)
            h2 = self._h_sel2
            k = int(h2[2])
            self._spec = (self.scene.lod.spt_perm[h2[4:4 + k].numpy().astype(np.int64)],
                          self._h_droot2[:k].numpy().copy(), h2[4 + S1:4 + S1 + k].numpy().copy())
        return self._spec

    def _prefetch_next(self):
        """Copy-engine prefetch of the predicted next view's misses."""
        pred = self._pred
        if pred is None:
            return
        if isinstance(pred, str):
            pred = self._spec_table()
        if pred is not None:
            self.cache.prefetch(*pred, max_rows=self._pf_rows_cap)

    def _predict_next(self, iteration: int):
        """The scheduler's draw for iteration+1, from a copy of the RNG
        (the real sequence is untouched)."""
        g = np.random.Generator(type(self.rng.bit_generator)())
        g.bit_generator.state = self.rng.bit_generator.state
        return next_view(self.graph, self.current_view, iteration + 1, g)

    def _gather_view(self, cam: Camera, view: int | None = None):
        """Cut + cache decisions + prefix loads + compaction + row gather
        (trainer.py:319-347, cli._gather cli.py:111-136)."""
        sc = self.scene
        self._mark("start")
        nv = self._next_view
        pre, self._presel = self._presel, None
        pre = pre[1] if pre is not None and pre[0] == view else None
        spec_cam = self.views[nv][0] if (nv is not None and nv != view and nv not in self._hist
                                         and not self._pipelined) else None
        sel, n_up, n_pa, n_sp, dev_ids, prefix, d_root = self.select(cam, spec_cam, pre=pre)
        self._mark("select")
        spt_ids = sc.lod.spt_perm[dev_ids]
        S1 = max(sc.lod.S, 1)
        hd, hb = self._h_dist.numpy(), self._h_blk.numpy()
        loaded, hits = self.cache.step(spt_ids, d_root, prefix, hd, hb[:S1], hb[S1:])
        if view is not None:
            self._hist[view] = (spt_ids.copy(), d_root.copy(), prefix.copy())
        # the next view's predicted selection: its misses are prefetched by
        # the copy engines once this step's backward is queued (train_step)
        # or its frame is rendered (render_view)
        self._pred = self._hist.get(nv, self._spec) if nv is not None else None   # "pending": spec
        if self._pipelined and self._pred is not None and not isinstance(self._pred, str):
            # render with a known next view: its misses start copying now,
            # under this whole frame rather than only its blend
            self._prefetch_next()
            self._pred = None
        if n_sp:
            # the prefix at the cached distance is the entry's prefix_len
            self._h_pref.numpy()[:n_sp] = hb[S1:S1 + n_sp]
            # kernel uploads: the H2D copy engine is busy with the prefetch
            _lib.upload(self._d_dist, self._h_dist)
            _lib.upload(self._d_blk, self._h_blk)
            _lib.upload(self._d_pref, self._h_pref)
        self._mark("cache")
        cmp = sc.lod.compact(sel.counts[2:3], sel.spt_ids, self._d_dist, known_prefix=self._d_pref)
        _lib.readback(self._h_total[:1], cmp.total[:1])
        torch.cuda.current_stream().synchronize()
        self._mark("compact")
        n_sel = int(self._h_total[0])
        R = n_up + n_pa + n_sel
        rows = None if self.cfg.fuse_gather else \
            self._ensure("_rows", FLOATS_PER_GAUSSIAN * R, torch.float64)[:FLOATS_PER_GAUSSIAN * R]
        row_node = self._ensure("_row_node", R, torch.int32)[:max(R, 1)]
        plan = _lib.GatherPlan(
            master=_lib.ptr(sc.records), capacity=sc.cap, upper_ids=_lib.ptr(sel.upper),
            pass_ids=_lib.ptr(sel.passthrough), n_upper=n_up, n_pass=n_pa,
            sel_seg=_lib.ptr(cmp.sel_seg), sel_pos=_lib.ptr(cmp.sel_pos), sel_node=_lib.ptr(cmp.sel_node),
            n_sel=n_sel, seg_block=_lib.ptr(self._d_blk), seg_rows=_lib.ptr(self._d_blk[S1:]),
            master_stride=NODE_RECORD, spt_from_master=int(self.spt_from_master))
        self._plan, self._plan_R = plan, R
        if self.cfg.fuse_gather:
            rows = None          # the forward reads the rows through the plan
        else:
            _lib.check(_lib.lib().glod_gather_render_rows(C.byref(plan), _lib.ptr(rows), _lib.ptr(row_node),
                                                          _lib.stream_ptr()))
        self._mark("gather")
        self.last_stats = {"n_upper": n_up, "n_pass": n_pa, "n_spt": n_sp,
                           "prefix_total": int(prefix.sum()) if n_sp else 0}
        counters = {"gaussians_rendered": int(R), "gaussians_loaded_from_store": int(loaded),
                    "cache_hits": int(hits),
                    "bytes_streamed": int(loaded * sc.store.bytes_per_gaussian)}
        return R, rows, row_node, plan, None, counters

    def _forward(self, rows, row_node, plan, R: int, cam: Camera, image: torch.Tensor | None = None):
        if rows is None:
            return self.rast.forward_plan(plan, row_node, R, cam, image=image)
        return self.rast.forward(rows, R, cam, image=image)

    def gathered_rows(self) -> torch.Tensor:
        """Packed f64 render rows of the last view (K4 gather of its plan,
        23·R values) — what the rasteriser read.  After a train step the
        plan's sources hold the updated parameters."""
        R = self._plan_R
        rows = self._ensure("_rows", FLOATS_PER_GAUSSIAN * max(R, 1), torch.float64)
        row_node = self._ensure("_row_node", max(R, 1), torch.int32)
        _lib.check(_lib.lib().glod_gather_render_rows(C.byref(self._plan), _lib.ptr(rows), _lib.ptr(row_node),
                                                      _lib.stream_ptr()))
        return rows[:FLOATS_PER_GAUSSIAN * R]

    def render_view(self, view: int, image: torch.Tensor | None = None,
                    next_view: int | None = None) -> torch.Tensor:
        """Serve/bench path (cli.cmd_render, cli.py:139-189): cut + cache +
        gather + forward render of one view; no parameter updates.  With
        `next_view` (a camera path known one frame ahead) the copy engines
        prefetch that view's cache misses while this frame renders, as the
        training step does for the scheduler's next draw; decisions and
        counters are unchanged."""
        cam, _ = self.views[view]
        self._next_view = next_view if self.cfg.prefetch else None
        pipe = self.cfg.pipeline_render and next_view is not None and next_view != view
        self._pipelined = pipe
        try:
            R, rows, row_node, plan, _, counters = self._gather_view(cam, view)
        finally:
            self._pipelined = False
        if pipe:
            # this frame up to its tile sort, the next frame's select, then
            # this frame's blend: the next call's cache decisions overlap it
            self.rast.defer_blend(True)
            try:
                img = self._forward(rows, row_node, plan, R, cam, image=image)
            finally:
                self.rast.defer_blend(False)
            self._preselect(next_view)
            self.rast.blend()
            if self.cfg.prefetch and next_view not in self._hist:
                self._pred = "pending"          # the preselect's table (_spec_table)
        else:
            img = self._forward(rows, row_node, plan, R, cam, image=image)
        self.cache.end_step(-1, mark_dirty=False)
        self._prefetch_next()
        self._mark("forward")
        self._collect()
        self.last_render = counters
        return img

    def _upload_target(self, target: torch.Tensor):
        """Host (pinned) target → device on a side stream, double-buffered:
        the copy overlaps this step's cut, gather and forward render; the
        loss waits for it (event).  A buffer is refilled only after the
        loss that read it two steps ago."""
        dev = self.scene.device
        if getattr(self, "_tgt_bufs", None) is None or self._tgt_bufs[0].shape != target.shape:
            self._tgt_bufs = [torch.empty(target.shape, dtype=target.dtype, device=dev) for _ in range(2)]
            self._tgt_stream = torch.cuda.Stream(device=dev)
            self._tgt_used = [torch.cuda.Event(), torch.cuda.Event()]
            self._tgt_done = [torch.cuda.Event(), torch.cuda.Event()]
            self._tgt_slot = 1
        k = self._tgt_slot = 1 - self._tgt_slot
        with torch.cuda.stream(self._tgt_stream):
            self._tgt_stream.wait_event(self._tgt_used[k])
            self._tgt_bufs[k].copy_(target, non_blocking=True)
            self._tgt_done[k].record()
        self._target_dev = self._tgt_bufs[k]
        return self._tgt_bufs[k], self._tgt_done[k]

    def train_step(self, iteration: int) -> dict:
        cfg, sc = self.cfg, self.scene
        self.current_view = next_view(self.graph, self.current_view, iteration, self.rng)
        self._next_view = self._predict_next(iteration) if cfg.prefetch else None
        cam, _ = self.views[self.current_view]
        target = self.targets[self.current_view]
        tgt_ready = None
        if not self.device_targets:
            target, tgt_ready = self._upload_target(target)
        R, rows, row_node, plan, _, counters = self._gather_view(cam, self.current_view)
        L = _lib.lib()
        st = _lib.stream_ptr()
        image = self._forward(rows, row_node, plan, R, cam)
        self._mark("forward")
        if tgt_ready is not None:
            torch.cuda.current_stream().wait_event(tgt_ready)
        value, dimg = self.rast.loss(image, target, cfg.loss_lambda)
        if tgt_ready is not None:
            self._tgt_used[self._tgt_slot].record()
        self._mark("loss")
        _lib.readback(self._h_loss[:value.numel()], value)
        if getattr(self, "_loss_ev", None) is None:
            self._loss_ev = torch.cuda.Event()
        self._loss_ev.record()
        # the backward is enqueued before the host waits for the loss: the
        # non-finite check (trainer.py:360-367) only has to precede ADAM, the
        # first write to the parameters
        grads = self.rast.backward(dimg, self._ensure("_grads", FLOATS_PER_GAUSSIAN * max(R, 1), torch.float64))
        self._mark("backward")
        # the copy engines fetch the next view's misses during the backward
        # and ADAM; issued here, where the host would only wait
        self._prefetch_next()
        self._loss_ev.synchronize()
        loss_value = float(self._h_loss[0])
        if not np.isfinite(loss_value):
            raise NonFiniteLossError(f"iteration {iteration}: non-finite loss rendering view "
                                     f"{self.current_view} with {R} gaussians")
        bias, blen = self._bias_table(iteration)
        if self.distributed:
            # sparse exchange: owner sums + owner-sharded ADAM + replication
            # of the updated rows (parallel.py)
            self.xchg.reduce(row_node[:max(R, 1)], grads, R)
            self._mark("exchange")
            ids, G, n_own = self.xchg.owned()
            _lib.check(L.glod_adam_step_records(_lib.ptr(sc.records), sc.cap, _lib.ptr(ids), _lib.ptr(G),
                                                None, n_own, n_own, self.lrs, _lib.ptr(bias), blen, None, st))
            self._mark("adam")
            self.xchg.allgather_params(sc.records, NODE_RECORD)
            self._mark("replicate")
        else:
            _lib.check(L.glod_adam_step_records(_lib.ptr(sc.records), sc.cap, _lib.ptr(row_node),
                                                _lib.ptr(grads), None, R, R, self.lrs, _lib.ptr(bias), blen,
                                                C.byref(plan), st))
            self._mark("adam")
        self.cache.end_step(iteration, mark_dirty=True)
        self._mark("scatter_flush")
        self._collect()
        self.iteration = iteration
        self.last_stats["n_instances"] = self.rast.stats()["n_instances"]
        self._last_grads = grads
        self._last_image = image
        self._last_rows = row_node[:R]
        out = {"iteration": iteration, "view": self.current_view, "loss": loss_value}
        out.update(counters)
        return out


# ---------------------------------------------------------------------------
# Drop-in at the reference's signature: train_step(state, iteration)
# ---------------------------------------------------------------------------
@dataclass
class OptimizerState:
    """trainer.OptimizerState (trainer.py:93-124): per-node ADAM moments
    mirroring every attribute array, plus per-node step counts."""

    m: dict
    v: dict
    step: np.ndarray

    @staticmethod
    def zeros(attrs) -> "OptimizerState":
        m = {n: np.zeros_like(np.asarray(getattr(attrs, n), dtype=np.float64)) for n, _ in SECTIONS}
        v = {n: np.zeros_like(np.asarray(getattr(attrs, n), dtype=np.float64)) for n, _ in SECTIONS}
        return OptimizerState(m=m, v=v, step=np.zeros(len(attrs), dtype=np.int64))


@dataclass
class TrainState:
    """trainer.TrainState (trainer.py:127-146), field for field.  The
    reference's own TrainState objects are accepted as well (duck-typed)."""

    config: TrainConfig
    hierarchy: object
    hspt: object
    scene: object
    cache: object
    graph: object
    views: list
    opt: OptimizerState
    rng: np.random.Generator
    extent: float
    skybox_ids: np.ndarray
    current_view: int = 0
    iteration: int = 0

    @property
    def mean_lr(self) -> float:
        return self.config.learning_rates["means"] * self.extent


def _config_of(c) -> TrainConfig:
    """Our TrainConfig from a reference (or our own) TrainConfig."""
    if isinstance(c, TrainConfig):
        return c
    cc = c.cache
    return TrainConfig(
        total_iterations=c.total_iterations, init_iterations=c.init_iterations, loss_lambda=c.loss_lambda,
        learning_rates=dict(c.learning_rates), lod=LodConfig(float(c.lod.threshold), c.lod.metric),
        cache=CacheConfig(budget_bytes=cc.budget_bytes, d_min=cc.d_min, d_max=cc.d_max,
                          flush_interval=cc.flush_interval),
        scheduler_k=c.scheduler_k, scheduler_exploration=c.scheduler_exploration,
        scheduler_random_every=c.scheduler_random_every, seed=c.seed, densify_interval=c.densify_interval,
        dead_opacity_threshold=c.dead_opacity_threshold, spawns_per_densify=c.spawns_per_densify,
        skybox_points=c.skybox_points, size_threshold=c.size_threshold, min_subtree=c.min_subtree)


def _moment(blk, name):
    return np.asarray(blk[name] if isinstance(blk, dict) else getattr(blk, name), dtype=np.float64)


def _flush_host_cache(state):
    """A warm reference cache is flushed into its store first (the device
    cache starts empty): dirty blocks written back in LRU order, exactly
    what the reference's tick_and_maybe_flush does at a flush."""
    cache = state.cache
    entries = getattr(cache, "entries", None)
    if entries:
        for e in list(entries.values()):
            if e.dirty:
                state.scene.write_back(e.block)
        entries.clear()
        cache.resident_bytes = 0


def _trainer_of(state) -> "Trainer":
    tr = getattr(state, "_device_trainer", None)
    if tr is not None and tr._state_key == (id(state.hspt), id(state.scene)):
        return tr
    from .hspt import Hspt
    _flush_host_cache(state)
    h, hs = Hierarchy.from_any(state.hierarchy), Hspt.from_any(state.hspt)
    store = HostStore.from_scene(state.scene)
    tr = Trainer(h, hs, state.views, _config_of(state.config), extent=float(state.extent), store=store,
                 graph=state.graph, rng=state.rng)
    tr.current_view, tr.iteration = int(state.current_view), int(state.iteration)
    tr.load_optimizer(state.opt)
    tr._state_key = (id(state.hspt), id(state.scene))
    state._device_trainer = tr
    return tr


def train_step(state, iteration: int) -> dict:
    """trainer.train_step(state, iteration) (trainer.py:312-378) on the
    device.  The first call uploads the state (hierarchy values, ADAM
    moments and steps, the scene store; a warm host cache is flushed into
    the store first) into a per-state device Trainer; later calls only run
    steps.  The scheduler draws advance `state.rng` itself, and
    `state.current_view` / `state.iteration` follow the reference.  The
    device is authoritative for parameters, moments, store and cache:
    `sync_state(state)` copies them back (a cache flush point, like
    save_checkpoint's, trainer.py:464-465) before host code reads
    `state.hierarchy.attrs`, `state.opt` or the scene."""
    tr = _trainer_of(state)
    out = tr.train_step(iteration)
    state.current_view, state.iteration = tr.current_view, iteration
    return out


def sync_state(state) -> None:
    """Device → reference state: flush the device cache (dirty blocks written
    back to the store), then copy the master attribute values into
    `state.hierarchy.attrs`, the moments/steps into `state.opt` and the
    store sections into `state.scene`'s backing."""
    tr = getattr(state, "_device_trainer", None)
    if tr is None:
        return
    tr.flush_cache()
    torch.cuda.synchronize()
    sc = tr.scene
    rec = sc.records.cpu().numpy()
    off = 0
    h = state.hierarchy
    for name, cols in SECTIONS:
        vals = rec[:, off:off + cols]
        getattr(h.attrs, name)[...] = vals.reshape(getattr(h.attrs, name).shape)
        for k, blk in enumerate((state.opt.m, state.opt.v)):
            mv = rec[:, REC_MV + 2 * off + k:REC_MV + 2 * (off + cols):2]
            if isinstance(blk, dict):
                blk[name][...] = mv.reshape(blk[name].shape)
            else:
                getattr(blk, name)[...] = mv.reshape(getattr(blk, name).shape)
        off += cols
    state.opt.step[...] = rec.view(np.int64)[:, REC_STEP]
    sc.store.to_scene(state.scene)
