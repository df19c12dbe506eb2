"""Seeded synthetic scenes for tests and benchmarks (host tooling).

The reference's LoD metric m_d = T / max(s) grows toward the leaves of a
moment-matched hierarchy, which makes every view cut degenerate to the root
(SURVEY §0.4).  Non-trivial cuts need node scales decoupled from depth, as
in the reference's own stress fixture `random_scale_hierarchy`
(pkg/tests/conftest.py:26-31).  `designed_scene` builds that shape at any
size:

  * leaves: a city-like slab of Gaussians (x, z ∈ ±extent, y ∈ [0, height])
  * hierarchy: median split + moment-matched merges (hierarchy.build_hierarchy)
  * upper tree (depth < D): tiny isotropic scales, so m_d > any view distance
    and the upper BFS always descends to the cut (never "taken")
  * cut roots (depth D, or deeper for a fraction of branches that end up as
    passthrough subtrees): slightly smaller scales so the volume-threshold
    partition of build_hspt cuts exactly there
  * everything below: i.i.d. log-uniform per-axis scales, so SPT selections
    and passthrough cuts are non-trivial at typical view distances.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .core import AttributeArrays, Camera, LodConfig, rotmat_to_quat
from .hierarchy import Hierarchy, build_hierarchy, node_depths
from .hspt import Hspt, build_hspt, build_hspt_host


def city_leaves(rng, n, extent=100.0, height=20.0, sh_sigma=0.05) -> AttributeArrays:
    a = AttributeArrays.zeros(n)
    a.means = np.stack([rng.uniform(-extent, extent, n), rng.uniform(0.0, height, n),
                        rng.uniform(-extent, extent, n)], axis=1)
    a.scales = np.exp(rng.uniform(np.log(0.01), np.log(0.1), (n, 3)))
    q = rng.normal(size=(n, 4))
    a.rotations = q / np.linalg.norm(q, axis=1, keepdims=True)
    a.opacities = rng.uniform(0.2, 0.95, n)
    a.base_colors = rng.uniform(0.05, 0.95, (n, 3))
    a.sh_rest = rng.normal(0.0, sh_sigma, (n, 9))
    return a


def city_block_leaves(rng, n, extent=100.0, height=20.0, blocks=8, street=0.15,
                      sh_sigma=0.05) -> AttributeArrays:
    """G-city (test_acceptance.py:180-193 `_city_scene` style):
    leaves on a blocks × blocks grid of city blocks separated by streets
    (`street` = street width / block pitch), each block a random-height
    building footprint, plus a thin ground layer in the streets."""
    a = city_leaves(rng, n, extent, height, sh_sigma)
    pitch = 2.0 * extent / blocks
    half = 0.5 * pitch * (1.0 - street)
    bx = rng.integers(0, blocks, n)
    bz = rng.integers(0, blocks, n)
    cx = -extent + (bx + 0.5) * pitch
    cz = -extent + (bz + 0.5) * pitch
    bh = rng.uniform(0.3, 1.0, (blocks, blocks)) * height
    ground = rng.uniform(size=n) < 0.1
    x = np.where(ground, rng.uniform(-extent, extent, n), cx + rng.uniform(-half, half, n))
    z = np.where(ground, rng.uniform(-extent, extent, n), cz + rng.uniform(-half, half, n))
    y = np.where(ground, rng.uniform(0.0, 0.02 * height, n), rng.uniform(0.0, 1.0, n) * bh[bx, bz])
    a.means = np.stack([x, y, z], axis=1)
    return a


@dataclass
class SceneSpec:
    n_leaves: int
    seed: int = 0
    extent: float | None = None     # None: 100 * (n / 1e7)^(1/3) (constant density)
    height: float | None = None
    spt_leaves: int = 4096          # target leaves per SPT subtree
    pass_fraction: float = 0.05     # share of cut branches that become passthrough
    min_subtree: int = 32
    threshold: float | None = None  # LoD T (runtime and SPT keys); None: extent / 4
    s_lo: float = 0.03
    s_hi: float = 0.3
    metric: str = "max_scale"
    relabel: bool = True            # node ids in store slot order (see relabel_slot_order)
    layout: str = "slab"            # "slab" (city_leaves) or "blocks" (G-city, city_block_leaves)


def scene_extent(n_leaves: int) -> float:
    return 100.0 * (n_leaves / 1e7) ** (1.0 / 3.0)


def designed_scene(spec: SceneSpec, device=None):
    """(Hierarchy, Hspt, LodConfig) with non-degenerate LoD cuts."""
    rng = np.random.default_rng(spec.seed)
    extent = spec.extent if spec.extent is not None else scene_extent(spec.n_leaves)
    height = spec.height if spec.height is not None else 0.2 * extent
    leaves = (city_block_leaves(rng, spec.n_leaves, extent, height) if spec.layout == "blocks"
              else city_leaves(rng, spec.n_leaves, extent, height))
    h = build_hierarchy(leaves, device=device)
    del leaves
    depth = node_depths(h)
    max_depth = int(depth.max())
    D = max(1, int(round(math.log2(max(spec.n_leaves / spec.spt_leaves, 1.0)))))
    D = min(D, max_depth - 1) if max_depth > 1 else 0
    T = spec.threshold if spec.threshold is not None else 0.25 * extent
    cfg = LodConfig(T, spec.metric)
    # upper nodes must never be "taken": m_d = T / s_up beyond every view
    view_range = 40.0 * extent
    s_up = T / view_range
    s_cut = 0.8 * s_up
    thr = 0.9 * s_up ** 3
    cap = h.capacity
    scales = np.exp(rng.uniform(np.log(spec.s_lo), np.log(spec.s_hi), (cap, 3)))
    is_upper = depth < D
    is_cut = depth == D
    # passthrough branches: some depth-D nodes keep descending until their
    # subtrees fall below min_subtree nodes; those become passthrough roots
    if spec.pass_fraction > 0 and D < len(h.levels()):
        lvlD = np.nonzero(is_cut)[0]
        frontier = lvlD[rng.uniform(size=lvlD.size) < spec.pass_fraction]
        counts = h.subtree_node_counts()
        while frontier.size:
            stop = (counts[frontier] < spec.min_subtree) | (h.children[frontier, 0] == -1)
            is_cut[frontier] = stop
            go = frontier[~stop]
            is_upper[go] = True
            frontier = h.children[go].ravel().astype(np.int64)
            is_cut[frontier] = True
    scales[is_upper] = s_up
    scales[is_cut] = s_cut
    h.attrs.scales = scales
    # scene tooling: the device build (K12) when a GPU is present, the numpy
    # restatement in CPU-only test contexts
    import torch
    build = build_hspt if torch.cuda.is_available() else build_hspt_host
    hspt = build(h, thr, spec.min_subtree, cfg)
    if spec.relabel:
        h = relabel_slot_order(h, hspt)
        hspt = build(h, thr, spec.min_subtree, cfg)
    return h, hspt, cfg


def relabel_slot_order(h: Hierarchy, hspt: Hspt) -> Hierarchy:
    """Renumber nodes so that node id == store slot (store.py:143-154: every
    non-SPT node first in ascending id, then each SPT's records in record
    order).  A data-layout choice for HBM: SPT cut prefixes become
    contiguous id ranges, so the render rows a view selects (and the ADAM
    updates of their master rows) are nearly sequential in memory.  Ties in
    the SPT record order (siblings share key_parent, broken by node id) keep
    their order because new ids increase along the records; rebuilding the
    HSPT on the result reproduces the same partition and record order."""
    from .store import slot_order
    order = slot_order(h, hspt)                      # slot -> old id
    new_of = np.full(h.capacity, -1, dtype=np.int64)
    new_of[order] = np.arange(order.size)
    n = order.size
    attrs = h.attrs.take(order)
    par = h.parent[order].astype(np.int64)
    ch = h.children[order].astype(np.int64)
    par = np.where(par >= 0, new_of[np.maximum(par, 0)], -1)
    ch = np.where(ch >= 0, new_of[np.maximum(ch, 0)], -1)
    return Hierarchy(attrs=attrs, parent=par.astype(np.int32), children=ch.astype(np.int32),
                     root=int(new_of[h.root]))


def look_at(position, target, focal, resolution, near=0.1) -> Camera:
    position = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - position
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 1.0, 0.0])
    if abs(fwd @ up) > 0.99:
        up = np.array([1.0, 0.0, 0.0])
    right = np.cross(up, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd], axis=1)
    w, hh = resolution
    return Camera(position=position, orientation=rotmat_to_quat(rot), focal=focal,
                  principal_point=(w / 2.0, hh / 2.0), resolution=resolution, near=near)


def orbit_views(n, radius, height, resolution=(1920, 1080), focal=None, seed=0,
                jitter=0.0, target_jitter=0.0):
    """Aerial orbit looking at the scene centre (test_acceptance.py:296-301
    style), `n` poses evenly around the circle with optional jitter."""
    rng = np.random.default_rng(seed)
    w, hh = resolution
    f = focal if focal is not None else (0.75 * w, 0.75 * w)
    cams = []
    for i in range(n):
        ang = 2 * np.pi * i / n + rng.uniform(-jitter, jitter)
        pos = np.array([radius * np.cos(ang), height, radius * np.sin(ang)])
        pos += rng.normal(0.0, jitter * radius * 0.05, 3)
        tgt = rng.normal(0.0, target_jitter, 3)
        cams.append(look_at(pos, tgt, f, resolution))
    return cams


def street_views(n, extent, resolution=(1920, 1080), blocks=8, eye=1.7, seed=0):
    """Street-level cameras (test_acceptance.py:216-219 style): eye height
    `eye`, walking along the streets between the city blocks and looking
    down the street."""
    rng = np.random.default_rng(seed)
    w, hh = resolution
    pitch = 2.0 * extent / blocks
    cams = []
    for i in range(n):
        k = rng.integers(1, blocks)
        t = rng.uniform(-0.9 * extent, 0.9 * extent)
        along_x = i % 2 == 0
        street = -extent + k * pitch
        pos = np.array([t, eye, street]) if along_x else np.array([street, eye, t])
        d = np.array([1.0, 0.0, 0.0]) if along_x else np.array([0.0, 0.0, 1.0])
        d = d * (1 if rng.uniform() < 0.5 else -1)
        cams.append(look_at(pos, pos + 10.0 * d + np.array([0.0, 0.3, 0.0]), (0.6 * w, 0.6 * w),
                            resolution, near=0.1))
    return cams
