"""Densification: trainer.densify (trainer.py:411-443)
with hierarchy.densify_spawn / respawn_dead / split_attributes
(hierarchy.py:269-361) and OptimizerState.grow_to / reset_nodes
(trainer.py:108-124).

The tree surgery is sequential, RNG-driven host work (a few thousand leaf
edits every `densify_interval` = 500 iterations), so it stays on the host
and consumes the scheduler RNG exactly like the reference (same draws, same
order: `rng.choice` for opacity-weighted leaf sampling, `rng.integers(2)`
per split).  What follows it is device work: the HSPT rebuild on the
mutated hierarchy (K12, `hspt.build_hspt` with the surface-area metric,
hspt.py:161-165) and the re-layout of the store and node records
(`Trainer.densify`).
"""
from __future__ import annotations

import numpy as np

from .core import AttributeArrays, quat_to_rotmat
from .hierarchy import NONE, Hierarchy

SPLIT_OFFSET = 0.6
SPLIT_SHRINK = 1.6


class InvalidTargetError(ValueError):
    pass


class CannotRespawnRootError(ValueError):
    pass


def split_attributes(attrs: AttributeArrays, leaf: int, rng: np.random.Generator) -> AttributeArrays:
    """Two children at ± SPLIT_OFFSET·s_max along the dominant axis, shrunk
    along it; opacity 1 − √(1 − σ) floored at σ/2 (hierarchy.py:269-294)."""
    g_scale = attrs.scales[leaf]
    k = int(np.argmax(g_scale))
    v = quat_to_rotmat(attrs.rotations[leaf])[:, k]
    offset = SPLIT_OFFSET * g_scale[k] * v
    sign = 1.0 if rng.integers(2) == 0 else -1.0
    means = np.stack([attrs.means[leaf] + sign * offset, attrs.means[leaf] - sign * offset])
    scales = np.stack([g_scale, g_scale])
    scales[:, k] /= SPLIT_SHRINK
    sigma = float(attrs.opacities[leaf])
    op = 1.0 - np.sqrt(max(1.0 - min(sigma, 1.0), 0.0))
    op = min(max(op, 0.5 * sigma), 1.0)
    return AttributeArrays(means=means, scales=scales, rotations=np.stack([attrs.rotations[leaf]] * 2),
                           opacities=np.array([op, op]), base_colors=np.stack([attrs.base_colors[leaf]] * 2),
                           sh_rest=np.stack([attrs.sh_rest[leaf]] * 2))


def _grow(h: Hierarchy, extra: int) -> list:
    old = h.capacity
    block = AttributeArrays.zeros(extra, dtype=np.float64)
    if block.sh_rest.shape[1] != h.attrs.sh_rest.shape[1]:
        block.sh_rest = np.zeros((extra, h.attrs.sh_rest.shape[1]))
    h.attrs = AttributeArrays.concat([h.attrs, block])
    h.parent = np.concatenate([h.parent, np.full(extra, NONE, dtype=np.int32)])
    h.children = np.concatenate([h.children, np.full((extra, 2), NONE, dtype=np.int32)])
    return list(range(old, old + extra))


def _trim(h: Hierarchy, cap: int) -> None:
    h.attrs = h.attrs.take(slice(0, cap))
    h.parent = h.parent[:cap].copy()
    h.children = h.children[:cap].copy()


def _alloc2(h: Hierarchy) -> list:
    slots = []
    while h.free and len(slots) < 2:
        slots.append(h.free.pop())
    if len(slots) < 2:
        slots += _grow(h, 2 - len(slots))
    return sorted(slots)


def densify_spawn(h: Hierarchy, leaf: int, rng: np.random.Generator):
    """hierarchy.py:318-327."""
    if h.children[leaf, 0] != NONE:
        raise InvalidTargetError(f"node {leaf} is internal, cannot spawn")
    left, right = _alloc2(h)
    h.attrs.put(np.array([left, right]), split_attributes(h.attrs, leaf, rng))
    h.children[leaf] = (left, right)
    h.parent[left] = leaf
    h.parent[right] = leaf
    return left, right


def respawn_dead(h: Hierarchy, dead_leaf: int, target_leaf: int, rng: np.random.Generator):
    """hierarchy.py:330-361: the sibling replaces the parent; the two freed
    slots become the target's children."""
    if dead_leaf == h.root:
        raise CannotRespawnRootError("root cannot be respawned")
    if h.children[dead_leaf, 0] != NONE:
        raise InvalidTargetError(f"node {dead_leaf} is not a leaf")
    if h.children[target_leaf, 0] != NONE:
        raise InvalidTargetError(f"target {target_leaf} is not a leaf")
    p = int(h.parent[dead_leaf])
    l, r = h.children[p]
    sibling = int(r if l == dead_leaf else l)
    if target_leaf in (dead_leaf, p):
        raise InvalidTargetError("target must be a distinct live leaf")
    g = int(h.parent[p])
    if g == NONE:
        h.root = sibling
        h.parent[sibling] = NONE
    else:
        gl, _ = h.children[g]
        h.children[g, 0 if gl == p else 1] = sibling
        h.parent[sibling] = g
    left, right = sorted((dead_leaf, p))
    h.attrs.put(np.array([left, right]), split_attributes(h.attrs, target_leaf, rng))
    h.children[left] = (NONE, NONE)
    h.children[right] = (NONE, NONE)
    h.children[target_leaf] = (left, right)
    h.parent[left] = target_leaf
    h.parent[right] = target_leaf


def sample_leaves(h: Hierarchy, count: int, rng: np.random.Generator, exclude=()) -> np.ndarray:
    """Distinct leaves ∝ opacity (trainer.py:381-392)."""
    leaves = h.leaf_ids
    if exclude:
        leaves = leaves[~np.isin(leaves, np.asarray(list(exclude)))]
    if leaves.size == 0 or count == 0:
        return np.empty(0, dtype=np.int64)
    w = np.maximum(h.attrs.opacities[leaves], 1e-12)
    p = w / w.sum()
    return rng.choice(leaves, size=min(count, leaves.size), replace=False, p=p)


class Moments:
    """OptimizerState-shaped host view: m, v as AttributeArrays-like dicts
    keyed by attribute name, per-node step (trainer.py:94-124)."""

    def __init__(self, m: AttributeArrays, v: AttributeArrays, step: np.ndarray):
        self.m, self.v, self.step = m, v, step

    def grow_to(self, n: int):
        if n == self.step.size:
            return
        if n < self.step.size:            # densify_tree's trim of unused pre-grown slots
            for blk in (self.m, self.v):
                for name, arr in blk.arrays():
                    setattr(blk, name, arr[:n].copy())
            self.step = self.step[:n].copy()
            return
        extra = n - self.step.size
        for blk in (self.m, self.v):
            for name, arr in blk.arrays():
                setattr(blk, name, np.concatenate([arr, np.zeros((extra,) + arr.shape[1:])]))
        self.step = np.concatenate([self.step, np.zeros(extra, dtype=np.int64)])

    def reset_nodes(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        for blk in (self.m, self.v):
            for name, arr in blk.arrays():
                arr[ids] = 0.0
        self.step[ids] = 0


def _choice1(rng: np.random.Generator, a: np.ndarray, p: np.ndarray):
    """rng.choice(a, size=1, replace=False, p=p)[0] with numpy's exact
    arithmetic and draws (one rng.random((1,)), cumsum, normalise by the
    last value, searchsorted 'right' — numpy/random/_generator.pyx),
    without the argument validation passes (tests/test_densify.py checks
    the two agree, index and generator state)."""
    x = rng.random((1,))
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    return a[int(cdf.searchsorted(x, side="right")[0])]


def densify_tree(h: Hierarchy, opt: Moments, rng: np.random.Generator, dead_opacity_threshold: float = 0.005,
                 spawns_per_densify: int | None = None) -> dict:
    """The host part of trainer.densify (trainer.py:411-440), in the
    reference's order: respawn every dead leaf into an opacity-sampled
    target, then spawn children under sampled leaves; moments of new /
    respawned nodes are zeroed.

    Same draws, same tree and the same slot ids as the reference, without
    its per-edit O(capacity) passes: the sorted leaf list and its weights
    are updated in place across respawns (each draw still normalises and
    accumulates the whole distribution, exactly as numpy's choice does),
    and the arrays grow once for all spawns (slot ids assigned as the
    reference's allocator would: free slots first, then new ones in
    order) instead of twice per spawn."""
    leaves = h.leaf_ids
    dead = leaves[h.attrs.opacities[leaves] < dead_opacity_threshold]
    wl = np.maximum(h.attrs.opacities[leaves], 1e-12)
    respawned = 0
    for d in dead:
        d = int(d)
        if h.children[d, 0] != NONE or d == h.root:
            continue                      # structure changed under a previous respawn
        parent = int(h.parent[d])
        # sample_leaves(h, 1, rng, exclude={d, parent}): parent is internal
        i = int(np.searchsorted(leaves, d))
        lv, w = np.delete(leaves, i), np.delete(wl, i)
        if lv.size == 0:
            continue
        target = int(_choice1(rng, lv, w / w.sum()))
        respawn_dead(h, d, target, rng)
        opt.reset_nodes([d, parent])
        respawned += 1
        # leaves: the target is internal now, the old parent a leaf; d and
        # the parent carry the split attributes
        j = int(np.searchsorted(leaves, target))
        leaves, wl = np.delete(leaves, j), np.delete(wl, j)
        k = int(np.searchsorted(leaves, parent))
        leaves, wl = np.insert(leaves, k, parent), np.insert(wl, k, max(float(h.attrs.opacities[parent]), 1e-12))
        wl[int(np.searchsorted(leaves, d))] = max(float(h.attrs.opacities[d]), 1e-12)
    n_spawn = spawns_per_densify if spawns_per_densify is not None else max(h.leaf_count // 200, 0)
    spawned = 0
    picks = sample_leaves(h, n_spawn, rng)
    # the reference's allocator (_alloc2) pops free slots first and grows by
    # the shortfall: grow once by the total shortfall, hand out the new ids
    # in the same order, trim what a failed spawn would leave unused
    cap0 = h.capacity
    need = max(0, 2 * len(picks) - len(h.free))
    if need:
        _grow(h, need)
        opt.grow_to(h.capacity)
    nxt = cap0
    for leaf in picks:
        leaf = int(leaf)
        if h.children[leaf, 0] != NONE:
            raise InvalidTargetError(f"node {leaf} is internal, cannot spawn")
        slots = []
        while h.free and len(slots) < 2:
            slots.append(h.free.pop())
        while len(slots) < 2:
            slots.append(nxt)
            nxt += 1
        left, right = sorted(slots)
        h.attrs.put(np.array([left, right]), split_attributes(h.attrs, leaf, rng))
        h.children[leaf] = (left, right)
        h.parent[left] = leaf
        h.parent[right] = leaf
        opt.reset_nodes([left, right])
        spawned += 1
    if nxt < h.capacity:
        _trim(h, nxt)
    opt.grow_to(h.capacity)
    return {"spawned": spawned, "respawned": respawned}
