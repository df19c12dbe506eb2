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


def densify_tree(h: Hierarchy, opt: Moments, rng: np.random.Generator, dead_opacity_threshold: float = 0.005,
                 spawns_per_densify: int | None = None) -> dict:
    """The host part of trainer.densify (trainer.py:411-440), in the
    reference's order: respawn every dead leaf into an opacity-sampled
    target, then spawn children under sampled leaves; moments of new /
    respawned nodes are zeroed."""
    leaves = h.leaf_ids
    dead = leaves[h.attrs.opacities[leaves] < dead_opacity_threshold]
    respawned = 0
    for d in dead:
        d = int(d)
        if h.children[d, 0] != NONE or d == h.root:
            continue                      # structure changed under a previous respawn
        parent = int(h.parent[d])
        targets = sample_leaves(h, 1, rng, exclude={d, parent})
        if targets.size == 0:
            continue
        respawn_dead(h, d, int(targets[0]), rng)
        opt.reset_nodes([d, parent])
        respawned += 1
    n_spawn = spawns_per_densify if spawns_per_densify is not None else max(h.leaf_count // 200, 0)
    spawned = 0
    for leaf in sample_leaves(h, n_spawn, rng):
        left, right = densify_spawn(h, int(leaf), rng)
        opt.grow_to(h.capacity)
        opt.reset_nodes([left, right])
        spawned += 1
    opt.grow_to(h.capacity)
    return {"spawned": spawned, "respawned": respawned}
