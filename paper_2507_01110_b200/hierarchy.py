"""Binary Gaussian hierarchy container + a data-parallel builder.

`Hierarchy` mirrors the reference container (hierarchy.py:51-134: SoA
attributes, int32 parent/children with NONE=-1, index-stable slots).

`build_hierarchy` is host tooling used to make synthetic scenes on the GPU
box (the reference cannot travel there). It follows the reference's
construction (hierarchy.py:192-241): top-down median split on the longest
bounding-box axis, then opacity·volume-weighted moment-matched merges
deepest level first (hierarchy.py:136-176).  Unlike the reference's
per-node Python stack it processes a whole tree level at once with two
stable sorts, in torch, so a 10M-leaf tree builds in seconds on a GPU (or
in a CPU process for small test scenes).  Node numbering is level order
(leaves keep ids 0..n-1, root = n as in the reference), so ids differ from
the reference's DFS numbering — parity tests that need the reference's
exact trees load them from `tests/golden/`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .core import AttributeArrays, EmptySceneError

NONE = -1


@dataclass
class CutSet:
    node_ids: np.ndarray

    def __len__(self):
        return int(self.node_ids.size)


@dataclass
class Hierarchy:
    attrs: AttributeArrays
    parent: np.ndarray      # (cap,) int32, NONE for the root
    children: np.ndarray    # (cap, 2) int32, NONE/NONE for leaves
    root: int
    free: list = field(default_factory=list)

    @property
    def capacity(self) -> int:
        return int(self.parent.shape[0])

    @property
    def node_count(self) -> int:
        return self.capacity - len(self.free)

    @property
    def is_leaf(self) -> np.ndarray:
        return self.children[:, 0] == NONE

    @property
    def leaf_ids(self) -> np.ndarray:
        mask = self.is_leaf.copy()
        if self.free:
            mask[np.asarray(self.free, dtype=np.int64)] = False
        return np.nonzero(mask)[0]

    @property
    def leaf_count(self) -> int:
        return int(self.leaf_ids.size)

    def levels(self):
        """Reachable nodes grouped by depth, root first."""
        out = []
        frontier = np.array([self.root], dtype=np.int64)
        while frontier.size:
            out.append(frontier)
            ch = self.children[frontier]
            frontier = ch[ch[:, 0] != NONE].ravel().astype(np.int64)
        return out

    def bfs_order(self) -> np.ndarray:
        lv = self.levels()
        return np.concatenate(lv) if lv else np.empty(0, dtype=np.int64)

    def subtree_node_counts(self) -> np.ndarray:
        counts = np.zeros(self.capacity, dtype=np.int64)
        for lvl in reversed(self.levels()):
            counts[lvl] += 1
            up = lvl[self.parent[lvl] != NONE]
            counts += np.bincount(self.parent[up], weights=counts[up],
                                  minlength=self.capacity).astype(np.int64)
        return counts

    def subtree_nodes(self, node: int) -> np.ndarray:
        out = []
        frontier = np.array([node], dtype=np.int64)
        while frontier.size:
            out.append(frontier)
            ch = self.children[frontier]
            frontier = ch[ch[:, 0] != NONE].ravel().astype(np.int64)
        return np.concatenate(out)

    @staticmethod
    def from_any(h) -> "Hierarchy":
        """Accept a reference `glod.hierarchy.Hierarchy` at the boundary."""
        if isinstance(h, Hierarchy):
            return h
        a = h.attrs
        attrs = AttributeArrays(a.means, a.scales, a.rotations, a.opacities,
                                a.base_colors, a.sh_rest)
        return Hierarchy(attrs=attrs, parent=np.asarray(h.parent, dtype=np.int32),
                         children=np.asarray(h.children, dtype=np.int32),
                         root=int(h.root), free=list(h.free))


# --------------------------------------------------------------------------
# builder (torch, device-agnostic)
# --------------------------------------------------------------------------

def _quat_to_rotmat_t(q: torch.Tensor) -> torch.Tensor:
    q = q / torch.linalg.norm(q, dim=-1, keepdim=True)
    w, x, y, z = q.unbind(-1)
    return torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        -1).reshape(q.shape[:-1] + (3, 3))


def _rotmat_to_quat_t(m: torch.Tensor) -> torch.Tensor:
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    d0, d1, d2 = m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]
    pick = torch.argmax(torch.stack([tr, d0, d1, d2], 1), 1)
    cands = []
    r = torch.sqrt(torch.clamp(1.0 + tr, min=1e-300)); s = 0.5 / r
    cands.append(torch.stack([0.5 * r, (m[:, 2, 1] - m[:, 1, 2]) * s,
                              (m[:, 0, 2] - m[:, 2, 0]) * s, (m[:, 1, 0] - m[:, 0, 1]) * s], 1))
    r = torch.sqrt(torch.clamp(1.0 + d0 - d1 - d2, min=1e-300)); s = 0.5 / r
    cands.append(torch.stack([(m[:, 2, 1] - m[:, 1, 2]) * s, 0.5 * r,
                              (m[:, 0, 1] + m[:, 1, 0]) * s, (m[:, 0, 2] + m[:, 2, 0]) * s], 1))
    r = torch.sqrt(torch.clamp(1.0 - d0 + d1 - d2, min=1e-300)); s = 0.5 / r
    cands.append(torch.stack([(m[:, 0, 2] - m[:, 2, 0]) * s, (m[:, 0, 1] + m[:, 1, 0]) * s,
                              0.5 * r, (m[:, 1, 2] + m[:, 2, 1]) * s], 1))
    r = torch.sqrt(torch.clamp(1.0 - d0 - d1 + d2, min=1e-300)); s = 0.5 / r
    cands.append(torch.stack([(m[:, 1, 0] - m[:, 0, 1]) * s, (m[:, 0, 2] + m[:, 2, 0]) * s,
                              (m[:, 1, 2] + m[:, 2, 1]) * s, 0.5 * r], 1))
    q = torch.stack(cands, 1).gather(1, pick.view(-1, 1, 1).expand(-1, 1, 4))[:, 0]
    q = q * torch.where(q[:, :1] < 0, -1.0, 1.0)
    return q / torch.linalg.norm(q, dim=1, keepdim=True)


def _eigh_batched(cov: torch.Tensor, sweeps: int = 8):
    """Symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations,
    vectorised over the batch (cusolver's batched syev rejects large
    batches).  Returns ascending eigenvalues and column eigenvectors like
    torch.linalg.eigh."""
    A = cov.clone()
    n = A.shape[0]
    V = torch.eye(3, dtype=A.dtype, device=A.device).expand(n, 3, 3).clone()
    for _ in range(sweeps):
        for p, q in ((0, 1), (0, 2), (1, 2)):
            apq = A[:, p, q]
            app, aqq = A[:, p, p], A[:, q, q]
            nz = apq.abs() > 1e-300
            tau = (aqq - app) / torch.where(nz, 2.0 * apq, torch.ones_like(apq))
            t = torch.sign(tau) / (tau.abs() + torch.sqrt(1.0 + tau * tau))
            t = torch.where(tau == 0, torch.ones_like(t), t)
            t = torch.where(nz, t, torch.zeros_like(t))
            c = 1.0 / torch.sqrt(1.0 + t * t)
            s_ = t * c
            J = torch.eye(3, dtype=A.dtype, device=A.device).expand(n, 3, 3).clone()
            J[:, p, p] = c
            J[:, q, q] = c
            J[:, p, q] = s_
            J[:, q, p] = -s_
            A = J.transpose(1, 2) @ A @ J
            V = V @ J
    vals = torch.diagonal(A, dim1=1, dim2=2)
    order = torch.argsort(vals, dim=1)
    vals = vals.gather(1, order)
    vecs = V.gather(2, order[:, None, :].expand(-1, 3, -1))
    return vals, vecs


def _merge_level(A: dict, dst, a, b):
    """Moment-matched merge of children (a, b) into dst (hierarchy.py:136-176)."""
    wa = A["opacities"][a] * torch.prod(A["scales"][a], 1)
    wb = A["opacities"][b] * torch.prod(A["scales"][b], 1)
    tot = wa + wb
    zero = tot <= 0
    wa = torch.where(zero, 0.5, wa)
    wb = torch.where(zero, 0.5, wb)
    tot = wa + wb
    fa = (wa / tot)[:, None]
    fb = (wb / tot)[:, None]
    mean = fa * A["means"][a] + fb * A["means"][b]
    ra = _quat_to_rotmat_t(A["rotations"][a])
    rb = _quat_to_rotmat_t(A["rotations"][b])
    ca = (ra * A["scales"][a][:, None, :] ** 2) @ ra.transpose(1, 2)
    cb = (rb * A["scales"][b][:, None, :] ** 2) @ rb.transpose(1, 2)
    da = A["means"][a] - mean
    db = A["means"][b] - mean
    cov = (fa[..., None] * (ca + da[:, :, None] * da[:, None, :])
           + fb[..., None] * (cb + db[:, :, None] * db[:, None, :]))
    cov = 0.5 * (cov + cov.transpose(1, 2))
    vals, vecs = _eigh_batched(cov)
    flip = torch.linalg.det(vecs) < 0
    vecs[:, :, 2] = torch.where(flip[:, None], -vecs[:, :, 2], vecs[:, :, 2])
    A["means"][dst] = mean
    A["scales"][dst] = torch.sqrt(torch.clamp(vals, min=1e-18))
    A["rotations"][dst] = _rotmat_to_quat_t(vecs)
    A["opacities"][dst] = torch.maximum(A["opacities"][a], A["opacities"][b])
    A["base_colors"][dst] = fa * A["base_colors"][a] + fb * A["base_colors"][b]
    A["sh_rest"][dst] = fa * A["sh_rest"][a] + fb * A["sh_rest"][b]


def build_hierarchy(leaves: AttributeArrays, device=None) -> Hierarchy:
    """Median-split + moment-matched binary hierarchy over `leaves`."""
    n = len(leaves)
    if n == 0:
        raise EmptySceneError("cannot build a hierarchy from zero Gaussians")
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() and n > 200_000 else torch.device("cpu"))
    total = 2 * n - 1
    A = {}
    for name, arr in leaves.arrays():
        arr = np.asarray(arr, dtype=np.float64)
        full = torch.zeros((total,) + arr.shape[1:], dtype=torch.float64, device=dev)
        full[:n] = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        A[name] = full
    A["rotations"][n:, 0] = 1.0
    A["scales"][n:] = 1.0
    parent = torch.full((total,), NONE, dtype=torch.int64, device=dev)
    children = torch.full((total, 2), NONE, dtype=torch.int64, device=dev)
    if n == 1:
        return _to_host(A, parent, children, 0)

    means = A["means"][:n]
    perm = torch.arange(n, device=dev)                 # leaves grouped by segment
    seg_start = torch.zeros(1, dtype=torch.int64, device=dev)
    seg_len = torch.full((1,), n, dtype=torch.int64, device=dev)
    seg_slot = torch.full((1,), n, dtype=torch.int64, device=dev)
    next_slot = n + 1
    levels = []                                        # internal slots per depth
    while seg_len.numel():
        levels.append(seg_slot)
        nseg = seg_len.numel()
        seg_of = torch.repeat_interleave(torch.arange(nseg, device=dev), seg_len)
        offs = torch.arange(seg_of.numel(), device=dev) - torch.repeat_interleave(
            torch.cumsum(seg_len, 0) - seg_len, seg_len)
        pos = seg_start[seg_of] + offs                 # positions in perm
        pts = means[perm[pos]]
        lo = torch.full((nseg, 3), float("inf"), dtype=torch.float64, device=dev)
        hi = torch.full((nseg, 3), -float("inf"), dtype=torch.float64, device=dev)
        idx3 = seg_of[:, None].expand(-1, 3)
        lo = lo.scatter_reduce(0, idx3, pts, "amin")
        hi = hi.scatter_reduce(0, idx3, pts, "amax")
        axis = torch.argmax(hi - lo, 1)
        key = pts.gather(1, axis[seg_of][:, None])[:, 0]
        o1 = torch.sort(key, stable=True).indices
        o2 = torch.sort(seg_of[o1], stable=True).indices
        order = o1[o2]
        perm[pos] = perm[pos[order]]
        half = seg_len // 2
        sizes = torch.stack([half, seg_len - half], 1)               # (nseg, 2)
        starts = torch.stack([seg_start, seg_start + half], 1)
        internal = sizes >= 2
        n_new = int(internal.sum())
        new_slots = torch.full_like(sizes, NONE)
        new_slots[internal] = torch.arange(next_slot, next_slot + n_new, device=dev)
        next_slot += n_new
        kid = torch.where(internal, new_slots, perm[starts.clamp(max=n - 1)])
        children[seg_slot] = kid
        parent[kid.reshape(-1)] = seg_slot.repeat_interleave(2)
        seg_start = starts[internal]
        seg_len = sizes[internal]
        seg_slot = new_slots[internal]
    for slots in reversed(levels):
        _merge_level(A, slots, children[slots, 0], children[slots, 1])
    return _to_host(A, parent, children, n)


def _to_host(A, parent, children, root) -> Hierarchy:
    attrs = AttributeArrays(*(A[name].cpu().numpy() for name in
                              ("means", "scales", "rotations", "opacities",
                               "base_colors", "sh_rest")))
    return Hierarchy(attrs=attrs, parent=parent.cpu().numpy().astype(np.int32),
                     children=children.cpu().numpy().astype(np.int32), root=int(root))


def node_depths(h: Hierarchy) -> np.ndarray:
    depth = np.full(h.capacity, -1, dtype=np.int32)
    for d, lvl in enumerate(h.levels()):
        depth[lvl] = d
    return depth
