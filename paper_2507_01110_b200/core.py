"""Host-side domain types of the per-view hot path.

These mirror the reference package's value types one-to-one (field names,
argument meaning, validation errors) so callers written against the
reference (`glod.core`, /root/reference/pkg/src/glod/core.py) can pass the
same objects here.  They are plain numpy containers: the device never sees
them directly — `device.py` packs them into the flat buffers the C-ABI
(`include/glod_b200.h`) takes.

Reference anchors:
  AttributeArrays   core.py:59-167   (SoA block, canonical section order)
  LodConfig         core.py:170-179
  quat_to_rotmat    core.py:182-202
  rotmat_to_quat    core.py:205-256  (host tooling: scene generation)
  Camera            core.py:259-291
  Frustum           core.py:294-328
  min_distance_batch core.py:356-361 (host tooling; the device has its own)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MAX_SCALE = "max_scale"
SURFACE_AREA = "surface_area"
LOWPASS_FLOOR = 0.3          # px^2 added to the projected covariance diagonal
SH_C1 = 0.4886025119029199   # degree-1 real SH normalisation

# Canonical attribute sections and their column counts (store.py:119-122).
SECTIONS = (("means", 3), ("scales", 3), ("rotations", 4), ("opacities", 1),
            ("base_colors", 3), ("sh_rest", 9))
FLOATS_PER_GAUSSIAN = sum(c for _, c in SECTIONS)   # 23
BYTES_PER_GAUSSIAN_F32 = 4 * FLOATS_PER_GAUSSIAN     # 92 (store.py:125-127)


class InvalidParameterError(ValueError):
    pass


class EmptySceneError(ValueError):
    pass


@dataclass
class AttributeArrays:
    """N Gaussians as six arrays (means, scales, rotations (w,x,y,z),
    opacities, base_colors, sh_rest) — the layout the reference passes
    between its hierarchy, store and renderer."""

    means: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    base_colors: np.ndarray
    sh_rest: np.ndarray

    def __len__(self):
        return int(self.means.shape[0])

    @property
    def sh_degree(self) -> int:
        return int(round(np.sqrt(self.sh_rest.shape[1] // 3 + 1))) - 1

    @staticmethod
    def zeros(n: int, sh_degree: int = 1, dtype=np.float64) -> "AttributeArrays":
        rot = np.zeros((n, 4), dtype=dtype)
        rot[:, 0] = 1.0
        return AttributeArrays(
            means=np.zeros((n, 3), dtype=dtype),
            scales=np.ones((n, 3), dtype=dtype),
            rotations=rot,
            opacities=np.zeros(n, dtype=dtype),
            base_colors=np.zeros((n, 3), dtype=dtype),
            sh_rest=np.zeros((n, 3 * ((sh_degree + 1) ** 2 - 1)), dtype=dtype))

    def arrays(self):
        return [(name, getattr(self, name)) for name, _ in SECTIONS]

    def take(self, idx) -> "AttributeArrays":
        return AttributeArrays(*(getattr(self, n)[idx] for n, _ in SECTIONS))

    def put(self, idx, block: "AttributeArrays"):
        for n, _ in SECTIONS:
            getattr(self, n)[idx] = getattr(block, n)

    def copy(self) -> "AttributeArrays":
        return AttributeArrays(*(getattr(self, n).copy() for n, _ in SECTIONS))

    def astype(self, dtype) -> "AttributeArrays":
        return AttributeArrays(*(getattr(self, n).astype(dtype) for n, _ in SECTIONS))

    @staticmethod
    def concat(blocks) -> "AttributeArrays":
        blocks = list(blocks)
        return AttributeArrays(*(np.concatenate([getattr(b, n) for b in blocks])
                                 for n, _ in SECTIONS))

    def packed(self, dtype=np.float64) -> np.ndarray:
        """Flat section-major buffer [means(3N) | scales(3N) | rot(4N) |
        opac(N) | base(3N) | sh(9N)] — the device "attribute block" layout."""
        return np.concatenate([np.ascontiguousarray(getattr(self, n), dtype=dtype).reshape(-1)
                               for n, _ in SECTIONS])

    @staticmethod
    def from_packed(buf: np.ndarray, n: int) -> "AttributeArrays":
        out, off = [], 0
        for _, cols in SECTIONS:
            part = buf[off:off + cols * n]
            out.append(part.reshape(n, cols) if cols > 1 else part.copy())
            off += cols * n
        return AttributeArrays(*out)


@dataclass(frozen=True)
class LodConfig:
    threshold: float
    metric: str = MAX_SCALE

    def __post_init__(self):
        if not self.threshold > 0:
            raise InvalidParameterError("LoD threshold must be > 0")
        if self.metric not in (MAX_SCALE, SURFACE_AREA):
            raise InvalidParameterError(f"unknown LoD metric {self.metric!r}")

    @property
    def metric_code(self) -> int:
        return 0 if self.metric == MAX_SCALE else 1


def quat_to_rotmat(q: np.ndarray) -> np.ndarray:
    """(w,x,y,z) → R, normalising first; (4,)→(3,3) or (N,4)→(N,3,3).
    Same elementwise formula as core.py:182-202 (bit-identical: no BLAS)."""
    q = np.asarray(q, dtype=np.float64)
    one = q.ndim == 1
    q = np.atleast_2d(q)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    r = np.empty((q.shape[0], 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r[0] if one else r


def rotmat_to_quat(m: np.ndarray) -> np.ndarray:
    """Batched Shepperd conversion, w ≥ 0 (core.py:205-256). Host tooling
    only (scene generation / hierarchy merge), never on the per-view path."""
    m = np.asarray(m, dtype=np.float64)
    one = m.ndim == 2
    m = m.reshape(-1, 3, 3)
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    pick = np.argmax(np.stack([tr, m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], 1), 1)
    q = np.empty((m.shape[0], 4))
    d = np.stack([m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], 1)
    for c in range(4):
        sel = pick == c
        if not sel.any():
            continue
        a = m[sel]
        if c == 0:
            r = np.sqrt(1.0 + tr[sel])
            s = 0.5 / r
            q[sel] = np.stack([0.5 * r, (a[:, 2, 1] - a[:, 1, 2]) * s,
                               (a[:, 0, 2] - a[:, 2, 0]) * s,
                               (a[:, 1, 0] - a[:, 0, 1]) * s], 1)
        elif c == 1:
            r = np.sqrt(1.0 + d[sel, 0] - d[sel, 1] - d[sel, 2])
            s = 0.5 / r
            q[sel] = np.stack([(a[:, 2, 1] - a[:, 1, 2]) * s, 0.5 * r,
                               (a[:, 0, 1] + a[:, 1, 0]) * s,
                               (a[:, 0, 2] + a[:, 2, 0]) * s], 1)
        elif c == 2:
            r = np.sqrt(1.0 - d[sel, 0] + d[sel, 1] - d[sel, 2])
            s = 0.5 / r
            q[sel] = np.stack([(a[:, 0, 2] - a[:, 2, 0]) * s,
                               (a[:, 0, 1] + a[:, 1, 0]) * s, 0.5 * r,
                               (a[:, 1, 2] + a[:, 2, 1]) * s], 1)
        else:
            r = np.sqrt(1.0 - d[sel, 0] - d[sel, 1] + d[sel, 2])
            s = 0.5 / r
            q[sel] = np.stack([(a[:, 1, 0] - a[:, 0, 1]) * s,
                               (a[:, 0, 2] + a[:, 2, 0]) * s,
                               (a[:, 1, 2] + a[:, 2, 1]) * s, 0.5 * r], 1)
    q *= np.where(q[:, 0] < 0, -1.0, 1.0)[:, None]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q[0] if one else q


@dataclass
class Camera:
    """Pinhole camera; `orientation` (w,x,y,z) maps camera→world, camera
    space is x right / y down / z forward (core.py:259-291)."""

    position: np.ndarray
    orientation: np.ndarray
    focal: tuple
    principal_point: tuple
    resolution: tuple
    near: float = 0.01
    far: float = 1e6

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        q = np.asarray(self.orientation, dtype=np.float64)
        n = np.linalg.norm(q)
        if not np.isfinite(n) or n < 1e-12:
            raise InvalidParameterError("degenerate camera orientation")
        self.orientation = q / n
        if not (0 < self.near < self.far):
            raise InvalidParameterError("camera requires 0 < near < far")
        if self.resolution[0] < 1 or self.resolution[1] < 1:
            raise InvalidParameterError("camera resolution must be >= 1")

    @property
    def world_to_cam(self) -> np.ndarray:
        return quat_to_rotmat(self.orientation).T

    def to_camera_space(self, points: np.ndarray) -> np.ndarray:
        return (np.asarray(points, dtype=np.float64) - self.position) @ self.world_to_cam.T

    @staticmethod
    def from_any(cam) -> "Camera":
        """Accept a reference `glod.core.Camera` (or anything shaped like
        one) — the drop-in boundary takes the caller's camera object."""
        if isinstance(cam, Camera):
            return cam
        return Camera(position=cam.position, orientation=cam.orientation,
                      focal=tuple(cam.focal), principal_point=tuple(cam.principal_point),
                      resolution=tuple(cam.resolution), near=cam.near, far=cam.far)


# Camera-space frustum planes (nx, ny, nz, d): apex, far, left, right, top,
# bottom (core.py:312-319). The far plane's d is filled in per camera.
def _camera_planes(cam: Camera):
    fx, fy = cam.focal
    cx, cy = cam.principal_point
    w, h = cam.resolution
    lo_x, hi_x = (0.0 - cx) / fx, (w - cx) / fx
    lo_y, hi_y = (0.0 - cy) / fy, (h - cy) / fy
    return ((0.0, 0.0, -1.0, 0.0), (0.0, 0.0, 1.0, -cam.far),
            (-1.0, 0.0, lo_x, 0.0), (1.0, 0.0, -hi_x, 0.0),
            (0.0, -1.0, lo_y, 0.0), (0.0, 1.0, -hi_y, 0.0))


@dataclass(frozen=True)
class Frustum:
    """Six outward world-space planes; outside plane k iff n·p + d > 0."""

    planes: np.ndarray

    @staticmethod
    def from_camera(cam: Camera) -> "Frustum":
        # Computed on the host with the same numpy BLAS calls as the
        # reference (core.py:320-328: per-plane gemv `r @ n` and ddot
        # `n @ position`), so the device receives bit-identical planes.
        rot = quat_to_rotmat(cam.orientation)
        planes = np.empty((6, 4))
        for k, (a, b, c, d) in enumerate(_camera_planes(cam)):
            n_cam = np.array([a, b, c])
            n_cam = n_cam / np.linalg.norm(n_cam)
            n_world = rot @ n_cam
            planes[k, :3] = n_world
            planes[k, 3] = d / np.linalg.norm([a, b, c]) - n_world @ cam.position
        return Frustum(planes=planes)


def min_distance_batch(scales: np.ndarray, cfg: LodConfig) -> np.ndarray:
    """LoD metric m_d (core.py:356-361): T/max(s) or T/sqrt(s1s2+s1s3+s2s3)."""
    s = np.asarray(scales, dtype=np.float64)
    if cfg.metric == MAX_SCALE:
        return cfg.threshold / np.max(s, axis=-1)
    return cfg.threshold / np.sqrt(s[..., 0] * s[..., 1] + s[..., 0] * s[..., 2]
                                   + s[..., 1] * s[..., 2])


def covariance_from_batch(scales: np.ndarray, rotations: np.ndarray) -> np.ndarray:
    r = quat_to_rotmat(rotations)
    return np.einsum("nij,nj,nkj->nik", r, np.asarray(scales, dtype=np.float64) ** 2, r)
