"""Drop-in rasteriser API (mirrors renderer.py of the reference) on the GPU.

`render_forward` / `render` / `backward` / `loss` / `psnr` take and return
the reference's types (numpy float64 images, GaussianGradients) and run the
CUDA kernels of csrc/raster.cu and csrc/loss.cu through the C-ABI.
`Rasterizer` is the device-level interface the trainer and bench use:
packed f64 attribute blocks and f32 images stay in HBM.

Reference anchors: constants renderer.py:17-25, InvalidInputError :28,
GaussianGradients :32-46, RenderContext :59-64, render_forward :117-166,
render :169-171, backward :197-304, loss :322-360, psnr :363-368.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import SECTIONS, AttributeArrays, Camera, quat_to_rotmat

ALPHA_CLAMP = 0.99
TRANSMITTANCE_EPS = 1e-4
FOOTPRINT_SIGMA = 3.0
Q_CUTOFF = 2.0 * (FOOTPRINT_SIGMA + 1.0) ** 2
SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


class InvalidInputError(ValueError):
    pass


@dataclass
class GaussianGradients:
    means: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    base_colors: np.ndarray
    sh_rest: np.ndarray

    @staticmethod
    def zeros(n: int, sh_cols: int = 9) -> "GaussianGradients":
        return GaussianGradients(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 4)),
                                 np.zeros(n), np.zeros((n, 3)), np.zeros((n, sh_cols)))

    @staticmethod
    def from_packed(buf: np.ndarray, n: int) -> "GaussianGradients":
        a = AttributeArrays.from_packed(buf, n)
        return GaussianGradients(a.means, a.scales, a.rotations, a.opacities, a.base_colors,
                                 a.sh_rest)


@dataclass
class RenderContext:
    attrs: AttributeArrays
    cam: Camera
    image: np.ndarray
    splats: list            # reference field; holds the device state handle here
    _dev: object = None


def camera_struct(cam: Camera) -> _lib.Camera:
    c = _lib.Camera()
    c.position[:] = [float(x) for x in cam.position]
    c.w2c[:] = [float(x) for x in quat_to_rotmat(cam.orientation).T.reshape(-1)]
    c.fx, c.fy = (float(f) for f in cam.focal)
    c.cx, c.cy = (float(p) for p in cam.principal_point)
    c.near_plane = float(cam.near)
    c.width, c.height = (int(r) for r in cam.resolution)
    return c


class Rasterizer:
    """One glod_raster context: forward state is kept for `backward`."""

    def __init__(self):
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.glod_raster_create(C.byref(h)))
        self._h = h
        self._loss_scratch = None
        self.last_n = 0
        self.cam = None

    def __del__(self):
        try:
            if self._h:
                _lib.load().glod_raster_destroy(self._h)
        except Exception:
            pass

    def forward(self, attrs_packed: torch.Tensor, n: int, cam: Camera, image: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
        w, h = cam.resolution
        if image is None:
            image = torch.empty((h, w, 3), dtype=torch.float32, device=attrs_packed.device)
        self._cam_struct = camera_struct(cam)
        self.cam = cam
        self.last_n = int(n)
        self._attrs = attrs_packed     # must stay alive for backward
        _lib.check(_lib.lib().glod_render_forward(self._h, _lib.ptr(attrs_packed), int(n),
                                                  C.byref(self._cam_struct), _lib.ptr(image),
                                                  _lib.stream_ptr(stream)))
        return image

    def forward_plan(self, plan, row_node: torch.Tensor, n: int, cam: Camera, image: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
        """`forward` of the render set a gather plan describes, read in place
        (glod_render_forward_plan: the K4 gather fused into the preprocess);
        fills row_node.  The plan's arrays must stay valid until `backward`."""
        w, h = cam.resolution
        if image is None:
            image = torch.empty((h, w, 3), dtype=torch.float32, device=row_node.device)
        self._cam_struct = camera_struct(cam)
        self.cam = cam
        self.last_n = int(n)
        self._attrs = (plan, row_node)
        _lib.check(_lib.lib().glod_render_forward_plan(self._h, C.byref(plan), _lib.ptr(row_node),
                                                       C.byref(self._cam_struct), _lib.ptr(image),
                                                       _lib.stream_ptr(stream)))
        return image

    def defer_blend(self, enable: bool):
        """While on, `forward`/`forward_plan` stop before the compositing
        kernel; `blend` enqueues it (glod_render_defer_blend)."""
        _lib.check(_lib.lib().glod_render_defer_blend(self._h, int(bool(enable))))

    def blend(self, stream=None):
        _lib.check(_lib.lib().glod_render_blend(self._h, _lib.stream_ptr(stream)))

    def backward(self, dl_dimage: torch.Tensor, grads: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if grads is None:
            grads = torch.empty(23 * max(self.last_n, 1), dtype=torch.float64, device=dl_dimage.device)
        _lib.check(_lib.lib().glod_render_backward(self._h, _lib.ptr(dl_dimage.contiguous()),
                                                   _lib.ptr(grads), _lib.stream_ptr(stream)))
        return grads

    def blend_timing(self, enable: bool | None = None) -> dict:
        """CUDA-event durations of the blend kernels since the last call
        (measurement only); `enable` then resets and switches timing."""
        ms = (C.c_double * 3)()
        n = (C.c_int64 * 3)()
        _lib.check(_lib.lib().glod_render_kernel_timing(self._h, -1 if enable is None else int(bool(enable)),
                                                        ms, n))
        return {"fwd_ms": ms[0], "bwd_ms": ms[1], "fwd_launches": n[0], "bwd_launches": n[1],
                "pre_ms": ms[2], "pre_launches": n[2]}

    def stats(self) -> dict:
        s = _lib.RenderStats()
        _lib.check(_lib.lib().glod_render_stats_get(self._h, C.byref(s)))
        return {"n_gaussians": s.n_gaussians, "n_instances": s.n_instances,
                "tiles": (s.tiles_x, s.tiles_y), "depth_full_sort": bool(s.depth_full_sort)}

    def loss(self, rendered: torch.Tensor, target: torch.Tensor, lam: float = 0.2,
             value: torch.Tensor | None = None, grad: torch.Tensor | None = None, stream=None):
        h, w, _ = rendered.shape
        need = int(_lib.lib().glod_loss_scratch_bytes(w, h))
        if self._loss_scratch is None or self._loss_scratch.numel() < need:
            self._loss_scratch = torch.empty(need, dtype=torch.uint8, device=rendered.device)
        if value is None:
            value = torch.empty(3, dtype=torch.float64, device=rendered.device)
        if grad is None:
            grad = torch.empty_like(rendered)
        _lib.check(_lib.lib().glod_loss_l1_ssim(_lib.ptr(rendered), _lib.ptr(target), w, h, float(lam),
                                                _lib.ptr(value), _lib.ptr(grad),
                                                _lib.ptr(self._loss_scratch), self._loss_scratch.numel(),
                                                _lib.stream_ptr(stream)))
        return value, grad


_RAST: dict = {}


def _rasterizer() -> Rasterizer:
    dev = torch.cuda.current_device()
    r = _RAST.get(dev)
    if r is None:
        r = _RAST[dev] = Rasterizer()
    return r


def _packed_device(attrs) -> tuple[torch.Tensor, int]:
    a = attrs if isinstance(attrs, AttributeArrays) else AttributeArrays(
        attrs.means, attrs.scales, attrs.rotations, attrs.opacities, attrs.base_colors, attrs.sh_rest)
    n = len(a)
    if a.sh_rest.ndim != 2 or a.sh_rest.shape[1] != 9:
        sh = np.zeros((n, 9))
        k = min(9, a.sh_rest.shape[1] if a.sh_rest.ndim == 2 else 0)
        sh[:, :k] = a.sh_rest[:, :k]
        a = AttributeArrays(a.means, a.scales, a.rotations, a.opacities, a.base_colors, sh)
    buf = torch.from_numpy(a.packed(np.float64)).cuda()
    return buf, n


def render_forward(attrs, cam) -> RenderContext:
    """Drop-in for renderer.render_forward (renderer.py:117-166)."""
    cam = Camera.from_any(cam)
    buf, n = _packed_device(attrs)
    r = _rasterizer()
    img = r.forward(buf, n, cam)
    ctx = RenderContext(attrs=attrs, cam=cam, image=img.double().cpu().numpy(), splats=[], _dev=r)
    ctx._packed = buf
    ctx._n = n
    return ctx


def render(attrs, cam) -> np.ndarray:
    return render_forward(attrs, cam).image


def backward(ctx: RenderContext, dl_dimage: np.ndarray) -> GaussianGradients:
    """Drop-in for renderer.backward (renderer.py:197-304)."""
    w, h = ctx.cam.resolution
    if dl_dimage.shape != (h, w, 3):
        raise InvalidInputError("upstream gradient does not match image size")
    n = ctx._n
    if n == 0:
        return GaussianGradients.zeros(0)
    r = ctx._dev
    if r.last_n != n or r._attrs is not ctx._packed:
        r.forward(ctx._packed, n, ctx.cam)      # restore forward state
    up = torch.from_numpy(np.ascontiguousarray(dl_dimage, dtype=np.float32)).cuda()
    g = r.backward(up)
    return GaussianGradients.from_packed(g.cpu().numpy(), n)


def loss(rendered: np.ndarray, target: np.ndarray, lam: float = 0.2):
    """Drop-in for renderer.loss (renderer.py:322-360); GPU fp64 windows."""
    if rendered.shape != target.shape:
        raise InvalidInputError("image dimensions differ")
    if not 0.0 <= lam <= 1.0:
        raise InvalidInputError("lambda must lie in [0, 1]")
    x = torch.from_numpy(np.ascontiguousarray(rendered, dtype=np.float32)).cuda()
    y = torch.from_numpy(np.ascontiguousarray(target, dtype=np.float32)).cuda()
    value, grad = _rasterizer().loss(x, y, lam)
    return float(value[0].item()), grad.double().cpu().numpy()


def psnr(rendered: np.ndarray, target: np.ndarray) -> float:
    mse = float(np.mean((np.asarray(rendered, dtype=np.float64) - np.asarray(target, dtype=np.float64)) ** 2))
    return float("inf") if mse == 0 else -10.0 * np.log10(mse)
