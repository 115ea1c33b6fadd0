"""Reference-facing rasterizer API (reference raster.py:39-432), backed by the
CUDA pipeline in engine.py.  Same names, argument meaning and errors:

* ``render_arrays(camera, arrays) -> Image``            (raster.py:194)
* ``render_arrays_backward(camera, arrays, grad_image, trainable=None) -> dict``
                                                          (raster.py:207-348)
* ``render`` / ``render_backward`` with lifespans       (raster.py:355-396)
* ``project(gaussian, camera) -> Splat2D | None``       (raster.py:176-191)

Arithmetic differences from the fp64 reference (documented tolerances, see
DESIGN.md): projection, cull, bbox and depth order are fp64; per-pixel
blending and its backward run in fp32.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from .core import (Camera, Gaussian, GaussianArrays, InvalidParameterError, Lifespan, SplatError,
                   is_active)
from .engine import Store, ViewPipeline, device

NEAR_PLANE = 0.01           # raster.py:31
COV2D_DILATION = 0.3        # raster.py:34
PSNR_IDENTICAL = math.inf   # raster.py:36
GRAD_KEYS = ("mean", "log_scale", "quat", "opacity_logit", "color")
# column slices of a 14-wide gradient row (include/swings.h)
GRAD_COLS = {"mean": slice(0, 3), "quat": slice(3, 7), "log_scale": slice(7, 10),
             "opacity_logit": 10, "color": slice(11, 14)}


class ConsistencyError(SplatError):
    """Forward and backward passes disagree about the active set (raster.py:39)."""


@dataclass(frozen=True)
class Splat2D:
    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    source_index: int


@dataclass
class Image:
    """(H, W, 3) float64 linear RGB (raster.py:55-73)."""

    pixels: np.ndarray

    def __post_init__(self):
        a = np.asarray(self.pixels, dtype=np.float64)
        if a.ndim != 3 or a.shape[2] != 3:
            raise InvalidParameterError(f"image must be (H, W, 3), got {a.shape}")
        self.pixels = a

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


_PIPE: ViewPipeline | None = None


def pipeline() -> ViewPipeline:
    global _PIPE
    if _PIPE is None:
        _PIPE = ViewPipeline()
    return _PIPE


def set_deterministic(flag: bool = True) -> None:
    """Fixed-order gradient accumulation in render_arrays_backward (no float
    atomics; bit-identical run to run, like the reference's single-threaded
    loops)."""
    pipeline().deterministic = bool(flag)


def set_alpha_floor(log2_floor: int | None = -28) -> None:
    """Alpha floor of the binning and rasterizer (ss_set_alpha_floor): blend
    a (splat, pixel) pair only when maha <= 64 (_kernels.py:39-41) and
    alpha G >= 2^log2_floor; each skipped contribution is below the floor,
    so images stay within ~2 |skipped| 2^floor of the reference (<= 3e-5 at
    the default -28).  None: the reference's rule alone."""
    from . import _lib as L

    v = 0 if log2_floor is None else int(log2_floor)
    L.check(L.lib().ss_set_alpha_floor(v), "set_alpha_floor")


def get_alpha_floor() -> int | None:
    from . import _lib as L

    v = int(L.lib().ss_get_alpha_floor())
    return None if v == 0 else v


def set_binning(mode: str = "counting") -> None:
    """Tile binning used by the forward: "counting" (default; chunked
    histograms + stable scatter, ss_bin_tiles) or "sort" (emit pairs + stable
    radix sort on tile ids).  Both give bit-identical tile lists."""
    modes = {"counting": 0, "sort": 1}
    if mode not in modes:
        raise InvalidParameterError(f"binning must be one of {sorted(modes)}, got {mode!r}")
    from . import _lib as L

    L.check(L.lib().ss_set_binning(modes[mode]), "set_binning")


def set_strips(forward: int = 4, backward: int = 4) -> None:
    """Pixels per lane of the raster kernels (2, 4 or 8; default 4): a warp
    covers 16 x (2 strip) pixels.  A tuning knob; results are unchanged
    within the fp32 tolerance (unequal strips disable the entry-use masks)."""
    from . import _lib as L

    L.check(L.lib().ss_set_raster_strips(int(forward), int(backward)), "set_raster_strips")


def _upload(arrays: GaussianArrays) -> Store:
    rows = torch.from_numpy(arrays.rows()).to(device())
    return Store(opt=None, mat=rows)


def render_arrays_device(camera: Camera, arrays: GaussianArrays) -> torch.Tensor:
    """render_arrays returning the float32 device image (no host copy)."""
    pipe = pipeline()
    return pipe.forward(_upload(arrays), None, len(arrays), camera)


def render_arrays(camera: Camera, arrays: GaussianArrays) -> Image:
    """Render already-active splats to a linear-RGB image (raster.py:194-204)."""
    if len(arrays) == 0:
        return Image(np.zeros((camera.height, camera.width, 3)))
    img = render_arrays_device(camera, arrays)
    return Image(img.double().cpu().numpy())


def render_arrays_backward(camera: Camera, arrays: GaussianArrays, grad_image: np.ndarray,
                           trainable: Optional[np.ndarray] = None) -> dict:
    """Optimization-space gradients of sum(grad_image * render) (raster.py:207-348)."""
    n = len(arrays)
    grad_image = np.ascontiguousarray(grad_image, dtype=np.float64)
    if grad_image.shape != (camera.height, camera.width, 3):
        raise InvalidParameterError(
            f"gradient image shape {grad_image.shape} does not match camera "
            f"({camera.height}, {camera.width}, 3)")
    out = {"mean": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "quat": np.zeros((n, 4)),
           "opacity_logit": np.zeros((n,)), "color": np.zeros((n, 3))}
    if n == 0:
        return out
    dev = device()
    pipe = pipeline()
    pipe.forward(_upload(arrays), None, n, camera)
    dimg = torch.from_numpy(grad_image.astype(np.float32)).to(dev)
    grads = torch.zeros((n, 14), dtype=torch.float32, device=dev)
    mask = None
    if trainable is not None:
        mask = torch.from_numpy(np.asarray(trainable, dtype=np.uint8)).to(dev)
    pipe.backward(dimg, grads, trainable_mask=mask, trainable_rows=n)
    g = grads.double().cpu().numpy()
    for k in GRAD_KEYS:
        out[k] = np.ascontiguousarray(g[:, GRAD_COLS[k]])
    return out


def project(gaussian: Gaussian, camera: Camera) -> Optional[Splat2D]:
    """Project one splat; None when culled (raster.py:176-191), through
    ss_project_splats (the same fp64 sequence as the batched projection)."""
    from . import _lib as L

    arr = GaussianArrays.from_gaussians([gaussian])
    rows = torch.from_numpy(arr.rows()).to(device())
    out = torch.empty((1, 7), dtype=torch.float64, device=device())
    store = Store(opt=None, mat=rows)
    cam = L.camera_struct(camera)
    L.check(L.lib().ss_project_splats(ctypes.byref(store.struct()), None, 1, ctypes.byref(cam),
                                      L.ptr(out), L.stream_ptr()), "project_splats")
    u, v, a, b, c, z, kept = out[0].cpu().numpy()
    if kept == 0.0:
        return None
    return Splat2D(mean2d=np.array([u, v]), cov2d=np.array([[a, b], [b, c]]), depth=float(z),
                   color=gaussian.color.copy(), opacity=float(gaussian.opacity), source_index=0)


def active_indices(gaussians: Sequence[Tuple[Gaussian, Lifespan]], frame: int) -> list:
    return [i for i, (_, ls) in enumerate(gaussians) if is_active(ls, frame)]


def render(camera: Camera, gaussians: Sequence[Tuple[Gaussian, Lifespan]], frame: int) -> Image:
    """Filter to the frame's active set, then blend (raster.py:355-359)."""
    idx = active_indices(gaussians, frame)
    return render_arrays(camera, GaussianArrays.from_gaussians([gaussians[i][0] for i in idx]))


def render_backward(camera: Camera, gaussians: Sequence[Tuple[Gaussian, Lifespan]], frame: int,
                    loss_gradient_image: np.ndarray, trainable: Optional[Sequence[bool]] = None,
                    expected_active: Optional[Sequence[int]] = None) -> dict:
    """Gradients aligned with the input list (raster.py:362-396)."""
    idx = active_indices(gaussians, frame)
    if expected_active is not None and list(expected_active) != idx:
        raise ConsistencyError("active set differs between forward and backward passes")
    arrays = GaussianArrays.from_gaussians([gaussians[i][0] for i in idx])
    sub_tr = None if trainable is None else np.asarray([trainable[i] for i in idx], dtype=bool)
    sub = render_arrays_backward(camera, arrays, loss_gradient_image, sub_tr)
    n = len(gaussians)
    out = {"mean": np.zeros((n, 3)), "log_scale": np.zeros((n, 3)), "quat": np.zeros((n, 4)),
           "opacity_logit": np.zeros((n,)), "color": np.zeros((n, 3))}
    if idx:
        sel = np.asarray(idx)
        for k in out:
            out[k][sel] = sub[k]
    return out


def psnr(a, b) -> float:
    """PSNR in dB over all channels; +inf when identical (raster.py:399-408)."""
    pa = a.pixels if isinstance(a, Image) else np.asarray(a, dtype=np.float64)
    pb = b.pixels if isinstance(b, Image) else np.asarray(b, dtype=np.float64)
    if pa.shape != pb.shape:
        raise InvalidParameterError(f"image dimensions differ: {pa.shape} vs {pb.shape}")
    mse = float(np.mean((pa - pb) ** 2))
    return PSNR_IDENTICAL if mse == 0.0 else 10.0 * math.log10(1.0 / mse)


def linear_to_srgb(x):
    """raster.py:411-413."""
    x = np.clip(x, 0.0, 1.0)
    return np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)


def srgb_to_linear(y):
    """raster.py:416-418."""
    y = np.clip(y, 0.0, 1.0)
    return np.where(y <= 0.04045, y / 12.92, np.power((y + 0.055) / 1.055, 2.4))


def srgb_u8_lut() -> np.ndarray:
    """Linear value of every 8-bit sRGB code (read_png's decode, raster.py:428-432)."""
    return srgb_to_linear(np.arange(256, dtype=np.float64) / 255.0)


def to_u8(image) -> np.ndarray:
    """write_png's quantisation (raster.py:421-425) without the PNG container."""
    px = image.pixels if isinstance(image, Image) else np.asarray(image, dtype=np.float64)
    return np.rint(linear_to_srgb(px) * 255.0).astype(np.uint8)


def write_png(image: Image, path) -> None:
    from PIL import Image as PILImage

    PILImage.fromarray(to_u8(image), mode="RGB").save(path, format="PNG")


def read_png_u8(path) -> np.ndarray:
    from PIL import Image as PILImage

    with PILImage.open(path) as im:
        return np.asarray(im.convert("RGB"), dtype=np.uint8)


def read_png(path) -> Image:
    return Image(srgb_to_linear(read_png_u8(path).astype(np.float64) / 255.0))
