"""ctypes binding of libswings.so (include/swings.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, ``lib()`` raises.  Torch tensors only provide device memory and the
current stream; every call passes raw pointers and sizes.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, Structure, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

import os

from ._build import VARIANTS, build, needs_build
from .core import InvalidParameterError

SS_OK, SS_ERR_INVALID, SS_ERR_CUDA, SS_ERR_CAPACITY, SS_ERR_WORKSPACE = 0, 1, 2, 3, 4
SS_ROW = 14
SS_GRAD_ROW = 14
SS_G2D_ROW = 12
SS_TILE = 16
SS_ABR_F32, SS_ABR_U8, SS_ABR_F64 = 0, 1, 2


class SSCamera(Structure):
    _fields_ = [("width", c_int32), ("height", c_int32), ("fx", c_double), ("fy", c_double),
                ("cx", c_double), ("cy", c_double), ("rot", c_double * 9), ("trans", c_double * 3)]


class SSStore(Structure):
    _fields_ = [("opt", c_void_p), ("n_opt", c_int64), ("mat", c_void_p), ("n_mat", c_int64)]


class SSGenStep(Structure):
    _fields_ = [("active", c_int32), ("pad", c_int32), ("bc1", c_double), ("bc2", c_double),
                ("gscale", c_double)]


class SSStepHyper(Structure):
    _fields_ = [("lr", c_double * 5), ("beta1", c_double), ("beta2", c_double), ("eps", c_double),
                ("opacity_reg", c_double), ("scale_reg", c_double), ("n_reg", c_double),
                ("noise_scale", c_double), ("gate_center", c_double),
                ("gate_sharpness", c_double), ("sgd", c_int32), ("sgld", c_int32),
                ("seed", c_uint64), ("counter", c_uint64)]


P = c_void_p
I32 = c_int32
I64 = c_int64


class SSView(Structure):
    _fields_ = [("rows", P), ("n", c_int32), ("pad0", c_int32), ("rec_a", P), ("rec_b", P),
                ("rec_c", P), ("depth_key", P), ("bbox", P), ("n_tiles", P), ("geom", P),
                ("tile_mask", P), ("order", P), ("offsets", P), ("keys", P), ("vals", P),
                ("keys_alt", P), ("vals_alt", P), ("pair_cap", c_int64), ("ranges", P),
                ("tile_order", P), ("img", P), ("t_final", P), ("n_contrib", P), ("ws", P),
                ("ws_bytes", c_size_t), ("ws_needed", c_size_t), ("n_pairs", c_int64),
                ("sorted_sel", c_int32), ("pad1", c_int32), ("events", P * 4),
                ("partial", P), ("rank", P), ("used", P), ("used_cap", c_int64),
                ("used_ok", c_int32), ("fwd_only", c_int32), ("order_ready", P), ("g2d_pre", P)]

class SSSplats2D(Structure):
    _fields_ = [("mean2d", P), ("inv2d", P), ("alpha", P), ("color", P), ("bbox", P),
                ("rank", P), ("n", c_int32), ("pad", c_int32)]


_SIGNATURES = {
    "ss_last_error": ([], ctypes.c_char_p),
    "ss_version": ([], c_int),
    "ss_device_sm_count": ([], c_int),
    "ss_compact_workspace_bytes": ([I64], c_size_t),
    "ss_compact_active": ([P, P, I64, I64, P, I32, I32, P, P, P, c_size_t, P], c_int),
    "ss_project_fwd": ([POINTER(SSStore), P, I32, POINTER(SSCamera), P, P, P, P, P, P, P, P, P],
                       c_int),
    "ss_binning_workspace_bytes": ([I32, I64, I32], c_size_t),
    "ss_depth_order": ([P, I32, P, P, c_size_t, P], c_int),
    "ss_tile_offsets": ([P, P, I32, P, P, c_size_t, P], c_int),
    "ss_emit_tile_pairs": ([P, P, P, P, P, I32, I32, P, P, P], c_int),
    "ss_sort_tile_pairs": ([P, P, P, P, I64, I32, POINTER(I32), P, c_size_t, P], c_int),
    "ss_tile_ranges": ([P, I64, I32, P, P], c_int),
    "ss_tile_order_workspace_bytes": ([I32], c_size_t),
    "ss_tile_order": ([P, I32, P, P, c_size_t, P], c_int),
    "ss_raster_fwd": ([P, P, P, P, P, I32, I32, P, P, P, P, P], c_int),
    "ss_raster_bwd": ([P, P, P, P, P, I32, I32, P, P, P, P, P, P], c_int),
    "ss_set_raster_strip": ([I32], c_int),
    "ss_set_raster_strips": ([I32, I32], c_int),
    "ss_set_binning": ([I32], c_int),
    "ss_get_binning": ([], c_int),
    "ss_set_alpha_floor": ([I32], c_int),
    "ss_write_small": ([P, P, c_size_t, P], c_int),
    "ss_raster_used_words": ([I64, I32], I64),
    "ss_project_splats": ([P, P, I32, P, P, P], c_int),
    "ss_reg_grads": ([P, P, I32, c_double, c_double, P, P, P, P], c_int),
    "ss_poll_wait_ns": ([], c_uint64),
    "ss_get_alpha_floor": ([], I32),
    "ss_bin_tiles_workspace_bytes": ([I64, I32], c_size_t),
    "ss_bin_tiles_supported": ([I64, I32], I32),
    "ss_bin_tiles": ([P, P, P, P, P, I32, I64, I32, I32, P, P, P, P, P, c_size_t, P], c_int),
    "ss_raster_partial_floats": ([I64], c_int64),
    "ss_raster_bwd_deterministic": ([P, P, P, P, P, I32, I32, P, P, P, P, P, P, P, P, P, I32, P, P,
                                     P, P], c_int),
    "ss_project_bwd": ([POINTER(SSStore), P, I32, POINTER(SSCamera), P, P, P, I64, P, P], c_int),
    "ss_loss_workspace_bytes": ([I32, I32], c_size_t),
    "ss_loss_l1_ssim": ([P, P, P, P, I32, I32, c_double, P, P, P, c_size_t, P], c_int),
    "ss_adam_sgld_step": ([P, P, P, P, I64, I32, P, POINTER(SSStepHyper), P, P], c_int),
    "ss_sgld": ([P, I64, I32, P, POINTER(SSStepHyper), P, P], c_int),
    "ss_relocate_workspace_bytes": ([I64], c_size_t),
    "ss_relocate": ([P, P, P, I64, I32, P, c_double, P, c_uint64, c_uint64, P, P, c_size_t, P],
                    c_int),
    "ss_to_direct": ([P, P, I64, P], c_int),
    "ss_memzero": ([P, c_size_t, P], c_int),
    "ss_to_srgb_u8": ([P, I64, P, P], c_int),
    "ss_render_fwd": ([POINTER(SSStore), POINTER(SSCamera), POINTER(SSView), P], c_int),
    "ss_render2d_fwd": ([POINTER(SSSplats2D), I32, I32, POINTER(SSView), P], c_int),
    "ss_render2d_bwd": ([POINTER(SSSplats2D), I32, I32, POINTER(SSView), P, P, P, P, P, P, P],
                        c_int),
    "ss_records_2d": ([POINTER(SSSplats2D), I32, I32, P, P, P, P, P, P, P, P, P], c_int),
    "ss_basis_to_2d": ([P, POINTER(SSSplats2D), P, P, P, P, P, P, P], c_int),
    "ss_render_bwd": ([POINTER(SSStore), POINTER(SSCamera), POINTER(SSView), P, P, P, I64, P, P],
                      c_int),
    "ss_side_sync": ([P], c_int),
    "ss_event_create": ([POINTER(P)], c_int),
    "ss_event_destroy": ([P], c_int),
    "ss_event_elapsed_ms": ([P, P, POINTER(ctypes.c_float)], c_int),
    "ss_encode_records": ([P, I64, I32, P, P, P], c_int),
    "ss_decode_records": ([P, I64, I32, P, P], c_int),
    "ss_abr_select": ([P, I64, I32, I32, I32, I64, P, P, P], c_int),
}

_LIB = None


class SwingsError(RuntimeError):
    """A CUDA-side failure reported by libswings.so."""


def lib():
    """Load libswings.so (building it first when sources are newer).
    SS_LIB_VARIANT=checked loads the bounds-checked build instead."""
    global _LIB
    if _LIB is None:
        variant = os.environ.get("SS_LIB_VARIANT", "")
        if needs_build(variant):
            build(variant=variant)
        handle = ctypes.CDLL(str(VARIANTS[variant][0]))
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = handle
    return _LIB


def exported_symbols():
    return list(_SIGNATURES)


def check(rc: int, what: str = "") -> None:
    if rc == SS_OK:
        return
    msg = lib().ss_last_error().decode(errors="replace")
    if rc == SS_ERR_INVALID:
        raise InvalidParameterError(f"{what}: {msg}")
    raise SwingsError(f"{what}: rc={rc}: {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def camera_struct(cam) -> SSCamera:
    c = SSCamera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    rot = [float(v) for v in cam.rotation.reshape(-1)]
    tr = [float(v) for v in cam.translation.reshape(-1)]
    c.rot = (c_double * 9)(*rot)
    c.trans = (c_double * 3)(*tr)
    return c
