"""ABR tail-drop subsampling (reference server.py:39-79) on
the GPU, with the reference's names, arguments and errors:

* ``abr_keep_indices(opacities, fraction)`` -- ascending indices of the
  ceil(fraction n) highest opacities, ties to the lower index (server.py:39-50)
* ``abr_subsample(records, fraction)`` -- (kept GaussianArrays, kept count)
  (server.py:53-56)
* ``subsample_slice_bytes(slice_bytes, fraction, profile)`` -- the wire-level
  tail drop: the kept records' original bytes under a new slice header
  (server.py:59-79)
* ``subsample_records_device(payload, n, profile, fraction)`` -- the same on a
  device-resident payload (a slice served from HBM), no host round trip.

The selection is one CTA of ``ss_abr_select`` (csrc/abr.cu): a radix select of
the threshold opacity, then an index-order compaction; no CPU fallback.
"""

from __future__ import annotations

import math
from typing import Tuple

import numpy as np
import torch

from . import _lib as L
from .codec import HEADER_SIZE, SliceHeader
from .core import GaussianArrays, InvalidParameterError
from .engine import device

# profile id -> (key kind, opacity byte offset) inside a wire record
_OPACITY_FIELD = {0: (L.SS_ABR_F32, 40), 1: (L.SS_ABR_U8, 16)}


def _check_fraction(fraction: float) -> None:
    if not (0.0 < fraction <= 1.0):
        raise InvalidParameterError(f"fraction {fraction} outside (0, 1]")


def _select(src: torch.Tensor, n: int, kind: int, stride: int, offset: int, kept_n: int,
            gather: bool):
    idx = torch.empty(max(kept_n, 1), dtype=torch.int32, device=src.device)
    out = torch.empty(max(kept_n, 1) * stride, dtype=torch.uint8, device=src.device) \
        if gather else None
    L.check(L.lib().ss_abr_select(L.ptr(src), n, kind, stride, offset, kept_n, L.ptr(idx),
                                  L.ptr(out), L.stream_ptr()), "abr_select")
    return idx[:kept_n], (out[: kept_n * stride] if gather else None)


def abr_keep_indices(opacities, fraction: float) -> np.ndarray:
    """Indices (ascending, so wire order is preserved) of the
    ceil(fraction * n) highest-opacity records; opacity ties keep the lower
    index (server.py:39-50)."""
    _check_fraction(fraction)
    op = np.ascontiguousarray(opacities, dtype=np.float64).reshape(-1)
    n = len(op)
    kept_n = int(math.ceil(fraction * n))
    if kept_n >= n:
        return np.arange(n)
    src = torch.from_numpy(op).to(device())
    idx, _ = _select(src, n, L.SS_ABR_F64, 8, 0, kept_n, gather=False)
    return idx.cpu().numpy().astype(np.int64)


def abr_subsample(records: GaussianArrays, fraction: float) -> Tuple[GaussianArrays, int]:
    """Tail-drop a decoded slice; returns (kept records, kept_count)
    (server.py:53-56)."""
    keep = abr_keep_indices(records.opacities, fraction)
    return records.take(keep), len(keep)


def subsample_records_device(payload: torch.Tensor, n: int, profile, fraction: float):
    """Kept record bytes (uint8 CUDA tensor, wire order) and kept count for a
    device-resident payload of n records of `profile`."""
    kind, offset = _OPACITY_FIELD[profile.profile_id]
    size = profile.bytes_per_record
    if payload.numel() != n * size:
        raise InvalidParameterError("slice payload does not match its header")
    if fraction >= 1.0:
        return payload, n
    _check_fraction(fraction)
    kept_n = int(math.ceil(fraction * n))
    if kept_n >= n:
        return payload, n
    _, out = _select(payload, n, kind, size, offset, kept_n, gather=True)
    return out, kept_n


def subsample_slice_bytes(slice_bytes: bytes, fraction: float, profile) -> bytes:
    """Tail-drop at the wire level: select original record bytes so the kept
    records are bit-identical to the full-quality slice (server.py:59-79)."""
    header = SliceHeader.from_bytes(slice_bytes)
    payload = slice_bytes[HEADER_SIZE:]
    size = profile.bytes_per_record
    if len(payload) % size or len(payload) // size != header.kept_count:
        raise InvalidParameterError("slice payload does not match its header")
    if fraction >= 1.0:
        return slice_bytes
    _check_fraction(fraction)
    n = header.kept_count
    dev = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(device()) if n else \
        torch.empty(0, dtype=torch.uint8, device=device())
    kept, kept_n = subsample_records_device(dev, n, profile, fraction)
    new_header = SliceHeader(target_frame=header.target_frame, slice_index=header.slice_index,
                             kept_count=kept_n)
    return new_header.to_bytes() + kept.cpu().numpy().tobytes()
