"""Render-only playback path (reference player.py:52-118).

``PlayerBuffer`` keeps the reference's slot semantics (swin_size slots of
slice_size decoded splats, one slot replaced per frame, render order
(birth, slot) with padding dropped) and mirrors the slots into a GPU store:

  rows   (swin * slice, 14) f64 direct space, slot s = rows [s*slice, (s+1)*slice)
  start / expire per row: the slot's lifespan for kept records, (0, 0) for
                          inert padding (never active)

so a frame renders as ss_compact_active over the slots in (birth, slot) order
followed by the forward rasterizer -- no host arrays.  Slices can be applied
from already-decoded payloads (the reference's UpdateEvent) or from raw slice
bytes decoded on the GPU (``apply_bytes``, ss_decode_records).

The reader thread, wall-clock pacing, HTTP source and PNG output of
``start_player`` (player.py:228-362) are outside the hot path.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .codec import DecodedSlice, HEADER_SIZE, QuantProfile, SliceHeader
from .core import Camera, GaussianArrays, Lifespan, SplatError, is_active, slice_slot


class ProtocolError(SplatError):
    """Stream protocol violation (player.py:31)."""


@dataclass
class UpdateEvent:
    target_frame: int
    slot: int
    payload: DecodedSlice


class _Slot:
    """One slot's splats.  Slots filled from wire bytes on the GPU keep only
    the device rows; the host GaussianArrays (API compatibility:
    active_arrays, uploads) are materialised on first access."""

    def __init__(self, arrays: Optional[GaussianArrays], valid: np.ndarray, lifespan: Lifespan,
                 make_arrays=None):
        self._arrays = arrays
        self._make = make_arrays
        self.valid = valid
        self.n_valid = int(np.count_nonzero(valid))  # counted once, not per rendered frame
        self.lifespan = lifespan

    @property
    def arrays(self) -> GaussianArrays:
        if self._arrays is None:
            self._arrays = self._make()
            self._make = None
        return self._arrays


class _DeviceSlots:
    def __init__(self, swin: int, slice_size: int):
        import torch

        from . import _lib as L
        from .engine import ViewPipeline, device

        self.L, self.torch = L, torch
        self.swin, self.sl = swin, slice_size
        dev = device()
        n = swin * slice_size
        self.rows = torch.zeros((n, 14), dtype=torch.float64, device=dev)
        self.start = torch.zeros(n, dtype=torch.int32, device=dev)
        self.expire = torch.zeros(n, dtype=torch.int32, device=dev)
        self.blk_map = torch.zeros(swin, dtype=torch.int32, device=dev)
        self.active_rows = torch.empty(n, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(2, dtype=torch.int32, device=dev)
        self.ws = torch.empty(int(L.lib().ss_compact_workspace_bytes(n)), dtype=torch.uint8,
                              device=dev)
        self.pipe = ViewPipeline()
        self.pipe.forward_only = True  # playback renders never run a backward

    def set_slot(self, slot: int, rows, kept: int, lifespan: Lifespan):
        r0 = slot * self.sl
        if rows is not None:
            self.rows[r0:r0 + rows.shape[0]].copy_(rows)
        self.start[r0:r0 + self.sl].zero_()
        self.expire[r0:r0 + self.sl].zero_()
        self.start[r0:r0 + kept].fill_(lifespan.start)
        self.expire[r0:r0 + kept].fill_(lifespan.expire)

    def render(self, order: List[int], n_active: int, frame: int, camera: Camera):
        from .engine import Store

        L = self.L
        from .device_model import write_small

        write_small(self.blk_map, np.asarray(order, dtype=np.int32))
        L.check(L.lib().ss_compact_active(L.ptr(self.start), L.ptr(self.expire), 0,
                                          self.swin * self.sl, L.ptr(self.blk_map), self.sl, frame,
                                          L.ptr(self.active_rows), L.ptr(self.counts),
                                          L.ptr(self.ws), self.ws.numel(), L.stream_ptr()),
                "compact_active")
        return self.pipe.forward(Store(opt=None, mat=self.rows), self.active_rows, n_active, camera)


class PlayerBuffer:
    """swin_size slots of slice_size decoded splats plus a frame counter
    (player.py:52-100).  Slot replacement is atomic w.r.t. rendering."""

    def __init__(self, init_slices: Sequence[DecodedSlice], swin_size: int):
        if len(init_slices) != swin_size:
            raise ProtocolError(
                f"genesis block has {len(init_slices)} slices, expected {swin_size}")
        self.swin_size = swin_size
        self._lock = threading.Lock()
        self.slots: List[_Slot] = [_Slot(s.gaussians, s.valid, s.lifespan) for s in init_slices]
        self.frame = 0
        self._dev: Optional[_DeviceSlots] = None

    # ---------------------------------------------------------- reference API
    def apply(self, event: UpdateEvent) -> None:
        if event.slot != slice_slot(event.target_frame, self.swin_size):
            raise ProtocolError(f"slot {event.slot} does not match target frame "
                                f"{event.target_frame} mod {self.swin_size}")
        s = event.payload
        with self._lock:
            self.slots[event.slot] = _Slot(s.gaussians, s.valid, s.lifespan)
            if self._dev is not None:
                self._upload(event.slot)

    def advance(self, frame: int) -> None:
        with self._lock:
            if frame < self.frame:
                raise ProtocolError("frame counter may not move backwards")
            self.frame = frame

    def _order(self, frame: int):
        entries = [(s.lifespan.birth, i) for i, s in enumerate(self.slots)
                   if is_active(s.lifespan, frame)]
        entries.sort()
        return [i for _, i in entries]

    def active_arrays(self, frame: Optional[int] = None) -> GaussianArrays:
        """Active, non-padding splats in (birth, slot) order (player.py:88-100)."""
        with self._lock:
            frame = self.frame if frame is None else frame
            order = self._order(frame)
            parts = [self.slots[i].arrays.take(np.nonzero(self.slots[i].valid)[0]) for i in order]
        return GaussianArrays.concat(parts)

    # ------------------------------------------------------------ device path
    def to_device(self) -> "_DeviceSlots":
        if self._dev is None:
            sl = max(len(s.valid) for s in self.slots)
            self._dev = _DeviceSlots(self.swin_size, sl)
            for i in range(self.swin_size):
                self._upload(i)
        return self._dev

    def _upload(self, slot: int):
        import torch

        s = self.slots[slot]
        kept_idx = np.nonzero(s.valid)[0]
        rows = torch.from_numpy(s.arrays.take(kept_idx).rows()).to(self._dev.rows.device)
        self._dev.set_slot(slot, rows, len(kept_idx), s.lifespan)

    def apply_bytes(self, raw: bytes, profile: QuantProfile, params) -> None:
        """Apply one slice straight from its wire bytes, decoding the records
        on the GPU (codec.py:323-350 semantics for kept records)."""
        from .codec import decode_records_device

        header = SliceHeader.from_bytes(raw)
        if header.kept_count > params.slice_size:
            raise ProtocolError(f"kept_count {header.kept_count} exceeds slice size")
        need = header.kept_count * profile.bytes_per_record
        rows = decode_records_device(raw[HEADER_SIZE:HEADER_SIZE + need], profile,
                                     header.kept_count)
        t = header.target_frame
        lifespan = Lifespan(t, t, t + params.swin_size)
        slot = slice_slot(t, self.swin_size)
        dev = self.to_device()
        kept = header.kept_count
        pad = params.slice_size - kept
        valid = np.zeros(params.slice_size, dtype=bool)
        valid[:kept] = True

        def host_arrays():
            from .codec import decode_records

            host = GaussianArrays.from_rows(rows.cpu().numpy()) if kept else GaussianArrays.empty()
            if pad:
                host = GaussianArrays.concat([host, decode_records(
                    b"\x00" * (pad * profile.bytes_per_record), profile, pad)])
            return host

        with self._lock:
            self.slots[slot] = _Slot(None, valid, lifespan, host_arrays)
            dev.set_slot(slot, rows, kept, lifespan)

    def render_device_u8(self, camera: Camera, frame: Optional[int] = None, out=None):
        """(H, W, 3) uint8 sRGB CUDA frame (write_png's quantisation) for display."""
        import torch

        from . import _lib as L

        img = self.render_device(camera, frame)
        if out is None:
            out = torch.empty(img.shape, dtype=torch.uint8, device=img.device)
        L.check(L.lib().ss_to_srgb_u8(L.ptr(img), img.numel(), L.ptr(out), L.stream_ptr()),
                "to_srgb_u8")
        return out

    def render_device(self, camera: Camera, frame: Optional[int] = None):
        """(H, W, 3) float32 CUDA image of `frame` (default: the buffer's frame)."""
        dev = self.to_device()
        with self._lock:
            frame = self.frame if frame is None else frame
            order = self._order(frame)
            n = sum(self.slots[i].n_valid for i in order)
            return dev.render(order, n, frame, camera)


def apply_update(buffer: PlayerBuffer, event: UpdateEvent) -> None:
    buffer.apply(event)


def render_frame(buffer: PlayerBuffer, camera: Camera):
    """Render the buffer's current frame (player.py:107-108) on the GPU."""
    from .raster import Image

    return Image(buffer.render_device(camera).double().cpu().numpy())


def render_offline(generations: Sequence[DecodedSlice], camera: Camera, frame: int):
    """Reference render of a frame from a container's generation set
    (player.py:111-118)."""
    from .raster import render_arrays

    parts = [g.gaussians.take(np.nonzero(g.valid)[0]) for g in generations
             if is_active(g.lifespan, frame)]
    return render_arrays(camera, GaussianArrays.concat(parts))
