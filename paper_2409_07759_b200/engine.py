"""Device-side per-view pipeline: projection -> binning -> raster forward,
and raster backward -> projection backward, over libswings.so.

This is the one place that sequences the C-ABI calls of a view; the
reference-facing API (raster.py, loss.py, train.py) and the trainer both go
through it.  Buffers are torch CUDA tensors grown on demand and reused.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib as L

TILE = L.SS_TILE


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2409_07759_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class Store:
    """Gaussian rows on the device: optimizable rows (log-scale, logit) and
    matured / direct-space rows (include/swings.h ss_store)."""

    opt: torch.Tensor | None
    mat: torch.Tensor | None

    @property
    def n_opt(self) -> int:
        return 0 if self.opt is None else int(self.opt.shape[0])

    @property
    def n_mat(self) -> int:
        return 0 if self.mat is None else int(self.mat.shape[0])

    def struct(self) -> L.SSStore:
        s = L.SSStore()
        s.opt = L.ptr(self.opt)
        s.n_opt = self.n_opt
        s.mat = L.ptr(self.mat)
        s.n_mat = self.n_mat
        return s


def _grow(t: torch.Tensor | None, shape, dtype, dev) -> torch.Tensor:
    n = shape[0]
    if t is None or t.shape[0] < n or t.dtype != dtype or tuple(t.shape[1:]) != tuple(shape[1:]):
        cap = max(n, 1)
        if t is not None and t.dtype == dtype and tuple(t.shape[1:]) == tuple(shape[1:]):
            cap = max(cap, int(t.shape[0] * 1.25))
        return torch.empty((cap, *shape[1:]), dtype=dtype, device=dev)
    return t


class ViewPipeline:
    """Reusable buffers + the call sequence for one view."""

    def __init__(self):
        self.dev = device()
        self._b = {}
        self.n = 0
        self.width = self.height = 0
        self.n_pairs = 0
        self.sel = 0
        self.events = None  # name -> [(start, end)] CUDA events when timing
        L.lib()

    def enable_timing(self, on: bool = True):
        self.events = {} if on else None

    def _mark(self, name):
        if self.events is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return (name, ev)

    def _done(self, tok):
        if tok is None:
            return
        name, start = tok
        end = torch.cuda.Event(enable_timing=True)
        end.record()
        self.events.setdefault(name, []).append((start, end))

    def kernel_ms(self) -> dict:
        """Total milliseconds per timed stage (synchronizes)."""
        torch.cuda.synchronize()
        return {k: sum(a.elapsed_time(b) for a, b in v) for k, v in (self.events or {}).items()}

    def _buf(self, name, shape, dtype):
        t = _grow(self._b.get(name), shape, dtype, self.dev)
        self._b[name] = t
        return t

    # ------------------------------------------------------------------ fwd
    def forward(self, store: Store, rows: torch.Tensor | None, n: int, cam, stream=None):
        """Project, bin and rasterize n active splats (row ids `rows`, or
        0..n-1 into `store` when rows is None).  Returns the (H, W, 3) float32
        image (a view into an internal buffer)."""
        lib = L.lib()
        sp = L.stream_ptr(stream)
        W, H = int(cam.width), int(cam.height)
        tiles_x, tiles_y = (W + TILE - 1) // TILE, (H + TILE - 1) // TILE
        n_tiles = tiles_x * tiles_y
        self.n, self.width, self.height = n, W, H
        self.n_tiles = n_tiles
        self.cam_struct = L.camera_struct(cam)
        self.store, self.store_struct, self.rows = store, store.struct(), rows
        nn = max(n, 1)
        rec_a = self._buf("rec_a", (nn, 4), torch.float32)
        rec_b = self._buf("rec_b", (nn, 4), torch.float32)
        rec_c = self._buf("rec_c", (nn,), torch.float32)
        dkey = self._buf("depth_key", (nn,), torch.int64)
        bbox = self._buf("bbox", (nn, 4), torch.int32)
        ntl = self._buf("n_tiles", (nn,), torch.int32)
        geom = self._buf("geom", (nn, 7), torch.float64)
        tmask = self._buf("tile_mask", (nn,), torch.int64)
        order = self._buf("order", (nn,), torch.int32)
        offsets = self._buf("offsets", (nn + 1,), torch.int32)
        ranges = self._buf("ranges", (n_tiles, 2), torch.int32)
        img = self._buf("img", (H * W * 3,), torch.float32)
        t_final = self._buf("t_final", (H * W,), torch.float32)
        n_contrib = self._buf("n_contrib", (H * W,), torch.int32)
        ws_bytes = int(lib.ss_binning_workspace_bytes(nn, 1, n_tiles))
        ws = self._buf("ws_bin", (ws_bytes,), torch.uint8)
        if n == 0:
            img[: H * W * 3].zero_()
            t_final[: H * W].fill_(1.0)
            n_contrib[: H * W].zero_()
            ranges.zero_()
            self.n_pairs = 0
            return img[: H * W * 3].view(H, W, 3)
        rp = L.ptr(rows)
        L.check(lib.ss_project_fwd(ctypes.byref(self.store_struct), rp, n, ctypes.byref(self.cam_struct),
                                   L.ptr(rec_a), L.ptr(rec_b), L.ptr(rec_c), L.ptr(dkey), L.ptr(bbox),
                                   L.ptr(ntl), L.ptr(geom), L.ptr(tmask), sp), "project_fwd")
        L.check(lib.ss_depth_order(L.ptr(dkey), n, L.ptr(order), L.ptr(ws), ws.numel(), sp),
                "depth_order")
        L.check(lib.ss_tile_offsets(L.ptr(order), L.ptr(ntl), n, L.ptr(offsets), L.ptr(ws),
                                    ws.numel(), sp), "tile_offsets")
        n_pairs = int(offsets[n].item())  # the one host sync of a view
        self.n_pairs = n_pairs
        pc = max(n_pairs, 1)
        keys = self._buf("keys", (pc,), torch.int32)
        vals = self._buf("vals", (pc,), torch.int32)
        keys_alt = self._buf("keys_alt", (pc,), torch.int32)
        vals_alt = self._buf("vals_alt", (pc,), torch.int32)
        ws_bytes = int(lib.ss_binning_workspace_bytes(nn, pc, n_tiles))
        ws = self._buf("ws_bin", (ws_bytes,), torch.uint8)
        L.check(lib.ss_emit_tile_pairs(L.ptr(order), L.ptr(offsets), L.ptr(bbox), L.ptr(geom),
                                       L.ptr(tmask), n, tiles_x, L.ptr(keys), L.ptr(vals), sp),
                "emit_tile_pairs")
        sel = ctypes.c_int32(0)
        L.check(lib.ss_sort_tile_pairs(L.ptr(keys), L.ptr(vals), L.ptr(keys_alt), L.ptr(vals_alt),
                                       n_pairs, n_tiles, ctypes.byref(sel), L.ptr(ws), ws.numel(),
                                       sp), "sort_tile_pairs")
        self.sel = sel.value
        sk, sv = (keys, vals) if sel.value == 0 else (keys_alt, vals_alt)
        self.sorted_keys, self.sorted_vals = sk, sv
        L.check(lib.ss_tile_ranges(L.ptr(sk), n_pairs, n_tiles, L.ptr(ranges), sp), "tile_ranges")
        tord = self._buf("tile_order", (n_tiles,), torch.int32)
        tws = self._buf("ws_tord", (int(lib.ss_tile_order_workspace_bytes(n_tiles)),), torch.uint8)
        L.check(lib.ss_tile_order(L.ptr(ranges), n_tiles, L.ptr(tord), L.ptr(tws), tws.numel(), sp),
                "tile_order")
        tok = self._mark("raster_fwd")
        L.check(lib.ss_raster_fwd(L.ptr(ranges), L.ptr(sv), L.ptr(rec_a), L.ptr(rec_b),
                                  L.ptr(rec_c), W, H, L.ptr(tord), L.ptr(img), L.ptr(t_final),
                                  L.ptr(n_contrib), sp), "raster_fwd")
        self._done(tok)
        return img[: H * W * 3].view(H, W, 3)

    # ------------------------------------------------------------------ bwd
    def backward(self, dimg: torch.Tensor, grads: torch.Tensor, trainable_mask=None,
                 trainable_rows: int | None = None, stream=None):
        """Accumulate optimization-space gradients of sum(dimg * image) into
        `grads` (rows x 14 float32, indexed by row id; caller zeroes)."""
        lib = L.lib()
        sp = L.stream_ptr(stream)
        n, W, H = self.n, self.width, self.height
        if n == 0 or self.n_pairs == 0:
            return
        g2d = self._buf("g2d", (n, L.SS_G2D_ROW), torch.float32)
        g2d[:n].zero_()
        b = self._b
        tok = self._mark("raster_bwd")
        L.check(lib.ss_raster_bwd(L.ptr(b["ranges"]), L.ptr(self.sorted_vals), L.ptr(b["rec_a"]),
                                  L.ptr(b["rec_b"]), L.ptr(b["rec_c"]), W, H,
                                  L.ptr(b["tile_order"]), L.ptr(dimg),
                                  L.ptr(b["t_final"]), L.ptr(b["n_contrib"]), L.ptr(g2d), sp),
                "raster_bwd")
        self._done(tok)
        if trainable_rows is None:
            trainable_rows = self.store.n_opt + self.store.n_mat
        L.check(lib.ss_project_bwd(ctypes.byref(self.store_struct), L.ptr(self.rows), n,
                                   ctypes.byref(self.cam_struct), L.ptr(g2d), L.ptr(b["depth_key"]),
                                   L.ptr(trainable_mask), int(trainable_rows), L.ptr(grads), sp),
                "project_bwd")

    def k_used(self) -> int:
        """SURVEY.md §8 K_used of the last view: per tile, the longest list
        prefix any pixel walked (its contributor prefix when it saturated,
        else the whole list), summed over tiles."""
        W, H, b = self.width, self.height, self._b
        if self.n_pairs == 0:
            return 0
        tx, ty = (W + TILE - 1) // TILE, (H + TILE - 1) // TILE
        rg = b["ranges"][: tx * ty].long()
        lens = (rg[:, 1] - rg[:, 0]).clamp(min=0)
        nc = b["n_contrib"][: W * H].view(H, W).long()
        sat = b["t_final"][: W * H].view(H, W) < 1e-4
        tile = ((torch.arange(H, device=nc.device) // TILE)[:, None] * tx
                + (torch.arange(W, device=nc.device) // TILE)[None, :])
        walked = torch.where(sat, nc, lens[tile])
        per = torch.zeros(tx * ty, dtype=torch.long, device=nc.device)
        per.scatter_reduce_(0, tile.reshape(-1), walked.reshape(-1), reduce="amax")
        return int(per.sum().item())

    # ------------------------------------------------------------ introspection
    def state(self) -> dict:
        """Host copies of the per-view intermediates (tests / diagnostics)."""
        n, b = self.n, self._b
        out = {
            "rec_a": b["rec_a"][:n].cpu(), "rec_b": b["rec_b"][:n].cpu(),
            "rec_c": b["rec_c"][:n].cpu(), "depth_key": b["depth_key"][:n].cpu(),
            "bbox": b["bbox"][:n].cpu(), "n_tiles": b["n_tiles"][:n].cpu(),
            "order": b["order"][:n].cpu(), "offsets": b["offsets"][: n + 1].cpu(),
            "n_pairs": self.n_pairs,
            "t_final": b["t_final"][: self.width * self.height].cpu(),
            "n_contrib": b["n_contrib"][: self.width * self.height].cpu(),
        }
        if self.n_pairs:
            out["keys"] = self.sorted_keys[: self.n_pairs].cpu()
            out["vals"] = self.sorted_vals[: self.n_pairs].cpu()
            out["ranges"] = b["ranges"][: self.n_tiles].cpu()
        return out


class LossBuffers:
    """Workspace for ss_loss_l1_ssim."""

    def __init__(self):
        self.dev = device()
        self._ws = None
        self._dimg = None
        self.sums = torch.zeros(2, dtype=torch.float64, device=self.dev)

    def run(self, pred: torch.Tensor, H: int, W: int, gt_u8=None, lut=None, gt_f32=None,
            ssim_weight: float = 0.2, stream=None):
        lib = L.lib()
        need = int(lib.ss_loss_workspace_bytes(W, H))
        self._ws = _grow(self._ws, (need,), torch.uint8, self.dev)
        self._dimg = _grow(self._dimg, (H * W * 3,), torch.float32, self.dev)
        L.check(lib.ss_loss_l1_ssim(L.ptr(pred), L.ptr(gt_u8), L.ptr(lut), L.ptr(gt_f32), W, H,
                                    float(ssim_weight), L.ptr(self._dimg), L.ptr(self.sums),
                                    L.ptr(self._ws), self._ws.numel(), L.stream_ptr(stream)),
                "loss_l1_ssim")
        return self._dimg[: H * W * 3].view(H, W, 3), self.sums
