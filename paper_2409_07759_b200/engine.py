"""Device-side per-view pipeline: projection -> binning -> raster forward,
and raster backward -> projection backward, over libswings.so.

This is the one place that sequences the C-ABI calls of a view; the
reference-facing API (raster.py, loss.py, train.py) and the trainer both go
through it.  Buffers are torch CUDA tensors grown on demand and reused.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
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


class Splats2D:
    """Device copies of _kernels' 2D splat arrays + the ss_splats2d struct."""

    def __init__(self, mean2d, inv2d, alpha, color, bbox, rank):
        self.t = [mean2d, inv2d, alpha, color, bbox, rank]  # keep alive
        self.n = int(alpha.numel())
        self.struct = L.SSSplats2D(L.ptr(mean2d), L.ptr(inv2d), L.ptr(alpha), L.ptr(color),
                                   L.ptr(bbox), L.ptr(rank), self.n, 0)


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
        self.deterministic = False  # fixed-order gradient sums (no float atomics)
        self.forward_only = False  # playback: no backward follows (ss_view.fwd_only)
        L.lib()

    def enable_timing(self, on: bool = True, sample: float = 1.0, seed: int = 0):
        """Record CUDA events around the raster kernels (inside the native
        driver, on the launch stream) for kernel_ms().  Event quads come from
        a pool that persists across calls (no event creation per view).

        `sample` < 1 times a seeded random subset of the views (each view with
        that probability): an event record between two kernels stops the
        second one launching early (PDL), so timing every view costs the step
        ~1.5 %; the sampled launches are an unbiased estimate of the mean."""
        self._event_pool = getattr(self, "_event_pool", [])
        self.events = {"_pending": []} if on else None
        self._sample = float(sample)
        self._sample_rng = np.random.default_rng(seed)

    def kernel_ms(self) -> dict:
        """Total milliseconds of raster_fwd / raster_bwd over the timed views,
        and under "views" how many views were timed (synchronizes)."""
        torch.cuda.synchronize()
        pend = (self.events or {}).get("_pending", [])
        out = {"raster_fwd": 0.0, "raster_bwd": 0.0, "views": len(pend)}
        ms = ctypes.c_float()
        for evs in (self.events or {}).get("_pending", []):
            for name, (a, b) in (("raster_fwd", (0, 1)), ("raster_bwd", (2, 3))):
                if L.lib().ss_event_elapsed_ms(evs[a], evs[b], ctypes.byref(ms)) == L.SS_OK:
                    out[name] += ms.value
        return out

    def _buf(self, name, shape, dtype):
        t = _grow(self._b.get(name), shape, dtype, self.dev)
        self._b[name] = t
        return t

    # ------------------------------------------------------------------ fwd
    def forward(self, store: Store, rows: torch.Tensor | None, n: int, cam, stream=None):
        """Project, bin and rasterize n active splats (row ids `rows`, or
        0..n-1 into `store` when rows is None) with one native call
        (ss_render_fwd).  Returns the (H, W, 3) float32 image (a view into an
        internal buffer)."""
        lib = L.lib()
        sp = L.stream_ptr(stream)
        self.cam_struct = L.camera_struct(cam)
        self.store, self.store_struct, self.rows = store, store.struct(), rows

        def call(v):
            v.rows = L.ptr(rows)
            v.n = n
            return lib.ss_render_fwd(ctypes.byref(self.store_struct),
                                     ctypes.byref(self.cam_struct), ctypes.byref(v), sp)

        return self._run_forward(n, int(cam.width), int(cam.height), call, stream)

    def forward2d(self, splats: "Splats2D", width: int, height: int, stream=None):
        """_kernels.blend_forward on device-resident 2D splats (ss_render2d_fwd)."""
        lib = L.lib()
        sp = L.stream_ptr(stream)
        self.splats2d = splats

        def call(v):
            v.rows = None
            v.n = splats.n
            return lib.ss_render2d_fwd(ctypes.byref(splats.struct), int(width), int(height),
                                       ctypes.byref(v), sp)

        return self._run_forward(splats.n, int(width), int(height), call, stream)

    def _run_forward(self, n: int, W: int, H: int, call, stream=None):
        # the previous forward's side-stream tile order may still read / write
        # buffers this call regrows: order it before any of them is freed
        L.check(L.lib().ss_side_sync(L.stream_ptr(stream)), "side_sync")
        tiles_x, tiles_y = (W + TILE - 1) // TILE, (H + TILE - 1) // TILE
        n_tiles = tiles_x * tiles_y
        self.n, self.width, self.height, self.n_tiles = n, W, H, n_tiles
        nn = max(n, 1)
        b = {}
        for name, shape, dt in (("rec_a", (nn, 4), torch.float32), ("rec_b", (nn, 4), torch.float32),
                                ("rec_c", (nn,), torch.float32), ("depth_key", (nn,), torch.int64),
                                ("bbox", (nn, 4), torch.int32), ("n_tiles", (nn,), torch.int32),
                                ("geom", (nn, 8), torch.float32), ("tile_mask", (nn,), torch.int64),
                                ("order", (nn,), torch.int32), ("offsets", (nn + 1,), torch.int32),
                                ("ranges", (n_tiles, 2), torch.int32),
                                ("tile_order", (n_tiles,), torch.int32),
                                ("img", (H * W * 3,), torch.float32),
                                ("t_final", (H * W,), torch.float32),
                                ("n_contrib", (H * W,), torch.int32)):
            b[name] = self._buf(name, shape, dt)
        if "keys" not in self._b:
            cap = max(1 << 16, 16 * nn)
            for name in ("keys", "vals", "keys_alt", "vals_alt"):
                self._b[name] = torch.empty(cap, dtype=torch.int32, device=self.dev)
            self._b["ws_bin"] = torch.empty(1 << 20, dtype=torch.uint8, device=self.dev)
        v = L.SSView()
        v.fwd_only = 1 if self.forward_only else 0
        if not self.forward_only:
            # the backward's basis-sum buffer: zero-filled by the forward on
            # the library's side stream (ss_view.g2d_pre), not at the
            # backward's start
            v.g2d_pre = L.ptr(self._buf("g2d", (nn, L.SS_G2D_ROW), torch.float32))
        timed = self.events is not None and (self._sample >= 1.0
                                             or self._sample_rng.random() < self._sample)
        for _ in range(4):
            for name in ("rec_a", "rec_b", "rec_c", "depth_key", "bbox", "n_tiles", "geom",
                         "tile_mask", "order", "offsets", "ranges", "tile_order", "img", "t_final",
                         "n_contrib"):
                setattr(v, name, L.ptr(b[name]))
            for name in ("keys", "vals", "keys_alt", "vals_alt"):
                setattr(v, name, L.ptr(self._b[name]))
            v.pair_cap = self._b["keys"].numel()
            # entry-use masks (forward -> backward), sized for the pair capacity
            words = int(L.lib().ss_raster_used_words(v.pair_cap, n_tiles))
            um = self._b.get("used")
            if um is None or um.numel() < words:
                if um is not None:
                    um.record_stream(stream if stream is not None else torch.cuda.current_stream())
                self._b["used"] = um = torch.empty(words, dtype=torch.int32, device=self.dev)
            v.used = L.ptr(um)
            v.used_cap = um.numel()
            v.ws = L.ptr(self._b["ws_bin"])
            v.ws_bytes = self._b["ws_bin"].numel()
            if timed:
                evs = self._new_events()
                for i in range(4):
                    v.events[i] = evs[i]
            rc = call(v)
            if rc in (L.SS_ERR_CAPACITY, L.SS_ERR_WORKSPACE) and timed:
                self.events["_pending"].pop()  # this attempt recorded nothing
            # kernels queued by the failed attempt may still use the old
            # buffers on `stream`: keep them alive in the caching allocator
            # until that stream passes this point
            s_ = stream if stream is not None else torch.cuda.current_stream()
            if rc == L.SS_ERR_CAPACITY:
                cap = int(v.n_pairs * 1.25) + 1024
                for name in ("keys", "vals", "keys_alt", "vals_alt"):
                    self._b[name].record_stream(s_)
                    self._b[name] = torch.empty(cap, dtype=torch.int32, device=self.dev)
                continue
            if rc == L.SS_ERR_WORKSPACE:
                self._b["ws_bin"].record_stream(s_)
                self._b["ws_bin"] = torch.empty(int(v.ws_needed * 1.25), dtype=torch.uint8,
                                                device=self.dev)
                continue
            L.check(rc, "render_fwd")
            break
        else:
            raise L.SwingsError("render_fwd: could not size buffers")
        self.view = v
        self.n_pairs = int(v.n_pairs)
        self.sel = int(v.sorted_sel)
        sk, sv = (("keys", "vals") if self.sel == 0 else ("keys_alt", "vals_alt"))
        self.sorted_keys, self.sorted_vals = self._b[sk], self._b[sv]
        return b["img"][: H * W * 3].view(H, W, 3)

    def backward2d(self, dimg: torch.Tensor, g_mean2d, g_inv2d, g_alpha, g_color, stream=None):
        """_kernels.blend_backward for the view forward2d left: adds into the
        fp64 device gradient arrays (ss_render2d_bwd)."""
        if self.n == 0 or self.n_pairs == 0:
            return
        g2d = self._buf("g2d", (self.n, L.SS_G2D_ROW), torch.float32)
        sp = self.splats2d
        L.check(L.lib().ss_render2d_bwd(ctypes.byref(sp.struct), self.width, self.height,
                                        ctypes.byref(self.view), L.ptr(dimg), L.ptr(g2d),
                                        L.ptr(g_mean2d), L.ptr(g_inv2d), L.ptr(g_alpha),
                                        L.ptr(g_color), L.stream_ptr(stream)), "render2d_bwd")

    def _new_events(self):
        pending = self.events.setdefault("_pending", [])
        if len(pending) < len(self._event_pool):
            evs = self._event_pool[len(pending)]
        else:
            evs = []
            for _ in range(4):
                e = ctypes.c_void_p()
                L.check(L.lib().ss_event_create(ctypes.byref(e)), "event_create")
                evs.append(e.value)
            self._event_pool.append(evs)
        pending.append(evs)
        return evs

    # ------------------------------------------------------------------ bwd
    def backward(self, dimg: torch.Tensor, grads: torch.Tensor, trainable_mask=None,
                 trainable_rows: int | None = None, stream=None):
        """Accumulate optimization-space gradients of sum(dimg * image) into
        `grads` (rows x 14 float32, indexed by row id) with one native call
        (ss_render_bwd): every active trainable row is written (zeros when it
        reaches no pixel); rows outside the view are left to the caller."""
        n = self.n
        if n == 0:
            return
        g2d = self._buf("g2d", (n, L.SS_G2D_ROW), torch.float32)
        if self.deterministic and self.n_pairs > 0:
            nf = int(L.lib().ss_raster_partial_floats(self.n_pairs))
            part = self._buf("partial", (max(nf, 1),), torch.float32)
            rank = self._buf("rank", (max(n, 1),), torch.int32)
            self.view.partial, self.view.rank = L.ptr(part), L.ptr(rank)
        else:
            self.view.partial, self.view.rank = None, None
        if trainable_rows is None:
            trainable_rows = self.store.n_opt + self.store.n_mat
        L.check(L.lib().ss_render_bwd(ctypes.byref(self.store_struct), ctypes.byref(self.cam_struct),
                                      ctypes.byref(self.view), L.ptr(dimg), L.ptr(g2d),
                                      L.ptr(trainable_mask), int(trainable_rows), L.ptr(grads),
                                      L.stream_ptr(stream)), "render_bwd")

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
            # tile id of every list entry, from the ranges (both binning paths
            # leave the lists contiguous in tile order)
            rg = b["ranges"][: self.n_tiles].long()
            lens = (rg[:, 1] - rg[:, 0]).clamp(min=0)
            out["keys"] = torch.repeat_interleave(
                torch.arange(self.n_tiles, device=rg.device), lens).to(torch.int32).cpu()
            out["vals"] = self.sorted_vals[: self.n_pairs].cpu()
            out["ranges"] = b["ranges"][: self.n_tiles].cpu()
        return out


class LossBuffers:
    """Workspace for ss_loss_l1_ssim.  The two loss sums alternate between two
    device slots, so a reader copying one view's sums (e.g. to the host on a
    side stream, read back one view later) never races the next view's loss."""

    def __init__(self):
        self.dev = device()
        self._ws = None
        self._dimg = None
        self._sums = [torch.zeros(2, dtype=torch.float64, device=self.dev) for _ in range(2)]
        self._k = 0
        self.sums = self._sums[0]

    def run(self, pred: torch.Tensor, H: int, W: int, gt_u8=None, lut=None, gt_f32=None,
            ssim_weight: float = 0.2, stream=None):
        lib = L.lib()
        need = int(lib.ss_loss_workspace_bytes(W, H))
        self._ws = _grow(self._ws, (need,), torch.uint8, self.dev)
        self._dimg = _grow(self._dimg, (H * W * 3,), torch.float32, self.dev)
        self._k ^= 1
        self.sums = self._sums[self._k]
        L.check(lib.ss_loss_l1_ssim(L.ptr(pred), L.ptr(gt_u8), L.ptr(lut), L.ptr(gt_f32), W, H,
                                    float(ssim_weight), L.ptr(self._dimg), L.ptr(self.sums),
                                    L.ptr(self._ws), self._ws.numel(), L.stream_ptr(stream)),
                "loss_l1_ssim")
        return self._dimg[: H * W * 3].view(H, W, 3), self.sums
