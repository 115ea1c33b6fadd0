"""GPU-resident training state and the per-iteration step (train.py:374-417).

DeviceModel owns
  opt     (num_gs, 14) f64  optimizable rows, generation i = rows [i*sl, (i+1)*sl)
  m, v    (num_gs, 14) f64  Adam moments
  grads   (num_gs, 14) f32  optimization-space gradient (NCCL allreduce buffer)
  mat     ((swin+1)*sl, 14) f64  ring of matured, direct-space generations
  row_start / row_expire    per-row lifespans (opt rows, then matured ring rows)
and sequences the libswings.so calls of one training view.
"""

from __future__ import annotations

import ctypes
import logging

import numpy as np
import torch

from . import _lib as L
from .core import GaussianArrays
from .engine import LossBuffers, Store, ViewPipeline, device
from .raster import srgb_u8_lut

log = logging.getLogger("paper_2409_07759_b200.train")

GEN_DTYPE = np.dtype([("active", "<i4"), ("pad", "<i4"), ("bc1", "<f8"), ("bc2", "<f8"),
                      ("gscale", "<f8")])
assert GEN_DTYPE.itemsize == ctypes.sizeof(L.SSGenStep)
PARAM_KEYS = ("mean", "quat", "log_scale", "opacity_logit", "color")
COLS = {"mean": (0, 3), "quat": (3, 7), "log_scale": (7, 10), "opacity_logit": (10, 11),
        "color": (11, 14)}


def write_small(dst: torch.Tensor, host: np.ndarray) -> None:
    """Stream-ordered write of a small host array into device tensor `dst`
    (ss_write_small: the bytes travel as a kernel argument); falls back to a
    copy for tables over 2 KB."""
    host = np.ascontiguousarray(host)
    if host.nbytes <= 2048:
        L.check(L.lib().ss_write_small(L.ptr(dst), host.ctypes.data, host.nbytes, L.stream_ptr()),
                "write_small")
    else:
        dst.view(torch.uint8)[: host.nbytes].copy_(
            torch.from_numpy(host.view(np.uint8)).pin_memory(), non_blocking=True)
        torch.cuda.current_stream().synchronize()  # the pinned staging buffer is freed after


def _views(t: torch.Tensor) -> dict:
    out = {}
    for k, (a, b) in COLS.items():
        out[k] = t[:, a] if b - a == 1 else t[:, a:b]
    return out


def _pack(params: dict) -> np.ndarray:
    return np.concatenate([np.asarray(params["mean"]), np.asarray(params["quat"]),
                           np.asarray(params["log_scale"]),
                           np.asarray(params["opacity_logit"])[:, None],
                           np.asarray(params["color"])], axis=1).astype(np.float64)


def _unpack_into(params: dict, rows: np.ndarray) -> None:
    for k, (a, b) in COLS.items():
        src = rows[:, a] if b - a == 1 else rows[:, a:b]
        params[k][...] = src


def _hyper(cfg, n_reg: float, sgld: bool, seed: int, counter: int) -> L.SSStepHyper:
    h = L.SSStepHyper()
    h.lr = (ctypes.c_double * 5)(cfg.lr_mean, cfg.lr_quat, cfg.lr_log_scale,
                                 cfg.lr_opacity_logit, cfg.lr_color)
    h.beta1, h.beta2, h.eps = cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
    h.opacity_reg, h.scale_reg = cfg.opacity_reg, cfg.scale_reg
    h.n_reg = float(max(n_reg, 1))
    h.noise_scale = cfg.noise_lr * cfg.lr_mean
    h.gate_center, h.gate_sharpness = cfg.noise_gate_center, cfg.noise_gate_sharpness
    h.sgd = 1 if cfg.optimizer == "sgd" else 0
    h.sgld = 1 if sgld else 0
    h.seed = seed & 0xFFFFFFFFFFFFFFFF
    h.counter = counter & 0xFFFFFFFFFFFFFFFF
    return h


def philox_seed(rng_seed: int) -> int:
    """Philox key derived from TrainConfig.rng_seed (splitmix64)."""
    z = (int(rng_seed) + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


class DeviceModel:
    def __init__(self, state):
        cfg = state.config
        self.state, self.cfg = state, cfg
        self.dev = device()
        L.lib()
        sl, swin, num_gs = cfg.slice_size, cfg.swin_size, cfg.num_gs
        self.sl, self.swin, self.num_gs = sl, swin, num_gs
        dev = self.dev
        self.opt = torch.empty((num_gs, L.SS_ROW), dtype=torch.float64, device=dev)
        self.m = torch.zeros_like(self.opt)
        self.v = torch.zeros_like(self.opt)
        self.grads = torch.zeros((num_gs, L.SS_GRAD_ROW), dtype=torch.float32, device=dev)
        for i, gen in enumerate(state.slices):
            r0, r1 = i * sl, (i + 1) * sl
            self.opt[r0:r1] = torch.from_numpy(_pack(gen.params))
            self.m[r0:r1] = torch.from_numpy(_pack(gen.adam_m))
            self.v[r0:r1] = torch.from_numpy(_pack(gen.adam_v))
            gen.params = _views(self.opt[r0:r1])
            gen.adam_m = _views(self.m[r0:r1])
            gen.adam_v = _views(self.v[r0:r1])
            gen._rows = (self.opt, r0, r1)
        self.n_blocks = swin + 1
        self.mat = torch.zeros((self.n_blocks * sl, L.SS_ROW), dtype=torch.float64, device=dev)
        self.free_blocks = list(range(self.n_blocks))
        for mg in state.matured:  # host-only archive entries (state moved late)
            mg.block = self.free_blocks.pop(0)
            self.mat[mg.block * sl:(mg.block + 1) * sl] = torch.from_numpy(mg.arrays.rows())
        n_rows_all = num_gs + self.n_blocks * sl
        self.row_start = torch.zeros(n_rows_all, dtype=torch.int32, device=dev)
        self.row_expire = torch.zeros(n_rows_all, dtype=torch.int32, device=dev)
        self.blk_map = torch.zeros(self.n_blocks, dtype=torch.int32, device=dev)
        self.active_rows = torch.empty(n_rows_all, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(2, dtype=torch.int32, device=dev)
        lib = L.lib()
        self.ws_compact = torch.empty(int(lib.ss_compact_workspace_bytes(n_rows_all)),
                                      dtype=torch.uint8, device=dev)
        # per-step generation table, written to gen_dev through ss_write_small
        # (a kernel argument: no copy-engine op in the stream, and the host
        # buffer is free again as soon as the launch returns)
        self.gen_host = np.zeros(swin, dtype=GEN_DTYPE)
        self.gen_dev = torch.zeros(swin * GEN_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        self.reloc_ws = torch.empty(int(lib.ss_relocate_workspace_bytes(num_gs)),
                                    dtype=torch.uint8, device=dev)
        self.reloc_counts = torch.zeros(2, dtype=torch.int32, device=dev)
        self.eta = None
        self.pipe = ViewPipeline()
        self.lossbuf = LossBuffers()
        self.lut = torch.from_numpy(srgb_u8_lut().astype(np.float32)).to(dev)
        self.seed = philox_seed(cfg.rng_seed)
        self.store = Store(opt=self.opt, mat=self.mat)
        self.dirty = True
        self._rows_free = None  # event: the last view's backward no longer reads active_rows
        self._side = None       # side stream of the overlapped compaction
        self._life_sig = None
        self.last_sums = None
        self.last_counts = (0, 0)

    # ------------------------------------------------------------ bookkeeping
    def mark_lifespans_dirty(self):
        self.dirty = True

    def sync_lifespans(self):
        sig = (tuple((g.lifespan.start, g.lifespan.expire) for g in self.state.slices),
               tuple((m.block, m.lifespan.start, m.lifespan.expire) for m in self.state.matured))
        if sig == self._life_sig:
            # marked dirty but unchanged (e.g. a train_swin call on the same
            # window): row tables and compacted frames stay valid
            self.dirty = False
            return
        self._life_sig = sig
        sl, n_opt = self.sl, self.num_gs
        for i, gen in enumerate(self.state.slices):
            self.row_start[i * sl:(i + 1) * sl].fill_(gen.lifespan.start)
            self.row_expire[i * sl:(i + 1) * sl].fill_(gen.lifespan.expire)
        for mg in self.state.matured:
            r0 = n_opt + mg.block * sl
            self.row_start[r0:r0 + sl].fill_(mg.lifespan.start)
            self.row_expire[r0:r0 + sl].fill_(mg.lifespan.expire)
        blocks = [mg.block for mg in self.state.matured]
        if blocks:
            write_small(self.blk_map, np.asarray(blocks, dtype=np.int32))
        self.dirty = False

    def freeze(self, gen):
        """Direct-space snapshot of `gen` into a free matured block; returns
        (block, host GaussianArrays of the same bytes)."""
        block = self.free_blocks.pop(0)
        _, r0, r1 = gen._rows
        dst = self.mat[block * self.sl:(block + 1) * self.sl]
        L.check(L.lib().ss_to_direct(L.ptr(self.opt[r0:r1]), L.ptr(dst), r1 - r0, L.stream_ptr()),
                "to_direct")
        return block, GaussianArrays.from_rows(dst.cpu().numpy())

    def block_rows(self, block: int):
        return self.mat[block * self.sl:(block + 1) * self.sl]

    def release_block(self, block: int):
        if block >= 0:
            self.free_blocks.append(block)

    def _gen_table(self, stepped):
        cfg = self.cfg
        tab = self.gen_host
        for i, gen in enumerate(self.state.slices):
            e = tab[i]
            if stepped[i]:
                if cfg.optimizer == "adam":
                    gen.adam_t += 1
                t = max(gen.adam_t, 1)
                e["active"] = 1
                e["bc1"] = 1.0 - cfg.adam_beta1 ** t
                e["bc2"] = 1.0 - cfg.adam_beta2 ** t
                e["gscale"] = (cfg.gradient_scale_decay ** gen.windows_trained
                               if cfg.gradient_scaling else 1.0)
            else:
                e["active"] = 0
        write_small(self.gen_dev, tab)

    def compact(self, frame: int):
        """Active row ids of `frame` (a-2): optimizable rows of generations in
        state.slices order, then matured rows in archive order.  Returns
        (rows device tensor, n_active, n_active_optimizable).

        When the lifespan tables are unchanged since the previous view, the
        compaction runs on a side stream from the point where that view's
        backward released the row list (`_rows_free`), i.e. beside the
        previous step's optimizer; the caller's stream waits for it before
        the projection."""
        state, sl = self.state, self.sl
        side_ok = self._rows_free is not None and not self.dirty
        rows_free, self._rows_free = self._rows_free, None  # one use: set again by the next backward
        if self.dirty:
            self.sync_lifespans()
        live = lambda ls: ls.start <= frame < ls.expire  # noqa: E731
        n_opt = sl * sum(live(g.lifespan) for g in state.slices)
        n_mat = sl * sum(live(m.lifespan) for m in state.matured)
        lib = L.lib()
        main = torch.cuda.current_stream()
        if side_ok:
            if self._side is None:
                self._side = torch.cuda.Stream()
            self._side.wait_event(rows_free)
        s = self._side if side_ok else main
        L.check(lib.ss_compact_active(L.ptr(self.row_start), L.ptr(self.row_expire), self.num_gs,
                                      len(state.matured) * sl, L.ptr(self.blk_map), sl, frame,
                                      L.ptr(self.active_rows), L.ptr(self.counts),
                                      L.ptr(self.ws_compact), self.ws_compact.numel(),
                                      L.stream_ptr(s)), "compact_active")
        if side_ok:
            done = torch.cuda.Event()
            done.record(self._side)
            main.wait_event(done)
        n = n_opt + n_mat
        # recomputed every view, as the reference does (train.py:380-386);
        # the buffer is rewritten, in stream order, by the next view's call
        return self.active_rows[: max(n, 1)], n, n_opt

    # ------------------------------------------------------------------ step
    def train_step(self, draws, rank, dataset, it):
        """One training view (train.py:375-417).  `draws` are the (frame, view)
        samples of every data-parallel rank this iteration; this rank renders
        draws[rank]; generations active in any drawn frame are stepped."""
        from .train import stepped_generations

        stepped = stepped_generations(self.state.slices, [f for f, _ in draws])
        self._gen_table(stepped)
        # one rank, one view: every stepped row is active in this view and
        # ss_project_bwd writes all of them (zeros for culled rows), so the
        # gradient buffer needs no zero fill; with several ranks a stepped
        # generation may be inactive in this rank's frame
        dp = self.state.dp
        sums = self.view_gradients(draws[rank], dataset,
                                   zero_grads=dp is not None and dp.world_size > 1)
        if dp is not None:
            # only the stepped generations' rows are read by the step: reduce
            # their contiguous span (generation i = rows [i sl, (i+1) sl))
            gens = [i for i, st in enumerate(stepped) if st]
            if gens:
                lo, hi = gens[0] * self.sl, (gens[-1] + 1) * self.sl
                dp.allreduce_grads(self.grads[lo:hi])
        self.apply_step(stepped, it)
        return sums

    def view_gradients(self, draw, dataset, zero_grads: bool = True):
        """Forward, loss and backward of one (frame, view) draw: the
        optimization-space gradient lands in self.grads (zeroed first unless
        the caller knows every row it will read is active in this view).
        Returns the device loss sums."""
        frame, view = draw
        sp = L.stream_ptr()
        rows, n, n_opt_here = self.compact(frame)
        if zero_grads:
            L.check(L.lib().ss_memzero(L.ptr(self.grads), self.grads.numel() * 4, sp), "memzero")
        cam = dataset.cameras[view]
        # ground truth may still be in flight on a copy stream: only the loss
        # waits for it, the projection / binning / raster run meanwhile
        get_async = getattr(dataset, "device_frame_async", None)
        if get_async is not None:
            gt, gt_ready = get_async(frame, view)
        else:
            gt, gt_ready = dataset.device_frame(frame, view), None
        self.pipe.deterministic = self.state.deterministic
        img = self.pipe.forward(self.store, rows, n, cam)
        if gt_ready is not None:
            torch.cuda.current_stream().wait_event(gt_ready)
        dimg, sums = self.lossbuf.run(img, cam.height, cam.width, gt_u8=gt, lut=self.lut,
                                      ssim_weight=self.cfg.ssim_weight)
        self.pipe.backward(dimg, self.grads, trainable_rows=self.num_gs)
        # the row list is no longer read past this point: the next view's
        # compaction may start here (beside this step's optimizer)
        self._rows_free = torch.cuda.Event()
        self._rows_free.record()
        self.last_sums = sums
        self.last_counts = (n, n_opt_here)
        return sums

    def apply_step(self, stepped, it):
        """Fused Adam + gamma^w + projections + SGLD over the stepped
        generations (the table _gen_table wrote), relocation every
        relocate_period iterations (train.py:400-417)."""
        state, cfg = self.state, self.cfg
        lib = L.lib()
        sp = L.stream_ptr()
        n_reg = self.sl * sum(stepped)
        eta = None
        if state.noise_source == "numpy":
            eta = self._numpy_eta(stepped)
        h = _hyper(cfg, n_reg, True, self.seed, state.iteration)
        L.check(lib.ss_adam_sgld_step(L.ptr(self.opt), L.ptr(self.grads), L.ptr(self.m),
                                      L.ptr(self.v), self.num_gs, self.sl, L.ptr(self.gen_dev),
                                      ctypes.byref(h), L.ptr(eta), sp), "adam_sgld_step")
        if it % cfg.relocate_period == 0:
            self.relocate_device(cfg.dead_opacity_threshold)
        state.iteration += 1

    def _numpy_eta(self, stepped):
        """eta drawn per stepped generation in list order (train.py:255-258)."""
        if self.eta is None:
            self.eta = torch.zeros((self.num_gs, 3), dtype=torch.float64, device=self.dev)
        sl = self.sl
        for i, gen in enumerate(self.state.slices):
            if stepped[i]:
                e = self.state.rng.standard_normal((sl, 3))
                self.eta[i * sl:(i + 1) * sl].copy_(torch.from_numpy(e))
        return self.eta

    def relocate_device(self, threshold: float, uniforms_rng=None) -> int | None:
        """MCMC relocation over the generations flagged in the current gen
        table (train.py:267-318).  Philox uniforms unless the state draws from
        numpy, in which case the reference's choice() uniforms are consumed."""
        state = self.state
        lib = L.lib()
        sp = L.stream_ptr()
        uniforms = None
        if state.noise_source == "numpy":
            tab = self.gen_host
            rows = torch.cat([torch.arange(i * self.sl, (i + 1) * self.sl, device=self.dev)
                              for i in range(len(state.slices)) if tab[i]["active"]] or
                             [torch.zeros(0, dtype=torch.int64, device=self.dev)])
            alpha = 1.0 / (1.0 + torch.exp(-self.opt[rows, 10]))
            n_dead = int((alpha < threshold).sum().item())
            n_alive = int(rows.numel()) - n_dead
            if n_dead == 0:
                return 0
            if n_alive == 0:
                log.warning("relocation skipped: no alive splats above threshold %.4g", threshold)
                return 0
            uniforms = torch.from_numpy(state.rng.random(n_dead)).to(self.dev)
        L.check(lib.ss_relocate(L.ptr(self.opt), L.ptr(self.m), L.ptr(self.v), self.num_gs, self.sl,
                                L.ptr(self.gen_dev), float(threshold), L.ptr(uniforms), self.seed,
                                state.iteration, L.ptr(self.reloc_counts), L.ptr(self.reloc_ws),
                                self.reloc_ws.numel(), sp), "relocate")
        return None


# ---------------------------------------------------------------------------
# reference-API entry points on explicit generation lists (host or device)
# ---------------------------------------------------------------------------

def to_direct_host(params) -> GaussianArrays:
    t = torch.cat([params["mean"], params["quat"], params["log_scale"],
                   params["opacity_logit"][:, None], params["color"]], dim=1).contiguous()
    out = torch.empty_like(t)
    L.check(L.lib().ss_to_direct(L.ptr(t), L.ptr(out), t.shape[0], L.stream_ptr()), "to_direct")
    return GaussianArrays.from_rows(out.cpu().numpy())


class _Batch:
    """Concatenate the rows of a list of generations onto the device, run
    kernels on them, and write results back (numpy in place, or torch views)."""

    def __init__(self, gens):
        self.gens = gens
        self.sizes = [len(g.params["mean"]) for g in gens]
        dev = device()
        parts = []
        for g in gens:
            if g.on_device:
                parts.append(torch.cat([g.params[k].reshape(len(g.params["mean"]), -1)
                                        for k in PARAM_KEYS], 1))
            else:
                parts.append(torch.from_numpy(_pack(g.params)).to(dev))
        self.t = torch.cat(parts).contiguous() if parts else torch.zeros((0, 14), device=dev,
                                                                         dtype=torch.float64)

    def moments(self):
        dev = device()
        ms, vs = [], []
        for g in self.gens:
            if g.on_device:
                ms.append(torch.cat([g.adam_m[k].reshape(len(g.params["mean"]), -1)
                                     for k in PARAM_KEYS], 1))
                vs.append(torch.cat([g.adam_v[k].reshape(len(g.params["mean"]), -1)
                                     for k in PARAM_KEYS], 1))
            else:
                ms.append(torch.from_numpy(_pack(g.adam_m)).to(dev))
                vs.append(torch.from_numpy(_pack(g.adam_v)).to(dev))
        return torch.cat(ms).contiguous(), torch.cat(vs).contiguous()

    def write_back(self, t, which="params"):
        host = t.cpu().numpy()
        off = 0
        for g, n in zip(self.gens, self.sizes):
            tgt = getattr(g, which)
            block = host[off:off + n]
            if g.on_device:
                for k, (a, b) in COLS.items():
                    src = block[:, a] if b - a == 1 else block[:, a:b]
                    tgt[k].copy_(torch.from_numpy(np.ascontiguousarray(src)))
            else:
                _unpack_into(tgt, block)
            off += n


def _single_gen_table(active=1, bc1=1.0, bc2=1.0, gscale=1.0):
    tab = np.zeros(1, dtype=GEN_DTYPE)
    tab[0] = (active, 0, bc1, bc2, gscale)
    return torch.from_numpy(tab.view(np.uint8)).to(device())


def run_sgld(gens, current_mean_lr, noise_lr, rng, gate_center, gate_sharpness):
    if not gens:
        return
    b = _Batch(gens)
    n = b.t.shape[0]
    eta = np.concatenate([rng.standard_normal((s, 3)) for s in b.sizes])
    eta_t = torch.from_numpy(eta).to(device())
    h = L.SSStepHyper()
    h.noise_scale = noise_lr * current_mean_lr
    h.gate_center, h.gate_sharpness = gate_center, gate_sharpness
    h.sgld = 1
    L.check(L.lib().ss_sgld(L.ptr(b.t), n, max(n, 1), L.ptr(_single_gen_table()), ctypes.byref(h),
                            L.ptr(eta_t), L.stream_ptr()), "sgld")
    b.write_back(b.t)


def run_relocate(gens, threshold, rng) -> int:
    if not gens:
        return 0
    b = _Batch(gens)
    n = b.t.shape[0]
    alpha = 1.0 / (1.0 + torch.exp(-b.t[:, 10]))
    n_dead = int((alpha < threshold).sum().item())
    if n_dead == 0:
        return 0
    if n_dead == n:
        log.warning("relocation skipped: no alive splats above threshold %.4g", threshold)
        return 0
    u = torch.from_numpy(rng.random(n_dead)).to(device())
    m, v = b.moments()
    lib = L.lib()
    ws = torch.empty(int(lib.ss_relocate_workspace_bytes(n)), dtype=torch.uint8, device=device())
    counts = torch.zeros(2, dtype=torch.int32, device=device())
    L.check(lib.ss_relocate(L.ptr(b.t), L.ptr(m), L.ptr(v), n, n, L.ptr(_single_gen_table()),
                            float(threshold), L.ptr(u), 0, 0, L.ptr(counts), L.ptr(ws), ws.numel(),
                            L.stream_ptr()), "relocate")
    b.write_back(b.t)
    b.write_back(m, "adam_m")
    b.write_back(v, "adam_v")
    return n_dead


def run_optimizer_step(gen, grads, config):
    b = _Batch([gen])
    n = b.t.shape[0]
    g = torch.from_numpy(_pack({k: np.asarray(grads[k]) for k in PARAM_KEYS}).astype(np.float32))
    g = g.to(device())
    m, v = b.moments()
    if config.optimizer == "adam":
        gen.adam_t += 1
    t = max(gen.adam_t, 1)
    tab = _single_gen_table(1, 1.0 - config.adam_beta1 ** t, 1.0 - config.adam_beta2 ** t, 1.0)
    h = _hyper(config, 1, False, 0, 0)
    h.opacity_reg = h.scale_reg = 0.0
    L.check(L.lib().ss_adam_sgld_step(L.ptr(b.t), L.ptr(g), L.ptr(m), L.ptr(v), n, max(n, 1),
                                      L.ptr(tab), ctypes.byref(h), None, L.stream_ptr()),
            "adam_sgld_step")
    b.write_back(b.t)
    if config.optimizer == "adam":
        b.write_back(m, "adam_m")
        b.write_back(v, "adam_v")
