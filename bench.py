"""Benchmark: SwinGS window-training views/s at DyNeRF resolution on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one training view through the public API (train_swin): active-set
compaction -> projection -> tile binning -> raster forward -> L1+SSIM ->
raster backward -> projection backward -> [NCCL allreduce] -> fused Adam +
SGLD (+ MCMC relocation every 100 iterations, as the reference schedules it).

Workload (default, BASELINE.json configs[2], "DyNeRF-shaped synthetic"):
300-frame synthetic video, 20 arc cameras at 1352x1014, num_gs = 300k,
swin_size = 10.  Ground truth is the animated 300k-splat scene rendered by
the GPU forward; the model is initialised from the frame-0
point cloud as TrainConfig.init_points does.  Steps run in the window
[1, 11) after genesis + schedule_expire + mature(1), so every view mixes
optimizable and matured generations (the steady state).

Rank 0 prints one JSON line.  `value` is whole-job views/s with ground truth
resident in HBM; `e2e` is the same through train_swin with each step's
ground truth copied from pinned host memory and the loss read back.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    1: dict(name="synthetic tiny scene: 10k Gaussians, 64x64, 4 cameras, window=4, 20 frames",
            gt_n=10_000, frames=20, views=4, W=64, H=64, num_gs=10_000, swin=4, dynerf=False),
    2: dict(name="static single frame: 200k Gaussians, 1352x1014, 20 cameras",
            gt_n=200_000, frames=1, views=20, W=1352, H=1014, num_gs=200_000, swin=1, dynerf=True),
    3: dict(name="DyNeRF-shaped synthetic: 300 frames, 20 cameras at 1352x1014, 300k active "
                 "Gaussians, window=10",
            gt_n=300_000, frames=300, views=20, W=1352, H=1014, num_gs=300_000, swin=10,
            dynerf=True),
    4: dict(name="long video: 1200 frames, window=20, 1M Gaussians, 20 cameras",
            gt_n=1_000_000, frames=1200, views=20, W=1352, H=1014, num_gs=1_000_000, swin=20,
            dynerf=True),
}
METRIC = "window training views/sec (1352x1014)"
METRIC5 = "render-only streaming playback frames/sec (1920x1080)"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def _capture():
    """The latest committed ncu --set full capture of the raster kernels
    (profiles/r*_traffic.json), or None when its recorded source hash does
    not match the current csrc/raster.cu (the counters would be stale)."""
    import hashlib

    files = sorted((ROOT / "profiles").glob("r*_traffic.json"))
    if not files:
        return None, "no capture committed"
    d = json.loads(files[-1].read_text())
    src = ROOT / "paper_2409_07759_b200" / "csrc" / "raster.cu"
    sha = hashlib.sha256(src.read_bytes()).hexdigest()[:16]
    if d.get("raster_cu_sha16") != sha:
        return None, f"{files[-1].name} predates the current raster.cu (stale, not used)"
    return d, f"{files[-1].name} (ncu --set full of this raster.cu, sha {sha}, config 3)"


def load_traffic(kernels):
    """Per-launch DRAM bytes (read + write) of the given kernels from the
    committed capture of the CURRENT raster.cu, else None."""
    d, note = _capture()
    if d is None:
        return None, note
    try:
        return sum(d[k]["dram_bytes_read"] + d[k]["dram_bytes_write"] for k in kernels), note
    except KeyError:
        return None, note


def load_ncu_counters(kernels):
    """Issue-slot utilisation, SM / L2 / L1 throughput, occupancy and
    instructions per walked (warp, entry) of the given kernels from the same
    capture (the raster kernels are instruction-issue bound), else None."""
    d, note = _capture()
    if d is None:
        return None
    keys = ("issue_active_pct", "sm_throughput_pct", "l2_throughput_pct", "l1_throughput_pct",
            "l2_hit_rate_pct", "occupancy_pct", "warp_instructions",
            "warp_instructions_per_k_used_entry", "k_used")
    return {k: {q: d[k].get(q) for q in keys if q in d[k]} for k in kernels if k in d}


def load_peaks():
    if PEAKS.exists():
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits", "-lms", "200"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.samples.append([x.strip() for x in line.split(",")])
        p.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=3)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def build_workload(cfg_id: int, dp, init="gt", scene_ds=None):
    import torch

    from paper_2409_07759_b200 import synth, train

    c = CONFIGS[cfg_id]
    if scene_ds is not None:
        scene, ds = scene_ds
    elif c["dynerf"]:
        scene = synth.dynerf_scene(c["gt_n"], c["frames"], c["views"], c["W"], c["H"], seed=7)
        ds = synth.device_video(scene)
    else:
        cams = synth.arc_cameras(c["views"], c["W"], c["H"], arc_degrees=36.0)
        scene = synth.make_scene(7, c["frames"], cams, c["gt_n"])
        ds = synth.device_video(scene)
    pts = init_points(scene, c)
    tmp = tempfile.NamedTemporaryFile("w", suffix=".xyz", delete=False)
    np.savetxt(tmp, pts)
    tmp.close()
    cfg = train.TrainConfig(swin_size=c["swin"], num_gs=c["num_gs"], genesis_iterations=2,
                            window_iterations=2, relocate_period=100, rng_seed=0,
                            init_points=tmp.name)
    state = train.init_state(cfg)
    os.unlink(tmp.name)
    if init == "gt":
        means, quats, scales, opac, cols = gt_rows(scene, c)
        sl = cfg.slice_size
        for i, gen in enumerate(state.slices):
            r = slice(i * sl, (i + 1) * sl)
            gen.params["mean"][:] = means[r]
            gen.params["quat"][:] = quats[r]
            gen.params["log_scale"][:] = np.log(scales[r])
            gen.params["opacity_logit"][:] = train._logit(opac[r])
            gen.params["color"][:] = cols[r]
    state.dp = dp
    # genesis -> staggered lifespans -> first window slide (steady state)
    train.train_swin(0, cfg.swin_size, state, ds, iterations=2)
    st = 0
    if c["frames"] > 1:
        train.schedule_expire(state)
        train.mature(1, state, writer=None)
        st = 1
    window = (st, st + cfg.swin_size)
    # ground truth of the window resident in HBM before timing
    for f in range(window[0], min(window[1], c["frames"])):
        for v in range(c["views"]):
            ds.device_frame(f, v)
    torch.cuda.synchronize()
    return c, scene, ds, state, window


def gt_rows(scene, c):
    """Frame-0 ground-truth splats resampled to num_gs: (means, quats, scales,
    opacities, colors).  The default bench model starts here -- window training
    is warm-started from the previous window's trained model, so a converged
    state (not a random init) is the steady state being measured."""
    g0 = scene.gaussians_at(0)
    idx = np.arange(len(g0))
    rng = np.random.default_rng(0)
    if len(idx) < c["num_gs"]:
        idx = np.concatenate([idx, rng.integers(0, len(idx), c["num_gs"] - len(idx))])
    idx = idx[: c["num_gs"]]
    return (g0.means[idx], g0.quats[idx], g0.scales[idx], g0.opacities[idx], g0.colors[idx])


def init_points(scene, c):
    """x y z r g b of the frame-0 ground-truth splats, resampled to num_gs
    (the TrainConfig.init_points recipe both arms start from)."""
    g0 = scene.gaussians_at(0)
    pts = np.concatenate([g0.means, g0.colors], axis=1)
    rng = np.random.default_rng(0)
    if len(pts) < c["num_gs"]:
        pts = np.concatenate([pts, pts[rng.integers(0, len(pts), c["num_gs"] - len(pts))]])
    return pts[: c["num_gs"]]


class HostFeed:
    """Dataset view whose ground truth lives in pinned host memory and is
    copied to the GPU on every access (the e2e arm): the copy runs on a copy
    stream while the step's projection / binning / raster proceed, and only
    the loss waits for it (device_frame_async, the dataset API the trainer
    uses)."""

    def __init__(self, ds, window, views):
        import torch

        self.ds = ds
        self.cameras = ds.cameras
        self.total_frames = ds.total_frames
        self.host = {}
        for f in range(window[0], min(window[1], ds.total_frames)):
            for v in range(views):
                self.host[(f, v)] = ds.device_frame(f, v).cpu().pin_memory()
        self.h2d_bytes = 0
        self.torch = torch
        self.stream = torch.cuda.Stream()

    @property
    def n_views(self):
        return self.ds.n_views

    def device_frame_async(self, frame, view):
        torch = self.torch
        h = self.host[(frame, view)]
        self.h2d_bytes += h.numel()
        cur = torch.cuda.current_stream()
        with torch.cuda.stream(self.stream):
            d = h.to("cuda", non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        d.record_stream(cur)
        return d, ev

    def device_frame(self, frame, view):
        d, ev = self.device_frame_async(frame, view)
        self.torch.cuda.current_stream().wait_event(ev)
        return d


class LossReadback:
    """train_swin progress hook: every step's loss sums are copied to pinned
    host memory (non-blocking) and read one step later, as a training loop
    that logs the loss does; flush() reads the last one."""

    def __init__(self, model):
        import torch

        self.torch = torch
        self.model = model
        self.d2h_bytes = 0
        self.values = []
        self._pending = None
        self.stream = None

    def update(self, _n):
        torch = self.torch
        s = self.model.last_sums
        h = torch.empty(s.shape, dtype=s.dtype, pin_memory=True)
        # the copy runs on a side stream (a copy-engine op between the step's
        # kernels would stall the main stream's launch chain); the loss sums
        # alternate between two device slots and this view's copy is read
        # (synchronized) before the view after next can rewrite its slot
        if self.stream is None:
            self.stream = torch.cuda.Stream()
        ready = torch.cuda.Event()
        ready.record()
        self.stream.wait_event(ready)
        with torch.cuda.stream(self.stream):
            h.copy_(s, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        s.record_stream(self.stream)
        self.d2h_bytes += h.numel() * h.element_size()
        self._read()
        self._pending = (h, ev)

    def _read(self):
        if self._pending is not None:
            h, ev = self._pending
            ev.synchronize()
            self.values.append(float(h[0]))
            self._pending = None

    def flush(self):
        self._read()


def snapshot_state(state):
    """What train_swin changes on the window being benchmarked: the device
    store and Adam moments, per-generation step counters, the sampling RNG
    and the global iteration (Philox counter).  Restoring it replays the
    same views on the same model states."""
    dev = state.device
    return {"t": [t.clone() for t in (dev.opt, dev.m, dev.v)],
            "gens": [(g.adam_t, g.windows_trained) for g in state.slices],
            "rng": state.rng.bit_generator.state, "iteration": state.iteration}


def restore_state(state, snap):
    import torch

    dev = state.device
    for dst, src in zip((dev.opt, dev.m, dev.v), snap["t"]):
        dst.copy_(src)
    for g, (t, w) in zip(state.slices, snap["gens"]):
        g.adam_t, g.windows_trained = t, w
    state.rng.bit_generator.state = snap["rng"]
    state.iteration = snap["iteration"]
    torch.cuda.synchronize()


def time_steps(state, ds, window, steps, dp, progress=None):
    import torch

    from paper_2409_07759_b200 import train

    if dp is not None:
        dp.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    train.train_swin(window[0], window[1], state, ds, iterations=steps, progress=progress)
    if progress is not None and hasattr(progress, "flush"):
        progress.flush()  # the last step's result is read inside the timed region
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if dp is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dp.dist.all_reduce(t, op=dp.dist.ReduceOp.MAX)
        ms = float(t.item())
        dp.barrier()
    return ms


def count_launches(state, ds, window):
    """Kernels launched by one training step, from the torch profiler (ours =
    everything not emitted by torch's own ATen kernels)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2409_07759_b200 import train

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        train.train_swin(window[0], window[1], state, ds, iterations=1)
        torch.cuda.synchronize()
    ours = aten = 0
    names = {}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        n = e.name
        if "memcpy" in n.lower() or "memset" in n.lower():
            continue
        if "at::" in n or "at_cuda_detail" in n:
            aten += 1
        else:
            ours += 1
            names[n[:60]] = names.get(n[:60], 0) + 1
    return ours, aten, names


def roofline_pass(state, ds, window, steps):
    """Raster fwd+bwd kernel time (CUDA events on the launch stream) and
    K_used per view over `steps` extra (untimed) steps."""
    import torch

    from paper_2409_07759_b200 import train

    model = state.device
    pipe = model.pipe
    pipe.enable_timing(True)
    k_used, k_pairs, n_act = [], [], []

    class Hook:
        def update(self, _n):
            k_used.append(pipe.k_used())
            k_pairs.append(pipe.n_pairs)
            n_act.append(pipe.n)

    train.train_swin(window[0], window[1], state, ds, iterations=steps, progress=Hook())
    ms = pipe.kernel_ms()
    pipe.enable_timing(False)
    torch.cuda.synchronize()
    return ms, float(np.mean(k_used)), float(np.mean(k_pairs)), float(np.mean(n_act))


# --------------------------------------------------------------------------- CPU
def cpu_model_name() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class CpuTrainer:
    """The reference algorithm on the host -- oracle/ (the reference's fp64
    numpy stages and its two pixel loops in C, all host threads) -- training
    WHOLE 1352x1014 views of the bench workload, one view per step like
    train_swin (train.py:374-417): projection (raster.py:76-173) -> global
    (z, src) order -> blend forward (_kernels.py:20-53) -> L1 + SSIM + regs
    (loss.py:73-118) -> blend backward (_kernels.py:56-130) -> projection
    backward (raster.py:249-347) -> per-generation Adam (train.py:321-344)
    -> SGLD (train.py:246-264), relocation at it = 0 (train.py:416-417).

    Same model and window as the GPU arm: the ground-truth-init store after
    genesis + schedule_expire + mature(1), window [1, 1 + swin).  At frame f
    the active set is optimizable generations 0..f-1 (trained copies) then
    matured generations f..swin-1 (frozen init copies) -- the compaction
    order of train.py:380-386 -- so n_opt = f * slice.  The pixel loops walk
    tile lists (oracle.tile_bins: the reference's per-pixel sequence, the
    same images and gradients as the global walk), the only way a full view
    finishes in seconds.  Ground truth: the oracle's render of the animated
    scene at (f, v) for `n_gt` fixed draws, decoded through the u8 sRGB
    round trip as read_png does (rendered at setup, outside the timing)."""

    def __init__(self, c, threads, n_gt=4, seed=0):
        from paper_2409_07759_b200.synth import make_scene
        from oracle import splat_oracle as O

        self.O, self.c, self.threads = O, c, threads
        k = (300.0 / c["gt_n"]) ** (1 / 3) if c["dynerf"] else 1.0
        scene = make_scene(7, c["frames"], [], c["gt_n"], scale_range=(0.045 * k, 0.1 * k))
        means, quats, scales, opac, cols = gt_rows(scene, c)
        self.n, self.swin = c["num_gs"], c["swin"]
        self.sl = self.n // self.swin
        init = {"mean": means.copy(), "quat": quats.copy(), "log_scale": np.log(scales),
                "opacity_logit": O.logit(opac), "color": cols.copy()}
        self.mat = {k2: v.copy() for k2, v in init.items()}          # frozen copies
        self.opt = {k2: v.copy() for k2, v in init.items()}          # trained copies
        self.m = {k2: np.zeros_like(v) for k2, v in init.items()}
        self.v = {k2: np.zeros_like(v) for k2, v in init.items()}
        self.t = np.zeros(self.swin, dtype=np.int64)                  # per-generation adam_t
        self.cams = _arc_cams_np(c)
        self.rng = np.random.default_rng(seed)
        self.win = (1, 1 + self.swin) if c["frames"] > 1 else (0, 1)
        self.gt = []
        for _ in range(n_gt):
            f = int(self.rng.integers(self.win[0], min(self.win[1], c["frames"])))
            v = int(self.rng.integers(0, len(self.cams)))
            g = scene.gaussians_at(f)
            img = O.render_arrays(self.cams[v], g.means, g.quats, g.scales, g.opacities,
                                  g.colors, nthreads=threads, tiled=True)
            self.gt.append((f, v, O.linear_from_u8(O.u8_from_linear(img))))
        self.step_i = 0
        self.stats = []

    def _active(self, n_opt):
        sl = slice(0, n_opt)
        rest = slice(n_opt, self.n)
        out = {}
        for k2 in self.opt:
            out[k2] = np.concatenate([self.opt[k2][sl], self.mat[k2][rest]])
        return out

    def step(self, threads=None):
        O = self.O
        th = self.threads if threads is None else threads
        f, v, gt = self.gt[self.step_i % len(self.gt)]
        it = self.step_i
        self.step_i += 1
        cam = self.cams[v]
        n_opt = self.sl * (f - self.win[0] + 1) if self.c["frames"] > 1 else self.n
        a = self._active(n_opt)
        scales = np.exp(a["log_scale"])
        opac = O.sigmoid(a["opacity_logit"])
        cache = O.project_arrays(cam, a["mean"], a["quat"], scales, opac, a["color"])
        H, W = cam.height, cam.width
        bins = O.tile_bins(cache, W, H, floor_log2=None)  # the reference rule
        fw = O.blend_forward_tiled(cache, H, W, nthreads=th, bins=bins)
        _, gimg, reg = O.loss(fw["image"], gt, opac[:n_opt], scales[:n_opt])
        g2d = O.blend_backward_tiled(cache, bins, H, W, gimg, nthreads=th)
        trainable = np.zeros(self.n, dtype=bool)
        trainable[:n_opt] = True
        grads = O.projection_backward(cam, cache, self.n, *g2d, trainable=trainable)
        grads["opacity_logit"][:n_opt] += reg["opacity_logit"]
        grads["log_scale"][:n_opt] += reg["log_scale"]
        gens = list(range(n_opt // self.sl))
        views = []
        for gi in gens:
            r = slice(gi * self.sl, (gi + 1) * self.sl)
            p = {k2: self.opt[k2][r] for k2 in self.opt}
            mm = {k2: self.m[k2][r] for k2 in self.m}
            vv = {k2: self.v[k2][r] for k2 in self.v}
            self.t[gi] = O.optimizer_step(p, mm, vv, int(self.t[gi]),
                                          {k2: grads[k2][r] for k2 in grads})
            views.append((p, mm, vv))
        O.sgld_perturb([p for p, _, _ in views], 1.6e-4, 5e4,
                       [self.rng.standard_normal((self.sl, 3)) for _ in views])
        if it % 100 == 0:
            alpha = O.sigmoid(np.concatenate([p["opacity_logit"] for p, _, _ in views]))
            n_dead = int((alpha < 0.005).sum())
            O.relocate([p for p, _, _ in views], [mm for _, mm, _ in views],
                       [vv for _, _, vv in views], 0.005, self.rng.random(max(n_dead, 1)))
        self.stats.append((bins["K"], fw["K_used"]))


def cpu_crop_view(trainer, crop=256, n_crops=4, threads=1):
    """Crop-extrapolated s/view: the pixel loops + loss on
    `n_crops` crop cameras of crop x crop px (shifted principal point), scaled
    by P / P_crop, plus the per-splat stages at full size."""
    O = trainer.O
    c = trainer.c
    W, H = c["W"], c["H"]
    cam = trainer.cams[0]
    a = trainer._active(trainer.n)
    scales, opac = np.exp(a["log_scale"]), O.sigmoid(a["opacity_logit"])
    t0 = time.perf_counter()
    cache = O.project_arrays(cam, a["mean"], a["quat"], scales, opac, a["color"])
    p = len(cache["src"])
    O.projection_backward(cam, cache, trainer.n, np.zeros((p, 2)), np.zeros((p, 3)),
                          np.zeros(p), np.zeros((p, 3)))
    t_gauss = time.perf_counter() - t0
    xs, ys = [W // 4, 3 * W // 4], [H // 4, 3 * H // 4]
    centers = [(x, y) for y in ys for x in xs][:n_crops]
    t_pix, used = 0.0, 0
    rng = np.random.default_rng(1)
    for xc, yc in centers:
        cc = _Cam(crop, crop, cam.fx, cam.fy, cam.cx - (xc - crop // 2), cam.cy - (yc - crop // 2),
                  cam.rotation, cam.translation)
        t1 = time.perf_counter()
        cch = O.project_arrays(cc, a["mean"], a["quat"], scales, opac, a["color"])
        if cch is None:
            continue
        bins = O.tile_bins(cch, crop, crop, floor_log2=None)
        img = O.blend_forward_tiled(cch, crop, crop, nthreads=threads, bins=bins)["image"]
        gt = O.linear_from_u8(rng.integers(0, 256, (crop, crop, 3), dtype=np.uint8))
        _, gimg, _ = O.loss(img, gt, opac[:1], scales[:1])
        O.blend_backward_tiled(cch, bins, crop, crop, gimg, nthreads=threads)
        t_pix += time.perf_counter() - t1
        used += 1
    return t_gauss + t_pix / max(used, 1) * (W * H) / (crop * crop)


class _Cam:
    def __init__(self, width, height, fx, fy, cx, cy, rotation, translation):
        self.width, self.height, self.fx, self.fy, self.cx, self.cy = width, height, fx, fy, cx, cy
        self.rotation, self.translation = rotation, translation


def _arc_cams_np(c):
    n, W, H = c["views"], c["W"], c["H"]
    focal = 70.0 * W / 64 if c["dynerf"] else 70.0
    half = np.radians(36.0) / 2
    out = []
    for ang in (np.linspace(-half, half, n) if n > 1 else [0.0]):
        center = np.array([3 * np.sin(ang), 0.25 * np.sin(2.1 * ang), -3 * np.cos(ang)])
        fwd = -center / np.linalg.norm(center)
        right = np.cross([0.0, 1.0, 0.0], fwd)
        right /= np.linalg.norm(right)
        up = np.cross(fwd, right)
        R = np.stack([right, up, fwd])
        out.append(_Cam(W, H, focal, focal, W / 2, H / 2, R, -R @ center))
    return out


def build_player(n_total=1_000_000, swin=20, views=20, W=1920, H=1080, seed=7):
    """Config 5: a 1M-splat slot buffer (swin slots of n/swin decoded records)
    from the DyNeRF-shaped recipe, arc cameras at 1920x1080, focal 2100,
    70-degree arc (test_acceptance.py:385)."""
    from paper_2409_07759_b200 import player, synth
    from paper_2409_07759_b200.codec import DecodedSlice, SliceHeader
    from paper_2409_07759_b200.core import GaussianArrays, Lifespan

    cams = synth.arc_cameras(views, W, H, radius=3.0, focal=2100.0, arc_degrees=70.0)
    k = (300.0 / n_total) ** (1.0 / 3.0)
    scene = synth.make_scene(seed, 300, cams, n_total, scale_range=(0.045 * k, 0.1 * k))
    g0 = scene.gaussians_at(0)
    rng = np.random.default_rng(0)
    idx = np.concatenate([np.arange(len(g0)), rng.integers(0, len(g0), n_total - len(g0))])
    arr = g0.take(idx)
    sl = n_total // swin
    slices = []
    for s_ in range(swin):
        part = arr.take(np.arange(s_ * sl, (s_ + 1) * sl))
        ls = Lifespan(0, 0, 1 << 30)
        slices.append(DecodedSlice(SliceHeader(0, s_, sl), part, ls, np.ones(sl, bool)))
    buf = player.PlayerBuffer(slices, swin)
    buf.to_device()
    return buf, cams, arr, sl


def run_render_only(args, dp):
    """--config 5: frames/s of the render-only playback path (compaction over
    the slot buffer in (birth, slot) order -> projection -> binning -> raster
    forward) at 1920x1080, 1M splats; e2e adds per frame one slot update
    from wire bytes (H2D, GPU decode) and the frame read back to the host."""
    import torch

    from paper_2409_07759_b200 import codec
    from paper_2409_07759_b200.core import StreamParams

    world = 1 if dp is None else dp.world_size
    rank = 0 if dp is None else dp.rank
    buf, cams, arr, sl = build_player()
    W, H = cams[0].width, cams[0].height

    def frames(n, start=0):
        for i in range(n):
            buf.render_device(cams[(start + i * world + rank) % len(cams)], 0)

    frames(args.warmup)
    if args.profile_steps:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        frames(args.profile_steps)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return {"profiled_frames": args.profile_steps}
    from paper_2409_07759_b200.parallel import local_device_index

    with ClockSampler(local_device_index()) as clocks:
        if dp is not None:
            dp.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        frames(args.steps)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dp is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dp.dist.all_reduce(t, op=dp.dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"metric": METRIC5, "value": world * args.steps / (ms / 1e3), "unit": "frames/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (DyNeRF-shaped recipe, 1M splats in 20 slots)",
           "config": {"workload": "render-only streaming playback: 1M lifespan Gaussians, "
                                  "1920x1080 novel views", "width": W, "height": H,
                      "splats": len(arr), "slots": 20, "parallelism": f"replicas{world}",
                      "l2": "per-frame working set > 126 MB L2 (tile pairs); no explicit flush"},
           "clocks": clocks.summary()}
    # e2e: one slot update from wire bytes per frame + frame read back
    prof = codec.PROFILES[1]
    params = StreamParams(swin_size=20, num_gs=len(arr), fps=30.0, bytes_per_gaussian=30,
                          total_frames=1 << 20)
    blobs = []
    from paper_2409_07759_b200.core import Lifespan
    for s_ in range(4):
        part = arr.take(np.arange(s_ * sl, (s_ + 1) * sl))
        blobs.append(codec.pack_slice(part, Lifespan(s_, s_, s_ + 20), prof, 20))
    h2d = d2h = 0
    # display frames (uint8 sRGB, write_png's quantisation) copied to pinned
    # host buffers on a copy stream, double-buffered: frame i+1 renders while
    # frame i crosses PCIe; the host reads a frame once its copy event is done
    pinned = [torch.empty((H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
    dev_u8 = [torch.empty((H, W, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
    copy_stream = torch.cuda.Stream()
    done = [None, None]
    checksum = 0

    def frame(i):
        nonlocal checksum
        k = i % 2
        if done[k] is not None:           # buffer k's previous frame: consume it
            done[k].synchronize()
            checksum += int(pinned[k][0, 0, 0])
        blob = blobs[i % len(blobs)]
        buf.apply_bytes(blob, prof, params)
        buf.render_device_u8(cams[(i * world + rank) % len(cams)], 19, out=dev_u8[k])
        ready = torch.cuda.Event()
        ready.record()
        copy_stream.wait_event(ready)
        with torch.cuda.stream(copy_stream):
            pinned[k].copy_(dev_u8[k], non_blocking=True)
            done[k] = torch.cuda.Event()
            done[k].record(copy_stream)
        return len(blob), dev_u8[k].numel()

    def drain():
        for k in range(2):
            if done[k] is not None:
                done[k].synchronize()
        torch.cuda.current_stream().wait_stream(copy_stream)

    for i in range(args.warmup):        # staging buffers, streams, first decodes
        frame(i)
    drain()
    torch.cuda.synchronize()
    e0.record()
    for i in range(args.steps):
        bi, bo = frame(i)
        h2d += bi
        d2h += bo
    drain()
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    out["e2e"] = {"value": world * args.steps / (ms_e2e / 1e3), "unit": "frames/s",
                  "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                  "api": "PlayerBuffer.apply_bytes (wire bytes -> GPU decode) + render_device_u8 "
                         "(uint8 sRGB display frame) + pinned D2H on a copy stream"}
    pipe = buf.to_device().pipe
    pipe.enable_timing(True)
    ku = []
    for i in range(10):
        buf.render_device(cams[i % len(cams)], 0)
        ku.append(pipe.k_used())
    kms = pipe.kernel_ms()
    pipe.enable_timing(False)
    t_f = kms.get("raster_fwd", 0.0) / 10 / 1e3
    P = W * H
    b = 40.0 * float(np.mean(ku)) + 20.0 * P
    peak, kind = load_peaks()
    out["roofline"] = {"bound": "hbm", "achieved": b / t_f / 1e9, "peak": peak, "unit": "GB/s",
                       "frac": b / t_f / 1e9 / peak, "traffic": None, "kernel": "raster_fwd",
                       "peak_source": kind, "bytes_per_view": b, "K_used": float(np.mean(ku)),
                       "ms_per_view": {"raster_fwd": kms.get("raster_fwd", 0.0) / 10}}
    return out


def bracket_random_init(args, dp, scene, ds):
    """The same measurement from the reference's own init (init_state,
    train.py:207-235: frame-0 point cloud, opacity 0.1, nearest-neighbour
    scales) after the same genesis / schedule / mature(1) setup: the
    other end of the model-state range the headline's converged proxy sits
    at.  Same views and ground truth; W warm-up + K timed steps."""
    import torch

    from paper_2409_07759_b200 import train

    c, _, _, state, window = build_workload(args.config, dp, "random", scene_ds=(scene, ds))
    train.train_swin(window[0], window[1], state, ds, iterations=args.warmup)
    state.device.pipe.enable_timing(True)
    ms = time_steps(state, ds, window, args.steps, dp)
    kms = state.device.pipe.kernel_ms()
    state.device.pipe.enable_timing(False)
    out = {"init": "init_state from the frame-0 point cloud (train.py:207-235)",
           "value": args.steps / (ms / 1e3), "unit": "views/s", "ms_per_step": ms / args.steps,
           "ms_per_view": {k: kms.get(k, 0.0) / args.steps for k in ("raster_fwd", "raster_bwd")}}
    del state
    torch.cuda.empty_cache()
    return out


def workload_config(c, window, world, init):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": c["name"], "width": c["W"], "height": c["H"], "num_gs": c["num_gs"],
            "gt_gaussians": c["gt_n"], "swin_size": c["swin"], "window": list(window),
            "parallelism": f"dp{world}",
            "init": ("ground-truth splats (converged-model proxy)" if init == "gt"
                     else "init_state from the frame-0 point cloud"),
            "global_batch": world,
            "l2": "per-step working set > 126 MB L2 (tile pairs + optimizer state); "
                  "no explicit flush"}


def run_reference(args, c):
    """--impl reference: the reference algorithm (oracle/ port: fp64 numpy +
    the C pixel loops, all host threads) training whole 1352x1014 views of
    the same workload (CpuTrainer), W untimed + K timed steps; then, untimed,
    one whole view on ONE core and a 256^2-crop extrapolation for context."""
    from oracle import splat_oracle as O

    O.build_oracle()
    threads = O.default_threads()
    t0 = time.perf_counter()
    tr = CpuTrainer(c, threads)
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        tr.step()
    times = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        tr.step()
        times.append(time.perf_counter() - t1)
    total = float(np.sum(times))
    value = args.steps / total
    t1 = time.perf_counter()
    tr.step(threads=1)
    one_core_s = time.perf_counter() - t1
    crop_s = cpu_crop_view(tr, crop=256, n_crops=4, threads=threads)
    K = [k for k, _ in tr.stats]
    K_used = [u for _, u in tr.stats]
    sample = (f"whole {c['W']}x{c['H']} training views, {threads} threads: oracle port of the "
              f"reference (fp64; pixel loops in C over tile lists, numpy stages), "
              f"{total / args.steps:.2f} s/view")
    return {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) DyNeRF-shaped recipe, oracle-rendered ground truth)",
        "impl": "reference",
        "config": workload_config(c, tr.win, 1, "gt"),
        "cpu_baseline": {"value": value, "unit": "views/s", "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model_name(),
                         "one_core_s_per_view": one_core_s,
                         "crop256_extrapolated_s_per_view": crop_s,
                         "K_per_view": float(np.mean(K)), "K_used_per_view": float(np.mean(K_used)),
                         "setup_s": setup_s},
        "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def run_reference_render(args):
    """Config 5 on the host: the oracle's reference forward (global-order
    blend, fp64, all threads) over crop cameras of a 1920x1080 view of the 1M
    slot buffer, extrapolated by P / P_crop."""
    from oracle import splat_oracle as O
    from paper_2409_07759_b200.synth import make_scene

    O.build_oracle()
    threads = O.default_threads()
    n = 1_000_000
    k = (300.0 / n) ** (1.0 / 3.0)
    scene = make_scene(7, 300, [], n, scale_range=(0.045 * k, 0.1 * k))
    g0 = scene.gaussians_at(0)
    rng = np.random.default_rng(0)
    idx = np.concatenate([np.arange(len(g0)), rng.integers(0, len(g0), n - len(g0))])
    arr = g0.take(idx)
    W, H, f = 1920, 1080, 2100.0
    half = np.radians(70.0) / 2
    ang = -half
    center = np.array([3 * np.sin(ang), 0.25 * np.sin(2.1 * ang), -3 * np.cos(ang)])
    fwd = -center / np.linalg.norm(center)
    right = np.cross([0.0, 1.0, 0.0], fwd)
    right /= np.linalg.norm(right)
    R = np.stack([right, np.cross(fwd, right), fwd])
    crop = 96
    times = []
    for _ in range(max(args.steps, 1)):
        t_pix = 0.0
        t0 = time.perf_counter()
        cache = O.project_arrays(_Cam(W, H, f, f, W / 2, H / 2, R, -R @ center), arr.means,
                                 arr.quats, arr.scales, arr.opacities, arr.colors)
        t_gauss = time.perf_counter() - t0
        for xc, yc in [(W // 4, H // 4), (3 * W // 4, H // 4), (W // 4, 3 * H // 4),
                       (3 * W // 4, 3 * H // 4)]:
            cc = _Cam(crop, crop, f, f, W / 2 - (xc - crop // 2), H / 2 - (yc - crop // 2), R,
                      -R @ center)
            c2 = O.project_arrays(cc, arr.means, arr.quats, arr.scales, arr.opacities, arr.colors)
            t1 = time.perf_counter()
            if c2 is not None:
                O.blend_forward(c2, crop, crop, nthreads=threads)
            t_pix += time.perf_counter() - t1
        times.append(t_pix / 4 * (W * H) / (crop * crop) + t_gauss)
    tv = float(np.mean(times))
    v = 1.0 / tv
    return {"metric": METRIC5, "value": v, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tv * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "render-only streaming playback: 1M lifespan Gaussians, "
                                   "1920x1080 novel views", "threads": threads},
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": f"crop-extrapolated: 4 crops of {crop}^2 px"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="after warm-up run N steps between cudaProfilerStart/Stop and exit "
                         "(for ncu --profile-from-start off); prints no JSON")
    ap.add_argument("--strip", type=int, default=0, help="raster pixels per lane (2/4/8); 0 = library default")
    ap.add_argument("--strip-fwd", type=int, default=0, help="forward strip only (overrides --strip)")
    ap.add_argument("--init", default="gt", choices=["gt", "random"],
                    help="model state: ground-truth splats (converged proxy) or init_state")
    ap.add_argument("--binning", default="counting", choices=["counting", "sort"],
                    help="tile binning: chunked counting sort (default) or emit + radix pair sort")
    ap.add_argument("--timing-sample", type=float, default=0.25,
                    help="fraction of timed views whose raster launches carry CUDA events")
    ap.add_argument("--no-bracket", dest="bracket", action="store_false",
                    help="skip the random-init bracket measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "ours" and args.binning != "counting":
        from paper_2409_07759_b200 import raster

        raster.set_binning(args.binning)
    c = CONFIGS.get(args.config)
    rank = int(os.environ.get("RANK", "0"))
    if args.config == 5:
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps(run_reference_render(args)), flush=True)
            return
        import torch

        from paper_2409_07759_b200.parallel import init_from_env

        from paper_2409_07759_b200.parallel import local_device_index

        dp = init_from_env("nccl")
        torch.cuda.set_device(local_device_index())
        out = run_render_only(args, dp)
        if rank == 0:
            print(json.dumps(out), flush=True)
        return

    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args, c)), flush=True)
        return

    import torch

    from paper_2409_07759_b200.parallel import init_from_env

    dp = init_from_env("nccl")
    if args.strip:
        from paper_2409_07759_b200 import _lib

        _lib.check(_lib.lib().ss_set_raster_strip(args.strip), "set_raster_strip")
    if args.strip_fwd:
        from paper_2409_07759_b200 import _lib

        bwd = args.strip or 4
        _lib.check(_lib.lib().ss_set_raster_strips(args.strip_fwd, bwd), "set_raster_strips")
    from paper_2409_07759_b200.parallel import local_device_index

    local = local_device_index()  # LOCAL_RANK wrapped onto the visible GPUs
    torch.cuda.set_device(local)
    world = 1 if dp is None else dp.world_size
    c, scene, ds, state, window = build_workload(args.config, dp, args.init)
    from paper_2409_07759_b200 import train

    train.train_swin(window[0], window[1], state, ds, iterations=args.warmup)
    if args.profile_steps:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        train.train_swin(window[0], window[1], state, ds, iterations=args.profile_steps)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        pipe = state.device.pipe
        print(json.dumps({"profiled_steps": args.profile_steps, "n_pairs": pipe.n_pairs,
                          "K_used": pipe.k_used(), "n_active": pipe.n}))
        return
    # raster kernel times come from CUDA events recorded by the native driver
    # on the launch stream around the raster launches INSIDE the timed region,
    # on a seeded random quarter of the views (an event between two kernels
    # stops the second launching early, so timing every view would cost the
    # step ~1.5 %; the sample is an unbiased estimate of the mean launch)
    snap = snapshot_state(state)  # e2e and K_used replay the same trajectory
    state.device.pipe.enable_timing(True, sample=args.timing_sample)
    with ClockSampler(local) as clocks:
        ms = time_steps(state, ds, window, args.steps, dp)
    kms = state.device.pipe.kernel_ms()
    state.device.pipe.enable_timing(False)
    # K_used needs per-view host reads: measured over the first timed views
    # replayed from the snapshot (untimed)
    restore_state(state, snap)
    _, k_used, k_pairs, n_act = roofline_pass(state, ds, window, min(args.steps, 10))
    views_per_s = world * args.steps / (ms / 1e3)
    out = {
        "metric": METRIC, "value": views_per_s, "unit": "views/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SURVEY.md §8(d) DyNeRF-shaped recipe, GPU-rendered ground truth)",
        "config": workload_config(c, window, world, args.init),
        "clocks": clocks.summary(),
    }
    if not args.no_e2e:
        feed = HostFeed(ds, window, c["views"])
        rb = LossReadback(state.device)
        train.train_swin(window[0], window[1], state, feed, iterations=2, progress=rb)
        rb.flush()
        feed.h2d_bytes = 0
        rb.d2h_bytes = 0
        restore_state(state, snap)  # the same views and model states as `value`
        ms_e2e = time_steps(state, feed, window, args.steps, dp, progress=rb)
        if os.environ.get("SS_BENCH_RECHECK"):  # diagnostics: value again after the e2e arm
            restore_state(state, snap)
            ms_again = time_steps(state, ds, window, args.steps, dp)
            out["value_recheck"] = world * args.steps / (ms_again / 1e3)
        out["e2e"] = {"value": world * args.steps / (ms_e2e / 1e3), "unit": "views/s",
                      "h2d_bytes_per_step": feed.h2d_bytes // args.steps,
                      "d2h_bytes_per_step": rb.d2h_bytes // args.steps,
                      "api": "train.train_swin, ground truth from pinned host memory each step (copy stream), loss read back each step (one step lag)"}
    nview = max(kms.get("views", 0), 1)
    t_raster = (kms.get("raster_fwd", 0.0) + kms.get("raster_bwd", 0.0)) / nview / 1e3
    P = c["W"] * c["H"]
    b_raster = 116.0 * k_used + 52.0 * P
    peak, peak_kind = load_peaks()
    achieved = b_raster / t_raster / 1e9 if t_raster > 0 else 0.0
    traffic, traffic_note = load_traffic(["raster_fwd", "raster_bwd"])
    out["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                       "frac": achieved / peak, "traffic": traffic,
                       "traffic_source": traffic_note,
                       "ncu_counters": load_ncu_counters(["raster_fwd", "raster_bwd"]),
                       "issue_note": "the raster kernels are instruction-issue bound (ncu "
                                     "issue_active, profiles/): the HBM frac is low by design",
                       "kernel": "raster_fwd + raster_bwd", "peak_source": peak_kind,
                       "bytes_per_view": b_raster, "K_used": k_used, "K": k_pairs,
                       "timing": "kernel ms: CUDA events around the raster launches of "
                                 f"{kms.get('views', 0)} of the {args.steps} timed views (seeded "
                                 f"random sample, p={args.timing_sample}); K_used: the first 10 "
                                 "timed steps replayed from a snapshot",
                       "active_splats": n_act, "pixels": P,
                       "ms_per_view": {"raster_fwd": kms.get("raster_fwd", 0) / nview,
                                       "raster_bwd": kms.get("raster_bwd", 0) / nview}}
    ours, aten, names = count_launches(state, ds, window)
    out["gpu_launches"] = ours * args.steps
    out["gpu_launches_per_step"] = ours
    if args.bracket and world == 1 and args.init == "gt":
        out["bracket"] = bracket_random_init(args, dp, scene, ds)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import splat_oracle as O

        O.build_oracle()
        threads = O.default_threads()
        tr = CpuTrainer(c, threads, n_gt=2)
        t1 = time.perf_counter()
        for _ in range(2):
            tr.step()
        t = (time.perf_counter() - t1) / 2
        out["cpu_baseline"] = {"value": 1.0 / t, "unit": "views/s", "cores": threads,
                               "kind": "port", "cpu_model": cpu_model_name(),
                               "sample": f"2 whole {c['W']}x{c['H']} training views of this "
                                         f"workload through the oracle port of the reference "
                                         f"(fp64, all host threads), {t:.2f} s/view"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dp is not None:
        dp.barrier()


if __name__ == "__main__":
    main()
