"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference package is imported under the alias ``ref_splatstream`` from
/root/reference/pkg/src/splatstream.  Nothing at test time reads
/root/reference; the tests only read the .npz files written here.

Fixtures:
  raster_*.npz   render_arrays / render_arrays_backward / _project_arrays
                 outputs on small scenes (reference raster.py, _kernels.py)
  loss.npz       loss() / ssim_with_gradient() (reference loss.py)
  optim.npz      _optimizer_step / sgld_perturb / relocate with the numpy
                 draws the reference consumed (reference train.py)
  train_tiny.npz a few train_swin iterations on a tiny synthetic scene
  train_window.npz  genesis -> schedule_expire -> mature(1) -> window [1, 3)
                 -> mature(2) -> window [2, 4): matured rows in the views,
                 relocation inside a window, gamma^w < 1 on a surviving
                 generation (reference train.py:353-506)
  golden_render.npz  the frontend fixture model (golden_decode.json) rendered
                 at frame 3 from golden_camera.json with render_offline
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src/splatstream")
OUT = Path(__file__).resolve().parent


def load_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    spec = importlib.util.spec_from_file_location(
        "ref_splatstream", REF_SRC / "__init__.py", submodule_search_locations=[str(REF_SRC)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ref_splatstream"] = mod
    spec.loader.exec_module(mod)
    import ref_splatstream.raster  # noqa: F401
    import ref_splatstream.train  # noqa: F401
    import ref_splatstream.loss  # noqa: F401
    import ref_splatstream.player  # noqa: F401
    return mod


def random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def random_arrays(ref, rng, n, mean_lo=(-0.5, -0.5, 2.0), mean_hi=(0.5, 0.5, 4.0),
                  scale_lo=0.02, scale_hi=0.1, opacity_lo=0.1, opacity_hi=0.9):
    """Mirrors the reference's tests/conftest.py:12-20 recipe."""
    return ref.core.GaussianArrays(
        rng.uniform(mean_lo, mean_hi, size=(n, 3)),
        random_unit_quats(rng, n),
        np.exp(rng.uniform(np.log(scale_lo), np.log(scale_hi), size=(n, 3))),
        rng.uniform(opacity_lo, opacity_hi, size=n),
        rng.uniform(0.0, 1.0, size=(n, 3)),
    )


def cam_dict(cam):
    return dict(width=cam.width, height=cam.height, fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                rotation=cam.rotation, translation=cam.translation)


def save_raster_case(ref, name, cam, arrays, grad_img, trainable=None):
    cache = ref.raster._project_arrays(cam, arrays)
    img = ref.raster.render_arrays(cam, arrays).pixels
    grads = ref.raster.render_arrays_backward(cam, arrays, grad_img, trainable=trainable)
    out = dict(
        cam_wh=np.array([cam.width, cam.height]),
        cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        cam_R=cam.rotation, cam_T=cam.translation,
        means=arrays.means, quats=arrays.quats, scales=arrays.scales,
        opacities=arrays.opacities, colors=arrays.colors,
        image=img, grad_image=grad_img,
        trainable=np.ones(len(arrays), bool) if trainable is None else np.asarray(trainable),
        **{f"grad_{k}": v for k, v in grads.items()},
    )
    if cache is not None:
        x0, x1, y0, y1 = cache["bbox"]
        out.update(src=cache["src"], order=cache["order"], mean2d=cache["mean2d"],
                   inv2d=cache["inv2d"], z=cache["z"], bbox=np.stack([x0, x1, y0, y1], 1))
    np.savez_compressed(OUT / f"raster_{name}.npz", **out)
    print(f"raster_{name}: n={len(arrays)} kept={0 if cache is None else len(cache['src'])}")


def make_raster(ref):
    Camera = ref.core.Camera
    GaussianArrays = ref.core.GaussianArrays
    rng = np.random.default_rng(12345)
    ident = Camera(32, 32, 60.0, 60.0, 16.0, 16.0, np.eye(3), np.zeros(3))

    # 1. conftest-style random splats, identity camera (test_raster.py:207-212)
    arr = random_arrays(ref, rng, 30)
    save_raster_case(ref, "random30", ident, arr, rng.normal(size=(32, 32, 3)))

    # 2. frozen rows (test_raster.py:311-318)
    arr = random_arrays(ref, rng, 10)
    save_raster_case(ref, "frozen", ident, arr, np.ones((32, 32, 3)),
                     trainable=np.array([True] * 5 + [False] * 5))

    # 3. arc camera, synth-like volume, non-square image, cull on all sides
    cams = ref.synth.arc_cameras(3, 56, 40, radius=3.0, focal=70.0 * 56 / 64, arc_degrees=36.0)
    n = 400
    base = rng.uniform(-0.75, 0.75, size=(n, 3))
    base[:, 2] *= 0.6
    base[:20] *= 4.0  # some far off-screen / behind
    arr = GaussianArrays(base, random_unit_quats(rng, n),
                         np.exp(rng.uniform(np.log(0.03), np.log(0.08), size=(n, 3))),
                         rng.uniform(0.7, 0.98, size=n), rng.uniform(0.15, 1.0, size=(n, 3)))
    save_raster_case(ref, "arc400", cams[2], arr, rng.normal(size=(40, 56, 3)),
                     trainable=rng.uniform(size=n) < 0.7)

    # 4. saturating: opaque, dense -> the T < 1e-4 break and the 0.999 clamp engage
    n = 300
    arr = random_arrays(ref, rng, n, scale_lo=0.05, scale_hi=0.2, opacity_lo=0.9, opacity_hi=0.9999)
    cam = Camera(40, 36, 50.0, 55.0, 20.0, 17.5, np.eye(3), np.zeros(3))
    save_raster_case(ref, "saturate", cam, arr, rng.normal(size=(36, 40, 3)))

    # 5. depth ties broken by index (test_raster.py:223-231) + coincident splats
    G = ref.core.Gaussian
    gs = [G([0, 0, 2.0], [1, 0, 0, 0], [0.05] * 3, 0.5, [1.0, 0.0, 0.0]),
          G([0, 0, 2.0], [1, 0, 0, 0], [0.05] * 3, 0.5, [0.0, 1.0, 0.0]),
          G([0.01, 0, 2.0], [1, 0, 0, 0], [0.04] * 3, 0.3, [0.0, 0.0, 1.0]),
          G([0, 0, 2.5], [1, 0, 0, 0], [0.05] * 3, 0.3, [0.0, 1.0, 0.0])]
    cam33 = Camera(33, 33, 60.0, 60.0, 16.0, 16.0, np.eye(3), np.zeros(3))
    save_raster_case(ref, "ties", cam33, GaussianArrays.from_gaussians(gs),
                     rng.normal(size=(33, 33, 3)))

    # 6. larger rotated-camera scene, 1k splats at 96x80
    R = ref.core.quat_to_rotmat(random_unit_quats(rng, 1)[0])
    cam = Camera(96, 80, 90.0, 95.0, 47.5, 40.0, R, np.array([0.05, -0.1, 3.0]))
    n = 1000
    arr = GaussianArrays(rng.uniform(-0.6, 0.6, size=(n, 3)), random_unit_quats(rng, n),
                         np.exp(rng.uniform(np.log(0.01), np.log(0.06), size=(n, 3))),
                         rng.uniform(0.05, 0.99, size=n), rng.uniform(0.0, 1.0, size=(n, 3)))
    save_raster_case(ref, "rot1k", cam, arr, rng.normal(size=(80, 96, 3)))


def make_loss(ref):
    rng = np.random.default_rng(777)
    pred = rng.uniform(0.0, 1.0, size=(20, 24, 3))
    gt = rng.uniform(0.0, 1.0, size=(20, 24, 3))
    gt[3:6, 4:9] = pred[3:6, 4:9]   # exact ties -> sign(0) = 0
    n = 17
    opac = rng.uniform(0.01, 0.99, size=n)
    scales = rng.uniform(0.001, 0.2, size=(n, 3))
    arr = ref.core.GaussianArrays(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), scales,
                                  opac, np.zeros((n, 3)))
    br, grad, reg = sys.modules['ref_splatstream.loss'].loss(ref.raster.Image(pred), ref.raster.Image(gt), arr)
    ssim_v, ssim_g = sys.modules['ref_splatstream.loss'].ssim_with_gradient(pred, gt)
    np.savez_compressed(
        OUT / "loss.npz", pred=pred, gt=gt, opacities=opac, scales=scales, grad_image=grad,
        reg_opacity_logit=reg["opacity_logit"], reg_log_scale=reg["log_scale"],
        ssim_value=ssim_v, ssim_grad=ssim_g,
        breakdown=np.array([br.total, br.l1, br.ssim, br.photometric, br.opacity_term,
                            br.scale_term]))
    print("loss: ok")


def make_optim(ref):
    T = ref.train
    rng = np.random.default_rng(4242)
    out = {}
    ng, n = 3, 25
    gens = []
    for gi in range(ng):
        arr = random_arrays(ref, rng, n, opacity_lo=0.001, opacity_hi=0.95)
        params = {"mean": arr.means.copy(), "quat": arr.quats * rng.uniform(0.5, 2.0, (n, 1)),
                  "log_scale": np.log(arr.scales),
                  "opacity_logit": np.log(arr.opacities / (1 - arr.opacities)),
                  "color": arr.colors.copy()}
        params["color"][0] = [1.2, -0.1, 0.5]  # clip exercised
        params["log_scale"][1] = [-20.0, -14.0, -13.0]  # floor exercised
        gens.append(T.SliceGen(slot=gi, lifespan=ref.core.Lifespan(0, 0, 5), params=params))
    for gi, g in enumerate(gens):
        for k in T.PARAM_GROUPS:
            out[f"p0_{gi}_{k}"] = g.params[k].copy()
    cfg = T.TrainConfig(swin_size=5, num_gs=500)
    # two Adam steps per generation with fresh grads (+ pre-existing t for gen 2)
    gens[2].adam_t = 7
    for step in range(2):
        for gi, g in enumerate(gens):
            grads = {k: rng.normal(size=g.params[k].shape) * 10.0 ** rng.uniform(-6, -1)
                     for k in T.PARAM_GROUPS}
            grads["mean"][3] = 0.0
            for k in T.PARAM_GROUPS:
                out[f"g{step}_{gi}_{k}"] = grads[k]
            T._optimizer_step(g, grads, cfg)
            out[f"t{step}_{gi}"] = np.array(g.adam_t)
            for k in T.PARAM_GROUPS:
                out[f"p{step + 1}_{gi}_{k}"] = g.params[k].copy()
                out[f"m{step + 1}_{gi}_{k}"] = g.adam_m[k].copy()
                out[f"v{step + 1}_{gi}_{k}"] = g.adam_v[k].copy()
    # SGD step on a copy of gen 0
    sgd = T.SliceGen(slot=0, lifespan=ref.core.Lifespan(0, 0, 5),
                     params={k: v.copy() for k, v in gens[0].params.items()})
    grads = {k: out[f"g1_0_{k}"] for k in T.PARAM_GROUPS}
    T._optimizer_step(sgd, grads, T.TrainConfig(swin_size=5, num_gs=500, optimizer="sgd"))
    for k in T.PARAM_GROUPS:
        out[f"sgd_{k}"] = sgd.params[k].copy()
    # SGLD: replay the generator to capture eta in draw order
    seed = 99
    etas_rng = np.random.default_rng(seed)
    for gi, g in enumerate(gens):
        out[f"eta_{gi}"] = etas_rng.standard_normal((n, 3))
    T.sgld_perturb(gens, 1.6e-4, 5e4, np.random.default_rng(seed))
    for gi, g in enumerate(gens):
        out[f"sgld_mean_{gi}"] = g.params["mean"].copy()
    # relocation: capture the uniforms choice() consumes
    seed = 5
    alpha = np.concatenate([T._sigmoid(g.params["opacity_logit"]) for g in gens])
    n_dead = int((alpha < 0.3).sum())
    out["reloc_uniforms"] = np.random.default_rng(seed).random(n_dead)
    for gi, g in enumerate(gens):
        for k in T.PARAM_GROUPS:
            out[f"pre_reloc_{gi}_{k}"] = g.params[k].copy()
            out[f"pre_reloc_m_{gi}_{k}"] = g.adam_m[k].copy()
            out[f"pre_reloc_v_{gi}_{k}"] = g.adam_v[k].copy()
    moved = T.relocate(gens, 0.3, np.random.default_rng(seed))
    out["reloc_moved"] = np.array(moved)
    for gi, g in enumerate(gens):
        for k in T.PARAM_GROUPS:
            out[f"post_reloc_{gi}_{k}"] = g.params[k].copy()
            out[f"post_reloc_m_{gi}_{k}"] = g.adam_m[k].copy()
            out[f"post_reloc_v_{gi}_{k}"] = g.adam_v[k].copy()
    out["n_gens"] = np.array(ng)
    np.savez_compressed(OUT / "optim.npz", **out)
    print(f"optim: relocated {moved}")


def make_train_tiny(ref):
    """A few reference train_swin iterations (genesis) on a tiny synthetic scene,
    with the per-iteration (frame, view) draws recorded by replaying the rng."""
    T = ref.train
    tmp = Path(tempfile.mkdtemp(prefix="golden_train_"))
    scene, ds = ref.synth.synth_scene(seed=3, total_frames=4, n_views=2, n_gaussians=40,
                                      out_dir=tmp / "ds", width=24, height=20)
    cfg = T.TrainConfig(swin_size=2, num_gs=40, genesis_iterations=3, window_iterations=2,
                        relocate_period=2, rng_seed=11)
    state = T.init_state(cfg)
    out = {"cam_count": np.array(ds.n_views)}
    for gi, g in enumerate(state.slices):
        for k in T.PARAM_GROUPS:
            out[f"init_{gi}_{k}"] = g.params[k].copy()
    gts = np.stack([np.stack([ds.load(f, v).pixels for v in range(ds.n_views)])
                    for f in range(ds.total_frames)])
    out["gt"] = gts
    for vi, cam in enumerate(ds.cameras):
        out[f"cam{vi}_R"] = cam.rotation
        out[f"cam{vi}_T"] = cam.translation
        out[f"cam{vi}_f"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy])
        out[f"cam{vi}_wh"] = np.array([cam.width, cam.height])
    out["rng_state_after_init"] = np.frombuffer(
        json.dumps(state.rng.bit_generator.state).encode(), dtype=np.uint8)
    T.train_swin(0, cfg.swin_size, state, ds)
    for gi, g in enumerate(state.slices):
        for k in T.PARAM_GROUPS:
            out[f"final_{gi}_{k}"] = g.params[k].copy()
        out[f"final_t_{gi}"] = np.array(g.adam_t)
    np.savez_compressed(OUT / "train_tiny.npz", **out)
    print("train_tiny: ok")


def make_train_window(ref):
    """Reference train_swin past genesis: two window slides with maturation,
    relocation at it = 0 and 2 of each window and a generation that survives
    a slide (windows_trained = 1 -> gamma^w = 0.5 on its mean gradients)."""
    T = ref.train
    tmp = Path(tempfile.mkdtemp(prefix="golden_window_"))
    scene, ds = ref.synth.synth_scene(seed=5, total_frames=5, n_views=2, n_gaussians=60,
                                      out_dir=tmp / "ds", width=28, height=24)
    cfg = T.TrainConfig(swin_size=2, num_gs=60, genesis_iterations=3, window_iterations=4,
                        relocate_period=2, rng_seed=13)
    state = T.init_state(cfg)
    out = {"cam_count": np.array(ds.n_views)}
    gts = np.stack([np.stack([ds.load(f, v).pixels for v in range(ds.n_views)])
                    for f in range(ds.total_frames)])
    out["gt"] = gts
    for vi, cam in enumerate(ds.cameras):
        out[f"cam{vi}_R"] = cam.rotation
        out[f"cam{vi}_T"] = cam.translation
        out[f"cam{vi}_f"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy])
        out[f"cam{vi}_wh"] = np.array([cam.width, cam.height])

    def snap(tag):
        for gi, g in enumerate(state.slices):
            for k in T.PARAM_GROUPS:
                out[f"{tag}_{gi}_{k}"] = g.params[k].copy()
            out[f"{tag}_t_{gi}"] = np.array(g.adam_t)
            out[f"{tag}_w_{gi}"] = np.array(g.windows_trained)
            out[f"{tag}_life_{gi}"] = np.array([g.lifespan.birth, g.lifespan.start,
                                                g.lifespan.expire])
        out[f"{tag}_n_matured"] = np.array(len(state.matured))
        for mi, m in enumerate(state.matured):
            out[f"{tag}_mat_{mi}_rows"] = np.concatenate(
                [m.arrays.means, m.arrays.quats, m.arrays.scales, m.arrays.opacities[:, None],
                 m.arrays.colors], axis=1)
            out[f"{tag}_mat_{mi}_life"] = np.array([m.lifespan.birth, m.lifespan.start,
                                                    m.lifespan.expire])

    T.train_swin(0, cfg.swin_size, state, ds)
    snap("genesis")
    T.schedule_expire(state)
    T.mature(1, state, writer=None)
    T.train_swin(1, 1 + cfg.swin_size, state, ds)
    snap("w1")
    T.mature(2, state, writer=None)
    T.train_swin(2, 2 + cfg.swin_size, state, ds, iterations=3)
    snap("w2")
    np.savez_compressed(OUT / "train_window.npz", **out)
    print("train_window: ok")


def make_golden_render(ref):
    fx = Path("/root/reference/pkg/frontend/test/fixtures")
    gens_json = json.loads((fx / "golden_decode.json").read_text())
    cam_json = json.loads((fx / "golden_camera.json").read_text())
    frame = json.loads((fx / "golden_render.json").read_text())["frame"]
    cam = ref.core.Camera.from_matrix(cam_json["width"], cam_json["height"], cam_json["fx"],
                                      cam_json["fy"], cam_json["cx"], cam_json["cy"],
                                      np.array(cam_json["world_to_camera"]).reshape(4, 4))
    parts = []
    out = {}
    for gi, g in enumerate(gens_json):
        n = len(g["opacities"])
        arr = ref.core.GaussianArrays(np.array(g["means"]).reshape(n, 3),
                                      np.array(g["quats"]).reshape(n, 4),
                                      np.array(g["scales"]).reshape(n, 3),
                                      np.array(g["opacities"]),
                                      np.array(g["colors"]).reshape(n, 3))
        valid = np.array(g["valid"], bool)
        ls = ref.core.Lifespan(*g["lifespan"])
        out[f"gen{gi}_means"] = arr.means
        out[f"gen{gi}_quats"] = arr.quats
        out[f"gen{gi}_scales"] = arr.scales
        out[f"gen{gi}_opacities"] = arr.opacities
        out[f"gen{gi}_colors"] = arr.colors
        out[f"gen{gi}_valid"] = valid
        out[f"gen{gi}_lifespan"] = np.array(g["lifespan"])
        parts.append((arr, valid, ls))
    decoded = [type("G", (), {"gaussians": a, "valid": v, "lifespan": l})() for a, v, l in parts]
    img = ref.player.render_offline(decoded, cam, frame)
    out.update(n_gens=np.array(len(gens_json)), frame=np.array(frame), image=img.pixels,
               cam_wh=np.array([cam.width, cam.height]),
               cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
               cam_R=cam.rotation, cam_T=cam.translation)
    np.savez_compressed(OUT / "golden_render.npz", **out)
    print(f"golden_render: frame {frame}, {len(gens_json)} generations")


def make_codec(ref):
    """encode_records / pack_slice bytes for both profiles and a whole container
    (reference codec.py:215-232, 298-320, 365-406)."""
    C = sys.modules["ref_splatstream.codec"]
    rng = np.random.default_rng(31)
    out = {}
    n = 257
    arr = random_arrays(ref, rng, n, opacity_lo=0.0, opacity_hi=1.0)
    arr.quats[:5] = [[1, 0, 0, 0], [0, 1, 0, 0], [0.5, 0.5, 0.5, 0.5], [0.7071, 0, 0.7071, 0],
                     [-0.3, 0.1, 0.9, -0.2]]
    out.update(means=arr.means, quats=arr.quats, scales=arr.scales, opacities=arr.opacities,
               colors=arr.colors)
    for pid in (0, 1):
        prof = C.PROFILES[pid]
        out[f"records_p{pid}"] = np.frombuffer(C.encode_records(arr, prof), dtype=np.uint8)
        ls = ref.core.Lifespan(7, 7, 12)
        out[f"slice_p{pid}"] = np.frombuffer(C.pack_slice(arr, ls, prof, swin_size=5),
                                             dtype=np.uint8)
        dec = C.decode_records(C.encode_records(arr, prof), prof)
        out[f"decoded_p{pid}"] = np.concatenate([dec.means, dec.quats, dec.scales,
                                                 dec.opacities[:, None], dec.colors], 1)
    tmp = Path(tempfile.mkdtemp(prefix="golden_codec_"))
    man = C.Manifest(num_gs=20, swin_size=2, fps=30.0, total_frames=3, profile_id=1,
                     scene_bounds=(-1, -1, -1, 1, 1, 1), camera_count=2)
    part = arr.take(np.arange(10))
    with C.ContainerWriter(tmp / "c.swin", man) as w:
        for i, birth in enumerate([0, 0, 1, 2, 3]):
            w.write_slice(C.pack_slice(part, ref.core.Lifespan(birth, birth, birth + 2),
                                       C.PROFILES[1], swin_size=2,
                                       slice_index=(i if i < 2 else None)))
    out["container"] = np.frombuffer((tmp / "c.swin").read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "codec.npz", **out)
    print("codec: ok")


def make_abr(ref):
    """ABR tail-drop selection (reference server.py:39-79): abr_keep_indices on
    fp64 opacities with ties, and subsample_slice_bytes on wire slices of both
    profiles (u8 opacities tie heavily), at several quality fractions."""
    C = sys.modules["ref_splatstream.codec"]
    S = sys.modules["ref_splatstream.server"]
    rng = np.random.default_rng(41)
    out = {}
    fractions = np.array([0.013, 0.1, 0.37, 0.5, 0.77, 0.999, 1.0])
    out["fractions"] = fractions
    opac = rng.uniform(0, 1, 1001)
    opac[::7] = 0.25                      # a large tie class
    opac[5:40:3] = opac[4]                # ties at high opacity
    opac[100:110] = 0.0
    out["opac"] = opac
    for i, q in enumerate(fractions):
        out[f"keep_{i}"] = S.abr_keep_indices(opac, float(q)).astype(np.int64)
    n = 613
    arr = random_arrays(ref, rng, n, opacity_lo=0.0, opacity_hi=1.0)
    arr.opacities[::5] = 0.5
    arr.opacities[1:60:4] = arr.opacities[0]
    for pid in (0, 1):
        prof = C.PROFILES[pid]
        blob = C.pack_slice(arr, ref.core.Lifespan(9, 9, 14), prof, swin_size=5)
        out[f"slice_p{pid}"] = np.frombuffer(blob, dtype=np.uint8)
        for i, q in enumerate(fractions):
            out[f"sub_p{pid}_{i}"] = np.frombuffer(S.subsample_slice_bytes(blob, float(q), prof),
                                                   dtype=np.uint8)
    np.savez_compressed(OUT / "abr.npz", **out)
    print("abr: ok")


def main():
    ref = load_reference()
    import ref_splatstream.synth  # noqa: F401
    if len(sys.argv) > 1:  # regenerate selected fixtures only, e.g. `train_window`
        for name in sys.argv[1:]:
            globals()[f"make_{name}"](ref)
        return
    make_raster(ref)
    make_loss(ref)
    make_optim(ref)
    make_train_tiny(ref)
    make_train_window(ref)
    make_golden_render(ref)
    import ref_splatstream.codec  # noqa: F401
    make_codec(ref)
    import ref_splatstream.server  # noqa: F401
    make_abr(ref)


if __name__ == "__main__":
    main()
