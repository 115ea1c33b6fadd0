"""Race / bounds evidence without compute-sanitizer (closed on this GPU
pool: runs under it have left GPUs needing a reset).

  * the checked build (lib/libswings_checked.so, -DSS_CHECKED): device-side
    SS_DCHECKs on every scatter / emit / compaction / depth-order write
    position, tile range and reduction target trap on a violation; the
    raster, binning, compaction and view-driver GPU tests run through it in
    a subprocess and must pass with no check firing;
  * repetition: the kernels with cross-thread hand-offs -- warp-private
    shared staging and the batched reduction rows (raster.cu), the
    last-CTA done counter that publishes K to a host-mapped word (view.cu),
    the barrier-ranked binning scatter (binning.cu) -- run many times and
    their outputs (tile lists, images, deterministic gradients, compaction
    order) must be bit-identical every time.  A race shows up as a
    run-to-run difference.
"""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import arc_camera, synth_like

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

CHECKED_TESTS = [
    "tests/test_gpu_raster.py::test_forward_matches_golden",
    "tests/test_gpu_raster.py::test_backward_matches_golden",
    "tests/test_gpu_raster.py::test_huge_and_tiny_splats_tile_keys_and_image",
    "tests/test_gpu_raster.py::test_deterministic_backward_bit_identical",
    "tests/test_gpu_raster.py::test_binning_modes_agree",
    "tests/test_gpu_raster.py::test_wide_frame_chunked_binning",
    "tests/test_gpu_raster.py::test_depth_order_exact_on_adversarial_keys",
    "tests/test_gpu_raster.py::test_concurrent_views_from_two_threads",
    "tests/test_gpu_raster.py::test_config3_full_view_structural",
    "tests/test_gpu_trainer.py::test_compaction_bit_exact_through_window_slides",
    "tests/test_gpu_trainer.py::test_compaction_empty_and_large",
    "tests/test_gpu_trainer.py::test_deterministic_training_is_bit_reproducible",
]


def test_checked_build_runs_clean():
    env = dict(os.environ, SS_LIB_VARIANT="checked")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        *CHECKED_TESTS], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1500)
    out = r.stdout + r.stderr
    assert "SS_DCHECK failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]


def test_checked_build_is_the_one_loaded():
    code = ("import os; from paper_2409_07759_b200 import _lib; _lib.lib(); "
            "print([l for l in open('/proc/self/maps') if 'libswings' in l][0].split()[-1])")
    env = dict(os.environ, SS_LIB_VARIANT="checked")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().endswith("libswings_checked.so")


def test_repeated_views_are_bit_identical():
    """60 repetitions of forward + deterministic backward on a 60k-splat
    800x600 view: tile lists, image and gradients never change."""
    import paper_2409_07759_b200 as P
    from paper_2409_07759_b200 import raster as R

    n = 60_000
    arr = P.GaussianArrays(*synth_like(np.random.default_rng(2), n, (300.0 / 60_000) ** (1 / 3)))
    c = arc_camera(6, 20, 800, 600)
    cam = P.Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.rotation, c.translation)
    gdir = np.random.default_rng(3).normal(size=(600, 800, 3))
    R.set_deterministic(True)
    try:
        ref = None
        for rep in range(60):
            img = R.render_arrays(cam, arr).pixels
            st = R.pipeline().state()
            lists = (st["vals"].numpy().copy(), st["ranges"].numpy().copy(), st["n_pairs"])
            g = R.render_arrays_backward(cam, arr, gdir) if rep % 6 == 0 else None
            if ref is None:
                ref = (img, lists, g)
                continue
            assert np.array_equal(img, ref[0]), rep
            assert lists[2] == ref[1][2] and np.array_equal(lists[0], ref[1][0]), rep
            assert np.array_equal(lists[1], ref[1][1]), rep
            if g is not None:
                for k in g:
                    assert np.array_equal(g[k], ref[2][k]), (rep, k)
    finally:
        R.set_deterministic(False)


def test_repeated_compaction_and_pair_count_readback():
    """The mapped-word K readback and the compaction scan, 200 times: the
    same K and the same active rows every time (sequence-numbered words
    never return a stale K)."""
    import torch

    from paper_2409_07759_b200.engine import Store, ViewPipeline, device
    import paper_2409_07759_b200 as P

    arr = P.GaussianArrays(*synth_like(np.random.default_rng(4), 30_000, 0.3))
    rows = torch.from_numpy(arr.rows()).to(device())
    store = Store(opt=None, mat=rows)
    pipe = ViewPipeline()
    cams = []
    for i in range(5):
        c = arc_camera(i, 5, 320, 240)
        cams.append(P.Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.rotation,
                             c.translation))
    first = {}
    for rep in range(200):
        i = rep % 5
        img = pipe.forward(store, None, len(arr), cams[i])
        k = pipe.n_pairs
        if i not in first:
            first[i] = (k, img.clone())
        else:
            assert k == first[i][0], (rep, k, first[i][0])
            assert torch.equal(img, first[i][1]), rep
