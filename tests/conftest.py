import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running")


class Cam:
    """Duck-typed camera for the oracle (width, height, fx, fy, cx, cy, rotation, translation)."""

    def __init__(self, width, height, fx, fy, cx, cy, rotation, translation):
        self.width, self.height = int(width), int(height)
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.rotation = np.asarray(rotation, dtype=np.float64)
        self.translation = np.asarray(translation, dtype=np.float64)


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_cam(d, prefix="cam"):
    w, h = d[f"{prefix}_wh"]
    fx, fy, cx, cy = d[f"{prefix}_f"]
    return Cam(w, h, fx, fy, cx, cy, d[f"{prefix}_R"], d[f"{prefix}_T"])


RASTER_CASES = ["random30", "frozen", "arc400", "saturate", "ties", "rot1k"]


def random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def synth_like(rng, n, scale_k=1.0):
    """SURVEY.md §8(d) synthetic recipe (synth.py:92-147 distributions)."""
    base = rng.uniform(-0.75, 0.75, size=(n, 3))
    base[:, 2] *= 0.6
    quats = random_unit_quats(rng, n)
    scales = np.exp(rng.uniform(np.log(0.045 * scale_k), np.log(0.1 * scale_k), size=(n, 3)))
    opac = rng.uniform(0.7, 0.98, size=n)
    colors = rng.uniform(0.15, 1.0, size=(n, 3))
    return base, quats, scales, opac, colors


def arc_camera(i, n_views, width, height, radius=3.0, focal=None, arc_degrees=36.0):
    """synth.py:23-45 arc cameras (restated for tests)."""
    if focal is None:
        focal = 70.0 * width / 64
    half = np.radians(arc_degrees) / 2.0
    angs = [0.0] if n_views == 1 else np.linspace(-half, half, n_views)
    ang = angs[i]
    cy_off = 0.25 * np.sin(2.1 * ang)
    center = np.array([radius * np.sin(ang), cy_off, -radius * np.cos(ang)])
    fwd = -center / np.linalg.norm(center)
    up = np.array([0.0, 1.0, 0.0])
    right = np.cross(up, fwd)
    right /= np.linalg.norm(right)
    cam_up = np.cross(fwd, right)
    rot = np.stack([right, cam_up, fwd])
    return Cam(width, height, focal, focal, width / 2.0, height / 2.0, rot, -rot @ center)
