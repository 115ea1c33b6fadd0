"""B200-native SwinGS sliding-window training hot path.

A drop-in for the reference package ``splatstream`` on the path named in
BASELINE.json (active-set compaction -> EWA projection -> tile binning ->
alpha-blend forward -> L1+SSIM loss -> per-pixel backward -> Adam + SGLD +
MCMC relocation, plus the per-frame update export).  The host API mirrors
the reference's names and semantics; the compute runs in hand-written
sm_100a CUDA kernels (libswings.so, include/swings.h) with no CPU fallback.

    import paper_2409_07759_b200 as splatstream
"""

from .core import (Camera, Gaussian, GaussianArrays, InvalidParameterError, Lifespan, SplatError,
                   StateError, StreamParams, covariance, intensity, is_active, slice_slot)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-backed modules import torch and the CUDA library lazily.
    import importlib

    lazy = {
        "Image": "raster", "Splat2D": "raster", "project": "raster", "psnr": "raster",
        "read_png": "raster", "render": "raster", "render_backward": "raster",
        "render_arrays": "raster", "render_arrays_backward": "raster", "write_png": "raster",
        "ConsistencyError": "raster", "loss": "loss", "LossBreakdown": "loss",
        "TrainConfig": "train", "train_video": "train", "train_swin": "train",
        "init_state": "train", "FrameDataset": "dataset", "load_frame": "dataset",
        "synth_scene": "synth", "ContainerReader": "codec", "ContainerWriter": "codec",
        "Manifest": "codec", "PROFILE_FULL": "codec", "PROFILE_QUANT": "codec",
        "encode_records": "codec", "decode_records": "codec", "pack_slice": "codec",
        "unpack_slice": "codec", "read_container": "codec", "bandwidth": "codec",
        "render_offline": "player", "PlayerBuffer": "player",
    }
    if name in lazy:
        mod = importlib.import_module(f".{lazy[name]}", __name__)
        return getattr(mod, "loss" if name == "loss" else name)
    raise AttributeError(name)
