"""Time the device-resident ABR tail drop (subsample_records_device) on a
config-5-sized slice (50k records, both profiles), CUDA events over 200 calls.

    python tools/micro/abr_rate.py
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2409_07759_b200 import abr, codec  # noqa: E402
from paper_2409_07759_b200.core import GaussianArrays, Lifespan  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    n = 50_000
    q = rng.normal(size=(n, 4))
    arr = GaussianArrays(rng.uniform(-1, 1, (n, 3)), q / np.linalg.norm(q, axis=1, keepdims=True),
                         np.exp(rng.uniform(-5, -1, (n, 3))), rng.uniform(0, 1, n),
                         rng.uniform(0, 1, (n, 3)))
    out = {}
    for pid in (0, 1):
        prof = codec.PROFILES[pid]
        blob = codec.pack_slice(arr, Lifespan(3, 3, 8), prof, 5)
        dev = torch.frombuffer(bytearray(blob[codec.HEADER_SIZE:]), dtype=torch.uint8).cuda()
        for _ in range(10):
            abr.subsample_records_device(dev, n, prof, 0.5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            abr.subsample_records_device(dev, n, prof, 0.5)
        e1.record()
        torch.cuda.synchronize()
        out[f"profile{pid}_us_per_slice"] = round(e0.elapsed_time(e1) * 1e3 / 200, 1)
    print(json.dumps({"records": n, "fraction": 0.5, **out}))


if __name__ == "__main__":
    main()
