"""cProfile of the host side of 30 config-3 training steps (where Python time goes)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_07759_b200 import train  # noqa: E402

c, scene, ds, state, window = bench.build_workload(int(sys.argv[1]) if len(sys.argv) > 1 else 3, None, "gt")
train.train_swin(window[0], window[1], state, ds, iterations=5)
torch.cuda.synchronize()
t = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
train.train_swin(window[0], window[1], state, ds, iterations=30)
pr.disable()
torch.cuda.synchronize()
print("wall per step ms", (time.perf_counter() - t) / 30 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
