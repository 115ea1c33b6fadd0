"""How often the GPU runs dry at a training-step boundary (config 3): after
each step, an event is recorded behind the step's last kernel; when the host
reaches the next step head it queries that event.  "done" means the GPU had
already finished the previous step -- the host is the bottleneck there.
Also reports host wall time per phase (compaction, forward call, rest).

    python tools/host_behind.py [--steps 30]
"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2409_07759_b200 import device_model, train

    c, scene, ds, state, window = bench.build_workload(3, None, "gt")
    train.train_swin(window[0], window[1], state, ds, iterations=5)
    torch.cuda.synchronize()
    model = state.device
    stats = {"steps": 0, "gpu_idle_at_head": 0, "compact_miss": 0}
    phase = {"compact": 0.0, "forward": 0.0, "total": 0.0}
    orig_step, orig_compact, orig_fwd = model.train_step, model.compact, model.pipe.forward
    prev = {"ev": None}

    def compact(frame):
        t = time.perf_counter()
        miss = frame not in model._active_cache or model.dirty
        r = orig_compact(frame)
        phase["compact"] += time.perf_counter() - t
        stats["compact_miss"] += int(miss)
        return r

    def forward(*args, **kw):
        t = time.perf_counter()
        r = orig_fwd(*args, **kw)
        phase["forward"] += time.perf_counter() - t
        return r

    def step(*args, **kw):
        t = time.perf_counter()
        if prev["ev"] is not None and prev["ev"].query():
            stats["gpu_idle_at_head"] += 1
        r = orig_step(*args, **kw)
        ev = torch.cuda.Event()
        ev.record()
        prev["ev"] = ev
        stats["steps"] += 1
        phase["total"] += time.perf_counter() - t
        return r

    model.train_step, model.compact, model.pipe.forward = step, compact, forward
    t0 = time.perf_counter()
    train.train_swin(window[0], window[1], state, ds, iterations=a.steps)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    n = stats["steps"]
    print({**stats, "wall_ms_per_step": 1e3 * wall / n,
           **{f"host_{k}_ms_per_step": 1e3 * v / n for k, v in phase.items()}})


if __name__ == "__main__":
    main()
