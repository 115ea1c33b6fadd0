"""Where the GPU waits for the host: for each kernel of a few config-3 steps,
the lag between its host launch call and its GPU start (torch profiler with
CPU + CUDA activities, correlation ids).  Negative slack = the GPU was idle
waiting for this launch.

    python tools/launch_lag.py [--steps 3]
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2409_07759_b200 import train

    c, scene, ds, state, window = bench.build_workload(3, None, "gt")
    train.train_swin(window[0], window[1], state, ds, iterations=8)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        train.train_swin(window[0], window[1], state, ds, iterations=a.steps)
        torch.cuda.synchronize()
    path = ROOT / "gpurun_out" / "trace.json"
    prof.export_chrome_trace(str(path))
    tr = json.load(open(path))
    ev = tr["traceEvents"] if isinstance(tr, dict) else tr
    launches = {}
    kernels = []
    for e in ev:
        args = e.get("args", {})
        cid = args.get("correlation")
        if cid is None or "ts" not in e:
            continue
        if e.get("cat") in ("cuda_runtime", "cuda_driver"):
            launches[cid] = (e["ts"], e.get("dur", 0), e["name"])
        elif e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"):
            kernels.append((e["ts"], e.get("dur", 0), e["name"], cid))
    kernels.sort()
    rows = []
    prev_end = None
    for ts, dur, name, cid in kernels:
        if cid in launches and prev_end is not None:
            lts, ldur, lname = launches[cid]
            idle = ts - prev_end
            rows.append((idle, ts - (lts + ldur), name[:60], lname))
        prev_end = ts + dur if prev_end is None else max(prev_end, ts + dur)
    print("gpu_idle_us  launch_to_start_us  kernel  (launch call)")
    for idle, lag, name, lname in rows:
        if idle > 2.0:
            print(f"{idle:8.1f} {lag:8.1f}  {name}  ({lname})")


if __name__ == "__main__":
    main()
