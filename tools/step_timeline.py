"""Per-step GPU timeline of the config-3 training step (torch.profiler, CUPTI):
kernel time by name, GPU busy time vs the step's wall span, i.e. the idle gaps
that launch overhead and the per-view host sync leave.

    python tools/step_timeline.py [--steps 5] [--config 3]

With programmatic dependent launch (every library kernel) a kernel's CTAs
start early and wait for their predecessor inside the kernel, so per-kernel
durations here include that wait; the merged busy / idle totals stay valid.
Per-kernel times: the ncu launch list (profiles/) or bench.py's events.
"""

import argparse
import collections
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--e2e", action="store_true",
                    help="the bench's e2e arm: ground truth from pinned host memory + loss readback")
    ap.add_argument("--binning", default="counting", choices=["counting", "sort"])
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    from paper_2409_07759_b200 import raster, train

    raster.set_binning(a.binning)

    if a.config == 5:  # render-only playback frames (bench.run_render_only's path)
        buf, cams, arr, sl = bench.build_player()

        def run(n):
            for i in range(n):
                buf.render_device(cams[i % len(cams)], 0)
        run(5)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            run(a.steps)
            torch.cuda.synchronize()
    else:
        c, scene, ds, state, window = bench.build_workload(a.config, None, "gt")
        progress = None
        if a.e2e:
            ds = bench.HostFeed(ds, window, c["views"])
            progress = bench.LossReadback(state.device)
        train.train_swin(window[0], window[1], state, ds, iterations=5, progress=progress)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            train.train_swin(window[0], window[1], state, ds, iterations=a.steps, progress=progress)
            if progress is not None:
                progress.flush()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    spans = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    t0, t1 = spans[0][0], max(s[1] for s in spans)
    busy = 0
    cur_s, cur_e = spans[0][0], spans[0][1]
    for s, e, _ in spans[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    gaps = collections.Counter()
    prev_end = spans[0][1]
    prev_name = spans[0][2]
    for s_, e_, n_ in spans[1:]:
        if s_ > prev_end:
            gaps[(prev_name.split("(")[0][:40] + " -> " + n_.split("(")[0][:40])] += s_ - prev_end
        if e_ > prev_end:
            prev_end, prev_name = e_, n_
    by = collections.Counter()
    for s, e, n in spans:
        by[n.split("(")[0][:60]] += e - s
    out = {"steps": a.steps, "span_us_per_step": (t1 - t0) / a.steps,
           "gpu_busy_us_per_step": busy / a.steps,
           "idle_us_per_step": (t1 - t0 - busy) / a.steps,
           "gaps_us_per_step": {k: v / a.steps for k, v in gaps.most_common(12)},
           "kernels_us_per_step": {k: v / a.steps for k, v in by.most_common(25)}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
