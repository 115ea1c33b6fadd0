"""Time ss_loss_l1_ssim alone (SSIM fwd + bwd + reduce) on a config-3 sized
frame, CUDA events over 200 back-to-back calls, u8 ground truth.

    python tools/micro/loss_rate.py [--width 1352 --height 1014]
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2409_07759_b200.engine import LossBuffers  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=1352)
    ap.add_argument("--height", type=int, default=1014)
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    H, W = a.height, a.width
    g = torch.Generator(device="cuda").manual_seed(0)
    pred = torch.rand(H, W, 3, device="cuda", generator=g)
    gt = (torch.rand(H, W, 3, device="cuda", generator=g) * 255).to(torch.uint8)
    lut = torch.linspace(0, 1, 256, device="cuda")
    lb = LossBuffers()
    for _ in range(10):
        lb.run(pred, H, W, gt_u8=gt, lut=lut)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        lb.run(pred, H, W, gt_u8=gt, lut=lut)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    print(json.dumps({"us_per_loss": round(us, 2), "sums": lb.sums.tolist()}))


if __name__ == "__main__":
    main()
