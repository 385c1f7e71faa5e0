"""In-process A/B of two libvx builds on the DPT fused output head (3x3 conv 128 -> 32 + fp32 1x1 + activation)
of one 16-view chunk at 518^2, alternating A/B.

    python tools/ab_headout.py exp/libvx_a.so exp/libvx_b.so [--rounds 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--rounds", type=int, default=10)
    args = ap.parse_args()
    libs = [ops.load_library(p) for p in args.libs]
    Fr, H, C = 16, 518, 128
    x = torch.zeros(Fr, H + 2, H + 2, C, device="cuda", dtype=torch.bfloat16)
    x[:, 1:-1, 1:-1] = torch.randn(Fr, H, H, C, device="cuda").to(torch.bfloat16)
    w = (torch.randn(32, 9 * C, device="cuda") * 0.03).to(torch.bfloat16)
    b = torch.randn(32, device="cuda")
    hw, hb = torch.randn(3, 32, device="cuda") * 0.1, torch.randn(3, device="cuda")
    preds = [torch.empty(Fr, H, H, 2, device="cuda") for _ in range(2)]
    confs = [torch.empty(Fr, H, H, device="cuda") for _ in range(2)]
    ts = [[], []]
    for r in range(args.rounds):
        for idx in ((0, 1) if r % 2 == 0 else (1, 0)):
            ops._lib = libs[idx]
            run = lambda: ops.gemm_spatial(x.view(-1, C), w, b, Fr, H, H, conv3x3=True,  # noqa: E731
                                           head=(hw, hb, 1, preds[idx], confs[idx]))
            run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10):
                run()
            e.record()
            e.synchronize()
            ts[idx].append(s.elapsed_time(e) / 10)
    med = [sorted(t)[len(t) // 2] for t in ts]
    fl = 2.0 * Fr * (H + 2) * (H + 2) * 32 * 9 * C
    res = {"A_us": round(med[0] * 1e3, 1), "B_us": round(med[1] * 1e3, 1), "B_over_A": round(med[0] / med[1], 3),
           "A_tflops": round(fl / med[0] / 1e9, 1), "B_tflops": round(fl / med[1] / 1e9, 1),
           "pred_rel_diff": ((preds[0] - preds[1]).norm() / preds[0].norm()).item(),
           "conf_rel_diff": ((confs[0] - confs[1]).norm() / confs[0].norm()).item()}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
