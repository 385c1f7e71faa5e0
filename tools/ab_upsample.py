"""In-process A/B of two libvx builds on the DPT bilinear resizes of one 16-view chunk (the two big
ones: 148^2 -> 296^2 at C=256 into a padded buffer, 296^2 -> 518^2 at C=128 + pos-embed, padded).

    python tools/ab_upsample.py exp/libvx_a.so exp/libvx_b.so [--rounds 10]
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
    res = {}
    for (F, h, C, H, add) in ((16, 148, 256, 296, False), (16, 296, 128, 518, True), (16, 74, 256, 148, False)):
        x = torch.randn(F, h, h, C, device="cuda").to(torch.bfloat16)
        a = torch.randn(H, H, C, device="cuda").to(torch.bfloat16) if add else None
        out = torch.zeros(F, H + 2, H + 2, C, device="cuda", dtype=torch.bfloat16)
        outs, ts = [None, None], [[], []]
        for r in range(args.rounds):
            for idx in ((0, 1) if r % 2 == 0 else (1, 0)):
                ops._lib = libs[idx]
                ops.upsample_bilinear(x, (H, H), add=a, out=out, out_pad=True)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(10):
                    ops.upsample_bilinear(x, (H, H), add=a, out=out, out_pad=True)
                e.record()
                e.synchronize()
                ts[idx].append(s.elapsed_time(e) / 10)
                outs[idx] = out.clone()
        med = [sorted(t)[len(t) // 2] for t in ts]
        byt = F * (h * h + (H + 2) * (H + 2)) * C * 2 + (H * H * C * 2 if add else 0)
        key = f"{h}->{H}_C{C}" + ("_add" if add else "")
        res[key] = {"A_us": round(med[0] * 1e3, 1), "B_us": round(med[1] * 1e3, 1), "B_over_A": round(med[0] / med[1], 3),
                    "A_TBps": round(byt / med[0] / 1e9, 2), "B_TBps": round(byt / med[1] / 1e9, 2),
                    "bitwise_equal": bool(torch.equal(outs[0], outs[1]))}
        print(key, res[key], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
