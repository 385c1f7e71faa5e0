"""In-process A/B of two libvx builds on the attention layers (frame and global), alternating A/B so
clock and power drift hit both alike.

    python tools/ab_attn.py exp/libvx_a.so exp/libvx_b.so [--views 200] [--rounds 6] [--global-views 20 200]
Prints per-layer medians (ms, TFLOP/s) for A and B and B/A.
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--views", type=int, default=200, help="frame layer views")
    ap.add_argument("--global-views", type=int, nargs="*", default=[20, 200])
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--reps", type=int, default=0, help="launches per timed sample (default: 2 global / 10 frame)")
    ap.add_argument("--q-log2", default="", help="A,B flags: 1 = call B (or A) with q pre-scaled (VX_ATTN_Q_LOG2), e.g. 0,1")
    args = ap.parse_args()
    libs = [ops.load_library(p) for p in args.libs]
    ql2 = [f == "1" for f in args.q_log2.split(",")] if args.q_log2 else [False, False]
    N, H, d = 1374, 16, 64
    cases = [("frame", args.views, args.views, N)] + [("global", v, 1, v * N) for v in args.global_views]
    res = {}
    for name, views, nseq, L in cases:
        T = nseq * L
        q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
        fl = 4.0 * nseq * L * L * H * d
        reps = args.reps or (2 if nseq == 1 and T > 100000 else 10)
        ts = [[], []]
        for r in range(args.rounds):
            for li, lib in enumerate(libs if r % 2 == 0 else libs[::-1]):
                idx = li if r % 2 == 0 else 1 - li
                ops._lib = lib
                for _ in range(1):
                    ops.attention(q, k, v, o, nseq, L, L, q_log2=ql2[idx])
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(reps):
                    ops.attention(q, k, v, o, nseq, L, L, q_log2=ql2[idx])
                e.record()
                e.synchronize()
                ts[idx].append(s.elapsed_time(e) / reps)
        med = [sorted(t)[len(t) // 2] for t in ts]
        key = f"{name}_S{views}"
        res[key] = {"A_ms": round(med[0], 4), "B_ms": round(med[1], 4), "A_tflops": round(fl / med[0] / 1e9, 1),
                    "B_tflops": round(fl / med[1] / 1e9, 1), "B_over_A": round(med[0] / med[1], 4)}
        print(key, res[key], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
