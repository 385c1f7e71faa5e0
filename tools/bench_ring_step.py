"""Time one ring step of frame-sharded global attention (vx_attention_merge, mode 2) on one GPU.

Shape of rank r's step at S views over g ranks: Lq = Lk = (S/g) * 1374 tokens, 16 heads, d=64.
Prints ms per step and TFLOP/s (best of --reps after warm-up); VX_FMHA_SPLIT=0 disables the
KV-split tail for A/B runs.
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2509_25191_b200 import ops
    H, d = 16, 64
    res = {}
    for g in args.ranks:
        T = (args.views // g) * 1374
        q, k, v = (torch.randn(H, T, d, device="cuda").bfloat16() for _ in range(3))
        o_acc = torch.zeros(T, H * d, device="cuda")
        lse = torch.zeros(H, T, device="cuda")
        for _ in range(3):
            ops.attention_merge(q, k, v, 2, o_acc, lse, Lq=T, Lk=T)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ops.attention_merge(q, k, v, 2, o_acc, lse, Lq=T, Lk=T)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        res[f"g{g}"] = {"tokens": T, "ms": round(best, 3), "tflops": round(4.0 * H * T * T * d / best / 1e9, 1)}
    print(json.dumps({"split": os.environ.get("VX_FMHA_SPLIT", "1"), "views": args.views, **res}))


if __name__ == "__main__":
    main()
