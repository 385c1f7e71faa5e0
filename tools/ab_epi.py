"""In-process A/B of two library builds on store-heavy GEMM epilogues: fc1 (GELU, bf16 out, one 128-frame
chunk of rows) and the DPT 3x3 conv at 148^2 with two padded bf16 outputs (RCU conv2).

    python tools/ab_epi.py exp/libvx_a.so exp/libvx_b.so [--rounds 8]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("--rounds", type=int, default=8)
    args = ap.parse_args()
    libs = [ops.load_library(p) for p in args.libs]
    g = torch.Generator(device="cuda").manual_seed(0)
    M, C = 128 * 1374, 1024
    a = torch.randn(M, C, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(4 * C, C, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    b = torch.randn(4 * C, device="cuda", generator=g)
    h = torch.empty(M, 4 * C, device="cuda", dtype=torch.bfloat16)
    Fr, Hh, Cc = 16, 148, 256
    x = torch.zeros(Fr, Hh + 2, Hh + 2, Cc, device="cuda", dtype=torch.bfloat16)
    x[:, 1:-1, 1:-1] = torch.randn(Fr, Hh, Hh, Cc, device="cuda", generator=g).to(torch.bfloat16)
    wc = (torch.randn(Cc, 9 * Cc, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    bc = torch.randn(Cc, device="cuda", generator=g)
    o1, o2 = torch.zeros_like(x), torch.zeros_like(x)
    cases = {
        "fc1_gelu": (lambda: ops.gemm(a, w, ops.EPI_GELU, bias=b, out=h), 2.0 * M * C * 4 * C, lambda: h),
        "conv256_2out": (lambda: ops.gemm_spatial(x.view(-1, Cc), wc, bc, Fr, Hh, Hh, conv3x3=True, res1=x, res1_pad=True,
                                                  out1=o1, out1_pad=True, out2=o2, out2_pad=True),
                         2.0 * Fr * Hh * Hh * Cc * 9 * Cc, lambda: o1),
    }
    for name, (fn, fl, outf) in cases.items():
        ts, outs = [[], []], [None, None]
        for r in range(args.rounds):
            for idx in ((0, 1) if r % 2 == 0 else (1, 0)):
                ops._lib = libs[idx]
                fn()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(20):
                    fn()
                e.record()
                e.synchronize()
                ts[idx].append(s.elapsed_time(e) / 20)
                outs[idx] = outf().clone()
        med = [sorted(t)[len(t) // 2] for t in ts]
        print(name, {"A_ms": round(med[0], 4), "B_ms": round(med[1], 4), "B_over_A": round(med[0] / med[1], 4),
                     "A_TFLOPs": round(fl / med[0] / 1e9, 1), "B_TFLOPs": round(fl / med[1] / 1e9, 1),
                     "bitwise_equal": bool(torch.equal(outs[0], outs[1]))}, flush=True)


if __name__ == "__main__":
    main()
