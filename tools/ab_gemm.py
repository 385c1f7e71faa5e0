"""In-process A/B of two libvx builds on the residual-epilogue GEMMs (proj, fc2) at S views,
alternating A/B so clock and power drift hit both alike.

    python tools/ab_gemm.py exp/libvx_a.so exp/libvx_b.so [--views 200 20] [--rounds 8]
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
    ap.add_argument("--views", type=int, nargs="+", default=[200, 20])
    ap.add_argument("--rounds", type=int, default=8)
    args = ap.parse_args()
    libs = [ops.load_library(p) for p in args.libs]
    C = 1024
    res = {}
    for views in args.views:
        M = views * 1374
        x = torch.randn(M, C, device="cuda")
        kept = torch.empty(M, 2 * C, device="cuda", dtype=torch.bfloat16)
        # qkv: the fused per-head LayerNorm + 2D RoPE + head-major scatter epilogue
        H, d = 16, 64
        aq = torch.randn(M, C, device="cuda").to(torch.bfloat16)
        wq = (torch.randn(3 * C, C, device="cuda") * 0.02).to(torch.bfloat16)
        bq = torch.randn(3 * C, device="cuda")
        qq, kk, vv = (torch.empty(H, M, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        nw = tuple(torch.rand(d, device="cuda") + 0.5 for _ in range(4))
        from paper_2509_25191_b200.aggregator import rope_tables
        rope = tuple(t.cuda() for t in rope_tables(64, 38, 100.0))
        qkv_fn = lambda: ops.gemm(aq, wq, ops.EPI_QKV, bias=bq, qkv=(qq, kk, vv), qk_norm=nw, rope=rope,  # noqa: E731
                                  head_dim=d, tokens_total=M, tokens_per_frame=1374, patch_start=5, grid_w=37)
        reps = 10 if views >= 100 else 40
        ts, outs = [[], []], [None, None]
        for r in range(args.rounds):
            for idx in ((0, 1) if r % 2 == 0 else (1, 0)):
                ops._lib = libs[idx]
                qkv_fn()
                torch.cuda.synchronize()
                s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_.record()
                for _ in range(reps):
                    qkv_fn()
                e_.record()
                e_.synchronize()
                ts[idx].append(s_.elapsed_time(e_) / reps)
                outs[idx] = (qq.clone(), kk.clone(), vv.clone())
        med = [sorted(t)[len(t) // 2] for t in ts]
        fl = 2.0 * M * 3 * C * C
        diff = max(((a.float() - b.float()).norm() / b.float().norm()).item() for a, b in zip(outs[0], outs[1]))
        res[f"qkv_S{views}"] = {"A_ms": round(med[0], 4), "B_ms": round(med[1], 4), "B_over_A": round(med[0] / med[1], 4),
                                "A_TFLOPs": round(fl / med[0] / 1e9, 1), "B_TFLOPs": round(fl / med[1] / 1e9, 1),
                                "max_rel_diff": diff}
        print(f"qkv_S{views}", res[f"qkv_S{views}"], flush=True)
        del aq, wq, qq, kk, vv
        for name, K in (("fc2", 4 * C), ("fc2nokept", 4 * C), ("proj", C)):
            a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            w = (torch.randn(C, K, device="cuda") * 0.02).to(torch.bfloat16)
            bias = torch.randn(C, device="cuda")
            g = torch.rand(C, device="cuda") * 0.1
            kw = dict(bias=bias, resid=x, gamma=g, kept=kept[:, :C] if name == "fc2" else None)  # fc2nokept: layers not kept
            reps = 10 if views >= 100 else 40
            ts = [[], []]
            for r in range(args.rounds):
                order = (0, 1) if r % 2 == 0 else (1, 0)
                for idx in order:
                    ops._lib = libs[idx]
                    ops.gemm(a, w, ops.EPI_RESID, **kw)
                    torch.cuda.synchronize()
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    for _ in range(reps):
                        ops.gemm(a, w, ops.EPI_RESID, **kw)
                    e.record()
                    e.synchronize()
                    ts[idx].append(s.elapsed_time(e) / reps)
            med = [sorted(t)[len(t) // 2] for t in ts]
            byt = M * K * 2 + C * K * 2 + M * C * 8 + (M * C * 2 if name == "fc2" else 0)
            key = f"{name}_S{views}"
            res[key] = {"A_ms": round(med[0], 4), "B_ms": round(med[1], 4), "B_over_A": round(med[0] / med[1], 4),
                        "A_TBps": round(byt / med[0] / 1e9, 2), "B_TBps": round(byt / med[1] / 1e9, 2)}
            print(key, res[key], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
