"""Per-kernel timing of the vx ops at the VGGT-1B shapes, next to the same-box library
comparators (torch SDPA / cuBLAS).  CUDA events, warm-up, L2 flushed between reps.

    python tools/bench_kernels.py [--views 20] [--only attn|gemm|ln]
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402

FLUSH = None


def flush_l2():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    FLUSH.zero_()


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        flush_l2()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def attn(views, res):
    N, H, d = 1374, 16, 64
    T = views * N
    q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
    fl_g = 4.0 * T * T * H * d
    t = timeit(lambda: ops.attention(q, k, v, o, 1, T, T), reps=3 if views > 50 else 5)
    res[f"attn_global_S{views}"] = {"ms": t, "tflops": fl_g / t / 1e9}
    t = timeit(lambda: F.scaled_dot_product_attention(q[None], k[None], v[None]), reps=3 if views > 50 else 5)
    res[f"sdpa_global_S{views}"] = {"ms": t, "tflops": fl_g / t / 1e9}
    fl_f = 4.0 * views * N * N * H * d
    t = timeit(lambda: ops.attention(q, k, v, o, views, N, N))
    res[f"attn_frame_S{views}"] = {"ms": t, "tflops": fl_f / t / 1e9}
    qf = q.view(H, views, N, d).transpose(0, 1)
    kf, vf = k.view(H, views, N, d).transpose(0, 1), v.view(H, views, N, d).transpose(0, 1)
    t = timeit(lambda: F.scaled_dot_product_attention(qf, kf, vf))
    res[f"sdpa_frame_S{views}"] = {"ms": t, "tflops": fl_f / t / 1e9}


def gemm(views, res):
    M = views * 1374
    C = 1024
    x = torch.randn(M, C, device="cuda")
    a = torch.randn(M, 4096, device="cuda", dtype=torch.bfloat16)
    for name, N, K, epi in (("qkv", 3 * C, C, None), ("proj", C, C, ops.EPI_RESID), ("fc1", 4 * C, C, ops.EPI_GELU),
                            ("fc2", C, 4 * C, ops.EPI_RESID)):
        w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
        bias = torch.randn(N, device="cuda")
        A = a[:, :K]
        fl = 2.0 * M * N * K
        if epi is None:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            fn = lambda: ops.gemm(A, w, ops.EPI_BF16, bias=bias, out=out)
        elif epi == ops.EPI_RESID:
            g = torch.rand(N, device="cuda")
            fn = lambda: ops.gemm(A, w, ops.EPI_RESID, bias=bias, resid=x, gamma=g)
        else:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            fn = lambda: ops.gemm(A, w, epi, bias=bias, out=out)
        t = timeit(fn)
        res[f"gemm_{name}_S{views}"] = {"ms": t, "tflops": fl / t / 1e9}
        if name == "qkv":  # the real fused epilogue: per-head LayerNorm + 2D RoPE + scatter to [H, T, d]
            H, d = 16, 64
            q, k, v = (torch.empty(H, M, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
            nw = [torch.rand(d, device="cuda") + 0.5 for _ in range(4)]
            from paper_2509_25191_b200.aggregator import rope_tables
            rope = tuple(r.cuda() for r in rope_tables(64, 38, 100.0))
            fnq = lambda: ops.gemm(A, w, ops.EPI_QKV, bias=bias, qkv=(q, k, v), qk_norm=tuple(nw), rope=rope,
                                   head_dim=d, tokens_total=M, tokens_per_frame=1374, patch_start=5, grid_w=37)
            t = timeit(fnq)
            res[f"gemm_qkv_fused_S{views}"] = {"ms": t, "tflops": fl / t / 1e9}
        if name == "fc1":  # same GEMM without GELU: the epilogue's share
            out2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            t = timeit(lambda: ops.gemm(A, w, ops.EPI_BF16, bias=bias, out=out2))
            res[f"gemm_fc1_nogelu_S{views}"] = {"ms": t, "tflops": fl / t / 1e9}
        Ac = A.contiguous()
        t = timeit(lambda: torch.matmul(Ac, w.t()))
        res[f"cublas_{name}_S{views}"] = {"ms": t, "tflops": fl / t / 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, nargs="+", default=[20])
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ops.load_library()
    res = {}
    for v in args.views:
        if args.only in ("", "attn"):
            attn(v, res)
        if args.only in ("", "gemm"):
            gemm(v, res)
    for k, v in res.items():
        print(f"{k:28s} {v['ms']:10.3f} ms  {v['tflops']:8.1f} TFLOP/s")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
