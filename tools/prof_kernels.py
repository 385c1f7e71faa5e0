"""ncu driver: every vx kernel of the VGGT path once at the VGGT-1B S=20 shapes (after one warm-up).

    ncu --set full -k regex:'vx::' -o prof python tools/prof_kernels.py
Launch order (second pass is the profiled one): layernorm, gemm QKV, fmha frame, fmha global,
gemm proj (resid), gemm fc1 (gelu), gemm fc2 (resid), DPT 3x3 conv (148^2, 256->256),
DPT fused output head (518^2), upsample 296->518.
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402
from paper_2509_25191_b200.aggregator import rope_tables  # noqa: E402


def main(views=20):
    N, C, H, d = 1374, 1024, 16, 64
    T = views * N
    dev = "cuda"
    bf = torch.bfloat16
    x = torch.randn(T, C, device=dev)
    xn = torch.empty(T, C, device=dev, dtype=bf)
    w_ln = torch.ones(C, device=dev)
    b_ln = torch.zeros(C, device=dev)
    wqkv = (torch.randn(3 * C, C, device=dev) * 0.02).to(bf)
    bqkv = torch.zeros(3 * C, device=dev)
    q, k, v = (torch.empty(H, T, d, device=dev, dtype=bf) for _ in range(3))
    qn = [torch.ones(d, device=dev), torch.zeros(d, device=dev), torch.ones(d, device=dev), torch.zeros(d, device=dev)]
    cos, sin = rope_tables(d, 38, 100.0)
    rope = (cos.to(dev), sin.to(dev))
    o = torch.empty(T, C, device=dev, dtype=bf)
    wp = (torch.randn(C, C, device=dev) * 0.02).to(bf)
    w1 = (torch.randn(4 * C, C, device=dev) * 0.02).to(bf)
    w2 = (torch.randn(C, 4 * C, device=dev) * 0.02).to(bf)
    hbuf = torch.empty(T, 4 * C, device=dev, dtype=bf)
    g = torch.full((C,), 0.01, device=dev)
    Fr, hs, Fh = 8, 148, 256
    xin = torch.zeros(Fr, hs + 2, hs + 2, Fh, device=dev, dtype=bf)
    xin[:, 1:-1, 1:-1] = torch.randn(Fr, hs, hs, Fh, device=dev).to(bf)
    wc = (torch.randn(Fh, 9 * Fh, device=dev) * 0.02).to(bf)
    bc = torch.zeros(Fh, device=dev)
    yout = torch.zeros_like(xin)
    up_in = torch.randn(Fr, 296, 296, 128, device=dev).to(bf)
    wh = (torch.randn(32, 9 * 128, device=dev) * 0.02).to(bf)
    hw, hb = torch.randn(2, 32, device=dev) * 0.1, torch.zeros(2, device=dev)
    pred = torch.empty(Fr, 518, 518, 1, device=dev)
    conf = torch.empty(Fr, 518, 518, device=dev)
    for _ in range(2):
        ops.layernorm(x, w_ln, b_ln, 1e-5, out=xn)
        ops.gemm(xn, wqkv, ops.EPI_QKV, bias=bqkv, qkv=(q, k, v), qk_norm=qn, rope=rope, head_dim=d,
                 tokens_total=T, tokens_per_frame=N, patch_start=5, grid_w=37)
        ops.attention(q, k, v, o, views, N, N)
        ops.attention(q, k, v, o, 1, T, T)
        ops.gemm(o, wp, ops.EPI_RESID, bias=bc.new_zeros(C), resid=x, gamma=g)
        ops.gemm(xn, w1, ops.EPI_GELU, bias=torch.zeros(4 * C, device=dev), out=hbuf)
        ops.gemm(hbuf, w2, ops.EPI_RESID, bias=torch.zeros(C, device=dev), resid=x, gamma=g)
        ops.gemm_spatial(xin.view(-1, Fh), wc, bc, Fr, hs, hs, conv3x3=True, relu=True, out1=yout, out1_pad=True)
        u = ops.upsample_bilinear(up_in, (518, 518), out_pad=True)
        ops.gemm_spatial(u.view(-1, 128), wh, torch.zeros(32, device=dev), Fr, 518, 518, conv3x3=True,
                         head=(hw, hb, 0, pred, conf))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
