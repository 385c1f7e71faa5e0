"""Minimal driver for ncu: one global-attention launch at the S=20 VGGT-1B shape (+1 warm-up)."""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops
views = int(sys.argv[1]) if len(sys.argv) > 1 else 20
N, H, d = 1374, 16, 64
T = views * N
q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    ops.attention(q, k, v, o, 1, T, T)
torch.cuda.synchronize()
print("ok")
