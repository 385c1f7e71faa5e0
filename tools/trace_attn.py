"""Reads the clock64() trace of the VX_FMHA_TRACE debug build (tools/libvx_trace.so):
per KV iteration of CTA 0, softmax warps 4 (tile 0) and 12 (tile 1), and the MMA warp."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops
lib = ops.load_library(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvx_trace.so"))
ops._lib = lib
views = int(sys.argv[1]) if len(sys.argv) > 1 else 20
N, H, d = 1374, 16, 64
T = views * N
q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    ops.attention(q, k, v, o, 1, T, T)
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.int64)
lib.vx_fmha_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert lib.vx_fmha_trace_read(buf.ctypes.data, 4096) == 0
w4 = buf[:1024].reshape(64, 16)
mma = buf[1024:2048].reshape(64, 16)
w12 = buf[2048:3072].reshape(64, 16)
t0 = w4[8, 0]
names = ["it0", "s_full", "ldtm", "max", "bar", "exps", "p_free", "p_full"]
print("per-iteration deltas (clk), softmax warp 4 (tile 0, half 0):")
for j in range(8, 20):
    r = w4[j]
    print(j, " ".join(f"{names[s]}={r[s] - r[s - 1]:5d}" for s in range(1, 8)), f" period={w4[j + 1, 0] - r[0]}")
print("tile 1 (warp 12):")
for j in range(8, 20):
    r = w12[j]
    print(j, " ".join(f"{names[s]}={r[s] - r[s - 1]:5d}" for s in range(1, 8)), f" period={w12[j + 1, 0] - r[0]}")
print("MMA warp (relative to warp-4 iteration start): sfree0 sfree1 pfull0 pfull1")
for j in range(8, 20):
    print(j, [int(mma[j, s] - w4[j, 0]) for s in (8, 9, 10, 11)], " w12 start", int(w12[j, 0] - w4[j, 0]))
