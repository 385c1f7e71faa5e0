"""clock64 trace of the FMHA softmax / MMA schedule (diagnostic build with -DVX_FMHA_TRACE).

Builds exp/libvx_trace.so (fmha.cu with the trace stamps + the rest of the library), runs one
global-attention launch at the S=20 shape and prints, per tile and iteration of CTA 0's first
unit: wait-for-S, S->max, exps, tail (store P, rescale, arrive), and the MMA thread's view.
    python tools/trace_fmha.py build     # here (nvcc)
    python tools/trace_fmha.py run       # on the GPU box
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
EXP = os.path.join(ROOT, "exp")
LIB = os.path.join(EXP, "libvx_trace.so")


def build():
    from paper_2509_25191_b200 import build as b
    b.build()
    os.makedirs(EXP, exist_ok=True)
    obj = os.path.join(EXP, "fmha_trace.o")
    flags = list(b.FLAGS)
    i = flags.index("-Xptxas")
    del flags[i:i + 2]  # drop "-Xptxas -v"
    cmd = [b.NVCC, *b.ARCH, *flags, "-DVX_FMHA_TRACE", "-c", str(b.CSRC / "fmha.cu"), "-o", obj]
    subprocess.run(cmd, check=True)
    objs = [str(b.PKG / "build" / (s.stem + ".o")) for s in b.sources() if s.name != "fmha.cu"] + [obj]
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", LIB, *objs], check=True)
    print(LIB)


def run():
    import torch
    from paper_2509_25191_b200 import ops
    lib = ops.use_library(LIB)
    buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
    lib.vx_fmha_set_trace.argtypes = [ctypes.c_void_p]
    views = int(os.environ.get("VIEWS", "20"))
    T, H, d = views * 1374, 16, 64
    q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
    ops.attention(q, k, v, o, 1, T, T)
    torch.cuda.synchronize()
    assert lib.vx_fmha_set_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    ops.attention(q, k, v, o, 1, T, T)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype("int64")
    t0 = t[t > 0].min()
    print("per tile: j wait(S) S->max exps tail period   [clk]")
    for tile in range(4):
        rows = []
        for j in range(8, 40):
            b0 = (tile * 64 + j) * 8
            s = t[b0:b0 + 5] - t0
            nxt = t[(tile * 64 + j + 1) * 8] - t0
            rows.append((j, s[1] - s[0], s[2] - s[1], s[3] - s[2], s[4] - s[3], nxt - s[0]))
        import numpy as np
        a = np.array(rows)
        print(f"tile {tile}: mean wait {a[:,1].mean():.0f}  max {a[:,2].mean():.0f}  exps {a[:,3].mean():.0f}  "
              f"tail {a[:,4].mean():.0f}  period {a[:,5].mean():.0f}")
    print("iteration 20 timeline (clk from the first stamp):")
    for tile in range(4):
        b0 = (tile * 64 + 20) * 8
        print(f"  tile {tile}: wait@{t[b0]-t0} S@{t[b0+1]-t0} exps@{t[b0+2]-t0}..{t[b0+3]-t0} pfull@{t[b0+4]-t0}")
    for i in range(4):
        m0 = 4096 + (20 * 4 + i) * 2
        print(f"  mma tile {i}: p_full seen@{t[m0]-t0} S(j+1) committed@{t[m0+1]-t0}")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
