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


def run_boundary():
    """Frame-like launch (nseq sequences of L = 1536 tokens: 32 KV tiles per unit): per tile, the
    iterations around CTA 0's unit boundary (jj = 32 * unit + j) and the MMA thread's S(0) issue."""
    import numpy as np
    import torch
    from paper_2509_25191_b200 import ops
    lib = ops.use_library(LIB)
    buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
    lib.vx_fmha_set_trace.argtypes = [ctypes.c_void_p]
    L, nseq, H, d = 1536, 178, 16, 64
    T = nseq * L
    q, k, v = (torch.randn(H, T, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
    ops.attention(q, k, v, o, nseq, L, L, q_log2=True)
    torch.cuda.synchronize()
    assert lib.vx_fmha_set_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    ops.attention(q, k, v, o, nseq, L, L, q_log2=True)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype("int64")
    t0 = t[t > 0].min()
    z = lambda x: (x - t0) if x > 0 else -1  # noqa: E731
    for tile in range(4):
        print(f"tile {tile}: jj  wait@  S@  exps_done@  pfull@   [clk]  (period)")
        for jj in list(range(24, 40)):
            b0 = (tile * 64 + jj) * 8
            nxt = t[(tile * 64 + jj + 1) * 8] if jj + 1 < 64 else 0
            extra = ""
            if jj in (31, 63):
                extra = (f"  O final@{z(t[b0 + 5])} O read@{z(t[b0 + 7])} stores@{z(t[b0 + 2])}"
                         f" epilogue done@{z(t[b0 + 6])}")
            print(f"   {jj:3d} {z(t[b0]):8d} {z(t[b0 + 1]):8d} {z(t[b0 + 3]):8d} {z(t[b0 + 4]):8d}"
                  f"  ({(nxt - t[b0]) if nxt > 0 and t[b0] > 0 else -1}){extra}")
    print("producer unit0/1: q_empty seen", z(t[6230]), z(t[6231]),
          " k stage free j0/j1 (unit0, unit1):", z(t[6240]), z(t[6241]), z(t[6242]), z(t[6243]))
    print("MMA: q_full seen unit0/1:", z(t[6100]), z(t[6101]), " S(0) committed unit1:",
          [z(t[6004 + i]) for i in range(4)])
    for jj in (30, 31, 32, 33):
        print(f"  mma jj {jj}:", [(z(t[4096 + (jj * 4 + i) * 2]), z(t[4096 + (jj * 4 + i) * 2 + 1])) for i in range(4)])
    per = [np.mean([t[(tile * 64 + jj + 1) * 8] - t[(tile * 64 + jj) * 8] for jj in range(8, 28)]) for tile in range(4)]
    print("steady period per tile (jj 8-28):", [round(p) for p in per])


if __name__ == "__main__":
    {"build": build, "run": run, "run_boundary": run_boundary}[sys.argv[1]]()
