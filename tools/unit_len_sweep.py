"""Attention throughput against sequence length at a fixed token count (per-unit overhead probe):
nseq sequences of L tokens, 16 heads, d=64, q in log2 units, sustained (power-capped) samples.

    python tools/unit_len_sweep.py [L ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25191_b200 import ops  # noqa: E402

Ls = [int(x) for x in sys.argv[1:]] or [1374, 1536, 3072, 6144, 12288, 49152]
H, d, T = 16, 64, 200 * 1374
for L in Ls:
    nseq = max(1, T // L)
    Tt = nseq * L
    q, k, v = (torch.randn(H, Tt, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty(Tt, H * d, device="cuda", dtype=torch.bfloat16)
    fl = 4.0 * nseq * L * L * H * d
    reps = max(2, int(2e15 / fl))
    for _ in range(2):
        ops.attention(q, k, v, o, nseq, L, L, q_log2=True)
    torch.cuda.synchronize()
    best = []
    for r in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            ops.attention(q, k, v, o, nseq, L, L, q_log2=True)
        e.record()
        e.synchronize()
        best.append(s.elapsed_time(e) / reps)
    ms = sorted(best)[1]
    kv_tiles = -(-L // 48)
    print(f"L={L:6d} nseq={nseq:4d} kv_tiles/unit={kv_tiles:5d}  {ms:8.3f} ms  {fl / ms / 1e9:7.1f} TFLOP/s", flush=True)
