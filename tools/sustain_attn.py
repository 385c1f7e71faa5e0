"""Global-attention FMHA under sustained load (power-capped steady state, like inside bench.py).

Runs the S-view global attention back to back for --seconds and reports the mean launch time
over the second half of the window plus the median SM clock / board power sampled by nvidia-smi
during it.  The dispatcher reads its diagnostic env (VX_FMHA_EMU, VX_FMHA_CFG) once per process,
so alternate configurations from the shell: tools/sustain_attn.sh.
"""
from __future__ import annotations

import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import argparse
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def clocks_sampler(stop, out):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                "-i", "0"], capture_output=True, text=True, timeout=5)
            sm, pw = r.stdout.strip().split(",")[:2]
            out.append((float(sm), float(pw)))
        except Exception:
            pass
        time.sleep(0.25)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--label", default="")
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--seconds", type=float, default=12.0)
    args = ap.parse_args()
    import torch
    from paper_2509_25191_b200 import ops

    H, d, N = 16, 64, 1374
    T = args.views * N
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, T, d, device="cuda", generator=g).bfloat16() for _ in range(3))
    o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
    flops = 4.0 * H * T * T * d
    ops.attention(q, k, v, o, 1, T, T)
    torch.cuda.synchronize()
    times, samples = [], []
    stop = threading.Event()
    th = None
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < args.seconds:
        if th is None and time.perf_counter() - t0 > args.seconds / 2:
            th = threading.Thread(target=clocks_sampler, args=(stop, samples), daemon=True)
            th.start()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ops.attention(q, k, v, o, 1, T, T)
        e.record()
        e.synchronize()
        if th is not None:
            times.append(s.elapsed_time(e))
    stop.set()
    th.join()
    ms = sum(times) / max(len(times), 1)
    sm = sorted(x[0] for x in samples)
    pw = sorted(x[1] for x in samples)
    print(json.dumps({"label": args.label, "views": args.views, "ms": round(ms, 3),
                      "tflops": round(flops / ms / 1e9, 1), "sm_mhz": sm[len(sm) // 2] if sm else None,
                      "watts": pw[len(pw) // 2] if pw else None, "n": len(times)}), flush=True)


if __name__ == "__main__":
    main()
