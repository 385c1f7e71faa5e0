"""In-process A/B of cfg.q_chunk (or another chunk field, --field frame_chunk) on the 1B-shaped forward (one
GPU): whole q against q produced and attended a chunk of frames at a time, alternating so clock and power
drift hit every variant alike.

    python tools/ab_qchunk.py [--views 200] [--chunks 0 100 128] [--rounds 3] [--field q_chunk]
Prints per-variant median ms per forward, the global-attention phase and peak HBM, one JSON line.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--chunks", type=int, nargs="+", default=[0, 100, 128])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--field", default="q_chunk")
    args = ap.parse_args()
    from paper_2509_25191_b200 import profiling
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, args.views, 1).cuda()
    models = {c: VGGT(cfg.with_(**{args.field: c}), state_dict=sd) for c in args.chunks}
    for m in models.values():
        m(images)
    res = {c: {"ms": [], "attn_global_ms": [], "peak_gb": []} for c in args.chunks}
    for _ in range(args.rounds):
        for c, m in models.items():
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            timer = profiling.PhaseTimer()
            profiling.set_timer(timer)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = m(images)
            e.record()
            e.synchronize()
            profiling.set_timer(None)
            del out
            res[c]["ms"].append(s.elapsed_time(e))
            res[c]["attn_global_ms"].append(timer.summary()["attn_global"]["total_ms"])
            res[c]["peak_gb"].append(torch.cuda.max_memory_allocated() / 1e9)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    out = {str(c): {k: round(med(v), 2) for k, v in r.items()} for c, r in res.items()}
    print(json.dumps({"views": args.views, "field": args.field, **out}))


if __name__ == "__main__":
    main()
