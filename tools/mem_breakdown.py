"""Where the peak HBM of a VGGT forward goes (one GPU): bytes held between forwards (weights, the DPT
heads' cached zero-bordered buffers), the forward's peak, and the per-view slope from two view counts.

    python tools/mem_breakdown.py [--views 20 200]
Prints one JSON line.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, nargs="+", default=[20, 200])
    args = ap.parse_args()
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    res = {}
    for S in args.views:
        torch.cuda.empty_cache()
        model = VGGT(cfg, state_dict=sd)
        torch.cuda.synchronize()
        w = torch.cuda.memory_allocated()
        images = synthetic_images(cfg, S, 1).cuda()
        out = model(images)
        del out
        torch.cuda.synchronize()
        held = torch.cuda.memory_allocated() - w - images.numel() * 4
        cache = sum(b.numel() * b.element_size() for h in (model.depth_head, model.point_head)
                    for b in h._bufs.values())
        torch.cuda.reset_peak_memory_stats()
        out = model(images)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated()
        res[S] = {"weights_gb": w / 1e9, "held_between_forwards_gb": held / 1e9, "dpt_cache_gb": cache / 1e9,
                  "peak_gb": peak / 1e9}
        del out, model, images
    if len(args.views) >= 2:
        a, b = args.views[0], args.views[-1]
        res["slope_mb_per_view"] = (res[b]["peak_gb"] - res[a]["peak_gb"]) / (b - a) * 1e3
    print(json.dumps(res))


if __name__ == "__main__":
    main()
