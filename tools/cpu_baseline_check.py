"""Checks the per-unit CPU-baseline composition (oracle/cpu_baseline.py) against directly measured oracle
runs on the same host cores: a full 8-view forward of the 1B-shaped model and single global blocks at
S = 8 and 20 views.  Writes profiles/r02_cpu_baseline_check.json (run on the GPU box's host).

    python tools/cpu_baseline_check.py [--out profiles/r02_cpu_baseline_check.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_baseline_check.json"))
    ap.add_argument("--forward-views", type=int, default=8)
    ap.add_argument("--block-views", type=int, nargs="+", default=[8, 20])
    args = ap.parse_args()
    import torch
    from oracle import vggt_ref as R
    from oracle.cpu_baseline import compose, unit_times
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    out = {"threads": threads, "checks": []}
    with torch.no_grad():
        for S in args.block_views:
            N, C = cfg.tokens_per_frame, cfg.embed_dim
            x = torch.randn(1, S * N, C)
            gpos = R.positions(cfg).repeat(S, 1)
            blk = "aggregator.global_blocks.0"
            R.block(x[:, :N], sd, blk, cfg.num_heads, cfg.ln_eps, gpos[:N], cfg.rope_freq)  # warm-up
            t0 = time.perf_counter()
            R.block(x, sd, blk, cfg.num_heads, cfg.ln_eps, gpos, cfg.rope_freq)
            meas = time.perf_counter() - t0
            pred = compose(cfg, S, unit_times(cfg, sd, S, threads=threads))["global_block_s"]
            out["checks"].append({"what": f"global block, S={S}", "measured_s": meas, "composed_s": pred,
                                  "error_pct": 100 * (pred / meas - 1)})
            print(out["checks"][-1], flush=True)
        S = args.forward_views
        images = synthetic_images(cfg, S, 1)
        t0 = time.perf_counter()
        R.vggt_forward(images, sd, cfg)
        meas = time.perf_counter() - t0
        t = unit_times(cfg, sd, S, threads=threads)
        pred = compose(cfg, S, t)["forward_s"]
        out["checks"].append({"what": f"full forward, S={S}", "measured_s": meas, "composed_s": pred,
                              "error_pct": 100 * (pred / meas - 1), "units_s": t})
        print(out["checks"][-1], flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
