"""CPU baseline of the VGGT path: the fp32 oracle timed on the host cores, composed per unit.

TEST / BENCH INFRASTRUCTURE ONLY (like the rest of oracle/): used by bench.py's cpu_baseline leg and
its `--impl reference` arm (the reference ships no implementation of this path, so the
oracle restatement is the CPU path timed beside the GPU) and by tools/cpu_baseline_check.py.

A 200-view forward takes hours on a CPU, so one step times every kind of work unit of the S-view
forward AT ITS S-VIEW SHAPE on a bounded slice, and composes the forward from the unit counts:

  * patch-embed of one view;
  * one aggregator block on one view (its linears, norms, RoPE and 1374-token frame attention) and the
    frame attention alone, so a global block's per-view non-attention work is (block - attention);
  * global attention of Q of one view's queries (all 16 heads) against the FULL S*1374-token K/V of
    the S-view sequence — the operation that is 94% of the S = 200 forward, at its real key length;
  * the camera head over all S camera tokens (cheap: measured whole);
  * both DPT heads on one view.

forward(S) = S*(pe + 24*blk + 24*(blk - fattn) + 24*(1374/Q)*gattn_Q(S) + dpt) + camera(S).  The
composition is checked against directly measured forwards / global blocks by
tools/cpu_baseline_check.py (profiles/r02_cpu_baseline_check.json).
"""
from __future__ import annotations

import os
import time

import torch
import torch.nn.functional as F

from oracle import vggt_ref as R


def _best_of(fn, n=2):
    best = float("inf")
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


@torch.no_grad()
def unit_times(cfg, sd, S: int, q_rows: int = 512, threads: int | None = None, seed: int = 1) -> dict:
    """Seconds per work unit of an S-view forward (see the module docstring)."""
    threads = threads or (os.cpu_count() or 1)
    torch.set_num_threads(threads)
    N, C, H, d = cfg.tokens_per_frame, cfg.embed_dim, cfg.num_heads, cfg.head_dim
    g = torch.Generator().manual_seed(seed)
    img = torch.rand(1, 3, cfg.img_size, cfg.img_size, generator=g)
    x1 = torch.cat([R.special_tokens(sd, cfg, 1), R.patch_embed(img, sd, cfg)], dim=1)  # (1, N, C)
    pos = R.positions(cfg)
    t = {}
    t["patch_embed"] = _best_of(lambda: R.patch_embed(img, sd, cfg))
    blk = "aggregator.frame_blocks.0"
    t["block_1view"] = _best_of(lambda: R.block(x1, sd, blk, H, cfg.ln_eps, pos, cfg.rope_freq))
    qf = torch.randn(1, H, N, d, generator=g)
    t["frame_attn_1view"] = _best_of(lambda: F.scaled_dot_product_attention(qf, qf, qf))
    Q = min(q_rows, N)
    q = torch.randn(1, H, Q, d, generator=g)
    kv = torch.randn(1, H, S * N, d, generator=g)
    t["global_attn_q"] = _best_of(lambda: F.scaled_dot_product_attention(q, kv, kv))
    t["global_attn_q_rows"] = Q
    cam = torch.randn(S, 1, 2 * C, generator=g)
    t["camera_head"] = _best_of(lambda: R.camera_head(cam, sd, cfg), n=1 if S > 50 else 2)
    kept = {i: torch.randn(1, N, 2 * C, generator=g) for i in cfg.kept_layers}
    hw = (cfg.img_size, cfg.img_size)
    t["dpt_heads_1view"] = _best_of(lambda: (R.dpt_head(kept, sd, cfg, "depth_head.", "exp", hw),
                                             R.dpt_head(kept, sd, cfg, "point_head.", "inv_log", hw)), n=1)
    t["threads"] = threads
    return t


def compose(cfg, S: int, t: dict) -> dict:
    """Seconds of an S-view forward (and of one global block) from unit_times(cfg, sd, S)."""
    N, L = cfg.tokens_per_frame, cfg.depth
    lin = max(t["block_1view"] - t["frame_attn_1view"], 0.0)
    gattn_view = t["global_attn_q"] * N / t["global_attn_q_rows"]
    global_block = S * (lin + gattn_view)
    fwd = S * (t["patch_embed"] + L * t["block_1view"] + t["dpt_heads_1view"]) + L * global_block + t["camera_head"]
    return {"forward_s": fwd, "global_block_s": global_block, "frame_block_s": S * t["block_1view"],
            "global_attention_share": L * S * gattn_view / fwd}


def cpu_baseline(cfg, sd, S: int, threads: int | None = None) -> dict:
    """bench.py's cpu_baseline object for an S-view forward (value in views/s)."""
    t0 = time.perf_counter()
    t = unit_times(cfg, sd, S, threads=threads)
    c = compose(cfg, S, t)
    wall = time.perf_counter() - t0
    return {
        "value": S / c["forward_s"],
        "unit": "views/s",
        "cores": t["threads"],
        "kind": "port",
        "sample": (f"fp32 CPU oracle (oracle/vggt_ref.py) on {t['threads']} host threads, composed per work unit at "
                   f"the S={S} shapes: global attention of {t['global_attn_q_rows']} queries x 16 heads against "
                   f"the full {S * cfg.tokens_per_frame}-token K/V {t['global_attn_q']:.2f} s, one 1374-token block "
                   f"{t['block_1view'] * 1e3:.0f} ms (frame attention {t['frame_attn_1view'] * 1e3:.0f} ms), "
                   f"patch-embed {t['patch_embed'] * 1e3:.0f} ms and DPT heads {t['dpt_heads_1view']:.2f} s per "
                   f"view, camera head over all {S} views {t['camera_head']:.2f} s -> {c['forward_s']:.0f} s per "
                   f"forward ({100 * c['global_attention_share']:.1f}% global attention); composition checked "
                   f"against measured forwards in profiles/r02_cpu_baseline_check.json"),
        "forward_s": c["forward_s"],
        "units_s": t,
        "sample_wall_s": wall,
    }
