"""Timing of the scene-level kernels (csrc/scene.cu) at dense-view sizes, with CPU-oracle samples.

  unproject_depth_maps  S x 518 x 518 fp32 depth -> world points (16 B/pixel algorithmic traffic)
  pairwise_errors       n frames, all n(n-1) directed pairs (order_invariant)
  select_pairs          n frames, n(n-1)/2 view angles
  matched_points        the bench_ga scene (12.9M correspondences) with dense 480x640 depth maps

Prints one JSON line.  Device times: CUDA events around the op (inputs resident), best of 5.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def timed(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--frames", type=int, default=2000)
    args = ap.parse_args()
    import torch

    from oracle import scene_ref
    from paper_2509_25191_b200 import ops, scene

    res = {}
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs", 6541.5)
    # dense unprojection
    S, H, W = args.views, 518, 518
    depth = 1 + torch.rand(S, H, W, device="cuda")
    extri = torch.cat([torch.eye(3).expand(S, 3, 3), torch.randn(S, 3, 1)], -1).float().cuda().contiguous()
    intri = torch.tensor([[400.0, 0, 259], [0, 400.0, 259], [0, 0, 1]]).expand(S, 3, 3).contiguous().cuda()
    out = torch.empty(S, H, W, 3, device="cuda")
    ms = timed(lambda: ops.unproject_depth(depth, extri, intri, out))
    gbs = 16.0 * S * H * W / (ms * 1e-3) / 1e9
    a = time.perf_counter()
    scene_ref.unproject_depth_maps(depth[:2].cpu().numpy(), extri[:2].cpu().numpy(), intri[:2].cpu().numpy())
    cpu_per_view = (time.perf_counter() - a) / 2
    res["unproject"] = {"views": S, "ms": ms, "gbs": gbs, "frac_of_hbm": gbs / hbm,
                        "cpu_oracle_ms_per_view": 1e3 * cpu_per_view, "cpu_oracle_ms_total_extrapolated":
                        1e3 * cpu_per_view * S}
    # pairwise pose errors + pair selection at n frames
    n = args.frames
    rng = np.random.default_rng(0)
    q, _ = np.linalg.qr(rng.normal(size=(n, 3, 3)))
    Rp = torch.as_tensor(q, device="cuda").reshape(n, 9).contiguous()
    tp = torch.as_tensor(rng.normal(size=(n, 3)), device="cuda")
    Rg = Rp.clone()
    tg = tp + 0.01
    gt_of = torch.arange(n, device="cuda", dtype=torch.int32)
    ms = timed(lambda: ops.pairwise_errors(Rp, tp, Rg, tg, gt_of, True))
    m_cpu = 60
    a = time.perf_counter()
    scene_ref.pairwise_errors(q[:m_cpu], tp[:m_cpu].cpu().numpy(), q[:m_cpu], tg[:m_cpu].cpu().numpy(),
                              np.arange(m_cpu), True)
    cpu_pair_s = (time.perf_counter() - a) / (m_cpu * (m_cpu - 1))
    res["pairwise_errors"] = {"frames": n, "directed_pairs": n * (n - 1), "ms": ms,
                              "cpu_oracle_s_extrapolated": cpu_pair_s * n * (n - 1)}
    ms = timed(lambda: ops.select_pairs(Rp, 30.0))
    res["select_pairs"] = {"frames": n, "pairs": n * (n - 1) // 2, "ms": ms}
    # matched points on the GA bench scene with dense depth maps
    import bench_ga
    R, t, intr, pij, off, xi, xj = bench_ga.scene(200, 20000, 30.0, 4096)
    Kinv = np.stack([scene_ref.k_inverse(*x[:4]) for x in intr])
    K = int(off[-1])
    dmaps = (2 + torch.rand(len(R), 480, 640, device="cuda", dtype=torch.float32))
    args_dev = (dmaps.reshape(-1), torch.as_tensor(np.arange(len(R)) * 480 * 640, device="cuda"),
                torch.as_tensor(np.tile([480, 640], (len(R), 1)).astype(np.int32), device="cuda"),
                torch.arange(len(R), device="cuda", dtype=torch.int32),
                torch.as_tensor(R, device="cuda").reshape(-1, 9), torch.as_tensor(t, device="cuda"),
                torch.as_tensor(Kinv, device="cuda").reshape(-1, 9), torch.as_tensor(pij, device="cuda"),
                torch.as_tensor(off, device="cuda"), torch.as_tensor(xi, device="cuda"),
                torch.as_tensor(xj, device="cuda"), torch.rand(K, device="cuda", dtype=torch.float64), 0.3)
    ms = timed(lambda: ops.matched_points(*args_dev))
    res["matched_points"] = {"correspondences": K, "ms": ms,
                             "algorithmic_gbs": (40 + 56 + 1) * K / (ms * 1e-3) / 1e9}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
