"""Benchmark of the on-device Global-Alignment optimiser at dense-view scale.

Synthetic scene (this script's own generator, shaped like the reference's synth.generate orbit
layout, pkg/src/epialign/synth.py:105-175): n cameras on a ring looking at a point cloud, pairs
whose optical axes are within `--angle` degrees (pairing.select_pairs), up to `--cap`
correspondences per pair (pairing.MAX_CORRESPONDENCES = 4096), 0.5 px pixel noise, perturbed
cameras.  Runs `ga.align_arrays` (300 Adam iterations by default) and prints one JSON line:
whole-call wall time, device time of the iteration loop, per-iteration time, the pair kernel's
achieved HBM bandwidth (40 algorithmic bytes per correspondence: xy_i, xy_j, w), and a CPU
baseline: the oracle (oracle/ga_ref.py, the reference's algorithm on numpy) timed for a few
iterations on the host and extrapolated per iteration.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def look_at(c, target):
    z = target - c
    z /= np.linalg.norm(z)
    up = np.array([0.0, 0.0, 1.0])
    x = np.cross(up, z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])  # world -> camera rows
    return R, -R @ c


def scene(n, points, angle, cap, seed=0, fx=400.0, W=640, H=480):
    rng = np.random.default_rng(seed)
    ang = np.linspace(0, 2 * np.pi, n, endpoint=False)
    C = np.stack([4 * np.cos(ang), 4 * np.sin(ang), 0.3 * rng.normal(size=n)], 1)
    X = rng.normal(size=(points, 3))
    X = 1.5 * X / np.linalg.norm(X, axis=1, keepdims=True) * rng.uniform(0, 1, size=(points, 1)) ** (1 / 3)
    Rs, ts = [], []
    for c in C:
        R, t = look_at(c, 0.15 * rng.normal(size=3))
        Rs.append(R)
        ts.append(t)
    Rs, ts = np.stack(Rs), np.stack(ts)
    cx, cy = (W - 1) / 2, (H - 1) / 2
    Xc = np.einsum("nij,pj->npi", Rs, X) + ts[:, None, :]
    uv = np.stack([fx * Xc[..., 0] / Xc[..., 2] + cx, fx * Xc[..., 1] / Xc[..., 2] + cy], -1)
    vis = (Xc[..., 2] > 0.1) & (uv[..., 0] >= 0) & (uv[..., 0] < W) & (uv[..., 1] >= 0) & (uv[..., 1] < H)
    z = Rs[:, 2, :]
    cosang = np.clip(z @ z.T, -1, 1)
    pairs, offs, xi, xj = [], [0], [], []
    for i in range(n):
        for j in range(i + 1, n):
            if np.degrees(np.arccos(cosang[i, j])) > angle:
                continue
            both = np.flatnonzero(vis[i] & vis[j])[:cap]
            if len(both) < 8:
                continue
            pairs.append((i, j))
            xi.append(uv[i, both] + 0.5 * rng.normal(size=(len(both), 2)))
            xj.append(uv[j, both] + 0.5 * rng.normal(size=(len(both), 2)))
            offs.append(offs[-1] + len(both))
    # perturb the cameras (frame 0 kept as the gauge)
    Rp, tp = Rs.copy(), ts.copy()
    for f in range(1, n):
        a = rng.normal(size=3)
        a *= np.radians(0.5) / np.linalg.norm(a)
        K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
        th = np.linalg.norm(a)
        dR = np.eye(3) + np.sin(th) / th * K + (1 - np.cos(th)) / th ** 2 * K @ K
        Rp[f] = dR @ Rs[f]
        tp[f] = ts[f] + 0.01 * rng.normal(size=3)
    intr = np.tile([fx, fx, cx, cy, W, H], (n, 1)).astype(np.float64)
    return (Rp, tp, intr, np.array(pairs, dtype=np.int32), np.array(offs, dtype=np.int64), np.concatenate(xi),
            np.concatenate(xj))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--points", type=int, default=20000)
    ap.add_argument("--angle", type=float, default=30.0)
    ap.add_argument("--cap", type=int, default=4096)
    ap.add_argument("--iterations", type=int, default=300)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    import torch

    from paper_2509_25191_b200 import ga

    t0 = time.time()
    R, t, intr, pair_ij, offsets, xy_i, xy_j = scene(args.views, args.points, args.angle, args.cap)
    gen_s = time.time() - t0
    P, K = len(pair_ij), int(offsets[-1])
    cfg = ga.AlignerConfig(iterations=args.iterations)
    out = ga.align_arrays(R, t, intr, pair_ij, offsets, xy_i, xy_j, cfg)  # warm-up (module load, graph code paths)
    torch.cuda.synchronize()
    walls = []
    for _ in range(args.repeats):
        torch.cuda.synchronize()
        a = time.perf_counter()
        out = ga.align_arrays(R, t, intr, pair_ij, offsets, xy_i, xy_j, cfg)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - a)

    # device time of the iteration loop alone (one CUDA graph), and of the pair kernel
    Kinv = np.stack([ga._k_inverse(*x[:4]) for x in intr])
    prob = ga.DeviceProblem(R, t, Kinv, pair_ij, offsets, xy_i, xy_j, 1, False, 0)
    from paper_2509_25191_b200 import ops
    ops.ga_decode(prob.pb)
    T = args.iterations
    bc1 = torch.as_tensor([1 - 0.9 ** k for k in range(1, T + 1)], device="cuda", dtype=torch.float64)
    bc2 = torch.as_tensor([1 - 0.999 ** k for k in range(1, T + 1)], device="cuda", dtype=torch.float64)
    trace = torch.empty(T, device="cuda", dtype=torch.float64)
    sk = torch.zeros(1, device="cuda", dtype=torch.float64)
    prob.adam(0, T, 1e-3, bc1, bc2, trace, sk)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    prob.adam(0, T, 1e-3, bc1, bc2, trace, sk)
    e.record()
    torch.cuda.synchronize()
    loop_ms = s.elapsed_time(e)
    # pair kernel alone: loss/grad evaluations (pair + loss + frame kernels) minus nothing: report both
    grad = torch.empty(prob.n, prob.dim, device="cuda", dtype=torch.float64)
    for _ in range(3):
        ops.ga_loss_grad(prob.pb, grad)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20):
        ops.ga_loss_grad(prob.pb, grad)
    e.record()
    torch.cuda.synchronize()
    eval_ms = s.elapsed_time(e) / 20
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs") or 6541.5
    res = {
        "workload": f"GA align, {args.views} views, {P} pairs, {K} correspondences, {T} iterations",
        "views": args.views, "pairs": P, "correspondences": K, "iterations": T,
        "align_wall_s": min(walls) if walls else None, "align_wall_all_s": walls,
        "loop_device_ms": loop_ms, "iteration_us": 1000 * loop_ms / T,
        "eval_us": 1000 * eval_ms,
        "pair_kernel_hbm_gbps_lower_bound": 40.0 * K / (eval_ms * 1e-3) / 1e9,
        "hbm_peak_gbps": hbm,
        "final_loss": float(out["loss_trace"][-1]), "initial_loss": float(out["loss_trace"][0]),
        "median_px": [float(out["report"][0]), float(out["report"][1])],
        "scene_gen_s": gen_s,
    }
    if not args.no_cpu:
        from oracle import ga_ref
        centroid = np.stack([-R[f].T @ t[f] for f in range(len(R))]).mean(axis=0)
        t_c = np.stack([t[f] + R[f] @ centroid for f in range(len(R))])
        Kinv = np.stack([ga_ref.k_inverse(x) for x in intr])
        from oracle import build_ref
        cy = build_ref.load()  # the reference's compiled per-pair kernel, when oracle/_ref was built
        cprob = ga_ref.Problem(R, t_c, Kinv, pair_ij, offsets, xy_i, xy_j, 1, False, 0, kernels=cy)
        p = ga_ref.identity_params(len(R), False)
        w = np.ones(K)
        a = time.perf_counter()
        for _ in range(args.cpu_iters):
            cprob.loss_and_gradient(p, w)
        it_s = (time.perf_counter() - a) / args.cpu_iters
        res["cpu_baseline"] = {"iteration_s": it_s, "align_s_extrapolated": it_s * T, "cores": 1,
                               "kind": "reference-kernel" if cy is not None else "port",
                               "sample": f"oracle/ga_ref.py loss_and_gradient x{args.cpu_iters} on the same scene "
                                         f"(per-pair sums by the {'compiled reference Cython kernel' if cy else 'numpy restatement'}, "
                                         f"one host thread); align time = per-iteration x {T}"}
        if walls:
            res["speedup_vs_cpu_align"] = res["cpu_baseline"]["align_s_extrapolated"] / res["align_wall_s"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
