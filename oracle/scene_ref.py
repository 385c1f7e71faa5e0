"""CPU oracle of the scene-level consumers of the predictions.

TEST INFRASTRUCTURE ONLY (same rules as oracle/vggt_ref.py): imported by tests/ and bench
baselines, never by the product path.

Numpy restatements, on plain arrays, of
  pkg/src/epialign/pointcloud.py  sample_depth (:66-88), select_matched_points (:91-130)
  pkg/src/epialign/geometry.py    unproject (:341-348)
  pkg/src/epialign/pairing.py     select_pairs (:88-109)
  pkg/src/epialign/metrics.py     _direction_angle_deg (:79-86), pairwise_errors (:89-118),
                                  auc_at_30 (:121-134)
plus the dense depth -> world-point map of the VGGT outputs (world = R^T (z K^-1 [u, v, 1] - t)
per pixel, the same algebra as geometry.unproject).

Parity is PINNED: tests/golden/scene.npz holds inputs and outputs of the reference's own
functions (tests/golden/make_scene_golden.py, run against /root/reference), and
tests/test_scene.py checks these restatements against them.
"""
from __future__ import annotations

import numpy as np

ZERO_BASELINE_TOL = 1e-9   # metrics.py:22


def k_inverse(fx, fy, cx, cy):
    return np.array([[1.0 / fx, 0.0, -cx / fx], [0.0, 1.0 / fy, -cy / fy], [0.0, 0.0, 1.0]])


def sample_depth(values, u, v):
    """pointcloud.py:66-88."""
    h, w = values.shape
    x0 = int(np.floor(u))
    y0 = int(np.floor(v))
    xs = np.clip([x0, x0 + 1], 0, w - 1)
    ys = np.clip([y0, y0 + 1], 0, h - 1)
    q = values[np.ix_(ys, xs)]
    if (q > 0).all():
        fx = u - x0
        fy = v - y0
        top = q[0, 0] * (1 - fx) + q[0, 1] * fx
        bot = q[1, 0] * (1 - fx) + q[1, 1] * fx
        return float(top * (1 - fy) + bot * fy)
    xn = int(np.clip(round(u), 0, w - 1))
    yn = int(np.clip(round(v), 0, h - 1))
    val = float(values[yn, xn])
    return val if val > 0 else 0.0


def unproject(pixel, depth, R, t, Kinv):
    """geometry.py:341-348."""
    ray = Kinv @ np.array([pixel[0], pixel[1], 1.0])
    return R.T @ (depth * ray - t)


def select_matched_points(pair_ij, offsets, xy_i, xy_j, w, depths, R, t, intr, thr=0.3):
    """pointcloud.py:91-130; depths: dict frame -> (H, W) array. -> (points (2m,3), scores (2m,), skipped)."""
    pts, scores, skipped = [], [], 0
    for p, (i, j) in enumerate(pair_ij):
        a, b = offsets[p], offsets[p + 1]
        Ki, Kj = k_inverse(*intr[i][:4]), k_inverse(*intr[j][:4])
        for k in np.flatnonzero(w[a:b] > thr):
            m = a + k
            zi = sample_depth(depths[i], xy_i[m, 0], xy_i[m, 1])
            zj = sample_depth(depths[j], xy_j[m, 0], xy_j[m, 1])
            if zi <= 0 or zj <= 0:
                skipped += 1
                continue
            p_i = unproject(xy_i[m], zi, R[i], t[i], Ki)
            p_j = unproject(xy_j[m], zj, R[j], t[j], Kj)
            gap = float(np.linalg.norm(p_i - p_j))
            pts.extend([p_i, p_j])
            scores.extend([gap, gap])
    return np.array(pts).reshape(-1, 3), np.array(scores), skipped


def select_pairs(R, thr_deg):
    """pairing.py:88-109 -> (pairs (m, 2) sorted by (i, j), angles (m,))."""
    z = np.stack([r[2] for r in R])
    cos = np.clip(z @ z.T, -1.0, 1.0)
    ang = np.degrees(np.arccos(cos))
    n = len(R)
    pairs, angles = [], []
    for i in range(n):
        for j in range(i + 1, n):
            if ang[i, j] <= thr_deg:
                pairs.append((i, j))
                angles.append(ang[i, j])
    return np.array(pairs, dtype=np.int64).reshape(-1, 2), np.array(angles)


def _direction_angle_deg(a, b):
    na = np.linalg.norm(a)
    nb = np.linalg.norm(b)
    if na < ZERO_BASELINE_TOL or nb < ZERO_BASELINE_TOL:
        return 0.0, True
    c = float(np.clip((a @ b) / (na * nb), -1.0, 1.0))
    return float(np.degrees(np.arccos(c))), False


def pairwise_errors(Rp, tp, Rg, tg, gt_of, order_invariant=False):
    """metrics.py:89-118 -> (rre, rte, flags)."""
    n = len(Rp)
    directed = []
    for i in range(n):
        for j in range(i + 1, n):
            directed.append((i, j))
            if order_invariant:
                directed.append((j, i))
    rre = np.empty(len(directed))
    rte = np.empty(len(directed))
    flags = np.zeros(len(directed), dtype=bool)
    for k, (i, j) in enumerate(directed):
        gi, gj = gt_of[i], gt_of[j]
        dRp, dtp = Rp[i].T @ Rp[j], Rp[i].T @ (tp[j] - tp[i])
        dRg, dtg = Rg[gi].T @ Rg[gj], Rg[gi].T @ (tg[gj] - tg[gi])
        M = dRg.T @ dRp
        rre[k] = float(np.degrees(np.arccos(np.clip((np.trace(M) - 1.0) / 2.0, -1.0, 1.0))))
        rte[k], flags[k] = _direction_angle_deg(dtp, dtg)
    return rre, rte, flags


def auc_at_30(rre, rte):
    """metrics.py:121-134."""
    err = np.maximum(rre, rte)
    return float(np.maximum(0.0, 30.0 - err).sum() / (30.0 * err.size))


def unproject_depth_maps(depth, extrinsic, intrinsic):
    """Dense world-point maps: depth (S, H, W), extrinsic (S, 3, 4) world-to-camera, intrinsic (S, 3, 3)
    -> (S, H, W, 3) in float64 (geometry.py:341-348 per pixel, pixel (u, v) = (column, row))."""
    S, H, W = depth.shape
    v, u = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    out = np.empty((S, H, W, 3))
    for s in range(S):
        K = intrinsic[s].astype(np.float64)
        Kinv = k_inverse(K[0, 0], K[1, 1], K[0, 2], K[1, 2])
        ray = np.stack([Kinv[0, 0] * u + Kinv[0, 1] * v + Kinv[0, 2], Kinv[1, 0] * u + Kinv[1, 1] * v + Kinv[1, 2],
                        np.ones_like(u)], -1)
        cam = depth[s].astype(np.float64)[..., None] * ray
        R = extrinsic[s, :, :3].astype(np.float64)
        t = extrinsic[s, :, 3].astype(np.float64)
        out[s] = (cam - t) @ R
    return out
