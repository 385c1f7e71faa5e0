"""Generates tests/golden/scene.npz from the REFERENCE's own scene-level functions.

Imports epialign (pointcloud, pairing, metrics, synth, geometry) from /root/reference/pkg/src
(read-only; build container only) and records inputs + outputs of
  select_matched_points (pointcloud.py:91-130) on synthetic scenes with the reference's sparse
    depth maps and with dense smooth depth maps (bilinear path), several thresholds;
  sample_depth (pointcloud.py:66-88) at random sub-pixel locations incl. borders;
  select_pairs (pairing.py:88-109) on a 40-camera orbit at several thresholds;
  pairwise_errors / evaluate_poses (metrics.py:89-147) on perturbed rigs, both orders, with a
    zero-baseline pair.
Re-run: python tests/golden/make_scene_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from epialign.geometry import CameraFrame, CameraPose, CameraRig  # noqa: E402
from epialign.metrics import evaluate_poses  # noqa: E402
from epialign.pairing import select_pairs  # noqa: E402
from epialign.pointcloud import DepthMap, sample_depth, select_matched_points  # noqa: E402
from epialign.synth import SynthConfig, generate, perturb  # noqa: E402
from epialign.weighting import WeightTable  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scene.npz")


def rig_arrays(rig):
    R = np.stack([f.pose.R for f in rig.frames])
    t = np.stack([f.pose.t for f in rig.frames])
    intr = np.array([[f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy, f.intrinsics.width,
                      f.intrinsics.height] for f in rig.frames])
    return R, t, intr


def match_arrays(ms):
    pij = np.array([[p.frame_i, p.frame_j] for p in ms.pairs], dtype=np.int32)
    off = np.concatenate([[0], np.cumsum([len(p) for p in ms.pairs])]).astype(np.int64)
    return pij, off, np.concatenate([p.xy_i for p in ms.pairs]), np.concatenate([p.xy_j for p in ms.pairs])


def main():
    out = {}
    rng = np.random.default_rng(7)
    # --- matched points: sparse synthetic depth maps (nearest-pixel fallback path)
    scene = generate(SynthConfig(n_cameras=5, n_points=400, seed=3, width=160, height=120, focal_px=100.0))
    R, t, intr = rig_arrays(scene.rig)
    pij, off, xi, xj = match_arrays(scene.matches)
    w = rng.uniform(0, 1, size=off[-1])
    depths = np.stack([scene.depths[f].values for f in range(len(R))])
    out.update({"mp/R": R, "mp/t": t, "mp/intr": intr, "mp/pair_ij": pij, "mp/offsets": off, "mp/xy_i": xi,
                "mp/xy_j": xj, "mp/w": w, "mp/depth_sparse": depths})
    for name, dm in (("sparse", depths),):
        for thr in (0.0, 0.3, 0.7):
            cloud, sk = select_matched_points(scene.matches, WeightTable(w, 0.5, 1.0),
                                              {f: DepthMap(dm[f]) for f in range(len(R))}, scene.rig, thr)
            out[f"mp/{name}_{thr}/points"] = cloud.points
            out[f"mp/{name}_{thr}/consistency"] = cloud.consistency
            out[f"mp/{name}_{thr}/skipped"] = np.array(sk)
    # dense smooth depth maps with holes (bilinear path + invalid neighbourhoods)
    H, W = depths.shape[1:]
    yy, xx = np.mgrid[0:H, 0:W]
    dense = np.stack([3.0 + 0.5 * np.sin(xx / 37.0 + f) * np.cos(yy / 23.0 - f) for f in range(len(R))])
    holes = rng.uniform(size=dense.shape) < 0.02
    dense[holes] = 0.0
    out["mp/depth_dense"] = dense
    for thr in (0.3,):
        cloud, sk = select_matched_points(scene.matches, WeightTable(w, 0.5, 1.0),
                                          {f: DepthMap(dense[f]) for f in range(len(R))}, scene.rig, thr)
        out[f"mp/dense_{thr}/points"] = cloud.points
        out[f"mp/dense_{thr}/consistency"] = cloud.consistency
        out[f"mp/dense_{thr}/skipped"] = np.array(sk)
    # --- sample_depth at random locations incl. out-of-image borders and exact pixel centres
    uv = np.concatenate([rng.uniform(-1.5, W + 0.5, size=(400, 1)), rng.uniform(-1.5, H + 0.5, size=(400, 1))], 1)
    uv[:50] = np.round(uv[:50])
    uv[50:60, 0] += 0.5 - (uv[50:60, 0] % 1.0)  # exact .5 (round-half-even in the fallback)
    out["sd/uv"] = uv
    out["sd/sparse"] = np.array([sample_depth(DepthMap(depths[0]), u, v) for u, v in uv])
    out["sd/dense"] = np.array([sample_depth(DepthMap(dense[1]), u, v) for u, v in uv])
    # --- pair selection on a 40-camera orbit
    big = generate(SynthConfig(n_cameras=40, n_points=50, seed=11))
    Rb, tb, _ = rig_arrays(big.rig)
    out["sp/R"] = Rb
    for thr in (15.0, 30.0, 100.0, 180.0):
        sel = select_pairs(big.rig, thr)
        out[f"sp/{thr}/pairs"] = np.array(sel.pairs, dtype=np.int64).reshape(-1, 2)
        out[f"sp/{thr}/angles"] = sel.view_angle_deg
    # --- pose metrics on a perturbed rig, with a duplicated centre (zero baseline) and shuffled ids
    cfg = SynthConfig(n_cameras=12, n_points=100, seed=5, rot_sigma_deg=2.0, trans_sigma_frac=0.02)
    sc = generate(cfg)
    pred, _, _ = perturb(sc.rig, sc.matches, cfg)
    frames = list(pred.frames)
    frames[3] = CameraFrame(frames[3].frame_id, frames[3].intrinsics, CameraPose(frames[2].pose.R, frames[2].pose.t))
    order = rng.permutation(len(frames))
    pred = CameraRig(tuple(frames[k] for k in order))
    Rp, tp, _ = rig_arrays(pred)
    Rg, tg, _ = rig_arrays(sc.rig)
    gt_index = sc.rig.index_by_id()
    out["pe/Rp"], out["pe/tp"], out["pe/Rg"], out["pe/tg"] = Rp, tp, Rg, tg
    out["pe/gt_of"] = np.array([gt_index[f.frame_id] for f in pred.frames], dtype=np.int32)
    for oi in (False, True):
        m = evaluate_poses(pred, sc.rig, order_invariant=oi)
        out[f"pe/{int(oi)}/rre"] = m.rre_deg
        out[f"pe/{int(oi)}/rte"] = m.rte_deg
        out[f"pe/{int(oi)}/flags"] = m.zero_baseline_flags
        out[f"pe/{int(oi)}/summary"] = np.array([m.rre_mean, m.rte_mean, m.pair_count, m.auc_at_30])
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
