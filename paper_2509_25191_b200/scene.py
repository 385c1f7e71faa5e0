"""Scene-level consumers of the predictions on the device.

Drop-ins for the reference functions that turn VGGT outputs into what the Global-Alignment and
3DGS stages use, with the reference's argument meaning, return types and exceptions:

  select_matched_points   pkg/src/epialign/pointcloud.py:91-130 (+ sample_depth :66-88,
                          geometry.unproject :341-348): high-weight correspondences lifted
                          to world points with their endpoint disagreement;
  select_pairs            pkg/src/epialign/pairing.py:88-109: view-angle pair filter;
  pairwise_errors /       pkg/src/epialign/metrics.py:89-147: relative rotation / translation
  evaluate_poses / auc_at_30   direction errors over all frame pairs, AUC@30;
  unproject_depth_maps    dense world-point maps from VGGT depth + decoded cameras (the
                          depth-based point cloud used to initialise 3DGS).

Inputs are duck-typed like paper_2509_25191_b200.ga (the reference's objects work as-is); the
reference's result classes and exceptions are used when `epialign` is importable.  All per-element
work runs in csrc/scene.cu; the host only gathers inputs and compacts outputs (torch, on device).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops

try:  # the reference's own result types and exceptions when installed
    from epialign.errors import (EmptySequence, FrameMismatch, InsufficientFrames, InvalidDepth,  # type: ignore
                                 MissingDepthMap)
    from epialign.metrics import PoseMetrics  # type: ignore
    from epialign.pairing import PairSelection  # type: ignore
    from epialign.pointcloud import ScenePointCloud  # type: ignore
except ImportError:  # same names / fields as pkg/src/epialign/{errors,metrics,pairing,pointcloud}.py
    class EpialignError(Exception):
        pass

    class DataError(EpialignError):
        pass

    class NumericalError(EpialignError):
        pass

    class FrameMismatch(DataError):
        pass

    class EmptySequence(DataError):
        pass

    class InsufficientFrames(DataError):
        pass

    class MissingDepthMap(DataError):
        pass

    class InvalidDepth(NumericalError):
        pass

    @dataclass(frozen=True)
    class ScenePointCloud:
        points: np.ndarray
        colors: np.ndarray | None = None
        source: str = "external"
        consistency: np.ndarray | None = None

        def __len__(self) -> int:
            return self.points.shape[0]

    @dataclass(frozen=True)
    class PairSelection:
        pairs: tuple
        view_angle_deg: np.ndarray

        def __len__(self) -> int:
            return len(self.pairs)

        def as_set(self) -> set:
            return set(self.pairs)

    @dataclass(frozen=True)
    class PoseMetrics:
        rre_deg: np.ndarray
        rte_deg: np.ndarray
        rre_mean: float
        rte_mean: float
        pair_count: int
        auc_at_30: float | None
        zero_baseline_flags: np.ndarray


def _k_inverse(fx, fy, cx, cy):
    return np.array([[1.0 / fx, 0.0, -cx / fx], [0.0, 1.0 / fy, -cy / fy], [0.0, 0.0, 1.0]])


def _dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def _rig(rig):
    fr = list(rig.frames)
    R = np.stack([np.asarray(f.pose.R, dtype=np.float64) for f in fr])
    t = np.stack([np.asarray(f.pose.t, dtype=np.float64) for f in fr])
    Kinv = np.stack([_k_inverse(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy) for f in fr])
    return R, t, Kinv


# ------------------------------------------------------------------------------------------------
# matched points (pointcloud.py:91-130)

def select_matched_points_arrays(pair_ij, offsets, xy_i, xy_j, w, depth_maps, R, t, Kinv,
                                 weight_threshold: float = 0.3):
    """Array form: depth_maps = list/dict frame -> 2-D map (numpy or torch, fp32/fp64).

    Returns (points (2m, 3), consistency (2m,), skipped) as numpy, points in (pair, correspondence)
    order with the two endpoints of a correspondence adjacent, like the reference.
    """
    if weight_threshold < 0:
        raise ValueError("weight threshold must be >= 0")
    pair_ij = np.asarray(pair_ij, dtype=np.int32).reshape(-1, 2)
    for f in np.unique(pair_ij):
        if int(f) not in depth_maps:
            raise MissingDepthMap(f"no depth map for frame index {int(f)}")
    R, t, Kinv = (np.asarray(a, dtype=np.float64) for a in (R, t, Kinv))
    n = R.shape[0]
    if pair_ij.size and (int(pair_ij.min()) < -n or int(pair_ij.max()) >= n):
        # the reference fails on rig[frame] (IndexError); the kernel would read past the cameras
        bad = int(pair_ij.min()) if int(pair_ij.min()) < -n else int(pair_ij.max())
        raise IndexError(f"pair frame index {bad} outside the rig of {n} frames")
    neg = sorted({int(f) for f in np.unique(pair_ij) if f < 0})
    virt = {}
    if neg:  # rig[-k] wraps in the reference while the depth map stays keyed by -k: one virtual frame each
        virt = {f: n + i for i, f in enumerate(neg)}
        R = np.concatenate([R, R[neg]])
        t = np.concatenate([t, t[neg]])
        Kinv = np.concatenate([Kinv, Kinv[neg]])
        pair_ij = np.vectorize(lambda f: virt.get(int(f), int(f)), otypes=[np.int32])(pair_ij)
    keys = sorted(int(k) for k in depth_maps)
    def as_map(d):  # DepthMap-like (.values) or a plain 2-D array / tensor
        return torch.as_tensor(d if isinstance(d, (np.ndarray, torch.Tensor)) else d.values)

    maps = [as_map(depth_maps[k]) for k in keys]
    f32 = all(m.dtype == torch.float32 for m in maps)
    dt = torch.float32 if f32 else torch.float64
    slot = np.full(n + len(virt), 0, dtype=np.int32)
    for s, k in enumerate(keys):
        if 0 <= k < n:
            slot[k] = s
        elif k in virt:
            slot[virt[k]] = s
    hw = np.array([[m.shape[0], m.shape[1]] for m in maps], dtype=np.int32)
    moff = np.concatenate([[0], np.cumsum([m.numel() for m in maps])[:-1]]).astype(np.int64)
    depth = torch.cat([m.reshape(-1).to(device="cuda", dtype=dt) for m in maps])
    xy_i = _dev(np.asarray(xy_i, dtype=np.float64).reshape(-1, 2))
    xy_j = _dev(np.asarray(xy_j, dtype=np.float64).reshape(-1, 2))
    pts, gap, state = ops.matched_points(
        depth, _dev(moff, torch.int64), _dev(hw, torch.int32), _dev(slot, torch.int32), _dev(R).reshape(-1, 9),
        _dev(t).reshape(-1, 3), _dev(Kinv).reshape(-1, 9), _dev(pair_ij, torch.int32), _dev(offsets, torch.int64),
        xy_i, xy_j, _dev(np.asarray(w, dtype=np.float64).reshape(-1)), weight_threshold)
    if bool((state == 3).any().item()):
        raise InvalidDepth("depth must be positive and finite")
    keep = state == 1
    points = pts[keep].reshape(-1, 3).cpu().numpy()
    consistency = gap[keep].repeat_interleave(2).cpu().numpy()
    skipped = int((state == 2).sum().item())
    return points, consistency, skipped


def select_matched_points(matches, weights, depths, rig, weight_threshold: float = 0.3):
    """pointcloud.py:91-130 -> (ScenePointCloud(source="matched"), skipped)."""
    pairs = list(matches.pairs)
    pair_ij = np.array([[p.frame_i, p.frame_j] for p in pairs], dtype=np.int32).reshape(-1, 2)
    offsets = np.concatenate([[0], np.cumsum([len(p.xy_i) for p in pairs])]).astype(np.int64)
    cat = (lambda key: np.concatenate([np.asarray(getattr(p, key), dtype=np.float64).reshape(-1, 2) for p in pairs])
           if pairs else np.zeros((0, 2)))
    w = np.asarray(getattr(weights, "weights", weights), dtype=np.float64).reshape(-1)
    if w.shape[0] != offsets[-1]:
        raise ValueError("weight table does not match the match set size")
    R, t, Kinv = _rig(rig)
    points, consistency, skipped = select_matched_points_arrays(pair_ij, offsets, cat("xy_i"), cat("xy_j"), w, depths,
                                                                R, t, Kinv, weight_threshold)
    return ScenePointCloud(points, source="matched", consistency=consistency), skipped


# ------------------------------------------------------------------------------------------------
# dense depth -> world points

def unproject_depth_maps(depth: torch.Tensor, extrinsic: torch.Tensor, intrinsic: torch.Tensor) -> torch.Tensor:
    """World-point maps (S, H, W, 3) fp32 from depth (S, H, W[, 1]), world-to-camera extrinsic (S, 3, 4) and
    intrinsic (S, 3, 3) — VGGT's depth-based point cloud (pose.pose_encoding_to_extri_intri gives the cameras)."""
    if depth.dim() == 4:
        depth = depth[..., 0]
    return ops.unproject_depth(depth.float().contiguous(), extrinsic.float().contiguous(),
                               intrinsic.float().contiguous())


# ------------------------------------------------------------------------------------------------
# pair selection (pairing.py:88-109)

def select_pairs(rig, threshold_deg: float):
    """pairing.py:88-109 -> PairSelection(pairs sorted by (i, j), view angles in degrees)."""
    n = len(rig.frames)
    if n < 2:
        raise InsufficientFrames(f"need at least 2 frames, got {n}")
    if not (0.0 < threshold_deg <= 180.0):
        raise ValueError(f"threshold must be in (0, 180], got {threshold_deg}")
    R = _dev(np.stack([np.asarray(f.pose.R, dtype=np.float64) for f in rig.frames])).reshape(-1, 9)
    flag, angle = ops.select_pairs(R, threshold_deg)
    idx = torch.nonzero(flag, as_tuple=False).reshape(-1)
    ij = torch.triu_indices(n, n, 1, device=flag.device)  # row-major (i, j), the kernel's output order
    pairs = tuple(zip(ij[0, idx].tolist(), ij[1, idx].tolist()))
    return PairSelection(pairs, angle[idx].cpu().numpy())


# ------------------------------------------------------------------------------------------------
# pose metrics (metrics.py:68-147)

def _match_frames(pred, gt):
    if len(pred.frames) != len(gt.frames) or len(pred.frames) < 2:
        raise FrameMismatch(f"rigs must share >= 2 frames, got {len(pred.frames)} vs {len(gt.frames)}")
    gt_index = {f.frame_id: k for k, f in enumerate(gt.frames)}
    try:
        return [gt_index[f.frame_id] for f in pred.frames]
    except KeyError as exc:
        raise FrameMismatch(f"frame id {exc.args[0]!r} missing from ground truth") from None


def pairwise_errors_arrays(Rp, tp, Rg, tg, gt_of, order_invariant: bool = False):
    """-> (rre, rte, zero_baseline flags) as device tensors in the reference's directed-pair order."""
    rre, rte, flag = ops.pairwise_errors(_dev(Rp).reshape(-1, 9), _dev(tp).reshape(-1, 3), _dev(Rg).reshape(-1, 9),
                                         _dev(tg).reshape(-1, 3), _dev(gt_of, torch.int32), order_invariant)
    return rre, rte, flag.bool()


def pairwise_errors(pred, gt, order_invariant: bool = False):
    """metrics.py:89-118 -> PoseMetrics (auc_at_30 None)."""
    gt_of = _match_frames(pred, gt)
    Rp, tp, _ = _rig(pred)
    Rg, tg, _ = _rig(gt)
    rre, rte, flag = pairwise_errors_arrays(Rp, tp, Rg, tg, np.asarray(gt_of, dtype=np.int32), order_invariant)
    rre_n, rte_n = rre.cpu().numpy(), rte.cpu().numpy()
    return PoseMetrics(rre_deg=rre_n, rte_deg=rte_n, rre_mean=float(rre_n.mean()), rte_mean=float(rte_n.mean()),
                       pair_count=int(rre_n.shape[0]), auc_at_30=None, zero_baseline_flags=flag.cpu().numpy())


def auc_at_30(rre_deg, rte_deg) -> float:
    """metrics.py:121-134: exact area under the accuracy curve from 0 to 30 degrees."""
    rre = np.asarray(rre_deg, dtype=np.float64).reshape(-1)
    rte = np.asarray(rte_deg, dtype=np.float64).reshape(-1)
    if rre.shape != rte.shape:
        raise ValueError("RRE and RTE sequences must have equal length")
    if rre.size == 0:
        raise EmptySequence("cannot integrate an empty error sequence")
    err = np.maximum(rre, rte)
    return float(np.maximum(0.0, 30.0 - err).sum() / (30.0 * err.size))


def evaluate_poses(pred, gt, order_invariant: bool = False):
    """metrics.py:137-147."""
    m = pairwise_errors(pred, gt, order_invariant)
    return PoseMetrics(rre_deg=m.rre_deg, rte_deg=m.rte_deg, rre_mean=m.rre_mean, rte_mean=m.rte_mean,
                       pair_count=m.pair_count, auc_at_30=auc_at_30(m.rre_deg, m.rte_deg),
                       zero_baseline_flags=m.zero_baseline_flags)


__all__ = ["select_matched_points", "select_matched_points_arrays", "unproject_depth_maps", "select_pairs",
           "pairwise_errors", "pairwise_errors_arrays", "evaluate_poses", "auc_at_30"]
