"""Pose-encoding decode and the PredictionSet export (§8f-1).

`pose_encoding_to_extri_intri` follows the upstream absT_quaR_FoV convention:
enc = [T(3), quat XYZW(4), fov_h, fov_w]; extrinsic = [R | T] camera-from-world
(world-to-camera, the reference's convention `pkg/src/epialign/geometry.py:5-8`);
fx = (W/2)/tan(fov_w/2), fy = (H/2)/tan(fov_h/2), principal point (W/2, H/2).

`to_prediction_set` emits the arrays of the reference adapter's `PredictionSet`
npz schema (`pkg/adapter/src/epialign_adapter/export.py:54-99`,
`pkg/adapter/README.md:47-53`): intrinsics (N,3,3), rotations (N,3,3)
world-to-camera, translations (N,3), depth (N,H,W), float32.
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np
import torch


def quat_to_mat(q: torch.Tensor) -> torch.Tensor:
    """XYZW (scalar-last) quaternion -> rotation matrix, normalising."""
    q = q / q.norm(dim=-1, keepdim=True)
    x, y, z, w = q.unbind(-1)
    return torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
        2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
        2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y),
    ], dim=-1).reshape(q.shape[:-1] + (3, 3))


def pose_encoding_to_extri_intri(enc: torch.Tensor, image_size_hw: Tuple[int, int]):
    H, W = image_size_hw
    T = enc[..., :3]
    R = quat_to_mat(enc[..., 3:7])
    fy = (H / 2.0) / torch.tan(enc[..., 7] / 2.0)
    fx = (W / 2.0) / torch.tan(enc[..., 8] / 2.0)
    K = torch.zeros(enc.shape[:-1] + (3, 3), dtype=enc.dtype, device=enc.device)
    K[..., 0, 0] = fx
    K[..., 1, 1] = fy
    K[..., 0, 2] = W / 2.0
    K[..., 1, 2] = H / 2.0
    K[..., 2, 2] = 1.0
    return torch.cat([R, T[..., None]], dim=-1), K


def to_prediction_set(preds: Dict[str, torch.Tensor]) -> Dict[str, np.ndarray]:
    """VGGT output dict -> arrays of the epialign-adapter PredictionSet npz (float32)."""
    enc = preds["pose_enc"][0].float()
    H, W = preds["depth"].shape[2:4]
    ext, K = pose_encoding_to_extri_intri(enc, (H, W))
    return {
        "intrinsics": K.cpu().numpy().astype(np.float32),
        "rotations": ext[..., :3].cpu().numpy().astype(np.float32),
        "translations": ext[..., 3].cpu().numpy().astype(np.float32),
        "depth": preds["depth"][0, ..., 0].float().cpu().numpy().astype(np.float32),
    }


def save_prediction_set(preds: Dict[str, torch.Tensor], path) -> None:
    np.savez(path, **to_prediction_set(preds))
