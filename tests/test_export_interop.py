"""f1: the PredictionSet this package writes feeds the reference's own adapter unchanged.

`pose.save_prediction_set` writes the npz schema of `pkg/adapter/src/epialign_adapter/export.py:54-99`.
Here the reference adapter itself (imported from /root/reference in this container; skipped where
it is absent, e.g. on the GPU box) loads that file and runs its `export`: shape checks against
a manifest, the rotation acceptance rule (`export.py:111-128`), and the cameras.json / EPMT /
PFM writers (`formats.py:23-91`). The written files are then read back and compared with the
decoded poses. CPU only: the decode is host code and the predictions are synthetic,
shaped like the VGGT output dict.
"""
import json
import math
import sys

import numpy as np
import pytest
import torch

ADAPTER_SRC = "/root/reference/pkg/adapter/src"


@pytest.fixture(scope="module")
def adapter():
    if ADAPTER_SRC not in sys.path:
        sys.path.insert(0, ADAPTER_SRC)
    return pytest.importorskip("epialign_adapter", reason="reference adapter not present")


def _vggt_like_outputs(S=5, H=48, W=64, seed=0):
    """A VGGT output dict: pose_enc [1, S, 9] (T, quat XYZW, fov_h, fov_w), depth [1, S, H, W, 1]."""
    g = torch.Generator().manual_seed(seed)
    T = torch.randn(S, 3, generator=g)
    q = torch.randn(S, 4, generator=g)
    q = q / q.norm(dim=-1, keepdim=True)
    fov = torch.tensor([math.radians(50.0), math.radians(60.0)]).expand(S, 2)
    enc = torch.cat([T, q, fov], dim=-1)[None].float()
    depth = (1.0 + torch.rand(1, S, H, W, 1, generator=g)).float()
    return {"pose_enc": enc, "depth": depth}


def test_prediction_set_npz_exports_through_reference_adapter(adapter, tmp_path):
    from paper_2509_25191_b200.pose import pose_encoding_to_extri_intri, save_prediction_set

    S, H, W = 5, 48, 64
    out = _vggt_like_outputs(S, H, W)
    npz = tmp_path / "preds.npz"
    save_prediction_set(out, npz)

    preds = adapter.PredictionSet.load_npz(npz)
    frames = tuple(adapter.FrameSpec(f"frame_{i:04d}", "", W, H) for i in range(S))
    manifest = adapter.AdapterManifest("vggt", frames, str(tmp_path / "exported"))
    res = adapter.export(manifest, preds)
    assert len(res.depth_paths) == S and res.pair_count == 0

    ext, K = pose_encoding_to_extri_intri(out["pose_enc"][0].double(), (H, W))
    rig = json.loads(res.cameras_path.read_text())
    assert rig["convention"] == "world_to_camera" and len(rig["frames"]) == S
    for i, fr in enumerate(rig["frames"]):
        assert (fr["width"], fr["height"]) == (W, H)
        assert np.allclose([fr["fx"], fr["fy"], fr["cx"], fr["cy"]],
                           [K[i, 0, 0], K[i, 1, 1], K[i, 0, 2], K[i, 1, 2]], rtol=1e-6)
        # the adapter re-orthonormalises the float32 block: within float32 rounding of ours
        assert np.allclose(np.reshape(fr["R"], (3, 3)), ext[i, :, :3].numpy(), atol=1e-6)
        assert np.allclose(fr["t"], ext[i, :, 3].numpy(), atol=1e-6)
    # PFM: bottom-up rows, little-endian float32 (formats.py:80-86)
    for i, p in enumerate(res.depth_paths):
        blob = p.read_bytes()
        header = f"Pf\n{W} {H}\n-1.0\n".encode("ascii")
        assert blob.startswith(header)
        d = np.frombuffer(blob[len(header):], dtype="<f4").reshape(H, W)[::-1]
        assert np.array_equal(d, out["depth"][0, i, ..., 0].numpy())


def test_reflected_rotation_is_rejected_by_reference_adapter(adapter, tmp_path):
    """A decode that produced a reflection would abort the reference export (NonRotationExtrinsic);
    quaternion decode never does, but the schema check is the reference's, so exercise it."""
    from paper_2509_25191_b200.pose import to_prediction_set

    out = _vggt_like_outputs(3, 8, 8, seed=1)
    arrays = to_prediction_set(out)
    arrays["rotations"][1] = -arrays["rotations"][1]  # det = -1
    preds = adapter.PredictionSet(**arrays)
    frames = tuple(adapter.FrameSpec(str(i), "", 8, 8) for i in range(3))
    with pytest.raises(adapter.NonRotationExtrinsic):
        adapter.export(adapter.AdapterManifest("vggt", frames, str(tmp_path)), preds)
