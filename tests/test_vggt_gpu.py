"""End-to-end parity of the B200 path against the CPU oracle (north-star tolerances).

  * kept aggregator tokens and depth: relative (Frobenius) error <= 1e-2
  * decoded poses: rotation error <= 1e-2 rad, translation error <= 1 %
    (|dt| / max(|t_ref|, mean |t_ref|))
Same seeded weights (bf16-representable matrices) and synthetic images on both.
"""
import os

import numpy as np
import pytest
import torch

from oracle import vggt_ref as R
from paper_2509_25191_b200.config import vggt_1b, vggt_small, vggt_tiny
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images

pytestmark = pytest.mark.gpu

TOL_TOKENS = 1e-2
TOL_DEPTH = 1e-2
TOL_ROT = 1e-2
TOL_TRANS = 1e-2


def rel(a, b):
    a, b = a.detach().float().cpu(), b.detach().float().cpu()
    return ((a - b).norm() / b.norm()).item()


def _check(cfg, sd, images, ref, label):
    from paper_2509_25191_b200.vggt import VGGT
    model = VGGT(cfg, state_dict=sd)
    out = model(images.cuda())
    kept, psi = model.aggregator(images.cuda())
    assert psi == cfg.patch_start_idx
    report = {}
    for i in cfg.kept_layers:
        C = cfg.embed_dim
        got = kept[i][0]
        assert got.dtype == torch.bfloat16 and got.shape == ref["kept"][i].shape
        report[f"kept{i}"] = rel(got, ref["kept"][i])
        report[f"kept{i}_frame"] = rel(got[..., :C], ref["kept"][i][..., :C])
        report[f"kept{i}_global"] = rel(got[..., C:], ref["kept"][i][..., C:])
        assert report[f"kept{i}"] <= TOL_TOKENS, (label, report)
    report["depth"] = rel(out["depth"], ref["depth"])
    report["depth_conf"] = rel(out["depth_conf"], ref["depth_conf"])
    report["world_points"] = rel(out["world_points"], ref["world_points"])
    report["world_points_conf"] = rel(out["world_points_conf"], ref["world_points_conf"])
    ang, terr = R.pose_errors(out["pose_enc"][0].cpu(), ref["pose_enc"][0])
    report["rot_rad_max"] = ang.max().item()
    report["trans_rel_max"] = terr.max().item()
    print(label, {k: f"{v:.2e}" for k, v in report.items()})
    assert report["depth"] <= TOL_DEPTH, (label, report)
    assert report["world_points"] <= 2e-2, (label, report)
    assert report["rot_rad_max"] <= TOL_ROT, (label, report)
    assert report["trans_rel_max"] <= TOL_TRANS, (label, report)
    assert out["pose_enc"].shape == (1, images.shape[0], 9)
    assert out["depth"].shape == (1, images.shape[0], cfg.img_size, cfg.img_size, 1)
    assert out["world_points"].shape == (1, images.shape[0], cfg.img_size, cfg.img_size, 3)
    return report


def _oracle(cfg, sd, images):
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    ref = R.vggt_forward(images, sd, cfg)
    S = images.shape[0]
    x0 = torch.cat([R.special_tokens(sd, cfg, S), R.patch_embed(images, sd, cfg)], dim=1)
    ref["kept0_in"] = x0
    return ref


def test_tiny_against_golden():
    """configs[0] (d = 32) against the committed golden fixture."""
    cfg = vggt_tiny()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 8, 1)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "tiny_s8.npz"))
    ref = {"kept": {i: torch.from_numpy(g[f"kept_{i}"]) for i in cfg.kept_layers}}
    for k in ("pose_enc", "depth", "depth_conf", "world_points", "world_points_conf"):
        ref[k] = torch.from_numpy(g[k])[None]
    ref["kept0_in"] = torch.cat([R.special_tokens(sd, cfg, 8), R.patch_embed(images, sd, cfg)], dim=1)
    _check(cfg, sd, images, ref, "tiny")


@pytest.mark.parametrize("init_values", [0.01, 0.5])
def test_small_d64(init_values):
    cfg = vggt_small().with_(init_values=init_values)
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 5, 1)
    _check(cfg, sd, images, _oracle(cfg, sd, images), f"small(ls={init_values})")


def test_vggt1b_two_views():
    """VGGT-1B-shaped (24x2 blocks, dim 1024, 518x518), S = 2."""
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 2, 1)
    _check(cfg, sd, images, _oracle(cfg, sd, images), "1b-s2")


def test_frame_chunking_is_exact():
    """frame_chunk changes only the schedule: bit-identical aggregator tokens (the vx
    kernels are row-deterministic); heads within 1e-5 (cuDNN picks batch-dependent
    conv algorithms)."""
    from paper_2509_25191_b200.vggt import VGGT
    cfg = vggt_small()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 7, 1).cuda()
    ma = VGGT(cfg.with_(frame_chunk=7, head_chunk=7), state_dict=sd)
    mb = VGGT(cfg.with_(frame_chunk=2, head_chunk=3), state_dict=sd)
    ka, _ = ma.aggregator(images)
    kb, _ = mb.aggregator(images)
    for i in cfg.kept_layers:
        assert torch.equal(ka[i], kb[i])
    a, b = ma(images), mb(images)
    for k in ("pose_enc", "depth", "world_points"):
        torch.testing.assert_close(a[k], b[k], rtol=1e-5, atol=1e-5)


def test_prediction_set_export():
    from paper_2509_25191_b200.pose import to_prediction_set
    from paper_2509_25191_b200.vggt import VGGT
    cfg = vggt_tiny()
    out = VGGT(cfg)(synthetic_images(cfg, 4, 1).cuda())
    ps = to_prediction_set(out)
    assert ps["intrinsics"].shape == (4, 3, 3) and ps["rotations"].shape == (4, 3, 3)
    assert ps["translations"].shape == (4, 3) and ps["depth"].shape == (4, 112, 112)
    for Rm in ps["rotations"].astype(np.float64):
        # the adapter's acceptance rule (export.py:111-128)
        assert np.linalg.norm(Rm.T @ Rm - np.eye(3)) <= 1e-3 and np.linalg.det(Rm) > 0


@pytest.mark.gpu
def test_point_map_from_depth_matches_oracle():
    """VGGT.point_map_from_depth (vx_unproject_depth on the decoded cameras) vs the oracle's
    per-pixel unprojection of the same depth and cameras."""
    from oracle import scene_ref
    from paper_2509_25191_b200.pose import pose_encoding_to_extri_intri
    from paper_2509_25191_b200.vggt import VGGT
    cfg = vggt_tiny()
    model = VGGT(cfg)
    out = model(synthetic_images(cfg, 3, 1).cuda())
    pts = model.point_map_from_depth(out)
    assert pts.shape == (1, 3, cfg.img_size, cfg.img_size, 3)
    ext, K = pose_encoding_to_extri_intri(out["pose_enc"][0].float(), (cfg.img_size, cfg.img_size))
    ref = scene_ref.unproject_depth_maps(out["depth"][0, ..., 0].cpu().double().numpy(), ext.cpu().double().numpy(),
                                         K.cpu().double().numpy())
    got = pts[0].cpu().double().numpy()
    assert np.abs(got - ref).max() < 1e-4 * max(1.0, np.abs(ref).max())


@pytest.mark.gpu
def test_sharded_embed_matches_global_slice():
    """A frame shard that does not own global frame 0 (ranks > 0 under torchrun) embeds its views
    exactly like the same views of the whole batch (camera/register tokens index 1)."""
    from paper_2509_25191_b200.aggregator import DeviceWeights, alloc_workspace, embed
    cfg = vggt_tiny()
    W = DeviceWeights(make_state_dict(cfg, 0), cfg, torch.device("cuda"))
    imgs = synthetic_images(cfg, 6, 1).cuda()
    ws_all = alloc_workspace(cfg, 6)
    embed(W, imgs, ws_all, frame0_is_first=True)
    ws_shard = alloc_workspace(cfg, 3)
    embed(W, imgs[2:5].contiguous(), ws_shard, frame0_is_first=False)
    N = cfg.tokens_per_frame
    assert torch.equal(ws_shard.x[: 3 * N], ws_all.x[2 * N:5 * N])
    ws_head = alloc_workspace(cfg, 2)
    embed(W, imgs[:2].contiguous(), ws_head, frame0_is_first=True)
    assert torch.equal(ws_head.x[: 2 * N], ws_all.x[: 2 * N])


def test_vggt1b_eight_views():
    """VGGT-1B-shaped, S = 8: global attention has 16 x 22 = 352 work units (2 waves + 56), so its
    last wave runs KV-split, inside a full forward against the oracle."""
    cfg = vggt_1b()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 8, 3)
    _check(cfg, sd, images, _oracle(cfg, sd, images), "1b-s8")
