"""The DINOv2 patch embedding (SURVEY.md §8a a2', "DINO-based patch embedding"): what
upstream VGGT-1B checkpoints carry under aggregator.patch_embed.*.  The device path runs the encoder
in the aggregator's residual stream (aggregator.dinov2_encode); the oracle restates DINOv2's
forward_features (oracle/vggt_ref.py dinov2_patch_tokens).  Tolerances as the conv path's."""
import os

import pytest
import torch

from oracle import vggt_ref as R
from paper_2509_25191_b200.config import vggt_1b, vggt_small, vggt_tiny
from paper_2509_25191_b200.weights import check_state_dict, make_state_dict, param_shapes, synthetic_images


def _cfg(name):
    return {"tiny": vggt_tiny().with_(patch_embed="dinov2", dino_depth=2),
            "small": vggt_small().with_(patch_embed="dinov2", dino_depth=3),
            "1b": vggt_1b().with_(patch_embed="dinov2")}[name]


def test_dinov2_state_dict_names():
    cfg = _cfg("1b")
    shapes = param_shapes(cfg)
    assert shapes["aggregator.patch_embed.pos_embed"] == (1, 1 + 37 * 37, 1024)
    assert shapes["aggregator.patch_embed.register_tokens"] == (1, 4, 1024)
    assert shapes["aggregator.patch_embed.blocks.23.mlp.fc2.weight"] == (1024, 4096)
    assert "aggregator.patch_embed.proj.weight" not in shapes
    n = sum(torch.Size(s).numel() for k, s in shapes.items() if k.startswith("aggregator.patch_embed."))
    assert 300e6 < n < 310e6  # ViT-L/14: ~304M parameters


def test_dinov2_pos_embed_any_square_grid_accepted():
    cfg = _cfg("tiny")
    sd = make_state_dict(cfg, 0)
    sd["aggregator.patch_embed.pos_embed"] = torch.randn(1, 1 + 16 * 16, cfg.embed_dim)  # a 224-px table
    check_state_dict(sd, cfg)
    assert R.dino_pos_embed(sd["aggregator.patch_embed.pos_embed"], cfg.grid).shape == (1, 1 + 64, cfg.embed_dim)
    sd["aggregator.patch_embed.pos_embed"] = torch.randn(1, 1 + 15, cfg.embed_dim)
    with pytest.raises(ValueError):
        check_state_dict(sd, cfg)


def test_dinov2_oracle_depth0_is_normed_patch_embed():
    """With no encoder blocks the patch tokens are LayerNorm(conv(x) + pos[1:]) — the token assembly
    (cls / registers do not leak into patch rows)."""
    cfg = _cfg("tiny").with_(dino_depth=0)
    sd = make_state_dict(cfg, 0)
    img = synthetic_images(cfg, 2, 1)
    x = (img - torch.tensor(R.RESNET_MEAN).view(1, 3, 1, 1)) / torch.tensor(R.RESNET_STD).view(1, 3, 1, 1)
    d_ = "aggregator.patch_embed."
    t = torch.nn.functional.conv2d(x, sd[d_ + "patch_embed.proj.weight"], sd[d_ + "patch_embed.proj.bias"], stride=14)
    t = t.flatten(2).transpose(1, 2) + sd[d_ + "pos_embed"][:, 1:]
    want = torch.nn.functional.layer_norm(t, (cfg.embed_dim,), sd[d_ + "norm.weight"], sd[d_ + "norm.bias"], 1e-6)
    torch.testing.assert_close(R.patch_embed(img, sd, cfg), want)


def _rel(a, b):
    a, b = a.detach().float().cpu(), b.detach().float().cpu()
    return ((a - b).norm() / b.norm()).item()


@pytest.mark.gpu
@pytest.mark.parametrize("name,S,interp", [("tiny", 5, False), ("tiny", 3, True), ("small", 4, False),
                                           ("1b", 2, False)])
def test_dinov2_forward_matches_oracle(name, S, interp):
    from paper_2509_25191_b200.vggt import VGGT
    cfg = _cfg(name)
    sd = make_state_dict(cfg, 0)
    if interp:  # a checkpoint table for another resolution: bicubic interpolation at load
        g = torch.Generator().manual_seed(5)
        sd["aggregator.patch_embed.pos_embed"] = torch.randn(1, 1 + 16 * 16, cfg.embed_dim, generator=g) * 0.02
    images = synthetic_images(cfg, S, 1)
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    ref = R.vggt_forward(images, sd, cfg)
    m = VGGT(cfg, state_dict=sd)
    out = m(images.cuda())
    kept, _ = m.aggregator(images.cuda())
    rep = {f"kept{i}": _rel(kept[i][0], ref["kept"][i]) for i in cfg.kept_layers}
    rep.update({k: _rel(out[k], ref[k]) for k in ("depth", "depth_conf", "world_points", "world_points_conf")})
    ang, terr = R.pose_errors(out["pose_enc"][0].cpu(), ref["pose_enc"][0])
    rep["rot"], rep["trans"] = ang.max().item(), terr.max().item()
    print(name, S, interp, {k: f"{v:.2e}" for k, v in rep.items()})
    assert all(v <= 1e-2 for v in rep.values()), rep
