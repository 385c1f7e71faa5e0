"""External anchors for parts of the oracle (CPU).

The reference ships no implementation of the VGGT path, so the oracle
(oracle/vggt_ref.py) is a restatement.  Where an independent implementation of the same published
module is installed in this image, the restatement is checked against it on shared random weights:

  * DINOv2 ViT/14 with registers (a2'): `transformers` Dinov2WithRegistersModel — token assembly
    (cls + position embedding, registers after cls), pre-norm blocks with LayerScale, final norm;
  * the DPT fusion block (a14): `transformers` DPTFeatureFusionLayer / DPTPreActResidualLayer —
    pre-activation residual conv units, skip add, x2 bilinear (align_corners=True), 1x1 projection;
  * the DPT reassembly of each kept layer (a14): `transformers` DPTReassembleLayer — 1x1 projection,
    then ConvTranspose k = s = 4 / 2, identity, or 3x3 stride-2 conv.

These pin the block structure (pre-norm attention / MLP with LayerScale, exact GELU, SDPA scaling)
and the DPT reassembly / fusion arithmetic the aggregator and heads share; the VGGT-specific parts
(2D RoPE, q/k LayerNorm, camera head, the DPT UV pos-embed) remain restated, not pinned.
"""
import pytest
import torch

from oracle import vggt_ref as R
from paper_2509_25191_b200.config import vggt_tiny
from paper_2509_25191_b200.weights import make_state_dict

transformers = pytest.importorskip("transformers")


def test_dinov2_restatement_matches_transformers():
    from transformers import Dinov2WithRegistersConfig, Dinov2WithRegistersModel
    cfg = vggt_tiny().with_(patch_embed="dinov2", dino_depth=2)
    C, H = cfg.embed_dim, cfg.num_heads
    sd = make_state_dict(cfg, 0)
    hc = Dinov2WithRegistersConfig(hidden_size=C, num_hidden_layers=cfg.dino_depth, num_attention_heads=H,
                                   mlp_ratio=4, image_size=cfg.img_size, patch_size=cfg.patch_size,
                                   num_register_tokens=cfg.num_register_tokens, layer_norm_eps=cfg.dino_eps,
                                   layerscale_value=1.0, hidden_act="gelu", qkv_bias=True,
                                   attn_implementation="eager")
    model = Dinov2WithRegistersModel(hc).eval()
    d_ = "aggregator.patch_embed."
    m = {
        "embeddings.cls_token": sd[d_ + "cls_token"],
        "embeddings.mask_token": sd[d_ + "mask_token"].reshape(1, C),
        "embeddings.register_tokens": sd[d_ + "register_tokens"],
        "embeddings.position_embeddings": sd[d_ + "pos_embed"],
        "embeddings.patch_embeddings.projection.weight": sd[d_ + "patch_embed.proj.weight"],
        "embeddings.patch_embeddings.projection.bias": sd[d_ + "patch_embed.proj.bias"],
        "layernorm.weight": sd[d_ + "norm.weight"],
        "layernorm.bias": sd[d_ + "norm.bias"],
    }
    for i in range(cfg.dino_depth):
        b, e = f"{d_}blocks.{i}.", f"encoder.layer.{i}."
        qw, kw, vw = sd[b + "attn.qkv.weight"].chunk(3, 0)
        qb, kb, vb = sd[b + "attn.qkv.bias"].chunk(3, 0)
        m.update({
            e + "norm1.weight": sd[b + "norm1.weight"], e + "norm1.bias": sd[b + "norm1.bias"],
            e + "attention.attention.query.weight": qw, e + "attention.attention.query.bias": qb,
            e + "attention.attention.key.weight": kw, e + "attention.attention.key.bias": kb,
            e + "attention.attention.value.weight": vw, e + "attention.attention.value.bias": vb,
            e + "attention.output.dense.weight": sd[b + "attn.proj.weight"],
            e + "attention.output.dense.bias": sd[b + "attn.proj.bias"],
            e + "layer_scale1.lambda1": sd[b + "ls1.gamma"],
            e + "norm2.weight": sd[b + "norm2.weight"], e + "norm2.bias": sd[b + "norm2.bias"],
            e + "mlp.fc1.weight": sd[b + "mlp.fc1.weight"], e + "mlp.fc1.bias": sd[b + "mlp.fc1.bias"],
            e + "mlp.fc2.weight": sd[b + "mlp.fc2.weight"], e + "mlp.fc2.bias": sd[b + "mlp.fc2.bias"],
            e + "layer_scale2.lambda1": sd[b + "ls2.gamma"],
        })
    missing, unexpected = model.load_state_dict(m, strict=False)
    assert not unexpected and not [k for k in missing if "pooler" not in k], (missing, unexpected)
    g = torch.Generator().manual_seed(3)
    x = torch.randn(3, 3, cfg.img_size, cfg.img_size, generator=g)  # already ResNet-normalised
    with torch.no_grad():
        want = model(pixel_values=x).last_hidden_state[:, 1 + cfg.num_register_tokens:]
        got = R.dinov2_patch_tokens(x, sd, cfg)
    assert got.shape == want.shape
    torch.testing.assert_close(got, want, rtol=2e-5, atol=2e-5)


@pytest.mark.parametrize("with_skip", [False, True])
def test_dpt_fusion_block_matches_transformers(with_skip):
    from transformers import DPTConfig
    from transformers.models.dpt.modeling_dpt import DPTFeatureFusionLayer
    Fh = 64
    hc = DPTConfig(fusion_hidden_size=Fh, use_batch_norm_in_fusion_residual=False)
    layer = DPTFeatureFusionLayer(hc, align_corners=True).eval()
    g = torch.Generator().manual_seed(4)
    name = "depth_head.scratch.refinenet1"
    sd = {}
    for u, hf in ((1, layer.residual_layer1), (2, layer.residual_layer2)):
        for c, conv in ((1, hf.convolution1), (2, hf.convolution2)):
            sd[f"{name}.resConfUnit{u}.conv{c}.weight"] = torch.randn(Fh, Fh, 3, 3, generator=g) / 24
            sd[f"{name}.resConfUnit{u}.conv{c}.bias"] = torch.randn(Fh, generator=g) * 0.1
            conv.weight.data.copy_(sd[f"{name}.resConfUnit{u}.conv{c}.weight"])
            conv.bias.data.copy_(sd[f"{name}.resConfUnit{u}.conv{c}.bias"])
    sd[name + ".out_conv.weight"] = torch.randn(Fh, Fh, 1, 1, generator=g) / 8
    sd[name + ".out_conv.bias"] = torch.randn(Fh, generator=g) * 0.1
    layer.projection.weight.data.copy_(sd[name + ".out_conv.weight"])
    layer.projection.bias.data.copy_(sd[name + ".out_conv.bias"])
    x0 = torch.randn(2, Fh, 9, 11, generator=g)
    x1 = torch.randn(2, Fh, 9, 11, generator=g) if with_skip else None
    with torch.no_grad():
        want = layer(x0, x1)
        got = R._fusion(sd, name, x0, x1, size=None)
    torch.testing.assert_close(got, want, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("i,factor", [(0, 4), (1, 2), (2, 1), (3, 0.5)])
def test_dpt_reassemble_matches_transformers(i, factor):
    """Projection + resize of kept layer i (VGGT adds a UV pos-embed between them; anchored without it)."""
    from transformers import DPTConfig
    from transformers.models.dpt.modeling_dpt import DPTReassembleLayer
    Cin, Co = 96, 64
    hc = DPTConfig(hidden_size=Cin)
    layer = DPTReassembleLayer(hc, channels=Co, factor=factor).eval()
    g = torch.Generator().manual_seed(10 + i)
    head = "depth_head."
    sd = {f"{head}projects.{i}.weight": torch.randn(Co, Cin, 1, 1, generator=g) / 10,
          f"{head}projects.{i}.bias": torch.randn(Co, generator=g) * 0.1}
    layer.projection.weight.data.copy_(sd[f"{head}projects.{i}.weight"])
    layer.projection.bias.data.copy_(sd[f"{head}projects.{i}.bias"])
    if factor != 1:
        kshape = (Co, Co, factor, factor) if factor > 1 else (Co, Co, 3, 3)
        sd[f"{head}resize_layers.{i}.weight"] = torch.randn(*kshape, generator=g) / 20
        sd[f"{head}resize_layers.{i}.bias"] = torch.randn(Co, generator=g) * 0.1
        layer.resize.weight.data.copy_(sd[f"{head}resize_layers.{i}.weight"])
        layer.resize.bias.data.copy_(sd[f"{head}resize_layers.{i}.bias"])
    x = torch.randn(2, Cin, 9, 9, generator=g)
    with torch.no_grad():
        torch.testing.assert_close(R._reassemble(x, sd, head, i), layer(x), rtol=1e-5, atol=1e-5)
