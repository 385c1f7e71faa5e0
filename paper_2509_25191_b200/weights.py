"""Seeded random-init weights with the upstream `vggt` state_dict names.

There are no VGGT weights anywhere on disk, so every run uses
this deterministic init.  The state dict is generated on the CPU in fp32 and
the matrix weights (Linear / Conv) are rounded through bf16 once: the CPU
oracle computes with those values in fp32 and the CUDA path with the same
values in bf16, so weights are bit-identical between the two.
Parameters that stay fp32 on the device (LayerNorm, biases, LayerScale, special
tokens and the head "MLPs" VGGT-X keeps in fp32, `PAPER.md:81`) are not
rounded.

Init contract (oracle decision, documented in DESIGN.md):
  * Linear weights  N(0, 0.02) truncated at 2 sigma (upstream trunc_normal_).
  * biases / LN affine / LayerScale get small random perturbations so every
    epilogue term is exercised (upstream: zeros / ones / constant).
  * special tokens std 0.5 (upstream 1e-6) so they are on the patch scale.
  * CameraHead pose_branch.fc2 is scaled down and biased so that the decoded
    quaternion is well away from zero and the translation is non-trivial
    (SURVEY.md §7 "Decoded-pose tolerance with random weights").
"""
from __future__ import annotations

import zlib
from collections import OrderedDict

import torch

from .config import VGGTConfig

# parameters kept in fp32 on the device ("bf16 except MLP in heads")
FP32_PREFIXES = (
    "camera_head.pose_branch.",
    "camera_head.embed_pose.",
    "depth_head.scratch.output_conv2.2.",
    "point_head.scratch.output_conv2.2.",
)


def _gen(seed: int, name: str) -> torch.Generator:
    return torch.Generator().manual_seed(seed * 1000003 + zlib.crc32(name.encode()))


def _normal(shape, std, seed, name, mean=0.0, trunc=True):
    g = _gen(seed, name)
    t = torch.randn(shape, generator=g, dtype=torch.float32)
    if trunc:
        t.clamp_(-2.0, 2.0)
    return t.mul_(std).add_(mean)


def param_shapes(cfg: VGGTConfig) -> "OrderedDict[str, tuple]":
    """Upstream-named parameter shapes for aggregator + camera head + 2 DPT heads."""
    C, H = cfg.embed_dim, cfg.num_heads
    d = C // H
    hid = cfg.mlp_hidden
    P = cfg.patch_size
    s = OrderedDict()
    a = "aggregator."
    if cfg.patch_embed == "conv":
        s[a + "patch_embed.proj.weight"] = (C, 3, P, P)
        s[a + "patch_embed.proj.bias"] = (C,)
    else:  # DINOv2 ViT-L/14-reg (upstream vit_large as built by the VGGT aggregator)
        d_ = a + "patch_embed."
        s[d_ + "cls_token"] = (1, 1, C)
        s[d_ + "pos_embed"] = (1, 1 + cfg.num_patches, C)
        s[d_ + "register_tokens"] = (1, cfg.num_register_tokens, C)
        s[d_ + "mask_token"] = (1, C)
        s[d_ + "patch_embed.proj.weight"] = (C, 3, P, P)
        s[d_ + "patch_embed.proj.bias"] = (C,)
        for i in range(cfg.dino_depth):
            b = f"{d_}blocks.{i}."
            s[b + "norm1.weight"] = (C,)
            s[b + "norm1.bias"] = (C,)
            s[b + "attn.qkv.weight"] = (3 * C, C)
            s[b + "attn.qkv.bias"] = (3 * C,)
            s[b + "attn.proj.weight"] = (C, C)
            s[b + "attn.proj.bias"] = (C,)
            s[b + "ls1.gamma"] = (C,)
            s[b + "norm2.weight"] = (C,)
            s[b + "norm2.bias"] = (C,)
            s[b + "mlp.fc1.weight"] = (hid, C)
            s[b + "mlp.fc1.bias"] = (hid,)
            s[b + "mlp.fc2.weight"] = (C, hid)
            s[b + "mlp.fc2.bias"] = (C,)
            s[b + "ls2.gamma"] = (C,)
        s[d_ + "norm.weight"] = (C,)
        s[d_ + "norm.bias"] = (C,)
    s[a + "camera_token"] = (1, 2, 1, C)
    s[a + "register_token"] = (1, 2, cfg.num_register_tokens, C)
    for kind in ("frame_blocks", "global_blocks"):
        for i in range(cfg.depth):
            b = f"{a}{kind}.{i}."
            s[b + "norm1.weight"] = (C,)
            s[b + "norm1.bias"] = (C,)
            s[b + "attn.qkv.weight"] = (3 * C, C)
            s[b + "attn.qkv.bias"] = (3 * C,)
            s[b + "attn.q_norm.weight"] = (d,)
            s[b + "attn.q_norm.bias"] = (d,)
            s[b + "attn.k_norm.weight"] = (d,)
            s[b + "attn.k_norm.bias"] = (d,)
            s[b + "attn.proj.weight"] = (C, C)
            s[b + "attn.proj.bias"] = (C,)
            s[b + "ls1.gamma"] = (C,)
            s[b + "norm2.weight"] = (C,)
            s[b + "norm2.bias"] = (C,)
            s[b + "mlp.fc1.weight"] = (hid, C)
            s[b + "mlp.fc1.bias"] = (hid,)
            s[b + "mlp.fc2.weight"] = (C, hid)
            s[b + "mlp.fc2.bias"] = (C,)
            s[b + "ls2.gamma"] = (C,)
    # camera head (dim_in = 2C)
    D = 2 * C
    ch = "camera_head."
    s[ch + "token_norm.weight"] = (D,)
    s[ch + "token_norm.bias"] = (D,)
    s[ch + "trunk_norm.weight"] = (D,)
    s[ch + "trunk_norm.bias"] = (D,)
    s[ch + "empty_pose_tokens"] = (1, 1, 9)  # learnable iteration-0 input of embed_pose (upstream zeros)
    s[ch + "embed_pose.weight"] = (D, 9)
    s[ch + "embed_pose.bias"] = (D,)
    s[ch + "poseLN_modulation.1.weight"] = (3 * D, D)
    s[ch + "poseLN_modulation.1.bias"] = (3 * D,)
    s[ch + "pose_branch.fc1.weight"] = (D // 2, D)
    s[ch + "pose_branch.fc1.bias"] = (D // 2,)
    s[ch + "pose_branch.fc2.weight"] = (9, D // 2)
    s[ch + "pose_branch.fc2.bias"] = (9,)
    dh = int(D * cfg.mlp_ratio)
    for j in range(cfg.cam_trunk_depth):
        b = f"{ch}trunk.{j}."
        s[b + "norm1.weight"] = (D,)
        s[b + "norm1.bias"] = (D,)
        s[b + "attn.qkv.weight"] = (3 * D, D)
        s[b + "attn.qkv.bias"] = (3 * D,)
        s[b + "attn.proj.weight"] = (D, D)
        s[b + "attn.proj.bias"] = (D,)
        s[b + "ls1.gamma"] = (D,)
        s[b + "norm2.weight"] = (D,)
        s[b + "norm2.bias"] = (D,)
        s[b + "mlp.fc1.weight"] = (dh, D)
        s[b + "mlp.fc1.bias"] = (dh,)
        s[b + "mlp.fc2.weight"] = (D, dh)
        s[b + "mlp.fc2.bias"] = (D,)
        s[b + "ls2.gamma"] = (D,)
    # DPT heads
    F = cfg.dpt_features
    oc = cfg.dpt_out_channels
    for head, odim in (("depth_head.", 2), ("point_head.", 4)):
        s[head + "norm.weight"] = (D,)
        s[head + "norm.bias"] = (D,)
        for i in range(4):
            s[f"{head}projects.{i}.weight"] = (oc[i], D, 1, 1)
            s[f"{head}projects.{i}.bias"] = (oc[i],)
        s[head + "resize_layers.0.weight"] = (oc[0], oc[0], 4, 4)   # ConvTranspose2d (in, out, k, k)
        s[head + "resize_layers.0.bias"] = (oc[0],)
        s[head + "resize_layers.1.weight"] = (oc[1], oc[1], 2, 2)
        s[head + "resize_layers.1.bias"] = (oc[1],)
        s[head + "resize_layers.3.weight"] = (oc[3], oc[3], 3, 3)   # Conv2d stride 2
        s[head + "resize_layers.3.bias"] = (oc[3],)
        for i in range(4):
            s[f"{head}scratch.layer{i + 1}_rn.weight"] = (F, oc[i], 3, 3)
        for r in range(1, 5):
            rb = f"{head}scratch.refinenet{r}."
            units = (2,) if r == 4 else (1, 2)
            for u in units:
                for cv in (1, 2):
                    s[f"{rb}resConfUnit{u}.conv{cv}.weight"] = (F, F, 3, 3)
                    s[f"{rb}resConfUnit{u}.conv{cv}.bias"] = (F,)
            s[rb + "out_conv.weight"] = (F, F, 1, 1)
            s[rb + "out_conv.bias"] = (F,)
        s[head + "scratch.output_conv1.weight"] = (F // 2, F, 3, 3)
        s[head + "scratch.output_conv1.bias"] = (F // 2,)
        s[head + "scratch.output_conv2.0.weight"] = (cfg.dpt_head_features_2, F // 2, 3, 3)
        s[head + "scratch.output_conv2.0.bias"] = (cfg.dpt_head_features_2,)
        s[head + "scratch.output_conv2.2.weight"] = (odim, cfg.dpt_head_features_2, 1, 1)
        s[head + "scratch.output_conv2.2.bias"] = (odim,)
    return s


def _init_one(name: str, shape: tuple, cfg: VGGTConfig, seed: int) -> torch.Tensor:
    nd = len(shape)
    if name.endswith("camera_token") or name.endswith("register_token"):
        return _normal(shape, 0.5, seed, name, trunc=False)
    if name.endswith(("patch_embed.cls_token", "patch_embed.pos_embed", "patch_embed.register_tokens",
                      "patch_embed.mask_token")):
        return _normal(shape, 0.02, seed, name)
    if name == "camera_head.empty_pose_tokens":
        return torch.zeros(shape)  # upstream init; a trained checkpoint carries its own values
    if name.endswith(".gamma"):
        base = (cfg.cam_init_values if name.startswith("camera_head.") else
                cfg.dino_init_values if name.startswith("aggregator.patch_embed.") else cfg.init_values)
        return _normal(shape, 0.1 * base, seed, name, mean=base)
    if name == "camera_head.pose_branch.fc2.weight":
        return _normal(shape, 0.002, seed, name)
    if name == "camera_head.pose_branch.fc2.bias":
        # 4 refinement iterations accumulate ~4x this: t ~ (0.2,-0.2,1.0),
        # quat ~ (0,0,0,1) (XYZW), fov ~ 1 rad.
        return torch.tensor([0.05, -0.05, 0.25, 0.0, 0.0, 0.0, 0.25, 0.25, 0.25])
    if ".norm" in name or "_norm." in name or name.split(".")[-2].startswith("norm"):
        if name.endswith(".weight"):
            return _normal(shape, 0.05, seed, name, mean=1.0)
        return _normal(shape, 0.02, seed, name)
    if name.endswith(".bias"):
        return _normal(shape, 0.02, seed, name)
    if nd == 2:  # Linear
        return _normal(shape, 0.02, seed, name)
    if nd == 4:  # conv / conv-transpose / patch-embed
        if "patch_embed" in name:
            return _normal(shape, 0.02, seed, name)
        if "output_conv2.2" in name:
            fan_in = shape[1]
            return _normal(shape, 0.3 / fan_in ** 0.5, seed, name)
        if "resize_layers.0" in name or "resize_layers.1" in name:
            fan_in = shape[0]
        else:
            fan_in = shape[1] * shape[2] * shape[3]
        return _normal(shape, 1.0 / fan_in ** 0.5, seed, name)
    raise ValueError(name)


def is_bf16_param(name: str, shape: tuple) -> bool:
    if len(shape) < 2 or not name.endswith(".weight"):
        return False
    return not name.startswith(FP32_PREFIXES)


def check_state_dict(sd, cfg: VGGTConfig) -> None:
    """Every upstream-named parameter of this path must be present with its shape: a checkpoint that
    lacks one (e.g. camera_head.empty_pose_tokens) must not silently run with a made-up value."""
    missing = [k for k in param_shapes(cfg) if k not in sd]
    if missing:
        raise KeyError(f"state_dict lacks {len(missing)} parameter(s) of the VGGT path, e.g. {missing[:4]}")
    def ok(k, want):
        got = tuple(sd[k].shape)
        if k.endswith("patch_embed.pos_embed") and len(got) == 3:  # any square grid (interpolated at load)
            m = round((got[1] - 1) ** 0.5)
            return got[0] == 1 and m * m == got[1] - 1 and got[2] == want[2]
        return got == tuple(want)

    bad = [(k, tuple(sd[k].shape), s) for k, s in param_shapes(cfg).items() if not ok(k, s)]
    if bad:
        raise ValueError(f"state_dict shape mismatch: {bad[:4]}")


def make_state_dict(cfg: VGGTConfig, seed: int = 0) -> "OrderedDict[str, torch.Tensor]":
    """fp32 CPU state dict; bf16-device weights are already bf16-representable."""
    sd = OrderedDict()
    for name, shape in param_shapes(cfg).items():
        t = _init_one(name, shape, cfg, seed)
        assert tuple(t.shape) == tuple(shape), (name, t.shape, shape)
        if is_bf16_param(name, shape):
            t = t.to(torch.bfloat16).to(torch.float32)
        sd[name] = t.contiguous()
    return sd


def synthetic_images(cfg: VGGTConfig, num_views: int, seed: int = 1) -> torch.Tensor:
    """(S, 3, H, W) fp32 uniform [0, 1] views (SURVEY.md §8d synthetic inputs)."""
    g = torch.Generator().manual_seed(seed)
    return torch.rand(num_views, 3, cfg.img_size, cfg.img_size, generator=g)
