"""CPU fp32 oracle of the VGGT-X dense-view inference path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module,
and only as the checker / the timed CPU baseline.  The product package
(`paper_2509_25191_b200`) never imports it.

Parity status: UNPINNED against the reference.  `/root/reference` contains no
implementation of this path (`SPEC.md:12`, `SPEC.md:630`) and
no test pins any numeric VGGT output.  This file is a
from-scratch restatement of the upstream `vggt` architecture as frozen in
SURVEY.md Appendix A, with the VGGT-X modifications the paper describes:

  * `PAPER.md:79`  only the outputs of layers {4, 11, 17, 23} are kept
                   (`Aggregator.forward` returns a dict of kept layers);
  * `PAPER.md:81`  frame-wise work may be chunked into ceil(N/S) chunks
                   (`frame_chunk`), which must not change the result;
  * `PAPER.md:146` chunk S = 128.

Partial external anchors (tests/test_oracle_anchors.py): `dinov2_patch_tokens` equals the
`transformers` Dinov2WithRegistersModel, `_fusion` / `_rcu` its DPTFeatureFusionLayer and `_reassemble`
(without the UV pos-embed VGGT adds) its DPTReassembleLayer on shared random weights; nothing pins the
VGGT-specific parts (2D RoPE, q/k LayerNorm, camera head, UV pos-embed).

Everything runs in fp32 on the CPU with the seeded weights from
`paper_2509_25191_b200.weights` (matrix weights already bf16-representable).
The conventions reused from the reference are the world-to-camera extrinsic
(`pkg/src/epialign/geometry.py:5-8`) and the rotation-angle metric
(`pkg/src/epialign/geometry.py:280-283`, `metrics.py:111`), see `pose_errors`.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import torch
import torch.nn.functional as F

from paper_2509_25191_b200.config import VGGTConfig

RESNET_MEAN = (0.485, 0.456, 0.406)
RESNET_STD = (0.229, 0.224, 0.225)


# --------------------------------------------------------------------------
# elementary ops
# --------------------------------------------------------------------------
def layer_norm(x, w, b, eps):
    return F.layer_norm(x, (x.shape[-1],), w, b, eps)


def linear(x, sd, name):
    b = sd.get(name + ".bias")
    return F.linear(x, sd[name + ".weight"], b)


def positions(cfg: VGGTConfig) -> torch.Tensor:
    """a4: (y, x) patch grid + 1, special tokens at (0, 0); (P, 2) int64."""
    g = cfg.grid
    ys, xs = torch.meshgrid(torch.arange(g), torch.arange(g), indexing="ij")
    pos = torch.stack([ys.reshape(-1), xs.reshape(-1)], dim=-1) + 1
    special = torch.zeros(cfg.patch_start_idx, 2, dtype=torch.long)
    return torch.cat([special, pos], dim=0)


def rope_tables(head_dim: int, max_pos: int, freq: float):
    """a4: cos/sin tables (max_pos, head_dim/2) for one half of the head."""
    half = head_dim // 2
    exponents = torch.arange(0, half, 2, dtype=torch.float32) / half
    inv_freq = 1.0 / (freq ** exponents)
    ang = torch.arange(max_pos, dtype=torch.float32)[:, None] * inv_freq[None, :]
    ang = torch.cat([ang, ang], dim=-1)
    return ang.cos(), ang.sin()


def rope_2d(x: torch.Tensor, pos: torch.Tensor, freq: float) -> torch.Tensor:
    """x (..., T, d); pos (T, 2).  Vertical half uses y, horizontal half uses x."""
    d = x.shape[-1]
    cos, sin = rope_tables(d, int(pos.max()) + 1, freq)

    def one(v, p):
        c, s = cos[p], sin[p]
        h = v.shape[-1] // 2
        rot = torch.cat([-v[..., h:], v[..., :h]], dim=-1)
        return v * c + rot * s

    vert, hori = x.chunk(2, dim=-1)
    return torch.cat([one(vert, pos[:, 0]), one(hori, pos[:, 1])], dim=-1)


def attention(x, sd, name, num_heads, eps, pos=None, freq=100.0, qk_norm=True):
    """a6-a9 without the residual: qkv -> qk-LN -> RoPE -> SDPA -> proj.

    x: (B, T, C)
    """
    B, T, C = x.shape
    d = C // num_heads
    qkv = linear(x, sd, name + ".qkv").reshape(B, T, 3, num_heads, d).permute(2, 0, 3, 1, 4)
    q, k, v = qkv.unbind(0)
    if qk_norm:
        q = layer_norm(q, sd[name + ".q_norm.weight"], sd[name + ".q_norm.bias"], eps)
        k = layer_norm(k, sd[name + ".k_norm.weight"], sd[name + ".k_norm.bias"], eps)
    if pos is not None:
        q = rope_2d(q, pos, freq)
        k = rope_2d(k, pos, freq)
    o = F.scaled_dot_product_attention(q, k, v)
    o = o.transpose(1, 2).reshape(B, T, C)
    return linear(o, sd, name + ".proj")


def block(x, sd, name, num_heads, eps, pos=None, freq=100.0, qk_norm=True):
    """Pre-norm transformer block (a5-a10): x + ls1*attn(norm1 x); + ls2*mlp(norm2 x)."""
    h = layer_norm(x, sd[name + ".norm1.weight"], sd[name + ".norm1.bias"], eps)
    h = attention(h, sd, name + ".attn", num_heads, eps, pos, freq, qk_norm)
    x = x + sd[name + ".ls1.gamma"] * h
    h = layer_norm(x, sd[name + ".norm2.weight"], sd[name + ".norm2.bias"], eps)
    h = F.gelu(linear(h, sd, name + ".mlp.fc1"))
    h = linear(h, sd, name + ".mlp.fc2")
    return x + sd[name + ".ls2.gamma"] * h


# --------------------------------------------------------------------------
# Aggregator (a1-a3, a11, a16)
# --------------------------------------------------------------------------
def patch_embed(images, sd, cfg):
    """a1 + a2: ResNet normalisation then conv 14x14/14 (== im2col GEMM), or (a2') the DINOv2 encoder."""
    mean = torch.tensor(RESNET_MEAN).view(1, 3, 1, 1)
    std = torch.tensor(RESNET_STD).view(1, 3, 1, 1)
    x = (images - mean) / std
    if cfg.patch_embed == "dinov2":
        return dinov2_patch_tokens(x, sd, cfg)
    x = F.conv2d(x, sd["aggregator.patch_embed.proj.weight"], sd["aggregator.patch_embed.proj.bias"],
                 stride=cfg.patch_size)
    return x.flatten(2).transpose(1, 2)  # (S, P, C)


def dino_pos_embed(pos_embed, grid: int):
    """DINOv2 interpolate_pos_encoding for square inputs (upstream dinov2 vision_transformer, as built by
    the VGGT aggregator: bicubic, antialias, interpolate_offset 0): the stored (1, 1 + M*M, C) table
    unchanged when M == grid, else the patch part resized to grid x grid."""
    N = pos_embed.shape[1] - 1
    if N == grid * grid:
        return pos_embed
    M = int(math.sqrt(N))
    C = pos_embed.shape[-1]
    pos = pos_embed.float()
    patch = F.interpolate(pos[:, 1:].reshape(1, M, M, C).permute(0, 3, 1, 2), size=(grid, grid), mode="bicubic",
                          antialias=True)
    return torch.cat([pos[:, :1], patch.permute(0, 2, 3, 1).reshape(1, grid * grid, C)], dim=1)


def dinov2_patch_tokens(x, sd, cfg):
    """a2': DINOv2 ViT-L/14-reg forward_features -> x_norm_patchtokens (S, P, C).

    conv patch embed; cls token + (interpolated) learned position embedding; 4 register tokens inserted
    after cls (no position embedding); `dino_depth` pre-norm blocks (LayerNorm eps 1e-6, no RoPE, no
    qk-norm, LayerScale); final LayerNorm; patch tokens only."""
    d_ = "aggregator.patch_embed."
    S = x.shape[0]
    C = cfg.embed_dim
    t = F.conv2d(x, sd[d_ + "patch_embed.proj.weight"], sd[d_ + "patch_embed.proj.bias"], stride=cfg.patch_size)
    t = t.flatten(2).transpose(1, 2)
    t = torch.cat([sd[d_ + "cls_token"].expand(S, 1, C), t], dim=1) + dino_pos_embed(sd[d_ + "pos_embed"], cfg.grid)
    t = torch.cat([t[:, :1], sd[d_ + "register_tokens"].expand(S, -1, C), t[:, 1:]], dim=1)
    for i in range(cfg.dino_depth):
        t = block(t, sd, f"{d_}blocks.{i}", cfg.num_heads, cfg.dino_eps, None, qk_norm=False)
    t = layer_norm(t, sd[d_ + "norm.weight"], sd[d_ + "norm.bias"], cfg.dino_eps)
    return t[:, 1 + cfg.num_register_tokens:]


def special_tokens(sd, cfg, S):
    """a3: camera (1) + register (R) tokens; index 0 for frame 0, 1 for the rest."""
    cam = sd["aggregator.camera_token"][0]     # (2, 1, C)
    reg = sd["aggregator.register_token"][0]   # (2, R, C)
    idx = torch.ones(S, dtype=torch.long)
    idx[0] = 0
    return torch.cat([cam[idx], reg[idx]], dim=1)  # (S, 1+R, C)


def aggregator(images, sd, cfg: VGGTConfig, frame_chunk: Optional[int] = None,
               keep_all: bool = False) -> Dict[int, torch.Tensor]:
    """Returns {layer: (S, T, 2C)} for kept layers (all layers if keep_all).

    `frame_chunk` evaluates the frame blocks ceil(S/chunk) frames at a time
    (VGGT-X chunking, `PAPER.md:81`); results must not depend on it.
    """
    S = images.shape[0]
    T = cfg.tokens_per_frame
    C = cfg.embed_dim
    x = torch.cat([special_tokens(sd, cfg, S), patch_embed(images, sd, cfg)], dim=1)  # (S, T, C)
    pos = positions(cfg)
    gpos = pos.repeat(S, 1)
    keep = set(range(cfg.depth)) if keep_all else set(cfg.kept_layers)
    out = {}
    chunk = frame_chunk or S
    for i in range(cfg.depth):
        fb = f"aggregator.frame_blocks.{i}"
        parts = [block(x[s:s + chunk], sd, fb, cfg.num_heads, cfg.ln_eps, pos, cfg.rope_freq)
                 for s in range(0, S, chunk)]
        x = torch.cat(parts, dim=0)
        frame_out = x
        gb = f"aggregator.global_blocks.{i}"
        x = block(x.reshape(1, S * T, C), sd, gb, cfg.num_heads, cfg.ln_eps, gpos,
                  cfg.rope_freq).reshape(S, T, C)
        if i in keep:
            out[i] = torch.cat([frame_out, x], dim=-1)
    return out


# --------------------------------------------------------------------------
# Camera head (a12, a13)
# --------------------------------------------------------------------------
def activate_pose(enc):
    """trans linear, quat linear, fov relu (upstream absT_quaR_FoV)."""
    return torch.cat([enc[..., :7], F.relu(enc[..., 7:])], dim=-1)


def camera_head(tokens_last, sd, cfg: VGGTConfig) -> List[torch.Tensor]:
    """tokens_last: (S, T, 2C) kept layer depth-1 -> list of (S, 9) pose encodings."""
    D = 2 * cfg.embed_dim
    ch = "camera_head."
    tok = tokens_last[:, 0]  # camera token (S, D)
    tok = layer_norm(tok, sd[ch + "token_norm.weight"], sd[ch + "token_norm.bias"], cfg.ln_eps)
    S = tok.shape[0]
    pred = None
    outs = []
    for _ in range(cfg.cam_iters):
        # iteration 0 embeds the learnable (1, 1, 9) empty_pose_tokens (upstream CameraHead.forward)
        inp = sd[ch + "empty_pose_tokens"].reshape(1, 9).expand(S, 9) if pred is None else pred
        emb = linear(inp, sd, ch + "embed_pose")
        mod = linear(F.silu(emb), sd, ch + "poseLN_modulation.1")
        shift, scale, gate = mod.chunk(3, dim=-1)
        h = F.layer_norm(tok, (D,), None, None, 1e-6)
        h = gate * (h * (1 + scale) + shift) + tok
        h = h[None]
        for j in range(cfg.cam_trunk_depth):
            h = block(h, sd, f"{ch}trunk.{j}", cfg.cam_num_heads, cfg.ln_eps, None, qk_norm=False)
        h = h[0]
        h = layer_norm(h, sd[ch + "trunk_norm.weight"], sd[ch + "trunk_norm.bias"], cfg.ln_eps)
        delta = linear(F.gelu(linear(h, sd, ch + "pose_branch.fc1")), sd, ch + "pose_branch.fc2")
        pred = delta if pred is None else pred + delta
        outs.append(activate_pose(pred))
    return outs


def quat_to_mat(q):
    """XYZW quaternion -> rotation matrix (normalising)."""
    q = q / q.norm(dim=-1, keepdim=True)
    x, y, z, w = q.unbind(-1)
    return torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
        2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
        2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y),
    ], dim=-1).reshape(q.shape[:-1] + (3, 3))


def pose_encoding_to_extri_intri(enc, hw):
    """a13: (.., 9) -> extrinsic (.., 3, 4) world-to-camera, intrinsic (.., 3, 3)."""
    H, W = hw
    T = enc[..., :3]
    R = quat_to_mat(enc[..., 3:7])
    fov_h, fov_w = enc[..., 7], enc[..., 8]
    fy = (H / 2.0) / torch.tan(fov_h / 2.0)
    fx = (W / 2.0) / torch.tan(fov_w / 2.0)
    K = torch.zeros(enc.shape[:-1] + (3, 3), dtype=enc.dtype)
    K[..., 0, 0] = fx
    K[..., 1, 1] = fy
    K[..., 0, 2] = W / 2.0
    K[..., 1, 2] = H / 2.0
    K[..., 2, 2] = 1.0
    return torch.cat([R, T[..., None]], dim=-1), K


def pose_errors(enc, enc_ref):
    """Rotation angle (rad) and relative translation error per view.

    Angle: arccos((tr(R^T R_ref) - 1)/2) as `pkg/src/epialign/geometry.py:280-283`.
    Translation: |dt| / max(|t_ref|, mean |t_ref|).
    """
    R = quat_to_mat(enc[..., 3:7].double())
    Rr = quat_to_mat(enc_ref[..., 3:7].double())
    tr = (R.transpose(-1, -2) @ Rr).diagonal(dim1=-2, dim2=-1).sum(-1)
    ang = torch.arccos(((tr - 1) / 2).clamp(-1, 1))
    t, tref = enc[..., :3].double(), enc_ref[..., :3].double()
    nref = tref.norm(dim=-1)
    denom = torch.maximum(nref, nref.mean().expand_as(nref))
    return ang, (t - tref).norm(dim=-1) / denom


# --------------------------------------------------------------------------
# DPT head (a14)
# --------------------------------------------------------------------------
def _uv_grid(w, h, aspect):
    diag = (aspect ** 2 + 1.0) ** 0.5
    sx, sy = aspect / diag, 1.0 / diag
    xs = torch.linspace(-sx * (w - 1) / w, sx * (w - 1) / w, steps=w)
    ys = torch.linspace(-sy * (h - 1) / h, sy * (h - 1) / h, steps=h)
    uu, vv = torch.meshgrid(xs, ys, indexing="xy")
    return torch.stack([uu, vv], dim=-1)  # (h, w, 2)


def _sincos(dim, pos, omega0=100.0):
    omega = torch.arange(dim // 2, dtype=torch.float64) / (dim / 2.0)
    omega = 1.0 / omega0 ** omega
    out = pos.reshape(-1).double()[:, None] * omega[None]
    return torch.cat([out.sin(), out.cos()], dim=1).float()


def dpt_pos_embed(c, h, w, img_w, img_h, ratio=0.1):
    """UV sin/cos embedding (C, h, w) * 0.1 added to DPT feature maps."""
    uv = _uv_grid(w, h, img_w / img_h).reshape(-1, 2)
    emb = torch.cat([_sincos(c // 2, uv[:, 0]), _sincos(c // 2, uv[:, 1])], dim=-1)
    return (emb.reshape(h, w, c) * ratio).permute(2, 0, 1)


def _conv(x, sd, name, stride=1, padding=None):
    w = sd[name + ".weight"]
    pad = (w.shape[-1] // 2) if padding is None else padding
    return F.conv2d(x, w, sd.get(name + ".bias"), stride=stride, padding=pad)


def _rcu(x, sd, name):
    out = _conv(F.relu(x), sd, name + ".conv1")
    out = _conv(F.relu(out), sd, name + ".conv2")
    return out + x


def _fusion(sd, name, x0, x1=None, size=None):
    out = x0
    if x1 is not None:
        out = out + _rcu(x1, sd, name + ".resConfUnit1")
    out = _rcu(out, sd, name + ".resConfUnit2")
    if size is None:
        out = F.interpolate(out, scale_factor=2, mode="bilinear", align_corners=True)
    else:
        out = F.interpolate(out, size=size, mode="bilinear", align_corners=True)
    return _conv(out, sd, name + ".out_conv")


def _reassemble(x, sd, head, i, pos=None):
    """Kept layer i's token map (F, 2C, g, g) -> 1x1 projection (+ UV pos-embed) -> resize: ConvTranspose
    k = s = 4 (i = 0), k = s = 2 (i = 1), identity (i = 2), Conv 3x3 stride 2 (i = 3)."""
    x = _conv(x, sd, f"{head}projects.{i}", padding=0)
    if pos is not None:
        x = x + pos
    if i == 0:
        x = F.conv_transpose2d(x, sd[head + "resize_layers.0.weight"], sd[head + "resize_layers.0.bias"], stride=4)
    elif i == 1:
        x = F.conv_transpose2d(x, sd[head + "resize_layers.1.weight"], sd[head + "resize_layers.1.bias"], stride=2)
    elif i == 3:
        x = _conv(x, sd, head + "resize_layers.3", stride=2, padding=1)
    return x


def _dpt_chunk(layers, sd, head, cfg, img_hw):
    H, W = img_hw
    g = cfg.grid
    ps = cfg.patch_start_idx
    feats = []
    for i, x in enumerate(layers):
        x = x[:, ps:]
        x = layer_norm(x, sd[head + "norm.weight"], sd[head + "norm.bias"], cfg.ln_eps)
        x = x.permute(0, 2, 1).reshape(x.shape[0], -1, g, g)
        feats.append(_reassemble(x, sd, head, i, dpt_pos_embed(cfg.dpt_out_channels[i], g, g, W, H)))
    sc = head + "scratch."
    l1, l2, l3, l4 = [_conv(f, sd, f"{sc}layer{i + 1}_rn") for i, f in enumerate(feats)]
    out = _fusion(sd, sc + "refinenet4", l4, None, size=l3.shape[2:])
    out = _fusion(sd, sc + "refinenet3", out, l3, size=l2.shape[2:])
    out = _fusion(sd, sc + "refinenet2", out, l2, size=l1.shape[2:])
    out = _fusion(sd, sc + "refinenet1", out, l1, size=None)
    out = _conv(out, sd, sc + "output_conv1")
    out = F.interpolate(out, size=(H, W), mode="bilinear", align_corners=True)
    out = out + dpt_pos_embed(out.shape[1], H, W, W, H)
    out = F.relu(_conv(out, sd, sc + "output_conv2.0"))
    out = _conv(out, sd, sc + "output_conv2.2", padding=0)
    return out.permute(0, 2, 3, 1)  # (S, H, W, odim)


def dpt_head(kept: Dict[int, torch.Tensor], sd, cfg, head: str, activation: str,
             img_hw, chunk: Optional[int] = None):
    """a14: returns (preds (S,H,W,odim-1), conf (S,H,W)); frame-chunked."""
    layers = [kept[i] for i in cfg.kept_layers]
    S = layers[0].shape[0]
    chunk = chunk or S
    outs = [_dpt_chunk([l[s:s + chunk] for l in layers], sd, head, cfg, img_hw)
            for s in range(0, S, chunk)]
    fmap = torch.cat(outs, dim=0)
    xyz, conf = fmap[..., :-1], fmap[..., -1]
    if activation == "exp":
        pred = torch.exp(xyz)
    elif activation == "inv_log":
        pred = torch.sign(xyz) * torch.expm1(xyz.abs())
    else:
        raise ValueError(activation)
    return pred, 1 + conf.exp()


# --------------------------------------------------------------------------
# VGGT.forward (a15)
# --------------------------------------------------------------------------
@torch.no_grad()
def vggt_forward(images, sd, cfg: VGGTConfig, frame_chunk=None, head_chunk=None,
                 with_heads=True):
    """images (S,3,H,W) in [0,1] -> dict with the upstream VGGT output keys (B=1)."""
    images = images.float()
    kept = aggregator(images, sd, cfg, frame_chunk=frame_chunk)
    preds = {"kept": kept}
    if not with_heads:
        return preds
    hw = images.shape[-2:]
    pose_list = camera_head(kept[cfg.kept_layers[-1]], sd, cfg)
    preds["pose_enc"] = pose_list[-1][None]
    preds["pose_enc_list"] = [p[None] for p in pose_list]
    depth, dconf = dpt_head(kept, sd, cfg, "depth_head.", "exp", hw, head_chunk)
    pts, pconf = dpt_head(kept, sd, cfg, "point_head.", "inv_log", hw, head_chunk)
    preds["depth"] = depth[None]
    preds["depth_conf"] = dconf[None]
    preds["world_points"] = pts[None]
    preds["world_points_conf"] = pconf[None]
    preds["images"] = images[None]
    return preds


def forward_flops(cfg: VGGTConfig, S: int, with_heads: bool = True) -> float:
    """Algorithmic FLOPs of one forward."""
    N, C, L = cfg.tokens_per_frame, cfg.embed_dim, cfg.depth
    hid = cfg.mlp_hidden
    lin = 2 * N * (3 * C * C + C * C + 2 * C * hid)      # per view per block
    attn_frame = 4 * N * N * C
    attn_glob = 4 * S * N * N * C                          # per view
    patch = 2 * cfg.num_patches * cfg.patch_k * C
    f = S * (L * (2 * lin + attn_frame + attn_glob) + patch)
    if cfg.patch_embed == "dinov2":  # DINOv2 encoder blocks: frame-attention blocks (+1.01 TF/view)
        f += S * cfg.dino_depth * (lin + attn_frame)
    if with_heads:
        f += 2 * S * dpt_flops(cfg)
    return float(f)


def dpt_flops(cfg: VGGTConfig) -> float:
    g = cfg.grid
    D = 2 * cfg.embed_dim
    Fh = cfg.dpt_features
    oc = cfg.dpt_out_channels
    H = W = cfg.img_size
    sizes = [4 * g, 2 * g, g, (g + 1) // 2]
    f = 0
    for i in range(4):
        f += 2 * g * g * D * oc[i]
    f += 2 * g * g * oc[0] * oc[0] * 16 + 2 * g * g * oc[1] * oc[1] * 4
    f += 2 * sizes[3] ** 2 * oc[3] * oc[3] * 9
    for i in range(4):
        f += 2 * sizes[i] ** 2 * oc[i] * Fh * 9
    rcu = lambda s: 2 * 2 * s * s * Fh * Fh * 9
    f += rcu(sizes[3]) + sum(2 * rcu(sizes[i]) for i in range(3))
    outs = [sizes[2], sizes[1], sizes[0], 2 * sizes[0]]
    f += sum(2 * s * s * Fh * Fh for s in outs)
    f += 2 * (2 * sizes[0]) ** 2 * Fh * (Fh // 2) * 9
    f += 2 * H * W * (Fh // 2) * cfg.dpt_head_features_2 * 9
    return float(f)
