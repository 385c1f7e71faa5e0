"""Camera head and frame-chunked DPT heads on the device.

Precision policy ("bf16 except MLP in heads", `PAPER.md:81`):
  * camera-head trunk (4 blocks, dim 2C) and AdaLN modulation: bf16 GEMMs on the
    vx tcgen05 kernel with fp32 residual stream; the pose branch MLP, pose
    embedding and activation stay fp32;
  * DPT heads: LayerNorm + the four 1x1 projections run on the vx kernels
    (LN + tcgen05 GEMM, NHWC output); the conv / conv-transpose / bilinear
    stack runs in bf16 channels-last (cuDNN library kernels — a native
    implicit-GEMM conv is the next §8 row); bilinear resizes
    (+ fused pos-embed add) run on vx_upsample_bilinear; the final per-pixel
    1x1 output conv and the activations run in fp32.
  * heads are evaluated `head_chunk` frames at a time (VGGT-X chunking).
"""
from __future__ import annotations

import math
from typing import Dict, List

import torch
import torch.nn.functional as F

from . import ops
from .aggregator import DeviceWeights


# ---------------------------------------------------------------------------
# camera head
# ---------------------------------------------------------------------------
def _trunk_block(W: DeviceWeights, name: str, x: torch.Tensor, num_heads: int, eps: float):
    """Camera-trunk Block (no RoPE, no qk-norm) on fp32 residual x (S, D)."""
    S, D = x.shape
    d = D // num_heads
    xn = ops.layernorm(x, W[name + ".norm1.weight"], W[name + ".norm1.bias"], eps)
    qkv = ops.gemm(xn, W[name + ".attn.qkv.weight"], ops.EPI_BF16, bias=W[name + ".attn.qkv.bias"])
    q, k, v = qkv.view(S, 3, num_heads, d).permute(1, 2, 0, 3).unbind(0)
    # attention across the S camera tokens, head_dim 128: library SDPA (tiny: S x S per head)
    o = F.scaled_dot_product_attention(q[None], k[None], v[None])[0]
    o = o.permute(1, 0, 2).reshape(S, D).contiguous()
    ops.gemm(o, W[name + ".attn.proj.weight"], ops.EPI_RESID, bias=W[name + ".attn.proj.bias"], resid=x,
             gamma=W[name + ".ls1.gamma"])
    xn = ops.layernorm(x, W[name + ".norm2.weight"], W[name + ".norm2.bias"], eps)
    h = ops.gemm(xn, W[name + ".mlp.fc1.weight"], ops.EPI_GELU, bias=W[name + ".mlp.fc1.bias"])
    ops.gemm(h, W[name + ".mlp.fc2.weight"], ops.EPI_RESID, bias=W[name + ".mlp.fc2.bias"], resid=x,
             gamma=W[name + ".ls2.gamma"])
    return x


def activate_pose(enc: torch.Tensor) -> torch.Tensor:
    """absT_quaR_FoV: translation linear, quaternion linear, fov relu."""
    return torch.cat([enc[..., :7], F.relu(enc[..., 7:])], dim=-1)


def camera_head(W: DeviceWeights, cam_tokens: torch.Tensor) -> List[torch.Tensor]:
    """cam_tokens: (S, 2C) bf16/fp32 camera tokens of the last kept layer -> 4 x (S, 9) fp32."""
    cfg = W.cfg
    ch = "camera_head."
    eps = cfg.ln_eps
    S, D = cam_tokens.shape
    tok = ops.layernorm(cam_tokens, W[ch + "token_norm.weight"], W[ch + "token_norm.bias"], eps,
                        out_dtype=torch.float32)
    pred = None
    outs = []
    for _ in range(cfg.cam_iters):
        inp = torch.zeros(S, 9, device=tok.device) if pred is None else pred
        emb = F.linear(inp, W[ch + "embed_pose.weight"], W[ch + "embed_pose.bias"])
        mod = ops.gemm(F.silu(emb).to(torch.bfloat16), W[ch + "poseLN_modulation.1.weight"], ops.EPI_F32,
                       bias=W[ch + "poseLN_modulation.1.bias"])
        shift, scale, gate = mod.chunk(3, dim=-1)
        hn = ops.layernorm(tok, None, None, 1e-6, out_dtype=torch.float32)
        x = gate * (hn * (1 + scale) + shift) + tok
        x = x.contiguous()
        for j in range(cfg.cam_trunk_depth):
            _trunk_block(W, f"{ch}trunk.{j}", x, cfg.cam_num_heads, eps)
        xn = ops.layernorm(x, W[ch + "trunk_norm.weight"], W[ch + "trunk_norm.bias"], eps, out_dtype=torch.float32)
        hid = F.gelu(F.linear(xn, W[ch + "pose_branch.fc1.weight"], W[ch + "pose_branch.fc1.bias"]))
        delta = F.linear(hid, W[ch + "pose_branch.fc2.weight"], W[ch + "pose_branch.fc2.bias"])
        pred = delta if pred is None else pred + delta
        outs.append(activate_pose(pred))
    return outs


# ---------------------------------------------------------------------------
# DPT head
# ---------------------------------------------------------------------------
def _uv_grid(w, h, aspect):
    diag = (aspect ** 2 + 1.0) ** 0.5
    sx, sy = aspect / diag, 1.0 / diag
    xs = torch.linspace(-sx * (w - 1) / w, sx * (w - 1) / w, steps=w)
    ys = torch.linspace(-sy * (h - 1) / h, sy * (h - 1) / h, steps=h)
    uu, vv = torch.meshgrid(xs, ys, indexing="xy")
    return torch.stack([uu, vv], dim=-1)


def _sincos(dim, pos, omega0=100.0):
    omega = torch.arange(dim // 2, dtype=torch.float64) / (dim / 2.0)
    omega = 1.0 / omega0 ** omega
    out = pos.reshape(-1).double()[:, None] * omega[None]
    return torch.cat([out.sin(), out.cos()], dim=1).float()


def dpt_pos_embed(c, h, w, img_w, img_h, ratio=0.1):
    """(h, w, c) UV sin/cos embedding * ratio (channels-last)."""
    uv = _uv_grid(w, h, img_w / img_h).reshape(-1, 2)
    emb = torch.cat([_sincos(c // 2, uv[:, 0]), _sincos(c // 2, uv[:, 1])], dim=-1)
    return (emb.reshape(h, w, c) * ratio)


class DPTHeadDevice:
    def __init__(self, W: DeviceWeights, head: str, activation: str):
        self.W, self.head, self.activation = W, head, activation
        cfg = W.cfg
        dev = W.patch_w.device
        g = cfg.grid
        D = 2 * cfg.embed_dim
        H = Wd = cfg.img_size
        self.proj_w = [W[f"{head}projects.{i}.weight"].reshape(-1, D).contiguous() for i in range(4)]
        self.pos_small = [dpt_pos_embed(oc, g, g, Wd, H).to(dev) for oc in cfg.dpt_out_channels]
        self.pos_full = dpt_pos_embed(cfg.dpt_features // 2, H, Wd, Wd, H).to(dev).to(torch.bfloat16).contiguous()
        # bf16 channels-last conv weights
        self.cw = {}
        for k, v in W.t.items():
            if k.startswith(head) and v.dim() == 4 and "projects" not in k:
                if "output_conv2.2" in k:
                    self.cw[k] = v.float()
                else:
                    self.cw[k] = v.to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
        self.cb = {k: v for k, v in W.t.items() if k.startswith(head) and k.endswith(".bias")}

    def _conv(self, x, name, stride=1, padding=None, dtype=torch.bfloat16):
        w = self.cw[name + ".weight"]
        b = self.cb.get(name + ".bias")
        pad = (w.shape[-1] // 2) if padding is None else padding
        return F.conv2d(x, w, None if b is None else b.to(dtype), stride=stride, padding=pad)

    def _rcu(self, x, name):
        out = self._conv(F.relu(x), name + ".conv1")
        out = self._conv(F.relu(out), name + ".conv2")
        return out + x

    def _fusion(self, name, x0, x1=None, size=None):
        out = x0
        if x1 is not None:
            out = out + self._rcu(x1, name + ".resConfUnit1")
        out = self._rcu(out, name + ".resConfUnit2")
        h, w = out.shape[2:]
        size = (2 * h, 2 * w) if size is None else tuple(size)
        out = self._upsample(out, size)
        return self._conv(out, name + ".out_conv")

    @staticmethod
    def _upsample(x, size, add=None):
        """bilinear align_corners=True on channels-last bf16 via vx_upsample_bilinear."""
        nhwc = x.permute(0, 2, 3, 1)
        if not nhwc.is_contiguous():
            nhwc = nhwc.contiguous()
        return ops.upsample_bilinear(nhwc, size, add=add).permute(0, 3, 1, 2)

    def forward_chunk(self, layers: List[torch.Tensor]):
        """layers: 4 x (F, N, 2C) bf16 kept tokens -> (F, H, W, odim) fp32 pre-activation."""
        W, cfg, head = self.W, self.W.cfg, self.head
        g, ps = cfg.grid, cfg.patch_start_idx
        D = 2 * cfg.embed_dim
        Hh = Ww = cfg.img_size
        feats = []
        for i, x in enumerate(layers):
            Fr = x.shape[0]
            tok = x[:, ps:].reshape(Fr * g * g, D)
            xn = ops.layernorm(tok, W[head + "norm.weight"], W[head + "norm.bias"], cfg.ln_eps)
            y = ops.gemm(xn, self.proj_w[i], ops.EPI_BF16, bias=W[f"{head}projects.{i}.bias"])
            y = (y.view(Fr, g, g, -1) + self.pos_small[i].to(torch.bfloat16)).permute(0, 3, 1, 2)
            if i == 0:
                y = F.conv_transpose2d(y, self.cw[head + "resize_layers.0.weight"],
                                       self.cb[head + "resize_layers.0.bias"].to(torch.bfloat16), stride=4)
            elif i == 1:
                y = F.conv_transpose2d(y, self.cw[head + "resize_layers.1.weight"],
                                       self.cb[head + "resize_layers.1.bias"].to(torch.bfloat16), stride=2)
            elif i == 3:
                y = self._conv(y, head + "resize_layers.3", stride=2, padding=1)
            feats.append(y.contiguous(memory_format=torch.channels_last))
        sc = head + "scratch."
        l1, l2, l3, l4 = [self._conv(f, f"{sc}layer{i + 1}_rn") for i, f in enumerate(feats)]
        out = self._fusion(sc + "refinenet4", l4, None, size=l3.shape[2:])
        out = self._fusion(sc + "refinenet3", out, l3, size=l2.shape[2:])
        out = self._fusion(sc + "refinenet2", out, l2, size=l1.shape[2:])
        out = self._fusion(sc + "refinenet1", out, l1, size=None)
        out = self._conv(out, sc + "output_conv1")
        out = self._upsample(out, (Hh, Ww), add=self.pos_full)        # + UV pos-embed, fused
        out = F.relu(self._conv(out, sc + "output_conv2.0"))
        out = self._conv(out.float(), sc + "output_conv2.2", padding=0, dtype=torch.float32)
        return out.permute(0, 2, 3, 1)

    def __call__(self, kept: Dict[int, torch.Tensor], out_pred: torch.Tensor, out_conf: torch.Tensor,
                 chunk: int):
        cfg = self.W.cfg
        layers = [kept[i] for i in cfg.kept_layers]
        S = layers[0].shape[0]
        with torch.backends.cudnn.flags(enabled=True, allow_tf32=False):
            for s0 in range(0, S, chunk):
                s1 = min(S, s0 + chunk)
                fmap = self.forward_chunk([l[s0:s1] for l in layers])
                xyz, conf = fmap[..., :-1], fmap[..., -1]
                if self.activation == "exp":
                    out_pred[s0:s1] = torch.exp(xyz)
                else:
                    out_pred[s0:s1] = torch.sign(xyz) * torch.expm1(xyz.abs())
                out_conf[s0:s1] = 1 + conf.exp()
