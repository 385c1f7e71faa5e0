"""Camera head and frame-chunked DPT heads on the device.

Precision policy ("bf16 except MLP in heads", `PAPER.md:81`):
  * camera-head trunk (4 blocks, dim 2C, attention across the S camera tokens
    with head_dim 128 on the vx FMHA) and AdaLN modulation: bf16 GEMMs on the
    vx tcgen05 kernel with fp32 residual stream; the pose branch MLP, pose
    embedding and activation stay fp32;
  * DPT heads: entirely on the vx kernels — LayerNorm, 1x1 projections,
    conv-transposes (GEMM + pixel shuffle), implicit-GEMM 3x3 convolutions with
    fused ReLU / residual / skip epilogues, bilinear resizes (+ fused pos-embed),
    bf16 NHWC activations; the final per-pixel 1x1 output conv and the
    activations run in fp32 inside the last conv's epilogue.
  * heads are evaluated `head_chunk` frames at a time (VGGT-X chunking).
"""
from __future__ import annotations

from typing import Dict, List

import torch
import torch.nn.functional as F

from . import ops
from .aggregator import DeviceWeights


# ---------------------------------------------------------------------------
# camera head
# ---------------------------------------------------------------------------
def _trunk_block(W: DeviceWeights, name: str, x: torch.Tensor, num_heads: int, eps: float):
    """Camera-trunk Block (no RoPE, no qk-norm) on fp32 residual x (S, D), in place.

    The qkv GEMM epilogue scatters q/k/v head-major ([H, S, d], d = 128) for the vx FMHA, which
    attends across the S camera tokens (attention across frames)."""
    S, D = x.shape
    d = D // num_heads
    dev = x.device
    xn = ops.layernorm(x, W[name + ".norm1.weight"], W[name + ".norm1.bias"], eps)
    q, k, v = (torch.empty(num_heads, S, d, device=dev, dtype=torch.bfloat16) for _ in range(3))
    ops.gemm(xn, W[name + ".attn.qkv.weight"], ops.EPI_QKV, bias=W[name + ".attn.qkv.bias"], qkv=(q, k, v),
             head_dim=d, tokens_total=S)
    o = torch.empty(S, D, device=dev, dtype=torch.bfloat16)
    ops.attention(q, k, v, o, nseq=1, Lq=S, Lk=S)
    ops.gemm(o, W[name + ".attn.proj.weight"], ops.EPI_RESID, bias=W[name + ".attn.proj.bias"], resid=x,
             gamma=W[name + ".ls1.gamma"])
    xn = ops.layernorm(x, W[name + ".norm2.weight"], W[name + ".norm2.bias"], eps)
    h = ops.gemm(xn, W[name + ".mlp.fc1.weight"], ops.EPI_GELU, bias=W[name + ".mlp.fc1.bias"])
    ops.gemm(h, W[name + ".mlp.fc2.weight"], ops.EPI_RESID, bias=W[name + ".mlp.fc2.bias"], resid=x,
             gamma=W[name + ".ls2.gamma"])
    return x


def activate_pose(enc: torch.Tensor) -> torch.Tensor:
    """absT_quaR_FoV: translation linear, quaternion linear, fov relu (host reference of the
    VX_LF_POSE epilogue; used by the pose tools, not on the forward path)."""
    return torch.cat([enc[..., :7], F.relu(enc[..., 7:])], dim=-1)


def camera_head(W: DeviceWeights, cam_tokens: torch.Tensor) -> List[torch.Tensor]:
    """cam_tokens: (S, 2C) bf16/fp32 camera tokens of the last kept layer -> 4 x (S, 9) fp32.

    Upstream CameraHead.forward / trunk_fn: every iteration embeds the previous
    pose encoding (iteration 0: the learnable `empty_pose_tokens`), modulates the normalised camera
    tokens (AdaLN: shift / scale / gate), runs the 4-block trunk with attention across the S views,
    and adds the pose-branch delta.  All on libvx: fp32 SIMT linears for the pose embedding and the
    pose-branch MLP (kept fp32), the bf16 tcgen05 GEMM for the modulation and the trunk.
    """
    cfg = W.cfg
    ch = "camera_head."
    eps = cfg.ln_eps
    S, D = cam_tokens.shape
    dev = cam_tokens.device
    tok = ops.layernorm(cam_tokens, W[ch + "token_norm.weight"], W[ch + "token_norm.bias"], eps,
                        out_dtype=torch.float32)
    empty = W[ch + "empty_pose_tokens"].reshape(1, 9).expand(S, 9)
    pred = None
    outs = []
    for _ in range(cfg.cam_iters):
        emb = ops.linear_f32(empty if pred is None else pred, W[ch + "embed_pose.weight"], W[ch + "embed_pose.bias"],
                             ops.LF_SILU_BF16)
        mod = ops.gemm(emb, W[ch + "poseLN_modulation.1.weight"], ops.EPI_F32, bias=W[ch + "poseLN_modulation.1.bias"])
        x = ops.adaln_modulate(tok, mod, 1e-6)
        for j in range(cfg.cam_trunk_depth):
            _trunk_block(W, f"{ch}trunk.{j}", x, cfg.cam_num_heads, eps)
        xn = ops.layernorm(x, W[ch + "trunk_norm.weight"], W[ch + "trunk_norm.bias"], eps, out_dtype=torch.float32)
        hid = ops.linear_f32(xn, W[ch + "pose_branch.fc1.weight"], W[ch + "pose_branch.fc1.bias"], ops.LF_GELU)
        new = torch.empty(S, 9, device=dev, dtype=torch.float32)
        act = torch.empty(S, 9, device=dev, dtype=torch.float32)
        ops.linear_f32(hid, W[ch + "pose_branch.fc2.weight"], W[ch + "pose_branch.fc2.bias"], ops.LF_POSE, out=new,
                       prev=pred, act_out=act)
        pred = new
        outs.append(act)
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
    """Frame-chunked DPT head on the vx kernels (no library convolutions).

    Per chunk of F views: LayerNorm + 1x1 projections (+ UV pos-embed fused) ->
    conv-transpose as GEMM + pixel-shuffle epilogue (k4/s4, k2/s2), identity, 3x3/s2
    conv -> 3x3 layer_rn convs -> 4 fusion blocks (RCU = two implicit-GEMM 3x3 convs
    with ReLU / residual / skip adds fused in the epilogues, bilinear upsample, 1x1
    out_conv) -> 3x3 output_conv1 -> bilinear to H x W + pos-embed -> fused
    [3x3 conv -> ReLU -> fp32 1x1 -> exp / inv_log / expp1] writing the final maps.
    Activations are bf16 NHWC; 3x3-conv inputs live in zero-bordered buffers.
    """

    def __init__(self, W: DeviceWeights, head: str, activation: str):
        self.W, self.head, self.activation = W, head, activation
        self._bufs: Dict[tuple, torch.Tensor] = {}  # zero-bordered activation buffers, see _pad / prepare
        self._prepared = False
        self._zeroed = False
        self._dirty = False
        self._overlay: set = set()
        self._under_overlay: List[tuple] = []
        cfg = W.cfg
        dev = W.patch_w.device
        g = cfg.grid
        D = 2 * cfg.embed_dim
        H = Wd = cfg.img_size
        oc = cfg.dpt_out_channels
        bf = torch.bfloat16

        def conv_w(name):  # [out, in, 3, 3] -> [out, 9*in], K order (ky, kx, cin)
            w = W[name + ".weight"]
            return w.permute(0, 2, 3, 1).reshape(w.shape[0], -1).to(bf).contiguous()

        def lin_w(name):
            w = W[name + ".weight"]
            return w.reshape(w.shape[0], -1).to(bf).contiguous()

        def convT_w(name):  # [in, out, s, s] -> [(i*s + j)*out + c, in]
            w = W[name + ".weight"]
            return w.permute(2, 3, 1, 0).reshape(-1, w.shape[0]).to(bf).contiguous()

        self.b = {k: v.float().contiguous() for k, v in W.t.items() if k.startswith(head) and k.endswith(".bias")}
        self.proj_w = [lin_w(f"{head}projects.{i}") for i in range(4)]
        self.pos_small = [dpt_pos_embed(c, g, g, Wd, H).to(dev, bf).contiguous() for c in oc]
        self.pos_full = dpt_pos_embed(cfg.dpt_features // 2, H, Wd, Wd, H).to(dev, bf).contiguous()
        self.convT = [convT_w(head + "resize_layers.0"), convT_w(head + "resize_layers.1")]
        self.cw = {}
        for k in W.t:
            if k.startswith(head) and k.endswith(".weight") and W.t[k].dim() == 4:
                name = k[: -len(".weight")]
                if W.t[k].shape[-1] == 3:
                    self.cw[name] = conv_w(name)
                elif "out_conv" in name:
                    self.cw[name] = lin_w(name)
        hw = W[head + "scratch.output_conv2.2.weight"]
        self.head_w = hw.reshape(hw.shape[0], -1).float().contiguous()
        self.head_b = W[head + "scratch.output_conv2.2.bias"].float().contiguous()

    def buffer_plan(self) -> List[tuple]:
        """The (slot, H, W, C) of every zero-bordered buffer forward_chunk uses (see _pad)."""
        cfg = self.W.cfg
        g, oc, Fh, img = cfg.grid, cfg.dpt_out_channels, cfg.dpt_features, cfg.img_size
        sizes = [4 * g, 2 * g, g, (g + 1) // 2]
        sc = self.head + "scratch."
        plan = [("f0", sizes[0], sizes[0], oc[0]), ("f1", sizes[1], sizes[1], oc[1]), ("f2", g, g, oc[2]),
                ("y3", g, g, oc[3]), ("f3", sizes[3], sizes[3], oc[3])]
        plan += [(f"{n}{i}", sizes[i], sizes[i], Fh) for i in range(4) for n in ("l", "lr")]
        plan.append((f"{sc}refinenet4.resConfUnit2.h", sizes[3], sizes[3], Fh))
        for r, li in ((3, 2), (2, 1), (1, 0)):
            hs = sizes[li]
            plan += [(f"{sc}refinenet{r}.resConfUnit1.{n}", hs, hs, Fh) for n in ("h", "o", "o2")]
            plan.append((f"{sc}refinenet{r}.resConfUnit2.h", hs, hs, Fh))
        plan += [("oc1", 2 * sizes[0], 2 * sizes[0], Fh), ("u", img, img, Fh // 2)]
        return plan

    # buffers laid over others (see prepare): refinenet1's residual units run when every buffer of the
    # projections, layer_rn (but layer 1's) and refinenets 2-4 is dead; the last two buffers of a chunk
    # (oc1: refinenet1's output on the 296 grid, u: the output head's 518-grid input) when all are
    TAIL_SLOTS = ("oc1", "u")

    def _overlay_groups(self):
        sc = self.head + "scratch."
        rn1 = tuple(f"{sc}refinenet1.resConfUnit1.{n}" for n in ("h", "o", "o2")) + (f"{sc}refinenet1.resConfUnit2.h",)
        return rn1, self.TAIL_SLOTS

    def prepare(self, frames: int, dev) -> None:
        """Allocate this forward's zero-bordered buffers for chunks of up to `frames` views from the
        CURRENT stream's pool. VGGT.forward calls this on the main stream before the head streams wait on
        it and `release()`s after the main stream has waited for them, so the memory returns to the main
        stream's pool and the next forward's aggregator reuses it; nothing is held between forwards.

        One arena per head, laid out by liveness within a chunk: region 1 holds layer_rn 1's outputs (l0,
        lr0: read by refinenet1, the last fusion block), region 2 every other body buffer (projections,
        layer_rn 2-4, refinenets 2-4), refinenet1's residual-unit buffers sit over region 2 (all dead when
        refinenet1 runs), and the two tail buffers over everything from offset 0 (oc1 is consumed before
        u is written). 1B shape, 16-view chunks: 1.1 GB per head instead of 3.7 for separate buffers.
        Borders: all are zeroed by the head's first call on its own stream; an overlaid buffer's border
        is re-zeroed right before its producer writes it, and the buffers under an overlay get theirs
        re-zeroed at the start of the next chunk (the producing kernels overwrite every interior).
        """
        plan = self.buffer_plan()
        align = 512  # bf16 elements (1 KB)
        n_of = lambda H, W, C: -(-(frames * (H + 2) * (W + 2) * C) // align) * align  # noqa: E731
        rn1, tail = self._overlay_groups()
        region1 = [p for p in plan if p[0] in ("l0", "lr0")]
        region2 = [p for p in plan if p[0] not in ("l0", "lr0") + rn1 + tail]
        offs, off = {}, 0
        for p in region1:
            offs[p] = off
            off += n_of(*p[1:])
        base2 = off
        for p in region2:
            offs[p] = off
            off += n_of(*p[1:])
        o1 = base2
        for p in (p for p in plan if p[0] in rn1):
            offs[p] = o1
            o1 += n_of(*p[1:])
        for p in (p for p in plan if p[0] in tail):
            offs[p] = 0
        size = max([off, o1] + [offs[p] + n_of(*p[1:]) for p in plan])
        arena = torch.empty(size, device=dev, dtype=torch.bfloat16)
        self._bufs = {}
        for p in plan:
            slot, H, W, C = p
            n = frames * (H + 2) * (W + 2) * C
            self._bufs[p] = arena[offs[p]:offs[p] + n].view(frames, H + 2, W + 2, C)
        over = [(offs[p], offs[p] + n_of(*p[1:])) for p in plan if p[0] in rn1 + tail]
        self._overlay = set(rn1 + tail)
        self._under_overlay = [p for p in plan if p[0] not in self._overlay and
                               any(offs[p] < e and b < offs[p] + n_of(*p[1:]) for b, e in over)]
        self._prepared = True
        self._zeroed = False
        self._dirty = False

    @staticmethod
    def _zero_border(b: torch.Tensor) -> None:
        """Zero the border rows and columns of a [F, H+2, W+2, C] buffer: two strided fills."""
        _, H2, W2, C = b.shape
        b[:, 0::H2 - 1].zero_()                       # rows 0 and H+1
        b.reshape(-1, W2, C)[:, 0::W2 - 1].zero_()    # columns 0 and W+1 of every row (a view: contiguous)

    def _zero_borders(self) -> None:
        for b in self._bufs.values():
            self._zero_border(b)
        self._zeroed = True

    def release(self) -> None:
        self._bufs = {}
        self._prepared = False

    def _pad(self, slot: str, Fr: int, H: int, W: int, C: int, dev) -> torch.Tensor:
        """Zero-bordered NHWC buffer [Fr, H+2, W+2, C] for `slot`, reused across the frame chunks of a
        call: the producing kernels overwrite the whole interior, so borders are zeroed once per forward
        (and, for the buffers that share memory, as `prepare` describes) instead of zero-filling every
        buffer of every chunk."""
        key = (slot, H, W, C)
        buf = self._bufs.get(key)
        if buf is None or buf.shape[0] < Fr or buf.device != torch.device(dev):
            if self._prepared:  # buffer_plan() is out of step with forward_chunk
                raise RuntimeError(f"DPT buffer {key} x {Fr} views is not in the prepared plan")
            buf = torch.zeros(Fr, H + 2, W + 2, C, device=dev, dtype=torch.bfloat16)
            self._bufs[key] = buf
        if self._prepared and slot in self._overlay:  # over other buffers: re-zero, mark those dirty
            self._zero_border(buf[:Fr])
            self._dirty = True
        return buf[:Fr]

    def _rcu(self, name, x_raw, x_relu, Fr, hs, res2=None, res2_pad=False, dense_out=False):
        """ResidualConvUnit: conv2(relu(conv1(relu(x)))) + x (+ res2), relu(x) supplied padded."""
        Fh = self.W.cfg.dpt_features
        dev = x_raw.device
        h = self._pad(name + ".h", Fr, hs, hs, Fh, dev)
        ops.gemm_spatial(x_relu.view(-1, Fh), self.cw[name + ".conv1"], self.b[name + ".conv1.bias"], Fr, hs, hs,
                         conv3x3=True, relu=True, out1=h, out1_pad=True)
        if dense_out:
            o = torch.empty(Fr, hs, hs, Fh, device=dev, dtype=torch.bfloat16)
            o2 = None
        else:
            o = self._pad(name + ".o", Fr, hs, hs, Fh, dev)
            o2 = self._pad(name + ".o2", Fr, hs, hs, Fh, dev)
        ops.gemm_spatial(h.view(-1, Fh), self.cw[name + ".conv2"], self.b[name + ".conv2.bias"], Fr, hs, hs,
                         conv3x3=True, res1=x_raw, res1_pad=True, res2=res2, res2_pad=res2_pad,
                         out1=o, out1_pad=not dense_out, out2=o2, out2_pad=True)
        return o, o2

    def forward_chunk(self, layers: List[torch.Tensor], pred: torch.Tensor, conf: torch.Tensor):
        """layers: 4 x (F, N, 2C) bf16 kept tokens; writes pred (F,H,W,odim-1) and conf (F,H,W)."""
        W, cfg, head = self.W, self.W.cfg, self.head
        g, ps = cfg.grid, cfg.patch_start_idx
        D = 2 * cfg.embed_dim
        Hh = Ww = cfg.img_size
        oc = cfg.dpt_out_channels
        Fh = cfg.dpt_features
        Fr = layers[0].shape[0]
        dev = layers[0].device
        bf = torch.bfloat16
        empty = lambda *sh: torch.empty(*sh, device=dev, dtype=bf)
        pad = lambda slot, h_, w_, c_: self._pad(slot, Fr, h_, w_, c_, dev)
        if self._prepared and self._dirty:  # the previous chunk's overlaid buffers overwrote these borders
            for k in self._under_overlay:
                self._zero_border(self._bufs[k][:Fr])
            self._dirty = False
        sizes = [4 * g, 2 * g, g, (g + 1) // 2]
        feats = []
        for i, x in enumerate(layers):
            xn = ops.layernorm_tokens(x, ps, W[head + "norm.weight"], W[head + "norm.bias"], cfg.ln_eps)
            pb = self.b[f"{head}projects.{i}.bias"]
            if i < 2:  # 1x1 projection, then conv-transpose (k = s = 4 / 2) as GEMM + pixel shuffle
                y = empty(Fr, g, g, oc[i])
                ops.gemm_spatial(xn, self.proj_w[i], pb, Fr, g, g, out1=y, pos=self.pos_small[i])
                s = 4 if i == 0 else 2
                f = pad(f"f{i}", g * s, g * s, oc[i])
                ops.gemm_spatial(y.view(-1, oc[i]), self.convT[i], self.b[f"{head}resize_layers.{i}.bias"], Fr, g, g,
                                 shuffle=s, out1=f, out1_pad=True)
            elif i == 2:  # identity
                f = pad(f"f{i}", g, g, oc[i])
                ops.gemm_spatial(xn, self.proj_w[i], pb, Fr, g, g, out1=f, out1_pad=True, pos=self.pos_small[i])
            else:  # 3x3 stride-2 conv: stride-1 implicit GEMM keeping even pixels
                y = pad(f"y{i}", g, g, oc[i])
                ops.gemm_spatial(xn, self.proj_w[i], pb, Fr, g, g, out1=y, out1_pad=True, pos=self.pos_small[i])
                f = pad(f"f{i}", sizes[3], sizes[3], oc[i])
                ops.gemm_spatial(y.view(-1, oc[i]), self.cw[head + "resize_layers.3"],
                                 self.b[head + "resize_layers.3.bias"], Fr, g, g, conv3x3=True, subsample2=True,
                                 out1=f, out1_pad=True)
            feats.append(f)
        sc = head + "scratch."
        L = []
        for i, f in enumerate(feats):  # layer_rn 3x3 (no bias): raw + relu copies, padded
            hs = sizes[i]
            l, lr = pad(f"l{i}", hs, hs, Fh), pad(f"lr{i}", hs, hs, Fh)
            ops.gemm_spatial(f.view(-1, oc[i]), self.cw[f"{sc}layer{i + 1}_rn"], None, Fr, hs, hs, conv3x3=True,
                             out1=l, out1_pad=True, out2=lr, out2_pad=True)
            L.append((l, lr))

        def out_conv(r, o, hs, target, padded):
            # upstream: out_conv(interpolate(o)). A 1x1 conv commutes with bilinear resizing (both
            # linear; the resize weights sum to 1, so the bias passes through), so the conv runs at
            # the source resolution (~4x fewer pixels) and the resize writes the result, straight
            # into the zero-bordered buffer the next 3x3 conv reads when `padded`
            y = empty(Fr, hs, hs, Fh)
            ops.gemm_spatial(o.view(-1, Fh), self.cw[f"{sc}refinenet{r}.out_conv"],
                             self.b[f"{sc}refinenet{r}.out_conv.bias"], Fr, hs, hs, out1=y)
            if padded:
                return ops.upsample_bilinear(y, (target, target), out=pad(f"oc{r}", target, target, Fh), out_pad=True)
            return ops.upsample_bilinear(y, (target, target))

        # refinenet4: RCU2(l4) -> upsample to layer3 size -> out_conv
        o, _ = self._rcu(f"{sc}refinenet4.resConfUnit2", L[3][0], L[3][1], Fr, sizes[3], dense_out=True)
        x = out_conv(4, o, sizes[3], sizes[2], False)
        for r, li, target in ((3, 2, sizes[1]), (2, 1, sizes[0]), (1, 0, 2 * sizes[0])):
            hs = sizes[li]
            s_raw, s_relu = self._rcu(f"{sc}refinenet{r}.resConfUnit1", L[li][0], L[li][1], Fr, hs,
                                      res2=x, res2_pad=False)
            o, _ = self._rcu(f"{sc}refinenet{r}.resConfUnit2", s_raw, s_relu, Fr, hs, dense_out=True)
            x = out_conv(r, o, hs, target, padded=(r == 1))
        t = 2 * sizes[0]
        y = empty(Fr, t, t, Fh // 2)
        ops.gemm_spatial(x.view(-1, Fh), self.cw[sc + "output_conv1"], self.b[sc + "output_conv1.bias"], Fr, t, t,
                         conv3x3=True, out1=y)
        u = ops.upsample_bilinear(y, (Hh, Ww), add=self.pos_full, out_pad=True, out=pad("u", Hh, Ww, Fh // 2))
        act = 0 if self.activation == "exp" else 1
        ops.gemm_spatial(u.view(-1, Fh // 2), self.cw[sc + "output_conv2.0"], self.b[sc + "output_conv2.0.bias"],
                         Fr, Hh, Ww, conv3x3=True, head=(self.head_w, self.head_b, act, pred, conf))

    def __call__(self, kept: Dict[int, torch.Tensor], out_pred: torch.Tensor, out_conf: torch.Tensor,
                 chunk: int):
        cfg = self.W.cfg
        layers = [kept[i] for i in cfg.kept_layers]
        S = layers[0].shape[0]
        own = not self._prepared  # standalone call: buffers allocated lazily on this stream, dropped after
        if self._prepared and not self._zeroed:
            self._zero_borders()
        for s0 in range(0, S, chunk):
            s1 = min(S, s0 + chunk)
            self.forward_chunk([l[s0:s1] for l in layers], out_pred[s0:s1], out_conf[s0:s1])
        if own:
            self.release()
