"""Host orchestration of the VGGT Aggregator on the sm_100a kernels.

Upstream call stack replaced:
  Aggregator.forward -> normalize, patch_embed, special tokens, positions,
  24 x (frame_blocks[i], global_blocks[i]), output_list.
VGGT-X changes made native (`PAPER.md:79-81,146`):
  * only the kept layers {4, 11, 17, 23} are materialised; the fc2 residual
    epilogue of the frame / global block writes the bf16 copy straight into
    the kept buffer's left / right half (no intermediate cache, no concat);
  * bf16 GEMM / attention operands, fp32 inter-block residual stream
    (SURVEY.md §7 "Parity under bf16" design rule);
  * the frame-wise MLP is evaluated `frame_chunk` frames at a time so the
    4C-wide hidden activation never exists for all views at once.

HBM layout (T = S * tokens_per_frame rows, frame-major):
  x      fp32 [T, C]        residual stream
  xn     bf16 [T, C]        LayerNorm output (GEMM A operand)
  q,k,v  bf16 [H, T, d]     head-major: frame attention reads rows f*N..f*N+N-1
                            of each head, global attention all T rows (above cfg.q_chunk views
                            q holds one chunk of frames: _attention_q_chunked)
  o      bf16 [T, C]        attention output (proj A operand); the same buffer as xn
  h      bf16 [chunk*N, 4C] MLP hidden (per frame chunk)
  kept   bf16 [S, N, 2C]    per kept layer: [frame_out | global_out]
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, Optional

import torch

from . import ops
from .config import VGGTConfig
from .profiling import phase
from .weights import is_bf16_param


def rope_tables(head_dim: int, max_pos: int, freq: float):
    """cos/sin of pos * freq^(-2i/(d/2)), i < d/4, fp32 — one quarter of the head
    (the oracle's cat(angles, angles) duplicates it).  (max_pos, d/4) each."""
    half = head_dim // 2
    exponents = torch.arange(0, half, 2, dtype=torch.float32) / half
    inv_freq = 1.0 / (freq ** exponents)
    ang = torch.arange(max_pos, dtype=torch.float32)[:, None] * inv_freq[None, :]
    return ang.cos().contiguous(), ang.sin().contiguous()


def dino_pos_table(pos_embed: torch.Tensor, grid: int) -> torch.Tensor:
    """DINOv2 interpolate_pos_encoding for square views (upstream dinov2 as built by the VGGT aggregator:
    bicubic, antialias, offset 0), applied once at weight load: (1, 1 + M*M, C) -> [1 + grid*grid, C]."""
    C = pos_embed.shape[-1]
    pos = pos_embed.float().reshape(1, -1, C)
    N = pos.shape[1] - 1
    if N != grid * grid:
        M = round(N ** 0.5)
        patch = torch.nn.functional.interpolate(pos[:, 1:].reshape(1, M, M, C).permute(0, 3, 1, 2),
                                                size=(grid, grid), mode="bicubic", antialias=True)
        pos = torch.cat([pos[:, :1], patch.permute(0, 2, 3, 1).reshape(1, grid * grid, C)], dim=1)
    return pos[0]


class DeviceWeights:
    """Device copies of the state dict: bf16 matrix weights, fp32 everything else."""

    def __init__(self, sd: Dict[str, torch.Tensor], cfg: VGGTConfig, device="cuda"):
        self.cfg = cfg
        self.t: Dict[str, torch.Tensor] = {}
        for name, v in sd.items():
            dt = torch.bfloat16 if is_bf16_param(name, tuple(v.shape)) else torch.float32
            self.t[name] = v.to(device=device, dtype=dt).contiguous()
        a = "aggregator."
        C = cfg.embed_dim
        pe = a + ("patch_embed.proj." if cfg.patch_embed == "conv" else "patch_embed.patch_embed.proj.")
        self.patch_b = self.t[pe + "bias"]
        pw = sd[pe + "weight"].reshape(C, -1)
        pad = torch.zeros(C, cfg.patch_k_padded)
        pad[:, : cfg.patch_k] = pw
        self.patch_w = pad.to(device=device, dtype=torch.bfloat16)
        self.special = torch.cat([sd[a + "camera_token"][0], sd[a + "register_token"][0]], dim=1).to(
            device=device, dtype=torch.float32).contiguous()  # (2, 1+R, C)
        cos, sin = rope_tables(cfg.head_dim, cfg.grid + 1, cfg.rope_freq)
        self.rope = (cos.to(device), sin.to(device))
        if cfg.patch_embed == "dinov2":  # cls / registers / position table of the DINOv2 encoder (a2')
            d_ = a + "patch_embed."
            self.dino_cls = self.t[d_ + "cls_token"].reshape(C).contiguous()
            self.dino_reg = self.t[d_ + "register_tokens"].reshape(-1, C).contiguous()
            self.dino_pos = dino_pos_table(sd[d_ + "pos_embed"], cfg.grid).to(device=device,
                                                                               dtype=torch.float32).contiguous()

    def __getitem__(self, k):
        return self.t[k]


@dataclass
class Workspace:
    x: torch.Tensor
    xn: torch.Tensor
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    o: torch.Tensor
    h: torch.Tensor
    # q stored pre-scaled by log2(e)/sqrt(d) (the qkv epilogue's q_scale) and attention told so
    # (ops.attention(..., q_log2=True)): the FMHA then reads scores in log2 units directly. A global
    # attention hook receives q in this form.
    q_log2: bool = True


def alloc_workspace(cfg: VGGTConfig, S: int, device="cuda", rows_per_head: Optional[int] = None,
                    kv: Optional[tuple] = None, q_log2: bool = True, q_frames: Optional[int] = None) -> Workspace:
    """Per-forward buffers for S views.  `rows_per_head` (>= S * tokens_per_frame) is the per-head row
    stride of q/k/v; `kv` = (k, v) [H, rows_per_head, d] supplied by the frame-sharded ring (its send
    buffer: the QKV epilogue then writes the local K/V where the first ring step sends them from).
    `q_frames` < S: q holds that many frames only, and run_block produces and consumes it chunk by chunk
    (peak HBM: T x C bf16 less the chunk)."""
    T = S * cfg.tokens_per_frame
    R = rows_per_head or T
    if R < T:
        raise ValueError(f"rows_per_head {R} < {T} tokens")
    C, H, d = cfg.embed_dim, cfg.num_heads, cfg.head_dim
    chunk_rows = min(S, cfg.frame_chunk) * cfg.tokens_per_frame
    if kv is None:
        kv = tuple(torch.empty(H, R, d, device=device, dtype=torch.bfloat16) for _ in range(2))
    elif any(tuple(t.shape) != (H, R, d) or not t.is_contiguous() for t in kv):
        raise ValueError("kv buffers must be contiguous [H, rows_per_head, d]")
    # the LayerNorm output and the attention output share one buffer: in a block, xn (norm1) is dead once
    # the qkv GEMM has read it, before attention writes o, and o is dead once proj has read it, before
    # norm2 writes xn (one stream, in order) — T x C bf16 less peak HBM (2.8 GB at 1000 views)
    xn = torch.empty(T, C, device=device, dtype=torch.bfloat16)
    return Workspace(
        x=torch.empty(T, C, device=device, dtype=torch.float32),
        xn=xn,
        q=torch.empty(H, (q_frames * cfg.tokens_per_frame if q_frames and q_frames < S else R), d, device=device,
                      dtype=torch.bfloat16),
        k=kv[0],
        v=kv[1],
        o=xn,
        h=torch.empty(chunk_rows, cfg.mlp_hidden, device=device, dtype=torch.bfloat16),
        q_log2=q_log2,
    )


# attention hook: (q, k, v, o, nseq, L) for a global block; the multi-GPU path
# replaces it with the frame-sharded ring (ring.py)
GlobalAttnFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor], None]


def run_block(W: DeviceWeights, name: str, ws: Workspace, S: int, frame_attn: bool,
              kept_half: Optional[torch.Tensor], global_attn: Optional[GlobalAttnFn] = None,
              vggt_attn: bool = True, eps: Optional[float] = None):
    """One pre-norm Block on the whole residual stream.  vggt_attn: the
    aggregator's attention (q/k LayerNorm + 2D RoPE); False for the DINOv2 encoder blocks (a2')."""
    cfg = W.cfg
    N = cfg.tokens_per_frame
    T = S * N
    C = cfg.embed_dim
    eps = cfg.ln_eps if eps is None else eps
    with phase("layernorm"):
        ops.layernorm(ws.x, W[name + ".norm1.weight"], W[name + ".norm1.bias"], eps, out=ws.xn)
    extra = {}
    if vggt_attn:
        extra = dict(qk_norm=(W[name + ".attn.q_norm.weight"], W[name + ".attn.q_norm.bias"],
                              W[name + ".attn.k_norm.weight"], W[name + ".attn.k_norm.bias"]),
                     rope=W.rope, tokens_per_frame=N, patch_start=cfg.patch_start_idx, grid_w=cfg.grid,
                     eps=cfg.ln_eps)
    qs = ops.Q_LOG2_SCALE(cfg.head_dim) if ws.q_log2 else 0.0
    Rq = ws.q.shape[1]
    if Rq < T:  # chunked q (alloc_workspace q_frames): frame-aligned chunks of Rq rows
        _attention_q_chunked(W, name, ws, S, frame_attn, global_attn, extra, qs)
    else:
        with phase("gemm_qkv"):
            ops.gemm(ws.xn, W[name + ".attn.qkv.weight"], ops.EPI_QKV, bias=W[name + ".attn.qkv.bias"],
                     qkv=(ws.q, ws.k, ws.v), head_dim=cfg.head_dim, tokens_total=Rq, q_scale=qs, **extra)
        if frame_attn:
            with phase("attn_frame"):
                ops.attention(ws.q, ws.k, ws.v, ws.o, nseq=S, Lq=N, Lk=N, q_log2=ws.q_log2)
        elif global_attn is not None:
            with phase("attn_global"):
                global_attn(ws.q, ws.k, ws.v, ws.o)
        else:
            with phase("attn_global"):
                ops.attention(ws.q, ws.k, ws.v, ws.o, nseq=1, Lq=T, Lk=T, q_log2=ws.q_log2)
    with phase("gemm_proj"):
        ops.gemm(ws.o, W[name + ".attn.proj.weight"], ops.EPI_RESID, bias=W[name + ".attn.proj.bias"],
                 resid=ws.x, gamma=W[name + ".ls1.gamma"])
    with phase("layernorm"):
        ops.layernorm(ws.x, W[name + ".norm2.weight"], W[name + ".norm2.bias"], eps, out=ws.xn)
    rows = ws.h.shape[0]
    for r0 in range(0, T, rows):
        r1 = min(T, r0 + rows)
        hb = ws.h[: r1 - r0]
        with phase("gemm_fc1"):
            ops.gemm(ws.xn[r0:r1], W[name + ".mlp.fc1.weight"], ops.EPI_GELU, bias=W[name + ".mlp.fc1.bias"],
                     out=hb)
        with phase("gemm_fc2"):
            ops.gemm(hb, W[name + ".mlp.fc2.weight"], ops.EPI_RESID, bias=W[name + ".mlp.fc2.bias"],
                     resid=ws.x[r0:r1], gamma=W[name + ".ls2.gamma"],
                     kept=None if kept_half is None else kept_half[r0:r1])


def _attention_q_chunked(W: DeviceWeights, name: str, ws: Workspace, S: int, frame_attn: bool,
                         global_attn: Optional[GlobalAttnFn], extra: dict, qs: float):
    """qkv GEMM + attention with q held one chunk of frames at a time (ws.q has Rq = chunk rows per head).

    Frame blocks: per chunk, q/k/v of the chunk (k/v in the first H x Rq x d elements of the k/v buffers,
    idle in a frame block) and the chunk's frame attention. Global blocks: K and V of all tokens first
    (the qkv weight's rows C..3C, `col_offset` C), then per chunk its q (rows 0..C) and the attention of
    its queries against all keys. xn and o share a buffer: a chunk's xn rows are read (by its q GEMM)
    before its attention writes the same rows of o, and other chunks' rows are untouched."""
    cfg = W.cfg
    N = cfg.tokens_per_frame
    T = S * N
    C, H, d = cfg.embed_dim, cfg.num_heads, cfg.head_dim
    Rq = ws.q.shape[1]
    cf = Rq // N  # frames per chunk
    w = W[name + ".attn.qkv.weight"]
    b = W[name + ".attn.qkv.bias"]
    if global_attn is not None:
        raise ValueError("chunked q runs on one GPU only (the ring attends with the whole local q)")
    if frame_attn:
        kc = ws.k.view(-1)[: H * Rq * d].view(H, Rq, d)
        vc = ws.v.view(-1)[: H * Rq * d].view(H, Rq, d)
        for f0 in range(0, S, cf):
            r0, r1 = f0 * N, min(S, f0 + cf) * N
            with phase("gemm_qkv"):
                ops.gemm(ws.xn[r0:r1], w, ops.EPI_QKV, bias=b, qkv=(ws.q, kc, vc), head_dim=d, tokens_total=Rq,
                         q_scale=qs, **extra)
            with phase("attn_frame"):
                ops.attention(ws.q, kc, vc, ws.o[r0:r1], nseq=(r1 - r0) // N, Lq=N, Lk=N, q_log2=ws.q_log2)
        return
    with phase("gemm_qkv"):
        ops.gemm(ws.xn, w[C:], ops.EPI_QKV, bias=b[C:], qkv=(ws.q, ws.k, ws.v), head_dim=d,
                 tokens_total=ws.k.shape[1], q_scale=qs, embed_dim=C, col_offset=C, **extra)
    for f0 in range(0, S, cf):
        r0, r1 = f0 * N, min(S, f0 + cf) * N
        with phase("gemm_qkv"):
            ops.gemm(ws.xn[r0:r1], w[:C], ops.EPI_QKV, bias=b[:C], qkv=(ws.q, ws.k, ws.v), head_dim=d,
                     tokens_total=Rq, q_scale=qs, embed_dim=C, col_offset=0, **extra)
        with phase("attn_global"):
            ops.attention(ws.q, ws.k, ws.v, ws.o[r0:r1], nseq=1, Lq=r1 - r0, Lk=T, q_log2=ws.q_log2)


def embed(W: DeviceWeights, images: torch.Tensor, ws: Workspace, frame0_is_first: bool = True):
    """a1-a3: special tokens + ResNet-normalised conv patch-embed into the fp32 stream."""
    cfg = W.cfg
    S = images.shape[0]
    N = cfg.tokens_per_frame
    special = W.special
    if not frame0_is_first:  # a shard that does not own global frame 0 uses the "other" tokens
        special = special[1:2].expand(2, -1, -1).contiguous()
    with phase("embed"):
        a = ops.patchify(images, cfg.patch_size, cfg.patch_k_padded)
        ops.gemm(a, W.patch_w, ops.EPI_PATCH, bias=W.patch_b, resid=ws.x, tokens_per_frame=N,
                 patch_start=cfg.patch_start_idx)
        del a
        if cfg.patch_embed == "dinov2":
            dinov2_encode(W, ws, S)
        ops.special_tokens(ws.x, special, S, N)


def dinov2_encode(W: DeviceWeights, ws: Workspace, S: int):
    """a2': DINOv2 ViT-L/14-reg forward_features on the patch-embedded stream, in place.

    The encoder's tokens (cls + 4 registers + patches) have the aggregator's per-frame layout, so it runs
    in the aggregator's own residual stream: token assembly (cls + pos, registers, patches + pos), the
    `dino_depth` pre-norm blocks as frame-attention blocks without qk-norm / RoPE (LayerNorm eps 1e-6),
    then the final LayerNorm in place; the caller overwrites rows 0..4 of every frame with the
    aggregator's camera / register tokens, leaving x_norm_patchtokens as the patch rows."""
    cfg = W.cfg
    d_ = "aggregator.patch_embed."
    ops.dino_tokens(ws.x, W.dino_cls, W.dino_reg, W.dino_pos, S, cfg.tokens_per_frame)
    for i in range(cfg.dino_depth):
        run_block(W, f"{d_}blocks.{i}", ws, S, True, None, vggt_attn=False, eps=cfg.dino_eps)
    ops.layernorm(ws.x, W[d_ + "norm.weight"], W[d_ + "norm.bias"], cfg.dino_eps, out=ws.x)


def aggregator_forward(W: DeviceWeights, images: torch.Tensor, ws: Optional[Workspace] = None,
                       global_attn: Optional[GlobalAttnFn] = None, frame0_is_first: bool = True
                       ) -> Dict[int, torch.Tensor]:
    """images (S,3,H,W) fp32 on device -> {layer: (S, N, 2C) bf16} for cfg.kept_layers."""
    cfg = W.cfg
    S = images.shape[0]
    N = cfg.tokens_per_frame
    C = cfg.embed_dim
    if images.shape[-1] != cfg.img_size or images.shape[-2] != cfg.img_size:
        raise ValueError(f"images must be {cfg.img_size}x{cfg.img_size}, got {tuple(images.shape)}")
    if ws is None:
        ws = alloc_workspace(cfg, S, images.device)
    embed(W, images.float().contiguous(), ws, frame0_is_first)
    kept = {i: torch.empty(S * N, 2 * C, device=images.device, dtype=torch.bfloat16) for i in cfg.kept_layers}
    for i in range(cfg.depth):
        kb = kept.get(i)
        run_block(W, f"aggregator.frame_blocks.{i}", ws, S, True, None if kb is None else kb[:, :C])
        run_block(W, f"aggregator.global_blocks.{i}", ws, S, False, None if kb is None else kb[:, C:],
                  global_attn=global_attn)
    return {i: t.view(S, N, 2 * C) for i, t in kept.items()}
