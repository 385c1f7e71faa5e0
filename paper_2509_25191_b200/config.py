"""Frozen model / run configuration for the dense-view VGGT inference path.

The reference (VGGT-X, arXiv 2509.25191) describes this path only in prose:
`PAPER.md:79` (24 alternating frame/global "AA" layers; only layers 4, 11, 17
and 23 feed the dense heads), `PAPER.md:81` (bf16 everywhere except the head
MLPs; frame-wise work is chunked) and `PAPER.md:146` (chunk size 128).  The
architecture constants below are the upstream `vggt` values restated in
SURVEY.md Appendix A; the CPU oracle (`oracle/vggt_ref.py`) and the CUDA path
both read them from here so "identical weights" is exact.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class VGGTConfig:
    img_size: int = 518
    patch_size: int = 14
    embed_dim: int = 1024
    depth: int = 24
    num_heads: int = 16
    mlp_ratio: float = 4.0
    num_register_tokens: int = 4
    rope_freq: float = 100.0
    init_values: float = 0.01          # LayerScale init (upstream aggregator)
    ln_eps: float = 1e-5               # nn.LayerNorm default (blocks, qk-norm, heads)
    # VGGT-X "VGGT-": only these aggregator layers are materialised
    kept_layers: tuple = (4, 11, 17, 23)
    # camera head (upstream CameraHead(dim_in=2*embed_dim))
    cam_trunk_depth: int = 4
    cam_num_heads: int = 16
    cam_iters: int = 4
    cam_init_values: float = 0.01
    # DPT heads
    dpt_features: int = 256
    dpt_out_channels: tuple = (256, 512, 1024, 1024)
    dpt_head_features_2: int = 32
    # patch embedding (SURVEY.md §8a a2 / a2'): "conv" = Conv2d 14x14/14 as an im2col GEMM (the north
    # star's "patch-embed as a GEMM"); "dinov2" = the DINOv2 ViT-L/14-reg `forward_features` upstream
    # VGGT-1B checkpoints carry (aggregator.patch_embed.*), x_norm_patchtokens as the patch tokens
    patch_embed: str = "conv"
    dino_depth: int = 24
    dino_init_values: float = 1.0     # LayerScale of the DINOv2 blocks (init_values=1.0 upstream)
    dino_eps: float = 1e-6            # DINOv2 LayerNorm eps
    # memory discipline (VGGT-X "VGGT--")
    frame_chunk: int = 128             # frames per chunk for frame-wise MLP work
    head_chunk: int = 16               # frames per DPT-head chunk (16: -9% head time vs 8 for +4 GB, tools/exp_dpt_chunk.py)
    q_chunk: int = 256                 # above this many views (one GPU), q is produced and consumed this many frames
                                       # at a time: K/V for all tokens, then per chunk q + attention (0 = never)

    def __post_init__(self):
        # native DPT convs use 64-channel K blocks and 32-channel output chunks
        for c in (*self.dpt_out_channels, self.dpt_features, self.dpt_features // 2):
            if c % 64:
                raise ValueError(f"DPT channel counts must be multiples of 64 (got {c})")
        if self.dpt_head_features_2 != 32:
            raise ValueError("dpt_head_features_2 must be 32 (fused output head)")
        if self.patch_embed not in ("conv", "dinov2"):
            raise ValueError(f"patch_embed must be 'conv' or 'dinov2' (got {self.patch_embed!r})")
        if self.patch_embed == "dinov2" and self.num_register_tokens != 4:
            raise ValueError("the DINOv2-reg patch embedding has 4 register tokens (cls + 4 + patches = tokens_per_frame)")

    @property
    def grid(self) -> int:
        return self.img_size // self.patch_size

    @property
    def num_patches(self) -> int:
        return self.grid * self.grid

    @property
    def patch_start_idx(self) -> int:
        return 1 + self.num_register_tokens

    @property
    def tokens_per_frame(self) -> int:
        return self.patch_start_idx + self.num_patches

    @property
    def head_dim(self) -> int:
        return self.embed_dim // self.num_heads

    @property
    def mlp_hidden(self) -> int:
        return int(self.embed_dim * self.mlp_ratio)

    @property
    def patch_k(self) -> int:
        return 3 * self.patch_size * self.patch_size

    @property
    def patch_k_padded(self) -> int:
        # GEMM K must be a multiple of the 64-element (128 B) K block
        return (self.patch_k + 63) // 64 * 64

    def with_(self, **kw) -> "VGGTConfig":
        return replace(self, **kw)


def vggt_1b() -> VGGTConfig:
    """VGGT-1B-shaped aggregator (24x2 blocks, dim 1024) with conv patch-embed."""
    return VGGTConfig()


def vggt_tiny() -> VGGTConfig:
    """BASELINE.json configs[0]: depth 4, dim 128, 4 heads, 112x112 views."""
    return VGGTConfig(
        img_size=112, embed_dim=128, depth=4, num_heads=4,
        kept_layers=(0, 1, 2, 3),
        cam_num_heads=4, dpt_features=128, dpt_out_channels=(64, 64, 128, 128),
        dpt_head_features_2=32, frame_chunk=4, head_chunk=3,
    )


def vggt_small() -> VGGTConfig:
    """A mid-size config with d=64 heads (dim 256) used by GPU parity tests."""
    return VGGTConfig(
        img_size=126, embed_dim=256, depth=4, num_heads=4,
        kept_layers=(0, 1, 2, 3),
        cam_num_heads=4, dpt_features=128, dpt_out_channels=(64, 64, 128, 128),
        dpt_head_features_2=32, frame_chunk=4, head_chunk=3,
    )
