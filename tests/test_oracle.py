"""CPU oracle self-tests: goldens and invariances."""
import math
import os

import numpy as np
import pytest
import torch

from oracle import vggt_ref as R
from paper_2509_25191_b200.config import vggt_1b, vggt_tiny
from paper_2509_25191_b200.weights import make_state_dict, param_shapes, synthetic_images

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tiny_s8.npz")


@pytest.fixture(scope="module")
def tiny():
    cfg = vggt_tiny()
    return cfg, make_state_dict(cfg, 0), synthetic_images(cfg, 8, 1)


def test_golden_tiny(tiny):
    cfg, sd, images = tiny
    g = np.load(GOLDEN)
    assert abs(images.double().sum().item() - g["images_checksum"][0]) < 1e-6
    wsum = sum(v.double().sum().item() for v in sd.values())
    assert abs(wsum - g["weights_checksum"][0]) < 1e-6 * max(1.0, abs(wsum))
    p = R.vggt_forward(images, sd, cfg)
    for i in cfg.kept_layers:
        np.testing.assert_allclose(p["kept"][i].numpy(), g[f"kept_{i}"], rtol=1e-4, atol=1e-5)
    for k in ("pose_enc", "depth", "depth_conf", "world_points", "world_points_conf"):
        np.testing.assert_allclose(p[k][0].numpy(), g[k], rtol=1e-4, atol=1e-5)


def test_chunked_equals_unchunked(tiny):
    cfg, sd, images = tiny
    full = R.vggt_forward(images, sd, cfg)
    for fc, hc in ((1, 1), (3, 5), (128, 8)):
        p = R.vggt_forward(images, sd, cfg, frame_chunk=fc, head_chunk=hc)
        for i in cfg.kept_layers:
            torch.testing.assert_close(p["kept"][i], full["kept"][i], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(p["depth"], full["depth"], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(p["pose_enc"], full["pose_enc"], rtol=1e-5, atol=1e-5)


def test_kept_layers_are_slices_of_all_layers(tiny):
    cfg, sd, images = tiny
    cfg2 = cfg.with_(kept_layers=(1, 3))
    kept = R.aggregator(images, sd, cfg2)
    allk = R.aggregator(images, sd, cfg2, keep_all=True)
    assert sorted(kept) == [1, 3] and sorted(allk) == [0, 1, 2, 3]
    for i in kept:
        torch.testing.assert_close(kept[i], allk[i])


def test_single_view_frame_equals_global(tiny):
    """With S = 1 the global block attends over exactly the frame's tokens."""
    cfg, sd, images = tiny
    x = torch.randn(1, cfg.tokens_per_frame, cfg.embed_dim)
    pos = R.positions(cfg)
    a = R.block(x, sd, "aggregator.frame_blocks.0", cfg.num_heads, cfg.ln_eps, pos)
    sd2 = dict(sd)
    for k, v in sd.items():
        if k.startswith("aggregator.frame_blocks.0."):
            sd2[k.replace("frame_blocks", "global_blocks")] = v
    b = R.block(x, sd2, "aggregator.global_blocks.0", cfg.num_heads, cfg.ln_eps, pos)
    torch.testing.assert_close(a, b)


def test_global_attention_permutation_equivariance(tiny):
    """Frames 1..S-1 are exchangeable: permuting them permutes the outputs."""
    cfg, sd, images = tiny
    perm = torch.tensor([0, 3, 1, 2, 7, 6, 5, 4])
    a = R.aggregator(images, sd, cfg)
    b = R.aggregator(images[perm], sd, cfg)
    for i in cfg.kept_layers:
        torch.testing.assert_close(b[i], a[i][perm], rtol=1e-4, atol=1e-4)


def test_simulated_ring_equals_monolithic():
    """Split K/V into g blocks, merge partial results by log-sum-exp (ring math, no NCCL)."""
    from paper_2509_25191_b200.ring import lse_merge
    torch.manual_seed(0)
    H, T, d = 4, 300, 32
    q, k, v = (torch.randn(H, T, d) for _ in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v).permute(1, 0, 2).reshape(T, H * d)
    for g in (2, 3, 5):
        bounds = [(i * T // g, (i + 1) * T // g) for i in range(g)]
        o_acc = torch.zeros(T, H * d)
        lse_acc = torch.full((H, T), float("-inf"))
        for lo, hi in bounds:
            s = torch.einsum("hqd,hkd->hqk", q, k[:, lo:hi]) / math.sqrt(d)
            lse = torch.logsumexp(s, -1)
            o = torch.einsum("hqk,hkd->hqd", s.softmax(-1), v[:, lo:hi]).permute(1, 0, 2).reshape(T, H * d)
            lse_merge(o_acc, lse_acc, o, lse)
        torch.testing.assert_close(o_acc, ref, rtol=1e-5, atol=1e-5)


def test_rope_matches_rotation_definition():
    """RoPE is a rotation by pos*freq of (x_j, x_{j+d/4}) pairs in each half."""
    d = 64
    x = torch.randn(1, 5, d)
    pos = torch.tensor([[0, 0], [1, 2], [3, 4], [37, 37], [10, 1]])
    y = R.rope_2d(x, pos, 100.0)
    assert torch.allclose(y.norm(dim=-1), x.norm(dim=-1), atol=1e-5)
    torch.testing.assert_close(y[0, 0], x[0, 0])  # position (0, 0): identity
    q = d // 4
    inv = 1.0 / 100.0 ** (torch.arange(0, d // 2, 2).float() / (d // 2))
    th = pos[1, 0] * inv[0]
    exp0 = x[0, 1, 0] * math.cos(th) - x[0, 1, q] * math.sin(th)
    assert abs(y[0, 1, 0].item() - exp0.item()) < 1e-5


def test_pose_decode_conventions():
    enc = torch.tensor([[0.1, -0.2, 1.0, 0.0, 0.0, 0.0, 1.0, 1.0, 1.2]])
    ext, K = R.pose_encoding_to_extri_intri(enc, (518, 518))
    torch.testing.assert_close(ext[0, :, :3], torch.eye(3))
    torch.testing.assert_close(ext[0, :, 3], enc[0, :3])
    assert abs(K[0, 0, 0].item() - 259 / math.tan(0.6)) < 1e-3
    assert abs(K[0, 1, 1].item() - 259 / math.tan(0.5)) < 1e-3
    q = torch.nn.functional.normalize(torch.randn(100, 4), dim=-1)
    Rm = R.quat_to_mat(q)
    torch.testing.assert_close(Rm @ Rm.transpose(-1, -2), torch.eye(3).expand(100, 3, 3), atol=1e-5, rtol=0)
    assert (torch.linalg.det(Rm) > 0).all()
    ang, terr = R.pose_errors(enc, enc)
    assert ang.abs().max() < 1e-6 and terr.abs().max() < 1e-12


def test_flop_model_matches_survey():
    """Appendix B: 6.16 / 39.56 / 188.0 TFLOP per view at S = 20 / 200 / 1000."""
    cfg = vggt_1b()
    for S, tf in ((20, 6.16), (200, 39.56), (1000, 188.03)):
        per_view = R.forward_flops(cfg, S) / S / 1e12
        assert abs(per_view - tf) / tf < 0.01, (S, per_view)


def test_param_count_1b():
    cfg = vggt_1b()
    n = sum(math.prod(s) for s in param_shapes(cfg).values())
    assert 0.85e9 < n < 0.92e9, n
