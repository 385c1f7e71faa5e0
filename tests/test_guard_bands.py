"""Out-of-bounds and race checks of the shipped kernels without compute-sanitizer.

compute-sanitizer is closed on this GPU pool (profiles/r02_compute_sanitizer_refused.txt), so the
memcheck / racecheck questions are asked directly:

  * guard bands: every input and output of a C-ABI call is a view into a larger allocation whose
    margins hold a sentinel.  Output margins must be bit-identical afterwards (no out-of-bounds
    write); input margins hold NaN, so an out-of-bounds read that reaches a result shows up as a
    non-finite output.  The shapes are ragged on purpose (M, N, sequence lengths and pixel grids not
    multiples of the tiles; the 1374 = 2 x 512 + 350 frame layout; the KV-split tail; ring merges).
  * determinism: kernels whose work distribution is dynamic (the FMHA's atomic work tickets and
    KV-split tail) or concurrent (heads on side streams) must give bit-identical results run to run;
    a shared-memory or TMEM race shows up as run-to-run differences.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

G = 4096  # guard elements on each side


@pytest.fixture(scope="module")
def ops():
    from paper_2509_25191_b200 import ops as _ops
    _ops.load_library()
    return _ops


class Guarded:
    """A tensor of `shape` inside a flat buffer with G sentinel elements on both sides."""

    def __init__(self, shape, dtype, data=None, sentinel=float("nan")):
        n = math.prod(shape)
        self.buf = torch.full((n + 2 * G,), sentinel, device="cuda", dtype=dtype)
        self.t = self.buf[G:G + n].view(shape)
        if data is not None:
            self.t.copy_(data)
        self.margin0 = self._margins().clone()

    def _margins(self):
        return torch.cat([self.buf[:G], self.buf[-G:]]).view(torch.int8 if self.buf.element_size() == 1 else
                                                             {2: torch.int16, 4: torch.int32, 8: torch.int64}[
                                                                 self.buf.element_size()])

    def intact(self):
        return torch.equal(self._margins(), self.margin0)


def _rand(shape, dtype=torch.float32, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(dtype)


def _check_out(*outs):
    for o in outs:
        assert o.intact(), "write outside the output"
        assert torch.isfinite(o.t.float()).all(), "non-finite output: an out-of-bounds read reached it"


@pytest.mark.parametrize("epi", ["bf16", "gelu", "f32", "resid", "resid_kept"])
@pytest.mark.parametrize("M,N,K", [(300, 96, 192), (1374, 1024, 1024), (129, 4096, 64)])
def test_gemm_guard_bands(ops, epi, M, N, K):
    a = Guarded((M, K), torch.bfloat16, _rand((M, K), torch.bfloat16, seed=1))
    w = Guarded((N, K), torch.bfloat16, _rand((N, K), torch.bfloat16, 0.05, seed=2))
    bias = Guarded((N,), torch.float32, _rand((N,), seed=3))
    if epi in ("bf16", "gelu", "f32"):
        dt = torch.float32 if epi == "f32" else torch.bfloat16
        out = Guarded((M, N), dt, sentinel=-7.0)
        code = {"bf16": ops.EPI_BF16, "gelu": ops.EPI_GELU, "f32": ops.EPI_F32}[epi]
        ops.gemm(a.t, w.t, code, bias=bias.t, out=out.t)
        _check_out(out)
    else:
        x = Guarded((M, N), torch.float32, _rand((M, N), seed=4), sentinel=-7.0)
        gamma = Guarded((N,), torch.float32, _rand((N,), seed=5))
        kept = Guarded((M, N), torch.bfloat16, sentinel=-7.0) if epi == "resid_kept" else None
        ops.gemm(a.t, w.t, ops.EPI_RESID, bias=bias.t, resid=x.t, gamma=gamma.t, kept=None if kept is None else kept.t)
        _check_out(x, *(() if kept is None else (kept,)))
    for inp in (a, w, bias):
        assert inp.intact()


@pytest.mark.parametrize("mode", ["qknorm_rope_d64", "plain_d128"])
def test_gemm_qkv_guard_bands(ops, mode):
    from paper_2509_25191_b200.aggregator import rope_tables
    if mode == "qknorm_rope_d64":
        C, H, d, tpf, S = 256, 4, 64, 5 + 81, 3  # 9 x 9 patch grid + 5 special tokens
    else:
        C, H, d, tpf, S = 512, 4, 128, 1, 37
    M = S * tpf
    R = M + 70  # rows per head larger than the tokens (ring layout)
    x = Guarded((M, C), torch.bfloat16, _rand((M, C), torch.bfloat16, seed=6))
    w = Guarded((3 * C, C), torch.bfloat16, _rand((3 * C, C), torch.bfloat16, 0.05, seed=7))
    b = Guarded((3 * C,), torch.float32, _rand((3 * C,), seed=8))
    q, k, v = (Guarded((H, R, d), torch.bfloat16, torch.zeros(H, R, d, device="cuda"), sentinel=-7.0)
               for _ in range(3))
    kw = {}
    if mode == "qknorm_rope_d64":
        nw = [Guarded((d,), torch.float32, _rand((d,), seed=9 + i) * 0.1 + 1) for i in range(4)]
        cos, sin = rope_tables(d, 10, 100.0)
        kw = dict(qk_norm=tuple(t.t for t in nw), rope=(cos.cuda(), sin.cuda()), tokens_per_frame=tpf,
                  patch_start=5, grid_w=9)
    ops.gemm(x.t, w.t, ops.EPI_QKV, bias=b.t, qkv=(q.t, k.t, v.t), head_dim=d, tokens_total=R, **kw)
    _check_out(q, k, v)


@pytest.mark.parametrize("case", ["frame_1374", "global_kvsplit", "tiny_d32", "trunk_d128"])
def test_attention_guard_bands(ops, case):
    H, d, nseq, L = {"frame_1374": (16, 64, 3, 1374), "global_kvsplit": (16, 64, 1, 8 * 1374),
                     "tiny_d32": (4, 32, 5, 69), "trunk_d128": (16, 128, 1, 333)}[case]
    T = nseq * L
    q, k, v = (Guarded((H, T, d), torch.bfloat16, _rand((H, T, d), torch.bfloat16, seed=s)) for s in (10, 11, 12))
    out = Guarded((T, H * d), torch.bfloat16, sentinel=-7.0)
    lse = Guarded((H, T), torch.float32, sentinel=-7.0)
    ops.attention(q.t, k.t, v.t, out.t, nseq=nseq, Lq=L, Lk=L, lse=lse.t if d == 64 else None)
    _check_out(out, *((lse,) if d == 64 else ()))


def test_attention_merge_guard_bands(ops):
    H, d, Lq, shards = 16, 64, 2900, (2100, 3000, 700)
    q = Guarded((H, Lq, d), torch.bfloat16, _rand((H, Lq, d), torch.bfloat16, seed=13))
    o_acc = Guarded((Lq, H * d), torch.float32, sentinel=-7.0)
    lse = Guarded((H, Lq), torch.float32, sentinel=-7.0)
    out = Guarded((Lq, H * d), torch.bfloat16, sentinel=-7.0)
    for i, n in enumerate(shards):
        k = Guarded((H, n, d), torch.bfloat16, _rand((H, n, d), torch.bfloat16, seed=20 + i))
        v = Guarded((H, n, d), torch.bfloat16, _rand((H, n, d), torch.bfloat16, seed=30 + i))
        mode = 1 if i == 0 else (3 if i == len(shards) - 1 else 2)
        ops.attention_merge(q.t, k.t, v.t, mode, o_acc.t, lse.t, out=out.t, Lq=Lq, Lk=n)
    _check_out(out, lse)
    assert o_acc.intact()


def test_norm_patch_special_guard_bands(ops):
    x = Guarded((333, 1024), torch.float32, _rand((333, 1024), seed=40))
    w = Guarded((1024,), torch.float32, _rand((1024,), seed=41))
    b = Guarded((1024,), torch.float32, _rand((1024,), seed=42))
    y = Guarded((333, 1024), torch.bfloat16, sentinel=-7.0)
    ops.layernorm(x.t, w.t, b.t, 1e-5, out=y.t)
    _check_out(y)
    xt = Guarded((3, 74, 256), torch.float32, _rand((3, 74, 256), seed=43))
    yt = Guarded((3 * 69, 256), torch.bfloat16, sentinel=-7.0)
    ops.layernorm_tokens(xt.t, 5, w.t[:256], b.t[:256], 1e-5, out=yt.t)
    _check_out(yt)
    img = Guarded((2, 3, 126, 126), torch.float32, torch.rand(2, 3, 126, 126, device="cuda"))
    pa = Guarded((2 * 81, 640), torch.bfloat16, sentinel=-7.0)
    ops.patchify(img.t, 14, 640, out=pa.t)
    _check_out(pa)
    xs = Guarded((3 * 86, 256), torch.float32, torch.zeros(3 * 86, 256, device="cuda"), sentinel=-7.0)
    tok = Guarded((2, 5, 256), torch.float32, _rand((2, 5, 256), seed=44))
    ops.special_tokens(xs.t, tok.t, 3, 86)
    assert xs.intact()


@pytest.mark.parametrize("out_pad", [False, True])
def test_upsample_guard_bands(ops, out_pad):
    x = Guarded((3, 19, 19, 256), torch.bfloat16, _rand((3, 19, 19, 256), torch.bfloat16, seed=50))
    add = Guarded((37, 37, 256), torch.bfloat16, _rand((37, 37, 256), torch.bfloat16, seed=51))
    shape = (3, 39, 39, 256) if out_pad else (3, 37, 37, 256)
    out = Guarded(shape, torch.bfloat16, torch.zeros(shape, device="cuda"), sentinel=-7.0)
    ops.upsample_bilinear(x.t, (37, 37), add=add.t, out=out.t, out_pad=out_pad)
    _check_out(out)


@pytest.mark.parametrize("kind", ["conv3x3_res", "conv3x3_s2", "convT4", "head"])
def test_spatial_guard_bands(ops, kind):
    Fr, H, Cin = 2, 19, 128
    xp = torch.zeros(Fr, H + 2, H + 2, Cin, device="cuda", dtype=torch.bfloat16)
    xp[:, 1:-1, 1:-1] = _rand((Fr, H, H, Cin), torch.bfloat16, seed=60)
    a = Guarded(tuple(xp.shape), torch.bfloat16, xp)
    if kind == "convT4":
        a = Guarded((Fr * H * H, Cin), torch.bfloat16, _rand((Fr * H * H, Cin), torch.bfloat16, seed=61))
        w = Guarded((16 * 64, Cin), torch.bfloat16, _rand((16 * 64, Cin), torch.bfloat16, 0.05, seed=62))
        bias = Guarded((64,), torch.float32, _rand((64,), seed=63))
        out = Guarded((Fr, 4 * H + 2, 4 * H + 2, 64), torch.bfloat16, torch.zeros(Fr, 4 * H + 2, 4 * H + 2, 64,
                                                                                  device="cuda"), sentinel=-7.0)
        ops.gemm_spatial(a.t, w.t, bias.t, Fr, H, H, shuffle=4, out1=out.t, out1_pad=True)
        _check_out(out)
        return
    cout = 32 if kind == "head" else 256
    w = Guarded((cout, 9 * Cin), torch.bfloat16, _rand((cout, 9 * Cin), torch.bfloat16, 0.03, seed=64))
    bias = Guarded((cout,), torch.float32, _rand((cout,), seed=65))
    if kind == "head":
        hw = Guarded((4, 32), torch.float32, _rand((4, 32), seed=66) * 0.1)
        hb = Guarded((4,), torch.float32, _rand((4,), seed=67) * 0.1)
        pred = Guarded((Fr, H, H, 3), torch.float32, sentinel=-7.0)
        conf = Guarded((Fr, H, H), torch.float32, sentinel=-7.0)
        ops.gemm_spatial(a.t.view(-1, Cin), w.t, bias.t, Fr, H, H, conv3x3=True,
                         head=(hw.t, hb.t, 1, pred.t, conf.t))
        _check_out(pred, conf)
        return
    if kind == "conv3x3_s2":
        ho = (H + 1) // 2
        out = Guarded((Fr, ho + 2, ho + 2, cout), torch.bfloat16, torch.zeros(Fr, ho + 2, ho + 2, cout, device="cuda"),
                      sentinel=-7.0)
        ops.gemm_spatial(a.t.view(-1, Cin), w.t, bias.t, Fr, H, H, conv3x3=True, subsample2=True, out1=out.t,
                         out1_pad=True)
        _check_out(out)
        return
    res = Guarded((Fr, H + 2, H + 2, cout), torch.bfloat16, torch.zeros(Fr, H + 2, H + 2, cout, device="cuda"))
    res.t[:, 1:-1, 1:-1] = _rand((Fr, H, H, cout), torch.bfloat16, seed=68)
    out = Guarded((Fr, H, H, cout), torch.bfloat16, sentinel=-7.0)
    out2 = Guarded((Fr, H + 2, H + 2, cout), torch.bfloat16, torch.zeros(Fr, H + 2, H + 2, cout, device="cuda"),
                   sentinel=-7.0)
    ops.gemm_spatial(a.t.view(-1, Cin), w.t, bias.t, Fr, H, H, conv3x3=True, relu=True, res1=res.t, res1_pad=True,
                     out1=out.t, out2=out2.t, out2_pad=True)
    _check_out(out, out2)


def test_camera_head_kernels_guard_bands(ops):
    x = Guarded((37, 2048), torch.float32, _rand((37, 2048), seed=70))
    w = Guarded((1000, 2048), torch.float32, _rand((1000, 2048), seed=71) * 0.02)
    b = Guarded((1000,), torch.float32, _rand((1000,), seed=72))
    for epi, dt in ((ops.LF_F32, torch.float32), (ops.LF_GELU, torch.float32), (ops.LF_SILU_BF16, torch.bfloat16)):
        out = Guarded((37, 1000), dt, sentinel=-7.0)
        ops.linear_f32(x.t, w.t, b.t, epi, out=out.t)
        _check_out(out)
    w9 = Guarded((9, 2048), torch.float32, _rand((9, 2048), seed=73) * 0.02)
    prev = Guarded((37, 9), torch.float32, _rand((37, 9), seed=74))
    pred = Guarded((37, 9), torch.float32, sentinel=-7.0)
    act = Guarded((37, 9), torch.float32, sentinel=-7.0)
    ops.linear_f32(x.t, w9.t, b.t[:9], ops.LF_POSE, out=pred.t, prev=prev.t, act_out=act.t)
    _check_out(pred, act)
    tok = Guarded((37, 2048), torch.float32, _rand((37, 2048), seed=75))
    mod = Guarded((37, 6144), torch.float32, _rand((37, 6144), seed=76) * 0.1)
    y = Guarded((37, 2048), torch.float32, sentinel=-7.0)
    ops.adaln_modulate(tok.t, mod.t, 1e-6, out=y.t)
    _check_out(y)


# ---------------------------------------------------------------------------------------------------
# determinism (race check): dynamic FMHA work tickets, KV-split tail, concurrent head streams
def test_attention_bitwise_deterministic(ops):
    H, d, T = 16, 64, 8 * 1374  # last wave KV-split, 2+ waves of dynamically claimed units
    q, k, v = (_rand((H, T, d), torch.bfloat16, seed=s) for s in (80, 81, 82))
    outs = []
    for _ in range(5):
        o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
        ops.attention(q, k, v, o, nseq=1, Lq=T, Lk=T)
        outs.append(o)
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("cfg_name,S", [("tiny", 6), ("1b", 2)])
def test_forward_bitwise_deterministic(cfg_name, S):
    from paper_2509_25191_b200.config import vggt_1b, vggt_tiny
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import synthetic_images
    cfg = vggt_tiny() if cfg_name == "tiny" else vggt_1b()
    m = VGGT(cfg)
    x = synthetic_images(cfg, S, 1).cuda()
    a, b = m(x), m(x)
    for key in ("pose_enc", "depth", "depth_conf", "world_points", "world_points_conf"):
        assert torch.equal(a[key], b[key]), key
