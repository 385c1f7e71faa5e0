"""Small workloads of the shipped kernels for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py tiny_forward
    cases: tiny_forward, agg1b_s2, attention_kvsplit, ring_merge, camera_head_1b, all

Each case runs the product library (paper_2509_25191_b200/libvx.so) and checks the result loosely so
a sanitizer run also shows the kernels computed something sensible.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def tiny_forward():
    from paper_2509_25191_b200.config import vggt_tiny
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import synthetic_images
    cfg = vggt_tiny()
    m = VGGT(cfg)
    out = m(synthetic_images(cfg, 5, 1).cuda())
    torch.cuda.synchronize()
    assert torch.isfinite(out["depth"]).all() and torch.isfinite(out["pose_enc"]).all()


def agg1b_s2():
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import synthetic_images
    cfg = vggt_1b()
    m = VGGT(cfg)
    kept, _ = m.aggregator(synthetic_images(cfg, 2, 1).cuda())
    torch.cuda.synchronize()
    assert all(torch.isfinite(t.float()).all() for t in kept.values())


def _sdpa_ref(q, k, v, nseq, L):
    H, T, d = q.shape
    qs, ks, vs = (t.float().view(H, nseq, L, d).transpose(0, 1) for t in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)  # (nseq, H, L, d)
    return o.permute(0, 2, 1, 3).reshape(nseq * L, H * d)


def attention_kvsplit():
    """A global layer whose last wave runs KV-split (8 views: 16 x 22 units = 2 waves + 56), plus the
    ragged frame attention of the 1B shape (1374 = 2 x 512 + 350)."""
    from paper_2509_25191_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(0)
    for nseq, L, glob in ((1, 8 * 1374, True), (3, 1374, False)):
        T = nseq * L
        q, k, v = (torch.randn(16, T, 64, device="cuda", generator=g).bfloat16() for _ in range(3))
        o = torch.empty(T, 1024, device="cuda", dtype=torch.bfloat16)
        ops.attention(q, k, v, o, nseq=nseq, Lq=L, Lk=L)
        ref = _sdpa_ref(q, k, v, nseq, L)
        err = ((o.float() - ref).norm() / ref.norm()).item()
        assert err < 1e-2, (glob, err)


def ring_merge():
    """Three ring steps (modes 1, 2, 3) over unequal K/V shards against monolithic attention."""
    from paper_2509_25191_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(1)
    H, d = 16, 64
    Lq, shards = 3000, (2100, 3000, 900)
    q = torch.randn(H, Lq, d, device="cuda", generator=g).bfloat16()
    ks = [torch.randn(H, n, d, device="cuda", generator=g).bfloat16() for n in shards]
    vs = [torch.randn(H, n, d, device="cuda", generator=g).bfloat16() for n in shards]
    o_acc = torch.empty(Lq, H * d, device="cuda")
    lse = torch.empty(H, Lq, device="cuda")
    out = torch.empty(Lq, H * d, device="cuda", dtype=torch.bfloat16)
    for i, (k, v) in enumerate(zip(ks, vs)):
        mode = 1 if i == 0 else (3 if i == len(shards) - 1 else 2)
        ops.attention_merge(q, k, v, mode, o_acc, lse, out=out, Lq=Lq, Lk=k.shape[1])
    kf, vf = torch.cat(ks, 1).float(), torch.cat(vs, 1).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), kf, vf).permute(1, 0, 2).reshape(Lq, H * d)
    err = ((out.float() - ref).norm() / ref.norm()).item()
    assert err < 1e-2, err


def camera_head_1b():
    from paper_2509_25191_b200.aggregator import DeviceWeights
    from paper_2509_25191_b200.config import vggt_1b
    from paper_2509_25191_b200.heads import camera_head
    from paper_2509_25191_b200.weights import make_state_dict
    cfg = vggt_1b()
    W = DeviceWeights(make_state_dict(cfg, 0), cfg, "cuda")
    outs = camera_head(W, torch.randn(37, 2048, device="cuda"))
    torch.cuda.synchronize()
    assert all(torch.isfinite(o).all() for o in outs)


CASES = {f.__name__: f for f in (tiny_forward, agg1b_s2, attention_kvsplit, ring_merge, camera_head_1b)}

if __name__ == "__main__":
    names = sys.argv[1:] or ["all"]
    if names == ["all"]:
        names = list(CASES)
    for n in names:
        CASES[n]()
        print(f"{n}: ok", flush=True)
