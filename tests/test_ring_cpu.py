"""Frame-sharded ring schedule on CPU with gloo (world_size 2 and 3).

The ring (paper_2509_25191_b200/ring.py) is run with an injected fp32 torch
partial-attention function instead of the sm_100a kernel; the merged result
must equal monolithic global attention over all views, and the frame split /
camera-token all-gather must reproduce the global order.
"""
import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torch_partial(q, k, v, out, lse, Lq, Lk):
    H, _, d = q.shape
    s = torch.einsum("hqd,hkd->hqk", q[:, :Lq].float(), k[:, :Lk].float()) / math.sqrt(d)
    if lse is not None:
        lse.copy_(torch.logsumexp(s, -1))
    o = torch.einsum("hqk,hkd->hqd", s.softmax(-1), v[:, :Lk].float())
    out.copy_(o.permute(1, 0, 2).reshape(Lq, H * d))


def _worker(rank, world, port, S, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_25191_b200.config import vggt_tiny
        from paper_2509_25191_b200.ring import FrameShardedRing, frame_split
        cfg = vggt_tiny()
        N = cfg.tokens_per_frame
        H, d = 2, 8
        g = torch.Generator().manual_seed(0)
        T = S * N
        q, k, v = (torch.randn(H, T, d, generator=g) for _ in range(3))
        ring = FrameShardedRing(cfg, "cpu", partial_attention=_torch_partial)
        images = torch.arange(S, dtype=torch.float32).view(S, 1, 1, 1).expand(S, 3, 2, 2)
        local, f0, S_all = ring.local_frames(images, sharded_input=False)
        lo, hi = frame_split(S, world)[rank]
        assert f0 == lo and S_all == S and local.shape[0] == hi - lo
        assert torch.equal(local[:, 0, 0, 0], torch.arange(lo, hi, dtype=torch.float32))
        sl = slice(lo * N, hi * N)
        ql, kl, vl = (t[:, sl].contiguous() for t in (q, k, v))
        o = torch.empty(ql.shape[1], H * d)
        ring.global_attention(ql, kl, vl, o)
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v).permute(1, 0, 2).reshape(T, H * d)[sl]
        err = ((o - ref).norm() / ref.norm()).item()
        cam = local[:, 0, 0, 0].reshape(-1, 1).repeat(1, 4).contiguous()
        gathered = ring.all_gather_frames(cam)
        ok_gather = torch.equal(gathered[:, 0], torch.arange(S, dtype=torch.float32))
        result_q.put((rank, err, ok_gather))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,S", [(2, 4), (2, 5), (3, 7)])
def test_ring_matches_monolithic(world, S):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, ok in res:
        assert err < 1e-5, (rank, err)
        assert ok, rank


def test_frame_split_partitions():
    from paper_2509_25191_b200.ring import frame_split
    for S in (1, 7, 200, 1000, 1001):
        for g in (1, 2, 3, 8):
            if S < g:
                continue
            sp = frame_split(S, g)
            assert sp[0][0] == 0 and sp[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(sp, sp[1:]))
            sizes = [h - l for l, h in sp]
            assert max(sizes) - min(sizes) <= 1
