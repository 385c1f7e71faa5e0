"""The frame-sharded ring's fused-merge path (vx_attention_merge) on one GPU.

The NCCL exchange cannot run on a single device, so the g ranks are simulated one after another in
this process: `torch.distributed` is replaced by a stand-in whose batched send/recv hands rank r,
at ring step s, the K/V block that rank r - s - 1 owns — exactly what the real ring delivers.
Each simulated rank's output must equal monolithic attention over all views (this is the code path
`VGGT(dist=True)` runs on every rank of a multi-GPU box).
"""
import math

import pytest
import torch


class _FakeDist:
    """Minimal torch.distributed stand-in for one simulated rank of a g-rank ring."""

    def __init__(self, rank, world, blocks):
        self.rank, self.world, self.blocks = rank, world, blocks
        self.step = 0

    def is_initialized(self):
        return True

    def get_rank(self, group=None):
        return self.rank

    def get_world_size(self, group=None):
        return self.world

    def get_backend(self, group=None):
        return "nccl"  # device tensors go through P2POp directly (no host staging)

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            self.op, self.tensor, self.peer = op, tensor, peer

    def isend(self, *a, **k):
        pass

    def irecv(self, *a, **k):
        pass

    def batch_isend_irecv(self, ops):
        recv = [o for o in ops if o.op == self.irecv][0]
        src = (self.rank - self.step - 1) % self.world   # block held by the previous rank after this step
        k, v = self.blocks[src]
        n = k.shape[1]
        recv.tensor.zero_()
        recv.tensor[0, :, :n].copy_(k)
        recv.tensor[1, :, :n].copy_(v)
        self.step += 1

        class _Req:
            def wait(self):
                pass
        return [_Req()]


@pytest.mark.gpu
@pytest.mark.parametrize("S,world", [(6, 2), (7, 3), (9, 4)])
def test_ring_fused_merge_matches_global_attention(S, world, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2509_25191_b200 import ring as ring_mod
    from paper_2509_25191_b200.config import vggt_tiny

    cfg = vggt_tiny()
    N, H, d = cfg.tokens_per_frame, 2, 64
    T = S * N
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = ((torch.randn(H, T, d, device="cuda", generator=g)).bfloat16() for _ in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
    ref = ref.permute(1, 0, 2).reshape(T, H * d)
    split = ring_mod.frame_split(S, world)
    blocks = [(k[:, lo * N:hi * N].contiguous(), v[:, lo * N:hi * N].contiguous()) for lo, hi in split]
    for rank in range(world):
        fake = _FakeDist(rank, world, blocks)
        monkeypatch.setattr(ring_mod, "dist", fake)
        ring = ring_mod.FrameShardedRing(cfg, "cuda")
        assert ring.fused
        ring.split = split
        lo, hi = split[rank]
        sl = slice(lo * N, hi * N)
        o = torch.empty(hi * N - lo * N, H * d, device="cuda", dtype=torch.bfloat16)
        ring.global_attention(q[:, sl].contiguous(), k[:, sl].contiguous(), v[:, sl].contiguous(), o)
        err = ((o.float() - ref[sl]).norm() / ref[sl].norm()).item()
        assert err < 1e-2, (rank, err)
        assert fake.step == world - 1
