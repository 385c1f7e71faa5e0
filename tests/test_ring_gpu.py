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


@pytest.mark.gpu
def test_ring_over_nccl_loopback(tmp_path):
    """The ring's exchange through real NCCL P2P (ring.TorchDistComm, a world-size-1 group sending to
    itself; tests/nccl_loopback_worker.py): every virtual rank's merged output equals one attention
    call, over two layers, with the receive buffer zeroed before each transfer; and the whole
    VGGT(dist=True) forward over the same transport equals a single-GPU forward of rank 0's views."""
    import json
    import os
    import socket
    import subprocess
    import sys

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "loopback.json"
    env = dict(os.environ, OUT=str(out), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "nccl_loopback_worker.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert [c["world"] for c in res["ring"]] == [2, 3, 4]
    for c in res["ring"]:
        assert c["transfers"] == 2 * (c["world"] - 1), c  # g - 1 NCCL steps per layer, two layers
        assert max(c["rel_err"]) < 1e-2, c
    f = res["forward"]
    assert f["frame_offset"] == 0 and f["local_views"] == 3, f
    assert f["transfers"] == f["layers"], f  # one ring step per global layer at g = 2
    assert f["gathers"] >= 1, f  # the camera tokens
    for k in ("depth", "depth_conf", "world_points", "world_points_conf", "pose"):
        assert f[k] < 1e-2, (k, f)
    assert f["pose_copies"] < 1e-5, f
