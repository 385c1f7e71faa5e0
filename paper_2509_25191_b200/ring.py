"""Frame-sharded global attention: K/V ring over NCCL P2P (SURVEY.md §5 ring notes, §8e).

Rank r owns views [floor(r*S/g), floor((r+1)*S/g)) and computes everything that
is per-frame locally (patch-embed, frame blocks, all GEMMs / norms of the global
blocks, kept layers, DPT heads).  The only exchange on the data path is inside
global attention: g-1 ring steps, each sending this rank's current K/V block
(one packed [2, H, Tmax, d] bf16 buffer) to rank r+1 and receiving the next one
from rank r-1 while the FMHA kernel works on the current block.  Each step's
(O, lse) for the local queries is merged into a running fp32 (O, lse) with the
log-sum-exp rule inside the FMHA epilogue (vx_attention_merge: no separate
merge kernels; the last step writes the bf16 output).  Because RoPE positions are per frame and attention is
non-causal, every step has identical work (no zig-zag needed).

Every rank passes the full view batch (or its own slice); frame 0 carries the
"first frame" special tokens, so only the rank that owns global frame 0 uses
them (aggregator.embed(frame0_is_first=...)).

The attention / merge functions are injectable so the ring schedule is tested
on CPU with gloo (tests/test_ring_cpu.py) against monolithic attention.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist

from .config import VGGTConfig


def frame_split(S: int, world: int) -> List[Tuple[int, int]]:
    return [((r * S) // world, ((r + 1) * S) // world) for r in range(world)]


def lse_merge(o_acc: torch.Tensor, lse_acc: torch.Tensor, o_s: torch.Tensor, lse_s: torch.Tensor):
    """In-place fp32 merge of a partial attention result.

    o_acc (T, H*d) fp32, lse_acc (H, T) fp32; o_s (T, H*d), lse_s (H, T).
    """
    H = lse_acc.shape[0]
    T = lse_acc.shape[1]
    new = torch.logaddexp(lse_acc, lse_s)
    wa = torch.exp(lse_acc - new).t().unsqueeze(-1)  # (T, H, 1)
    wb = torch.exp(lse_s - new).t().unsqueeze(-1)
    oa = o_acc.view(T, H, -1)
    oa.mul_(wa).add_(o_s.view(T, H, -1).float() * wb)
    lse_acc.copy_(new)


def _vx_partial(q, k, v, out, lse, Lq, Lk):
    from . import ops
    ops.attention(q, k, v, out, nseq=1, Lq=Lq, Lk=Lk, lse=lse)


class FrameShardedRing:
    def __init__(self, cfg: VGGTConfig, device, group=None,
                 partial_attention: Optional[Callable] = None, merge: Callable = lse_merge):
        if not dist.is_initialized():
            raise RuntimeError("FrameShardedRing needs torch.distributed to be initialised (torchrun)")
        self.cfg = cfg
        self.device = torch.device(device)
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # default: vx_attention_merge (LSE merge fused into the FMHA epilogue); injected functions are
        # for the CPU (gloo) tests of the ring schedule
        self.fused = partial_attention is None
        self.partial = partial_attention or _vx_partial
        self.merge = merge
        self.split: Optional[List[Tuple[int, int]]] = None

    # -- frame partition ---------------------------------------------------
    def local_frames(self, images: torch.Tensor, sharded_input: bool):
        if sharded_input:
            n = torch.tensor([images.shape[0]], device=self.device if self.device.type == "cuda" else "cpu")
            sizes = [torch.zeros_like(n) for _ in range(self.world)]
            dist.all_gather(sizes, n, group=self.group)
            sizes = [int(s.item()) for s in sizes]
            offs = [sum(sizes[:r]) for r in range(self.world)]
            self.split = [(offs[r], offs[r] + sizes[r]) for r in range(self.world)]
            lo, _ = self.split[self.rank]
            return images, lo, sum(sizes)
        S = images.shape[0]
        if S < self.world:
            raise ValueError(f"{S} views cannot be sharded over {self.world} ranks")
        self.split = frame_split(S, self.world)
        lo, hi = self.split[self.rank]
        return images[lo:hi], lo, S  # a view: a host batch stays (pinned) host memory until the copy

    def tokens_of(self, r: int) -> int:
        lo, hi = self.split[r]
        return (hi - lo) * self.cfg.tokens_per_frame

    # -- global attention --------------------------------------------------
    def global_attention(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor):
        """q/k/v: local [H, T_local, d] bf16; o: [T_local, H*d] bf16 (written)."""
        H, Tl, d = q.shape
        g, r = self.world, self.rank
        if g == 1:
            self.partial(q, k, v, o, None, Tl, Tl)
            return
        Tmax = max(self.tokens_of(i) for i in range(g))
        bufs = [torch.empty(2, H, Tmax, d, device=q.device, dtype=q.dtype) for _ in range(2)]
        bufs[0][0, :, :Tl].copy_(k)
        bufs[0][1, :, :Tl].copy_(v)
        if self.fused:
            o_acc = torch.empty(Tl, H * d, device=q.device, dtype=torch.float32)
            lse_acc = torch.empty(H, Tl, device=q.device, dtype=torch.float32)
        else:
            o_acc = torch.zeros(Tl, H * d, device=q.device, dtype=torch.float32)
            lse_acc = torch.full((H, Tl), float("-inf"), device=q.device, dtype=torch.float32)
            o_s = torch.empty(Tl, H * d, device=q.device, dtype=o.dtype)
            lse_s = torch.empty(H, Tl, device=q.device, dtype=torch.float32)
        nxt, prv = (r + 1) % g, (r - 1) % g
        cur = 0
        for step in range(g):
            src = (r - step) % g            # owner of the K/V block held in bufs[cur]
            reqs = []
            if step < g - 1:
                ops_ = [dist.P2POp(dist.isend, bufs[cur], nxt, group=self.group),
                        dist.P2POp(dist.irecv, bufs[cur ^ 1], prv, group=self.group)]
                reqs = dist.batch_isend_irecv(ops_)
            Lk = self.tokens_of(src)
            kb = bufs[cur][0]
            vb = bufs[cur][1]
            if self.fused:  # one launch: partial attention + running log-sum-exp merge (+ final bf16 write)
                from . import ops
                mode = 1 if step == 0 else (3 if step == g - 1 else 2)
                ops.attention_merge(q, kb, vb, mode, o_acc, lse_acc, out=o, Lq=Tl, Lk=Lk)
            else:
                self.partial(q, kb, vb, o_s, lse_s, Tl, Lk)
                self.merge(o_acc, lse_acc, o_s, lse_s)
            for rq in reqs:
                rq.wait()
            cur ^= 1
        if not self.fused:
            o.copy_(o_acc)

    # -- camera tokens -----------------------------------------------------
    def all_gather_frames(self, x: torch.Tensor) -> torch.Tensor:
        """(S_local, D) -> (S, D) in global frame order (unequal shards padded)."""
        sizes = [hi - lo for lo, hi in self.split]
        m = max(sizes)
        pad = torch.zeros(m, *x.shape[1:], device=x.device, dtype=x.dtype)
        pad[: x.shape[0]].copy_(x)
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)], dim=0)
