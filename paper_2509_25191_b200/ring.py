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

Memory: the two packed ring buffers and the fp32 (O, lse) accumulators are
allocated once per forward (`begin`), and the QKV GEMM epilogue of every block
writes this rank's K/V straight into ring buffer 0 (`kv_buffers`), so a global
layer starts its first ring step without a copy.  The FMHA hands out its work
units through an atomic ticket counter, so the SMs an NCCL transfer kernel
occupies at the start of a ring step only delay the units they would have run.

Every rank passes the full view batch (or its own slice); frame 0 carries the
"first frame" special tokens, so only the rank that owns global frame 0 uses
them (aggregator.embed(frame0_is_first=...)).

The communicator (`TorchDistComm`: torch.distributed, NCCL on B200) and the
attention / merge functions are injectable, so the ring schedule is tested on
CPU with gloo (tests/test_ring_cpu.py) and the whole sharded forward with g
simulated ranks in threads on one GPU (tests/test_sharded_forward.py).
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


class TorchDistComm:
    """The ring's exchange over torch.distributed (NCCL P2P on B200, gloo in the CPU tests)."""

    def __init__(self, group=None):
        if not dist.is_initialized():
            raise RuntimeError("FrameShardedRing needs torch.distributed to be initialised (torchrun)")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves host memory only: device tensors are staged through host copies (synchronous);
        # NCCL (the B200 path) exchanges device memory directly and asynchronously
        self.stage = dist.get_backend(group) != "nccl"

    def sendrecv(self, send: torch.Tensor, recv: torch.Tensor, to: int, frm: int) -> list:
        """Start sending `send` to rank `to` and receiving `recv` from rank `frm`; returns requests to
        wait() on (torch orders the NCCL stream after the current stream at issue, and wait() orders
        the current stream after the transfer)."""
        if self.stage and send.is_cuda:
            hs, hr = send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)
            for q in dist.batch_isend_irecv([dist.P2POp(dist.isend, hs, to, group=self.group),
                                             dist.P2POp(dist.irecv, hr, frm, group=self.group)]):
                q.wait()
            recv.copy_(hr)
            return []
        ops_ = [dist.P2POp(dist.isend, send, to, group=self.group),
                dist.P2POp(dist.irecv, recv, frm, group=self.group)]
        return dist.batch_isend_irecv(ops_)

    def all_gather(self, outs: List[torch.Tensor], x: torch.Tensor) -> None:
        if self.stage and x.is_cuda:
            houts = [torch.empty(o.shape, dtype=o.dtype) for o in outs]
            dist.all_gather(houts, x.cpu(), group=self.group)
            for o, h in zip(outs, houts):
                o.copy_(h)
            return
        dist.all_gather(outs, x, group=self.group)


class FrameShardedRing:
    def __init__(self, cfg: VGGTConfig, device, group=None, comm=None,
                 partial_attention: Optional[Callable] = None, merge: Callable = lse_merge, q_log2: bool = False):
        self.cfg = cfg
        self.device = torch.device(device)
        self.comm = comm if comm is not None else TorchDistComm(group)
        self.rank = self.comm.rank
        self.world = self.comm.world
        # default: vx_attention_merge (LSE merge fused into the FMHA epilogue); injected functions are
        # for the CPU (gloo) tests of the ring schedule
        self.fused = partial_attention is None
        # q arrives pre-scaled by log2(e)/sqrt(d) (VGGT's aggregator); only the fused vx path reads it so
        if q_log2 and not self.fused:
            raise ValueError("q_log2 needs the fused vx ring step (no partial_attention)")
        self.q_log2 = q_log2
        self.partial = partial_attention or _vx_partial
        self.merge = merge
        self.split: Optional[List[Tuple[int, int]]] = None
        self._bufs = None  # (ring buffers [2, 2, H, Tmax, d], o_acc, lse_acc) of the current forward

    # -- frame partition ---------------------------------------------------
    def local_frames(self, images: torch.Tensor, sharded_input: bool):
        if sharded_input:
            n = torch.tensor([images.shape[0]], device=self.device if self.device.type == "cuda" else "cpu")
            sizes = [torch.zeros_like(n) for _ in range(self.world)]
            self.comm.all_gather(sizes, n)
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

    @property
    def rows_per_head(self) -> int:
        """Tmax: rows per head of the packed ring blocks (the largest shard's tokens)."""
        return max(self.tokens_of(i) for i in range(self.world))

    # -- per-forward buffers -------------------------------------------------
    def begin(self, H: Optional[int] = None, d: Optional[int] = None, dtype=torch.bfloat16):
        """Allocate (or reuse, when the shapes did not change) the two packed ring buffers and the fp32
        accumulators for this forward's shard."""
        H = H or self.cfg.num_heads
        d = d or self.cfg.head_dim
        Tmax, Tl = self.rows_per_head, self.tokens_of(self.rank)
        shape = (2, 2, H, Tmax, d)
        if (self._bufs is None or tuple(self._bufs[0].shape) != shape or self._bufs[0].dtype != dtype
                or self._bufs[1].shape[0] != Tl):
            bufs = torch.empty(shape, device=self.device, dtype=dtype)
            o_acc = torch.empty(Tl, H * d, device=self.device, dtype=torch.float32)
            lse_acc = torch.empty(H, Tmax, device=self.device, dtype=torch.float32)
            self._bufs = (bufs, o_acc, lse_acc)
        return self._bufs

    def kv_buffers(self) -> Tuple[torch.Tensor, torch.Tensor]:
        """K and V of ring buffer 0 ([H, Tmax, d] each): the QKV epilogue writes the local K/V here."""
        bufs = self._bufs[0]
        return bufs[0, 0], bufs[0, 1]

    # -- global attention --------------------------------------------------
    def global_attention(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor):
        """q/k/v: local [H, R, d] bf16 (rows 0..T_local-1 of each head valid, R >= T_local);
        o: [T_local, H*d] bf16 (written)."""
        H, _, d = q.shape
        g, r = self.world, self.rank
        Tl = self.tokens_of(r)
        if g == 1:
            if self.fused:
                from . import ops
                ops.attention(q, k, v, o, nseq=1, Lq=Tl, Lk=Tl, q_log2=self.q_log2)
            else:
                self.partial(q, k, v, o, None, Tl, Tl)
            return
        bufs, o_acc, lse_acc = self.begin(H, d, q.dtype)  # no-op after VGGT._aggregate's begin()
        if k.data_ptr() != bufs[0, 0].data_ptr():  # K/V not produced in place (tests, custom callers)
            bufs[0, 0, :, :Tl].copy_(k[:, :Tl])
            bufs[0, 1, :, :Tl].copy_(v[:, :Tl])
        if not self.fused:
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
                reqs = self.comm.sendrecv(bufs[cur], bufs[cur ^ 1], nxt, prv)
            Lk = self.tokens_of(src)
            kb = bufs[cur, 0]
            vb = bufs[cur, 1]
            if self.fused:  # one launch: partial attention + running log-sum-exp merge (+ final bf16 write)
                from . import ops
                mode = 1 if step == 0 else (3 if step == g - 1 else 2)
                ops.attention_merge(q, kb, vb, mode, o_acc, lse_acc, out=o, Lq=Tl, Lk=Lk, q_log2=self.q_log2)
            else:
                self.partial(q[:, :Tl], kb, vb, o_s, lse_s, Tl, Lk)
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
        self.comm.all_gather(outs, pad)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)], dim=0)
