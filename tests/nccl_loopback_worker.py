"""Worker for tests/test_ring_gpu.py::test_ring_over_nccl_loopback: the ring's global attention with its
K/V exchange going through real NCCL point-to-point transfers on one GPU.

NCCL needs one GPU per rank, so a multi-rank NCCL ring cannot run on a one-GPU box. What can run is
the same code path over a world-size-1 NCCL group in which rank 0 sends to itself: `LoopbackComm`
is ring.TorchDistComm (batch_isend_irecv of P2POps, NCCL stream ordering, work.wait()) that reports
a virtual rank r of g and delivers, at every ring step, this rank's own K/V block again. Attention
over g copies of one K/V block equals attention over the block once, so every virtual rank's merged
output must match a single ops.attention call. The receive buffer is zeroed before each transfer, so
a step whose FMHA read its block before the NCCL receive had landed would see zeros and fail.

The second half runs the whole sharded forward, VGGT(dist=True), over the same loopback (below).

Writes one JSON object to $OUT.
"""
import json
import math
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_25191_b200 import ops  # noqa: E402
from paper_2509_25191_b200.config import vggt_1b  # noqa: E402
from paper_2509_25191_b200.ring import FrameShardedRing, TorchDistComm  # noqa: E402


class LoopbackComm(TorchDistComm):
    def __init__(self, rank: int, world: int):
        super().__init__()
        if self.stage:
            raise RuntimeError("LoopbackComm needs the nccl backend")
        self.rank, self.world = rank, world
        self.transfers = 0
        self.gathers = 0

    def sendrecv(self, send, recv, to, frm):
        recv.zero_()  # on the current stream, before the NCCL receive is enqueued behind it
        self.transfers += 1
        return super().sendrecv(send, recv, 0, 0)

    def all_gather(self, outs, x):
        # a real NCCL all_gather over the one-rank group, its result handed to every virtual rank's slot
        got = [torch.zeros_like(x)]
        dist.all_gather(got, x)
        for o in outs:
            o.copy_(got[0])
        self.gathers += 1


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm()).item()


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    cfg = vggt_1b()
    H, d, N = cfg.num_heads, cfg.head_dim, cfg.tokens_per_frame
    gen = torch.Generator(device="cuda").manual_seed(0)
    res = []
    for g, vpr, q_log2 in ((2, 2, True), (3, 1, False), (4, 2, True)):
        T = vpr * N
        comm = LoopbackComm(g - 1, g)
        ring = FrameShardedRing(cfg, "cuda", comm=comm, q_log2=q_log2)
        ring.split = [(i * vpr, (i + 1) * vpr) for i in range(g)]
        ring.begin(H, d)
        errs = []
        for layer in range(2):  # two global layers: ring buffers and accumulators reused
            q, k, v = (torch.randn(H, T, d, device="cuda", generator=gen).bfloat16() for _ in range(3))
            if q_log2:  # as the aggregator's qkv epilogue stores it
                q = (q.float() * (math.log2(math.e) / math.sqrt(d))).bfloat16()
            o = torch.empty(T, H * d, device="cuda", dtype=torch.bfloat16)
            ring.global_attention(q, k, v, o)
            ref = torch.empty_like(o)
            ops.attention(q, k, v, ref, nseq=1, Lq=T, Lk=T, q_log2=q_log2)
            torch.cuda.synchronize()
            errs.append(rel(o, ref))
        res.append({"world": g, "views_per_rank": vpr, "q_log2": q_log2, "rel_err": errs,
                    "transfers": comm.transfers})
    # the whole sharded forward, VGGT(dist=True), as virtual rank 0 of 2 over 2 x 3 views: every ring step
    # and the camera-token gather deliver rank 0's own data again, and attention over duplicated keys equals
    # attention over them once, so rank 0's outputs equal a single-GPU forward of its 3 views, and the
    # gathered pose encodings repeat them
    from paper_2509_25191_b200.config import vggt_small
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    cfg = vggt_small().with_(init_values=0.5)
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 6, 1)
    ref = VGGT(cfg, state_dict=sd)(images[:3].cuda())
    comm = LoopbackComm(0, 2)
    out = VGGT(cfg, state_dict=sd, dist=True, comm=comm)(images)
    torch.cuda.synchronize()
    fwd = {k: rel(out[k][0], ref[k][0]) for k in ("depth", "depth_conf", "world_points", "world_points_conf")}
    fwd["pose"] = rel(out["pose_enc"][0, :3], ref["pose_enc"][0])
    fwd["pose_copies"] = rel(out["pose_enc"][0, 3:], out["pose_enc"][0, :3])
    fwd.update(frame_offset=out["frame_offset"], local_views=int(out["depth"].shape[1]),
               transfers=comm.transfers, gathers=comm.gathers, layers=cfg.depth)
    with open(os.environ["OUT"], "w") as f:
        json.dump({"ring": res, "forward": fwd}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
