"""The frame-sharded product path `VGGT(dist=True)` end to end, with g simulated ranks on one GPU.

A real multi-GPU run launches one process per B200 under torchrun and exchanges K/V blocks over NCCL
(ring.TorchDistComm).  This run has one GPU, so the g ranks run as g threads of one process, each with
its own VGGT instance and CUDA stream, and a thread communicator moves the ring blocks and the gathered
camera tokens between them: every exchange synchronises the sender's stream, hands the tensor over
through a barrier and copies it on the receiver's stream, so no rank's kernel ever waits on another
rank's kernel (the exchange is host-ordered, not overlapped).  Everything else — frame-0 token ownership,
the 2 x depth ring steps with the fused LSE merge, the camera-token all-gather, the per-rank DPT heads
and the global pose encoding — is the code a torchrun rank executes (alternating frame-wise
and global attention).

Checks: each rank's kept tokens, dense maps and confidences match the single-GPU forward's slice of the
same views within bf16 tolerance (the ring merges partial softmaxes in another order), and pose_enc is
bit-identical on every rank.
"""
import threading

import pytest
import torch

from paper_2509_25191_b200.config import vggt_small, vggt_tiny
from paper_2509_25191_b200.ring import frame_split
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images

pytestmark = pytest.mark.gpu


class ThreadHub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world, timeout=300)
        self.slots = [None] * world
        self.exchanges = 0


class ThreadComm:
    """rank / world / sendrecv / all_gather like ring.TorchDistComm, between threads of one process."""

    def __init__(self, hub: ThreadHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def sendrecv(self, send, recv, to, frm):
        torch.cuda.current_stream().synchronize()  # the block to send is complete
        self.hub.slots[to] = send
        self.hub.barrier.wait()
        recv.copy_(self.hub.slots[self.rank])  # the block rank `frm` sent to this rank
        torch.cuda.current_stream().synchronize()
        if self.rank == 0:
            self.hub.exchanges += 1
        self.hub.barrier.wait()  # every copy done before any sender reuses its buffer
        return []

    def all_gather(self, outs, x):
        torch.cuda.current_stream().synchronize()
        self.hub.slots[self.rank] = x
        self.hub.barrier.wait()
        for r, o in enumerate(outs):
            o.copy_(self.hub.slots[r].to(o.device))
        torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()


def rel(a, b):
    a, b = a.detach().float().cpu(), b.detach().float().cpu()
    return ((a - b).norm() / b.norm()).item()


def _sharded(cfg, sd, images, world, sharded_input=False):
    from paper_2509_25191_b200.vggt import VGGT
    hub = ThreadHub(world)
    res, errs = [None] * world, []
    split = frame_split(images.shape[0], world)

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                m = VGGT(cfg, state_dict=sd, dist=True, comm=ThreadComm(hub, r))
                x = images[split[r][0]:split[r][1]] if sharded_input else images
                out = m(x, sharded_input=sharded_input)
                kept, psi = m.aggregator(x, sharded_input=sharded_input)
                torch.cuda.current_stream().synchronize()
                res[r] = (out, kept)
        except BaseException as e:  # noqa: BLE001 - re-raised in the main thread
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res, hub, split


@pytest.mark.parametrize("cfg_name,world,S", [("tiny", 2, 5), ("tiny", 3, 4), ("small", 3, 7), ("small", 2, 6)])
def test_sharded_forward_matches_single_gpu(cfg_name, world, S):
    from paper_2509_25191_b200.vggt import VGGT
    cfg = vggt_tiny() if cfg_name == "tiny" else vggt_small().with_(init_values=0.5)
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, S, 1)  # host batch: every rank copies only its own frames
    single = VGGT(cfg, state_dict=sd)
    ref = single(images.cuda())
    ref_kept, _ = single.aggregator(images.cuda())
    res, hub, split = _sharded(cfg, sd, images, world)
    assert hub.exchanges == 2 * cfg.depth * (world - 1)  # forward + aggregator: g - 1 ring steps per global layer
    pose0 = res[0][0]["pose_enc"]
    C = cfg.embed_dim
    for r, (out, kept) in enumerate(res):
        lo, hi = split[r]
        assert out["frame_offset"] == lo
        assert torch.equal(out["pose_enc"], pose0), r  # global, identical on every rank
        assert out["depth"].shape[1] == hi - lo
        for i in cfg.kept_layers:
            got, want = kept[i][0], ref_kept[i][0, lo:hi]
            assert got.shape == want.shape
            assert rel(got[..., :C], want[..., :C]) < 1e-2, (r, i)
            assert rel(got[..., C:], want[..., C:]) < 1e-2, (r, i)
        for k in ("depth", "depth_conf", "world_points", "world_points_conf"):
            assert rel(out[k][0], ref[k][0, lo:hi]) < 1e-2, (r, k)
    assert rel(pose0, ref["pose_enc"]) < 1e-2


def test_sharded_input_unequal_shards():
    """Each rank passes only its own views (sharded_input=True) with unequal shard sizes."""
    from paper_2509_25191_b200.vggt import VGGT
    cfg = vggt_tiny()
    sd = make_state_dict(cfg, 0)
    images = synthetic_images(cfg, 7, 1)
    ref = VGGT(cfg, state_dict=sd)(images.cuda())
    res, _, split = _sharded(cfg, sd, images, 3, sharded_input=True)
    for r, (out, _) in enumerate(res):
        lo, hi = split[r]
        assert rel(out["depth"][0], ref["depth"][0, lo:hi]) < 1e-2
        assert torch.equal(out["pose_enc"], res[0][0]["pose_enc"])
