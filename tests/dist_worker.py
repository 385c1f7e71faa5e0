"""Worker for tests/test_multirank.py, launched by torch.distributed.run: the frame-sharded product
path through the real torch.distributed API (ring.TorchDistComm) with the gloo backend, so several
ranks can share one GPU (the exchange is staged through host memory; NCCL needs one GPU per rank).
Every rank compares its slice of the sharded forward with a single-process forward of the same views
and writes a JSON line to $OUT.<rank>."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm()).item()


def main():
    from paper_2509_25191_b200.config import vggt_small
    from paper_2509_25191_b200.ring import frame_split
    from paper_2509_25191_b200.vggt import VGGT
    from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
    dist.init_process_group("gloo")
    r, g = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cfg = vggt_small().with_(init_values=0.5)
    sd = make_state_dict(cfg, 0)
    S = int(os.environ.get("VIEWS", "7"))
    images = synthetic_images(cfg, S, 1)
    ref = VGGT(cfg, state_dict=sd)(images.cuda())
    m = VGGT(cfg, state_dict=sd, dist=True)
    out = m(images)
    lo, hi = frame_split(S, g)[r]
    res = {"rank": r, "world": g, "frame_offset": out["frame_offset"], "lo": lo, "hi": hi,
           "pose": out["pose_enc"].cpu().flatten().tolist()}
    for k in ("depth", "depth_conf", "world_points", "world_points_conf"):
        res[k] = rel(out[k][0], ref[k][0, lo:hi])
    res["pose_vs_single"] = rel(out["pose_enc"], ref["pose_enc"])
    with open(f"{os.environ['OUT']}.{r}", "w") as f:
        json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
