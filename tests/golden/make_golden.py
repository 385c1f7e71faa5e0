"""Generates tests/golden/tiny_s8.npz from the CPU oracle (configs[0]).

The reference holds no golden vectors for this path, so these
are this repo's own known-answer fixtures: weights seed 0, images seed 1,
fp32 CPU oracle.  Re-run: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.vggt_ref import vggt_forward  # noqa: E402
from paper_2509_25191_b200.config import vggt_tiny  # noqa: E402
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images  # noqa: E402


def main():
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    cfg = vggt_tiny()
    sd = make_state_dict(cfg, seed=0)
    images = synthetic_images(cfg, 8, seed=1)
    p = vggt_forward(images, sd, cfg)
    out = {f"kept_{i}": p["kept"][i].numpy() for i in cfg.kept_layers}
    for k in ("pose_enc", "depth", "depth_conf", "world_points", "world_points_conf"):
        out[k] = p[k][0].numpy()
    out["pose_enc_list"] = torch.stack([x[0] for x in p["pose_enc_list"]]).numpy()
    out["images_checksum"] = np.array([images.double().sum().item()])
    out["weights_checksum"] = np.array([sum(v.double().sum().item() for v in sd.values())])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tiny_s8.npz")
    np.savez_compressed(path, **out)
    print(path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
