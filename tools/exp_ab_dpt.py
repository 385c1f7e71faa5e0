"""A/B of two library builds (VX_LIB) on the DPT heads phase at 20 / 200 views (heads on side streams)."""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2509_25191_b200.config import vggt_1b
from paper_2509_25191_b200.vggt import VGGT
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
from paper_2509_25191_b200 import profiling
cfg = vggt_1b()
m = VGGT(cfg, state_dict=make_state_dict(cfg, 0))
for S in (20, 200):
    imgs = synthetic_images(cfg, S, 1).cuda()
    m(imgs); torch.cuda.synchronize()
    t = profiling.PhaseTimer(); profiling.set_timer(t)
    m(imgs); m(imgs)
    profiling.set_timer(None)
    print(os.environ.get("VX_LIB", "default")[-12:], S, round(t.summary()["heads"]["total_ms"] / 2, 2))
