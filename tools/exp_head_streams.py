"""DPT heads on two streams vs sequential (VX_HEAD_STREAMS), 20 and 200 views."""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2509_25191_b200.config import vggt_1b
from paper_2509_25191_b200.vggt import VGGT
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
from paper_2509_25191_b200 import profiling
cfg = vggt_1b()
sd = make_state_dict(cfg, 0)
m = VGGT(cfg, state_dict=sd)
for S in (20, 200):
    imgs = synthetic_images(cfg, S, 1).cuda()
    for hs in (False, True, False, True):
        m.head_streams = hs
        m(imgs); torch.cuda.synchronize()
        t = profiling.PhaseTimer(); profiling.set_timer(t)
        m(imgs)
        profiling.set_timer(None)
        print(S, "two streams" if hs else "sequential", round(t.summary()["dpt_heads"]["total_ms"], 2))
