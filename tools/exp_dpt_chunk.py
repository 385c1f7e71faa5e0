import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import sys, os, time, dataclasses
sys.path.insert(0, os.getcwd())
import torch
from paper_2509_25191_b200.config import vggt_1b
from paper_2509_25191_b200.vggt import VGGT
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images
from paper_2509_25191_b200 import profiling
S = 40
base = vggt_1b()
sd = make_state_dict(base, 0)
imgs = synthetic_images(base, S, 1).cuda()
for ch in (8, 16, 40):
    cfg = dataclasses.replace(base, head_chunk=ch)
    m = VGGT(cfg, state_dict=sd)
    m(imgs); torch.cuda.synchronize()
    t = profiling.PhaseTimer(); profiling.set_timer(t)
    m(imgs); m(imgs)
    profiling.set_timer(None)
    ph = t.summary()
    print(ch, {k: round(v["total_ms"] / 2, 2) for k, v in ph.items() if k in ("dpt_heads", "camera_head")}, round(torch.cuda.max_memory_allocated() / 1e9, 1))
    del m; torch.cuda.empty_cache(); torch.cuda.reset_peak_memory_stats()
