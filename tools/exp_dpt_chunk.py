"""DPT head chunk size sweep: heads-phase time (camera head concurrent with both DPT heads on side
streams) and peak HBM at S views.

    python tools/exp_dpt_chunk.py [S] [chunk ...]
"""
import _vxdiag  # noqa: F401  (VX_LIB=<path> binds a -DVX_DIAG build)
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_25191_b200 import profiling  # noqa: E402
from paper_2509_25191_b200.config import vggt_1b  # noqa: E402
from paper_2509_25191_b200.vggt import VGGT  # noqa: E402
from paper_2509_25191_b200.weights import make_state_dict, synthetic_images  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 40
chunks = [int(c) for c in sys.argv[2:]] or [8, 16, 32]
base = vggt_1b()
sd = make_state_dict(base, 0)
imgs = synthetic_images(base, S, 1).cuda()
for rep in range(2):
    for ch in chunks:
        cfg = dataclasses.replace(base, head_chunk=ch)
        m = VGGT(cfg, state_dict=sd)
        m(imgs)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        t = profiling.PhaseTimer()
        profiling.set_timer(t)
        m(imgs)
        m(imgs)
        profiling.set_timer(None)
        ph = t.summary()
        print(rep, ch, round(ph["heads"]["total_ms"] / 2, 2), "ms heads,", round(torch.cuda.max_memory_allocated() / 1e9, 1),
              "GB peak", flush=True)
        del m
        torch.cuda.empty_cache()
