"""cProfile of ga.align_arrays at the bench_ga scene: where the host time of one align call goes."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import torch  # noqa: E402

import bench_ga  # noqa: E402
from paper_2509_25191_b200 import ga  # noqa: E402

R, t, intr, pij, off, xi, xj = bench_ga.scene(200, 20000, 30.0, 4096)
cfg = ga.AlignerConfig()
ga.align_arrays(R, t, intr, pij, off, xi, xj, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
ga.align_arrays(R, t, intr, pij, off, xi, xj, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
