"""Imported by diagnostic tools: `VX_LIB=<path>` binds paper_2509_25191_b200.ops to another build of
libvx (e.g. the -DVX_DIAG library from paper_2509_25191_b200.build.build_diag, which honours the
VX_FMHA_CFG / VX_FMHA_EMU / VX_FMHA_SPLIT / VX_GEMM_PAIR variant switches).  The product library has
no run-time variant switches and the product path never reads VX_LIB."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

if os.environ.get("VX_LIB"):
    from paper_2509_25191_b200 import ops

    ops.use_library(os.environ["VX_LIB"])
