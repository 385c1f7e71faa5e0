"""Builds the reference's own native GA kernel into oracle/_ref/ (TEST INFRASTRUCTURE ONLY).

The reference's only compiled component is the Cython module
pkg/src/epialign/_kernels_cy.pyx (pair_residuals / pair_accumulate).  This recipe translates it
with Cython and compiles the generated C with gcc, reading the source where it lies under
/root/reference and writing only into oracle/_ref/ (git-ignored; it travels to the GPU box with
the snapshot).  It is used by tests/test_epipolar.py to check the numpy restatement
(oracle/epipolar_ref.py) against the real reference implementation, and by tools/bench_ga.py as
the reference CPU baseline of the per-pair kernels.  It is never imported by the product.

    python -m oracle.build_ref        # no-op when /root/reference is absent
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

SRC = Path("/root/reference/pkg/src/epialign/_kernels_cy.pyx")
OUT = Path(__file__).resolve().parent / "_ref"
SUFFIX = sysconfig.get_config_var("EXT_SUFFIX") or ".so"


def target() -> Path:
    return OUT / f"_kernels_cy{SUFFIX}"


def build(force: bool = False) -> Path | None:
    if not SRC.exists():
        return None
    so = target()
    if so.exists() and not force and so.stat().st_mtime >= SRC.stat().st_mtime:
        return so
    import numpy as np
    from Cython.Build import cythonize  # noqa: F401  (presence check)

    OUT.mkdir(exist_ok=True)
    c_file = OUT / "_kernels_cy.c"
    subprocess.run([sys.executable, "-m", "cython", "-3", "-o", str(c_file), str(SRC)], check=True,
                   capture_output=True)
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-fno-strict-aliasing", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
           *[f"-I{i}" for i in inc], str(c_file), "-o", str(so), "-lm"]
    subprocess.run(cmd, check=True, capture_output=True)
    c_file.unlink()  # keep only the binary
    return so


def load():
    """Import the compiled reference module from oracle/_ref (None when it was not built)."""
    so = target()
    if not so.exists():
        return None
    import importlib.util
    spec = importlib.util.spec_from_file_location("_kernels_cy", so)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    p = build(force="--force" in sys.argv)
    print(p if p else "reference sources absent: nothing to build")
