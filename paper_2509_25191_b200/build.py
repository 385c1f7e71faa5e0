"""Builds the in-tree C-ABI library `libvx.so` (sm_100a) with nvcc.

The library is compiled in place (next to this file) so it travels to the GPU
box with the repo snapshot; there is no JIT cache and no torch extension.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libvx.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", str(ROOT / "include")]


def sources():
    return sorted(CSRC.glob("*.cu"))


def headers():
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted((ROOT / "include").glob("*.h"))


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in sources() + headers())


# per-file flags: the fp64 GA kernels follow the reference's un-fused double arithmetic
# (pkg/src/epialign/_kernels_cy.pyx is compiled without FMA contraction on x86-64)
EXTRA = {"epipolar.cu": ["-fmad=false"], "ga.cu": ["-fmad=false"], "scene.cu": ["-fmad=false"]}


def _compile_one(src: Path, obj: Path, log):
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA.get(src.name, []), "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.write(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}\n")
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-4000:]}")


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor
    logpath = objdir / "nvcc.log"
    with open(logpath, "w") as log:
        objs = [objdir / (s.stem + ".o") for s in sources()]
        newest_header = max((p.stat().st_mtime for p in headers()), default=0.0)
        build_py = Path(__file__).stat().st_mtime

        def stale(src, obj):  # per-object rebuild: source, any header or this recipe newer than the object
            return force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_header,
                                                                          build_py)

        todo = [(s, o) for s, o in zip(sources(), objs) if stale(s, o)]
        with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            list(ex.map(lambda so: _compile_one(so[0], so[1], log), todo))
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.write(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}\n")
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, LIB)
    if verbose:
        print(logpath.read_text())
    return LIB


def build_diag(out: Path = ROOT / "exp" / "libvx_diag.so", defines=("VX_DIAG",)) -> Path:
    """The diagnostic library for tools/ (`-DVX_DIAG`: the run-time kernel-variant switches
    VX_FMHA_CFG / VX_FMHA_EMU / VX_FMHA_SPLIT / VX_GEMM_PAIR of DESIGN.md's A/B measurements).
    Never loaded by the product path; tools bind it with ops.use_library(path)."""
    out.parent.mkdir(parents=True, exist_ok=True)
    objdir = out.parent / (out.stem + "_obj")
    objdir.mkdir(exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    objs = []
    with open(objdir / "nvcc.log", "w") as log:
        for src in sources():
            obj = objdir / (src.stem + ".o")
            cmd = [NVCC, *ARCH, *FLAGS, *dflags, *EXTRA.get(src.name, []), "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log.write(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}\n")
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-4000:]}")
            objs.append(obj)
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr[-4000:]}")
    for o in objs:
        o.unlink()
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
