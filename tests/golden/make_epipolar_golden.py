"""Generates tests/golden/epipolar.npz from the REFERENCE's own numpy kernels.

Imports epialign._kernels_np from /root/reference/pkg/src (read-only; available in
the build container only) and records inputs + outputs for: random workloads in
both modes (pkg/tests/test_kernels.py:_workload), degenerate lines (F = e3 e3^T,
test_kernels.py:48-61) and the gradient dead zone (points on their epipolar lines,
test_kernels.py:64-87).  Re-run: python tests/golden/make_epipolar_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from epialign import _kernels_np as ref  # noqa: E402


def workload(rng, k):
    F = rng.normal(size=(3, 3))
    F /= np.linalg.norm(F)
    xi = rng.uniform(0, 640, size=(k, 2))
    xj = rng.uniform(0, 480, size=(k, 2))
    w = rng.uniform(0.1, 2.0, size=k)
    return F, xi, xj, w


def main():
    rng = np.random.default_rng(20250925)
    Fs, xis, xjs, ws, offs = [], [], [], [], [0]
    for p in range(24):
        k = int(rng.integers(1, 700)) if p % 6 else 500
        F, xi, xj, w = workload(rng, k)
        if p == 5:  # degenerate: every epipolar line has a zero image-plane normal
            F = np.zeros((3, 3))
            F[2, 2] = 1.0
        if p == 7:  # dead zone: put x' on its epipolar line
            lines = np.c_[xi, np.ones(k)] @ F.T
            t = rng.uniform(0, 1, size=k)
            for m in range(k):
                a, b, c = lines[m]
                if abs(b) > abs(a):
                    x = t[m] * 100.0
                    xj[m] = [x, -(a * x + c) / b]
                else:
                    y = t[m] * 100.0
                    xj[m] = [-(b * y + c) / a, y]
        if p == 11:  # partial degeneracy: some lines through the image-plane origin direction
            F[0, :] = 0.0
            F[1, :] = 0.0
            F[0, 2] = 1e-13
        Fs.append(F)
        xis.append(xi)
        xjs.append(xj)
        ws.append(w)
        offs.append(offs[-1] + k)
    out = {"F": np.stack(Fs), "offsets": np.array(offs, dtype=np.int64), "xy_i": np.concatenate(xis),
           "xy_j": np.concatenate(xjs), "w": np.concatenate(ws)}
    for mode in (0, 1):
        es, nd, acc, sk = [], [], [], []
        for p in range(len(Fs)):
            a, b = offs[p], offs[p + 1]
            e, n = ref.pair_residuals(Fs[p], out["xy_i"][a:b], out["xy_j"][a:b], mode)
            l, wsum, G, s = ref.pair_accumulate(Fs[p], out["xy_i"][a:b], out["xy_j"][a:b], out["w"][a:b], mode)
            es.append(e)
            nd.append(n)
            acc.append(np.r_[l, wsum, G.reshape(-1)])
            sk.append(s)
        out[f"e_{mode}"] = np.concatenate(es)
        out[f"ndeg_{mode}"] = np.array(nd)
        out[f"acc_{mode}"] = np.stack(acc)
        out[f"skip_{mode}"] = np.array(sk)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "epipolar.npz")
    np.savez_compressed(path, **out)
    print(path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
