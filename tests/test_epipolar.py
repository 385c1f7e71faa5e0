"""GA epipolar kernels: oracle pinned to the reference's own outputs,
CUDA path against the pinned oracle with the reference's tolerances
(pkg/tests/test_kernels.py:20-110): residuals rtol 1e-12 / atol 1e-15, loss and
weight sums rtol 1e-12, gradient rtol 1e-9 / atol 1e-12, degenerate lines and
dead zone exact, gradient vs central finite differences."""
import os

import numpy as np
import pytest

from oracle import epipolar_ref as R

GOLD = os.path.join(os.path.dirname(__file__), "golden", "epipolar.npz")
DEADZONE_PAIR = 7  # x' placed on its epipolar line: residuals are rounding noise (< 1e-9)


def _check_pair(p, g, mode, e, nd, l, ws, G, sk, a, b):
    ref = g[f"acc_{mode}"][p]
    assert nd == g[f"ndeg_{mode}"][p] and sk == g[f"skip_{mode}"][p]
    assert np.isclose(ws, ref[1], rtol=1e-12, atol=1e-300)
    if p == DEADZONE_PAIR:
        # reference semantics (pkg/tests/test_kernels.py:64-87): loss kept (~0), zero subgradient
        assert np.nanmax(e) < 1e-9 and l < 1e-8 and np.all(G == 0.0) and np.all(ref[2:] == 0.0)
        return
    assert np.allclose(e, g[f"e_{mode}"][a:b], rtol=1e-12, atol=1e-15, equal_nan=True)
    assert np.isclose(l, ref[0], rtol=1e-12, atol=1e-300)
    assert np.allclose(np.reshape(G, -1), ref[2:], rtol=1e-9, atol=1e-12)
REF_SRC = "/root/reference/pkg/src"


def _pairs(g):
    off = g["offsets"]
    for p in range(g["F"].shape[0]):
        a, b = off[p], off[p + 1]
        yield p, g["F"][p], g["xy_i"][a:b], g["xy_j"][a:b], g["w"][a:b], (a, b)


@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_matches_reference_golden(mode):
    g = np.load(GOLD)
    for p, F, xi, xj, w, (a, b) in _pairs(g):
        e, nd = R.pair_residuals(F, xi, xj, mode)
        l, ws, G, sk = R.pair_accumulate(F, xi, xj, w, mode)
        _check_pair(p, g, mode, e, nd, l, ws, G, sk, a, b)


def _compiled_reference():
    from oracle import build_ref
    build_ref.build()  # no-op when the sources are absent or the binary is current
    return build_ref.load()


@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_matches_compiled_reference_kernel(mode):
    """The restatement against the reference's own compiled Cython kernel (oracle/_ref, built from
    pkg/src/epialign/_kernels_cy.pyx by oracle/build_ref.py): residuals bit-identical, sums to
    rounding, on random workloads, degenerate lines and the dead zone."""
    cy = _compiled_reference()
    if cy is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    assert cy.IMPL == "compiled"
    rng = np.random.default_rng(11)
    g = np.load(GOLD)
    cases = [(F, xi, xj, w) for _, F, xi, xj, w, _ in _pairs(g)]
    for _ in range(6):
        F = rng.normal(size=(3, 3))
        F /= np.linalg.norm(F)
        k = int(rng.integers(1, 900))
        cases.append((F, rng.uniform(0, 640, (k, 2)), rng.uniform(0, 480, (k, 2)), rng.uniform(0.1, 2, k)))
    for F, xi, xj, w in cases:
        F, xi, xj, w = (np.ascontiguousarray(x, dtype=np.float64) for x in (F, xi, xj, w))
        e0, n0 = cy.pair_residuals(F, xi, xj, mode)
        e1, n1 = R.pair_residuals(F, xi, xj, mode)
        assert n0 == n1
        assert np.array_equal(np.isnan(e0), np.isnan(e1))
        assert np.array_equal(e0[~np.isnan(e0)], e1[~np.isnan(e1)])  # same formulas, same rounding
        l0, ws0, G0, sk0 = cy.pair_accumulate(F, xi, xj, w, mode)
        l1, ws1, G1, sk1 = R.pair_accumulate(F, xi, xj, w, mode)
        assert sk0 == sk1
        assert np.isclose(l0, l1, rtol=1e-12, atol=1e-300) and np.isclose(ws0, ws1, rtol=1e-12)
        assert np.allclose(G0, G1, rtol=1e-9, atol=1e-12 * max(1.0, np.abs(G0).max()))


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not mounted")
@pytest.mark.parametrize("mode", [0, 1])
def test_oracle_matches_reference_module_fresh(mode):
    import sys
    sys.path.insert(0, REF_SRC)
    from epialign import _kernels_np as ref
    rng = np.random.default_rng(7)
    for _ in range(5):
        F = rng.normal(size=(3, 3))
        F /= np.linalg.norm(F)
        xi, xj = rng.uniform(0, 640, (300, 2)), rng.uniform(0, 480, (300, 2))
        w = rng.uniform(0.1, 2, 300)
        e0, n0 = ref.pair_residuals(F, xi, xj, mode)
        e1, n1 = R.pair_residuals(F, xi, xj, mode)
        assert n0 == n1 and np.allclose(e0, e1, rtol=1e-12, atol=1e-15, equal_nan=True)
        a0, a1 = ref.pair_accumulate(F, xi, xj, w, mode), R.pair_accumulate(F, xi, xj, w, mode)
        assert np.isclose(a0[0], a1[0], rtol=1e-12) and np.isclose(a0[1], a1[1], rtol=1e-12)
        assert np.allclose(a0[2], a1[2], rtol=1e-9, atol=1e-12) and a0[3] == a1[3]


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_cuda_batched_matches_golden(mode):
    import torch
    from paper_2509_25191_b200 import epipolar as E
    g = np.load(GOLD)
    t = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt).cuda().contiguous()
    e, nd = E.pairs_residuals(t(g["F"]), t(g["offsets"], torch.int64), t(g["xy_i"]), t(g["xy_j"]), mode)
    l, ws, G, sk = E.pairs_accumulate(t(g["F"]), t(g["offsets"], torch.int64), t(g["xy_i"]), t(g["xy_j"]),
                                      t(g["w"]), mode)
    e, nd, l, ws, G, sk = (x.cpu().numpy() for x in (e, nd, l, ws, G, sk))
    for p, F, xi, xj, w, (a, b) in _pairs(g):
        _check_pair(p, g, mode, e[a:b], nd[p], l[p], ws[p], G[p], sk[p], a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_cuda_per_pair_dropin_matches_oracle(mode):
    from paper_2509_25191_b200 import epipolar as E
    rng = np.random.default_rng(11)
    for k in (1, 31, 500, 4096):
        F = rng.normal(size=(3, 3))
        F /= np.linalg.norm(F)
        xi, xj = rng.uniform(0, 640, (k, 2)), rng.uniform(0, 480, (k, 2))
        w = rng.uniform(0.1, 2, k)
        e, nd = E.pair_residuals(F, xi, xj, mode)
        e0, nd0 = R.pair_residuals(F, xi, xj, mode)
        assert nd == nd0 and np.allclose(e, e0, rtol=1e-12, atol=1e-15, equal_nan=True)
        l, ws, G, sk = E.pair_accumulate(F, xi, xj, w, mode)
        l0, ws0, G0, sk0 = R.pair_accumulate(F, xi, xj, w, mode)
        assert sk == sk0 and np.isclose(l, l0, rtol=1e-12) and np.isclose(ws, ws0, rtol=1e-12)
        assert np.allclose(G, G0, rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_cuda_gradient_matches_finite_differences(mode):
    from paper_2509_25191_b200 import epipolar as E
    rng = np.random.default_rng(3)
    F = rng.normal(size=(3, 3))
    F /= np.linalg.norm(F)
    xi, xj = rng.uniform(0, 640, (40, 2)), rng.uniform(0, 480, (40, 2))
    w = rng.uniform(0.1, 2, 40)
    _, _, G, _ = E.pair_accumulate(F, xi, xj, w, mode)
    h = 1e-7
    fd = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            Fp, Fm = F.copy(), F.copy()
            Fp[a, b] += h
            Fm[a, b] -= h
            fd[a, b] = (E.pair_accumulate(Fp, xi, xj, w, mode)[0] - E.pair_accumulate(Fm, xi, xj, w, mode)[0]) / (2 * h)
    assert np.abs(G - fd).max() < 1e-6 * np.abs(G).max()


@pytest.mark.gpu
def test_cuda_many_pairs_throughput_shape():
    """10k pairs x up to 4096 correspondences in one launch (an S = 1000 alignment step)."""
    import torch
    from paper_2509_25191_b200 import epipolar as E
    rng = np.random.default_rng(5)
    P = 10000
    ks = rng.integers(64, 512, P)
    off = np.r_[0, np.cumsum(ks)]
    K = int(off[-1])
    Fs = rng.normal(size=(P, 3, 3))
    Fs /= np.linalg.norm(Fs, axis=(1, 2), keepdims=True)
    xi, xj, w = rng.uniform(0, 640, (K, 2)), rng.uniform(0, 480, (K, 2)), rng.uniform(0.1, 2, K)
    t = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt).cuda().contiguous()
    l, ws, G, sk = E.pairs_accumulate(t(Fs), t(off, torch.int64), t(xi), t(xj), t(w), 1)
    for p in (0, 1234, P - 1):
        a, b = off[p], off[p + 1]
        l0, ws0, G0, sk0 = R.pair_accumulate(Fs[p], xi[a:b], xj[a:b], w[a:b], 1)
        assert np.isclose(l[p].item(), l0, rtol=1e-12) and np.allclose(G[p].cpu().numpy(), G0, rtol=1e-9, atol=1e-12)
