"""Global-Alignment optimiser: CPU oracle pinned to the reference's own outputs
(tests/golden/ga.npz, made by tests/golden/make_ga_golden.py from pkg/src/epialign), and the
device implementation (paper_2509_25191_b200.ga / csrc/ga.cu) checked against the same goldens.

Tolerances: the device sums each pair's correspondences in a different (parallel, fixed) order
than the reference's sequential Cython loop, so results agree to rounding, not bitwise; the
reference's own gradient tests use rtol 1e-9 (pkg/tests/test_kernels.py:20-45).
"""
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

from oracle import ga_ref

GOLD = Path(__file__).parent / "golden" / "ga.npz"


def _cases():
    g = np.load(GOLD)
    out = {}
    for c in g["cases"]:
        out[str(c)] = {k.split("/", 1)[1]: g[k] for k in g.files if k.startswith(str(c) + "/")}
    return out


CASES = _cases()
NAMES = sorted(CASES)


def _cfg(d):
    from paper_2509_25191_b200.ga import AlignerConfig
    it, lr0, lr1, lr2, b1, b2, focal, gauge, geo, alpha, wm, rew = d["cfg"]
    return AlignerConfig(iterations=int(it), lr0=lr0, lr1=lr1, lr2=lr2, b1=b1, b2=b2, optimize_focal=bool(focal),
                         gauge_frame=int(gauge), residual_mode="geometric" if geo else "algebraic", alpha=alpha,
                         weight_mode=["adaptive", "uniform", "confidence"][int(wm)], reweight_every=int(rew))


def _check_align(o, d, exact, rtol):
    if exact:  # a fixed point: the trace is rounding noise, only its size is meaningful
        assert np.all(np.abs(o["loss_trace"]) < 1e-9) and np.all(np.abs(d["loss_trace"]) < 1e-9)
        assert o["report"][1] < 1e-8
        assert np.abs(o["out_R"] - d["out_R"]).max() < 1e-8
        assert np.abs(o["out_t"] - d["out_t"]).max() < 1e-8
        return
    tr = np.abs(o["loss_trace"] - d["loss_trace"]) / np.abs(d["loss_trace"])
    assert tr.max() < rtol, tr.max()
    assert np.abs(o["out_R"] - d["out_R"]).max() < rtol
    assert np.abs(o["out_t"] - d["out_t"]).max() < rtol * max(1.0, np.abs(d["out_t"]).max())
    np.testing.assert_allclose(o["out_f"], d["out_f"], rtol=rtol)
    np.testing.assert_allclose(o["report"][:3], d["report"][:3], rtol=rtol)
    assert o["report"][3] == d["report"][3] and o["report"][4] == d["report"][4]
    np.testing.assert_allclose(o["rot_delta"], d["rot_delta"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(o["trans_delta"], d["trans_delta"], rtol=1e-6, atol=1e-12)


# ------------------------------------------------------------------------------------------------
# CPU: the oracle restatement against the reference's own outputs

@pytest.mark.parametrize("name", NAMES)
def test_oracle_align_matches_reference(name):
    d = CASES[name]
    if d["offsets"][-1] > 20000:
        pytest.skip("large case: covered on the GPU")
    o = ga_ref.align(d["R"], d["t"], d["intr"], d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], d["cfg"],
                     conf=d.get("conf"), weights=d.get("weights_in"))
    _check_align(o, d, name.startswith("exact"), 1e-10)


@pytest.mark.parametrize("name", [n for n in NAMES if "probe_grad" in CASES[n]])
def test_oracle_loss_gradient_matches_reference(name):
    d = CASES[name]
    focal = bool(d["cfg"][6])
    Kinv = np.stack([ga_ref.k_inverse(x) for x in d["intr"]])
    prob = ga_ref.Problem(d["R"], d["t"], Kinv, d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], int(d["cfg"][8]),
                          focal, int(d["cfg"][7]))
    e0, _, _ = prob.residuals(ga_ref.identity_params(len(d["R"]), focal))
    np.testing.assert_allclose(e0, d["probe_e0"], rtol=1e-10, atol=1e-12)
    w, _ = ga_ref.adaptive_weights(e0, 0.5)  # the probe uses the default alpha (make_ga_golden.py)
    np.testing.assert_allclose(w, d["probe_w"], rtol=1e-12)
    loss, grad, sk = prob.loss_and_gradient(d["probe_params"], d["probe_w"])
    assert loss == pytest.approx(d["probe_loss"][0], rel=1e-12)
    assert sk == d["probe_loss"][1]
    np.testing.assert_allclose(grad, d["probe_grad"], rtol=1e-9, atol=1e-12 * np.abs(d["probe_grad"]).max())


# ------------------------------------------------------------------------------------------------
# GPU: the device optimiser

@pytest.fixture(scope="module")
def ga():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2509_25191_b200 import ga as mod
    return mod


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_align_matches_reference(ga, name):
    d = CASES[name]
    o = ga.align_arrays(d["R"], d["t"], d["intr"], d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], _cfg(d),
                        conf=d.get("conf"), weights=d.get("weights_in"))
    _check_align(o, d, name.startswith("exact"), 1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in NAMES if "probe_grad" in CASES[n]])
def test_device_loss_gradient_matches_reference(ga, name):
    import torch
    d = CASES[name]
    focal = bool(d["cfg"][6])
    Kinv = np.stack([ga._k_inverse(*x[:4]) for x in d["intr"]])
    prob = ga.DeviceProblem(d["R"], d["t"], Kinv, d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], int(d["cfg"][8]),
                            focal, int(d["cfg"][7]))
    prob.set_params(ga.identity_params(len(d["R"]), focal))
    e0, st = prob.residuals()
    assert np.array_equal(np.isnan(e0), np.isnan(d["probe_e0"]))
    np.testing.assert_allclose(e0, d["probe_e0"], rtol=1e-10, atol=1e-12)
    w, _ = ga.adaptive_weights_device(torch.as_tensor(e0, device="cuda"), 0.5)
    np.testing.assert_allclose(w.cpu().numpy(), d["probe_w"], rtol=1e-12)
    prob.set_params(d["probe_params"])
    prob.set_weights(d["probe_w"])
    lg = prob.loss_and_gradient()
    assert lg.loss == pytest.approx(d["probe_loss"][0], rel=1e-12)
    assert lg.skipped == d["probe_loss"][1]
    np.testing.assert_allclose(lg.grad, d["probe_grad"], rtol=1e-9, atol=1e-12 * np.abs(d["probe_grad"]).max())
    assert np.all(lg.grad[int(d["cfg"][7])] == 0.0)  # gauge block exactly zero


@pytest.mark.gpu
def test_device_graph_and_stream_launch_agree_bitwise(ga):
    d = CASES["noisy5"]
    a = ga.align_arrays(d["R"], d["t"], d["intr"], d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], _cfg(d))
    b = ga.align_arrays(d["R"], d["t"], d["intr"], d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], _cfg(d),
                        use_graph=False)
    c = ga.align_arrays(d["R"], d["t"], d["intr"], d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], _cfg(d))
    assert np.array_equal(a["loss_trace"], b["loss_trace"]) and np.array_equal(a["loss_trace"], c["loss_trace"])
    assert np.array_equal(a["params"], c["params"])


# duck-typed objects with the reference's attribute names (pkg/src/epialign/geometry.py, pairing.py)
@dataclass(frozen=True)
class _Intr:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def scaled_focal(self, s):
        k = float(np.exp(s))
        return _Intr(self.fx * k, self.fy * k, self.cx, self.cy, self.width, self.height)


@dataclass(frozen=True)
class _Pose:
    R: np.ndarray
    t: np.ndarray


@dataclass(frozen=True)
class _Frame:
    frame_id: str
    intrinsics: _Intr
    pose: _Pose


@dataclass(frozen=True)
class _Rig:
    frames: tuple

    def __getitem__(self, i):
        return self.frames[i]


@dataclass(frozen=True)
class _PM:
    frame_i: int
    frame_j: int
    xy_i: np.ndarray
    xy_j: np.ndarray
    confidence: np.ndarray = None


@dataclass(frozen=True)
class _MS:
    pairs: tuple


def _objects(d):
    rig = _Rig(tuple(_Frame(f"f{k}", _Intr(*d["intr"][k][:4], int(d["intr"][k][4]), int(d["intr"][k][5])),
                            _Pose(d["R"][k], d["t"][k])) for k in range(len(d["R"]))))
    o = d["offsets"]
    ms = _MS(tuple(_PM(int(i), int(j), d["xy_i"][o[p]:o[p + 1]], d["xy_j"][o[p]:o[p + 1]],
                       None if "conf" not in d else d["conf"][o[p]:o[p + 1]])
                   for p, (i, j) in enumerate(d["pair_ij"])))
    return rig, ms


@pytest.mark.gpu
def test_device_align_object_api(ga):
    d = CASES["focal6"]
    rig, ms = _objects(d)
    refined, rep = ga.align(rig, ms, _cfg(d))
    assert refined[0] is rig[0]  # gauge frame returned untouched (test_aligner.py:224-230)
    np.testing.assert_allclose(rep.loss_trace, d["loss_trace"], rtol=1e-8)
    for k in range(1, len(rig.frames)):
        np.testing.assert_allclose(refined[k].pose.R, d["out_R"][k], atol=1e-8)
        assert refined[k].intrinsics.fx == pytest.approx(d["out_f"][k][0], rel=1e-8)
    assert rep.to_dict()["iterations"] == int(d["cfg"][0])
    e, st = ga.epipolar_residuals(rig, ms)
    assert e.shape == (d["offsets"][-1],) and st.degenerate_pairs == 0


@pytest.mark.gpu
def test_device_align_errors(ga):
    d = CASES["noisy5"]
    rig, ms = _objects(d)
    with pytest.raises(ga.InsufficientCorrespondences):
        ga.align(rig, _MS(()))
    p0 = ms.pairs[0]
    with pytest.raises(ga.InsufficientCorrespondences):
        ga.align(rig, _MS((_PM(p0.frame_i, p0.frame_j, p0.xy_i[:3], p0.xy_j[:3]),)))
    with pytest.raises(ga.ZeroTotalWeight):
        ga.align(rig, ms, weights=np.zeros(int(d["offsets"][-1])))
    with pytest.raises(ga.MissingConfidence):
        ga.align(rig, ms, ga.AlignerConfig(weight_mode="confidence"))
    with pytest.raises(ValueError):
        ga.align(rig, ms, ga.AlignerConfig(gauge_frame=99))


@pytest.mark.gpu
def test_device_align_dense_scene_matches_oracle(ga):
    """A denser synthetic scene than the goldens (80 views, every frame in > 32 pairs, so the per-frame
    CSR gather spans several warp strides) against the oracle restatement."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import bench_ga
    R, t, intr, pij, off, xi, xj = bench_ga.scene(80, 600, 80.0, 96, seed=3)
    cfgv = np.array([30, 5e-4, 1e-3, 1e-2, 2.5, 7.5, 0.0, 0, 1.0, 0.5, 0, 0])
    ref = ga_ref.align(R, t, intr, pij, off, xi, xj, cfgv)
    o = ga.align_arrays(R, t, intr, pij, off, xi, xj, ga.AlignerConfig(iterations=30))
    assert np.bincount(pij.reshape(-1)).max() > 32
    tr = np.abs(o["loss_trace"] - ref["loss_trace"]) / np.abs(ref["loss_trace"])
    assert tr.max() < 1e-8, tr.max()
    assert np.abs(o["out_R"] - ref["out_R"]).max() < 1e-8
    np.testing.assert_allclose(o["report"][:3], ref["report"][:3], rtol=1e-8)


def test_match_arrays_confidence_checked_on_live_pairs_only():
    """aligner.py:358-360 drops empty pairs before weighting.py:108-111 checks confidences, so an empty
    pair without confidences must not make weight_mode='confidence' fail."""
    from paper_2509_25191_b200.ga import _match_arrays
    d = CASES["focal6"]
    o = d["offsets"]
    rng = np.random.default_rng(0)
    pairs = [_PM(int(i), int(j), d["xy_i"][o[p]:o[p + 1]], d["xy_j"][o[p]:o[p + 1]], rng.random(o[p + 1] - o[p]))
             for p, (i, j) in enumerate(d["pair_ij"])]
    pairs.insert(1, _PM(0, 1, np.zeros((0, 2)), np.zeros((0, 2)), None))
    pij, off, xi, xj, conf = _match_arrays(_MS(tuple(pairs)))
    assert conf is not None and conf.shape == (int(off[-1]),)
    np.testing.assert_array_equal(conf, np.concatenate([p.confidence for p in pairs if len(p.xy_i)]))
    pairs[2] = _PM(pairs[2].frame_i, pairs[2].frame_j, pairs[2].xy_i, pairs[2].xy_j, None)
    assert _match_arrays(_MS(tuple(pairs)))[4] is None


@pytest.mark.gpu
def test_device_problem_status_does_not_stick(ga):
    """A DeviceProblem that raised on a degenerate 6D rotation evaluates valid parameters afterwards."""
    d = CASES["noisy5"]
    R, t, intr = d["R"], d["t"], d["intr"]
    Kinv = np.stack([np.linalg.inv(np.array([[x[0], 0, x[2]], [0, x[1], x[3]], [0, 0, 1.0]])) for x in intr])
    prob = ga.DeviceProblem(R, t, Kinv, d["pair_ij"], d["offsets"], d["xy_i"], d["xy_j"], 1, False, 0)
    good = ga.identity_params(len(R), False)
    bad = good.copy()
    bad[1, :6] = 0.0
    with pytest.raises(ga.DegenerateRotation6D):
        prob.set_params(bad)
    prob.set_params(good)
    lg = prob.loss_and_gradient()
    assert np.isfinite(lg.loss)
