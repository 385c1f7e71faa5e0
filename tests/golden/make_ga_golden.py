"""Generates tests/golden/ga.npz from the REFERENCE's own Global-Alignment optimiser.

Imports epialign (aligner, synth, pairing, weighting) from /root/reference/pkg/src
(read-only; available in the build container only), builds the synthetic scenes the
reference's own tests use (pkg/tests/test_aligner.py:_noisy_scene, :280-291, :313-323),
runs `epialign.aligner.align` and `loss_gradient` and records inputs + outputs:
cameras (R, t, intrinsics), pairs (frame indices, offsets, correspondences, optional
confidences), the config, and the report (loss trace, medians, learning rate, refined
poses, per-frame deltas, skip count).  Re-run: python tests/golden/make_ga_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from epialign.aligner import AlignerConfig, align, identity_params, loss_gradient  # noqa: E402
from epialign.pairing import MatchSet, PairMatches, select_pairs  # noqa: E402
from epialign.synth import SynthConfig, generate, perturb  # noqa: E402
from epialign.weighting import adaptive_weights, build_histogram  # noqa: E402
from epialign.aligner import epipolar_residuals  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ga.npz")


def _select(rig, matches, angle=100.0):
    sel = select_pairs(rig, angle).as_set()
    return MatchSet(tuple(p for p in matches.pairs if (p.frame_i, p.frame_j) in sel))


def _scene(freeze=None, **kw):
    cfg = SynthConfig(**kw)
    scene = generate(cfg)
    if freeze is None:
        rig, matches, _ = perturb(scene.rig, scene.matches, cfg)
    else:
        rig, matches, _ = perturb(scene.rig, scene.matches, cfg, freeze=freeze)
    return rig, _select(rig, matches)


def _pack(prefix, rig, matches, cfg, out, weights=None, probe=True):
    d = {}
    d["R"] = np.stack([f.pose.R for f in rig.frames])
    d["t"] = np.stack([f.pose.t for f in rig.frames])
    d["intr"] = np.array([[f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy,
                           f.intrinsics.width, f.intrinsics.height] for f in rig.frames])
    d["pair_ij"] = np.array([[p.frame_i, p.frame_j] for p in matches.pairs], dtype=np.int32).reshape(-1, 2)
    d["offsets"] = np.concatenate([[0], np.cumsum([len(p) for p in matches.pairs])]).astype(np.int64)
    d["xy_i"] = np.concatenate([p.xy_i for p in matches.pairs]) if matches.pairs else np.zeros((0, 2))
    d["xy_j"] = np.concatenate([p.xy_j for p in matches.pairs]) if matches.pairs else np.zeros((0, 2))
    if matches.has_confidence():
        d["conf"] = np.concatenate([p.confidence for p in matches.pairs])
    d["cfg"] = np.array([cfg.iterations, cfg.lr0, cfg.lr1, cfg.lr2, cfg.b1, cfg.b2, float(cfg.optimize_focal),
                         cfg.gauge_frame, 1.0 if cfg.residual_mode == "geometric" else 0.0, cfg.alpha,
                         {"adaptive": 0, "uniform": 1, "confidence": 2}[cfg.weight_mode], cfg.reweight_every])
    if weights is not None:
        d["weights_in"] = weights.weights
    refined, rep = align(rig, matches, cfg, weights=weights)
    d["out_R"] = np.stack([f.pose.R for f in refined.frames])
    d["out_t"] = np.stack([f.pose.t for f in refined.frames])
    d["out_f"] = np.array([[f.intrinsics.fx, f.intrinsics.fy] for f in refined.frames])
    d["loss_trace"] = rep.loss_trace
    d["report"] = np.array([rep.initial_median_px, rep.final_median_px, rep.learning_rate,
                            rep.dropped_pairs, rep.degenerate_correspondences])
    d["rot_delta"] = rep.rotation_delta_deg
    d["trans_delta"] = rep.translation_delta
    if probe:
        # one loss/gradient evaluation at a perturbed parameter block (adaptive weights at the input)
        rng = np.random.default_rng(len(prefix))
        p = identity_params(len(rig), cfg.optimize_focal) + rng.normal(0, 2e-3, size=(len(rig), cfg.param_dim))
        e0, _ = epipolar_residuals(rig, matches, cfg.residual_mode)
        wt = adaptive_weights(e0, build_histogram(e0))
        lg = loss_gradient(rig, matches, wt, p, cfg)
        d["probe_params"] = p
        d["probe_w"] = wt.weights
        d["probe_loss"] = np.array([lg.loss, lg.skipped])
        d["probe_grad"] = lg.grad
        d["probe_e0"] = e0
    for k, v in d.items():
        out[f"{prefix}/{k}"] = v


def main():
    out = {}
    cases = []
    # test_aligner.py:_noisy_scene defaults (5 cameras, 60 points, 1 deg, 0.5 px)
    rig, m = _scene(n_cameras=5, n_points=60, seed=9, rot_sigma_deg=1.0, trans_sigma_frac=0.005,
                    pixel_sigma_px=0.5)
    _pack("noisy5", rig, m, AlignerConfig(iterations=30), out)
    cases.append("noisy5")
    # test_aligner.py:280-291 (noise reduction, 300 iterations, gauge frozen)
    rig, m = _scene(freeze=(0,), n_cameras=10, n_points=300, seed=14, focal_px=1200.0, width=1600,
                    height=1200, rot_sigma_deg=0.8, trans_sigma_frac=0.002)
    _pack("noise10", rig, m, AlignerConfig(), out)
    cases.append("noise10")
    # test_aligner.py:313-323 (outliers; adaptive vs uniform)
    kw = dict(n_cameras=12, n_points=400, seed=17, focal_px=400.0, rot_sigma_deg=0.15,
              trans_sigma_frac=0.001, pixel_sigma_px=0.3, outlier_frac=0.10)
    rig, m = _scene(freeze=(0,), **kw)
    _pack("outlier12_adaptive", rig, m, AlignerConfig(weight_mode="adaptive"), out)
    _pack("outlier12_uniform", rig, m, AlignerConfig(weight_mode="uniform"), out, probe=False)
    cases += ["outlier12_adaptive", "outlier12_uniform"]
    # focal optimisation, algebraic residuals, periodic re-weighting, non-zero gauge
    rig, m = _scene(n_cameras=6, n_points=120, seed=21, rot_sigma_deg=0.5, trans_sigma_frac=0.003,
                    pixel_sigma_px=0.4)
    _pack("focal6", rig, m, AlignerConfig(iterations=100, optimize_focal=True), out)
    _pack("algebraic6", rig, m, AlignerConfig(iterations=50, residual_mode="algebraic"), out)
    _pack("reweight6", rig, m, AlignerConfig(iterations=60, reweight_every=10), out, probe=False)
    _pack("gauge6", rig, m, AlignerConfig(iterations=40, gauge_frame=2), out, probe=False)
    cases += ["focal6", "algebraic6", "reweight6", "gauge6"]
    # matcher confidences (confidence weights), plus an empty pair that align drops
    rng = np.random.default_rng(5)
    pairs = [PairMatches(p.frame_i, p.frame_j, p.xy_i, p.xy_j, rng.uniform(0.2, 1.0, size=len(p)))
             for p in m.pairs]
    pairs.insert(1, PairMatches(0, 5, np.zeros((0, 2)), np.zeros((0, 2)), np.zeros(0)))
    mc = MatchSet(tuple(pairs))
    _pack("confidence6", rig, mc, AlignerConfig(iterations=40, weight_mode="confidence"), out, probe=False)
    cases.append("confidence6")
    # exact scene = fixed point (test_aligner.py:212-221)
    scene = generate(SynthConfig(n_cameras=6, n_points=150, seed=7))
    _pack("exact6", scene.rig, _select(scene.rig, scene.matches), AlignerConfig(iterations=50), out,
          probe=False)
    cases.append("exact6")
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT), "bytes;", ", ".join(cases))


if __name__ == "__main__":
    main()
