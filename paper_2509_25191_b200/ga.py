"""Drop-in device implementation of the reference's Global-Alignment optimiser.

Mirrors `epialign.aligner` (pkg/src/epialign/aligner.py): `AlignerConfig` (:47-77),
`AlignmentReport` (:80-108), `LossGradient`, `identity_params` (:122-128),
`select_learning_rate` (:131-140), `align` (:348-443), `epipolar_residuals` (:285-290),
`weighted_epipolar_loss` (:293-305), `loss_at` (:308-318) and `loss_gradient` (:321-334), with the
same argument meaning, defaults, return types and exceptions.  Inputs are duck-typed: any rig with
`.frames[f].pose.R/.t` and `.intrinsics.fx/.fy/.cx/.cy` and any match set with
`.pairs[p].frame_i/.frame_j/.xy_i/.xy_j[/.confidence]` — the reference's own objects work as-is,
and the refined rig is rebuilt with the caller's frame/pose types.  When `epialign` is importable
its exception classes are raised, so existing `except` clauses keep working.

Everything inside the loop runs on the GPU (csrc/ga.cu via ops.ga_*): decode, per-pair epipolar
sums and chain rule, per-frame gradient, Adam, adaptive weights; the 300 iterations are one CUDA
graph.  Host work is the setup, two medians (for the learning-rate band and the report) and the
output assembly.  There is no CPU fallback.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import ops

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8
F_NORM_EPS = 1e-15
MIN_TOTAL_CORRESPONDENCES = 8
CLIP_RANGE = (0.0, 20.0)   # weighting.py:19
N_BINS = 100               # weighting.py:20
DEFAULT_ALPHA = 0.5        # weighting.py:22
MODE_ALGEBRAIC, MODE_GEOMETRIC = 0, 1

try:  # raise the reference's own exception types when it is installed
    from epialign.errors import (DegenerateRotation6D, EmptyResiduals, InsufficientCorrespondences,  # type: ignore
                                 MissingConfidence, ZeroTotalWeight)
except ImportError:  # same names and bases as pkg/src/epialign/errors.py:9-82
    class EpialignError(Exception):
        pass

    class DataError(EpialignError):
        pass

    class NumericalError(EpialignError):
        pass

    class InsufficientCorrespondences(DataError):
        pass

    class EmptyResiduals(DataError):
        pass

    class MissingConfidence(DataError):
        pass

    class ZeroTotalWeight(NumericalError):
        pass

    class DegenerateRotation6D(NumericalError):
        pass


def mode_id(name: str) -> int:
    """kernels.py:45-50."""
    if name == "algebraic":
        return MODE_ALGEBRAIC
    if name == "geometric":
        return MODE_GEOMETRIC
    raise ValueError(f"unknown residual mode {name!r}")


@dataclass(frozen=True)
class AlignerConfig:
    """aligner.py:47-77 (same fields, defaults and validation)."""

    iterations: int = 300
    lr0: float = 5e-4
    lr1: float = 1e-3
    lr2: float = 1e-2
    b1: float = 2.5
    b2: float = 7.5
    optimize_focal: bool = False
    gauge_frame: int = 0
    residual_mode: str = "geometric"
    alpha: float = 0.5
    weight_mode: str = "adaptive"    # adaptive | uniform | confidence
    reweight_every: int = 0          # 0 keeps the weights frozen

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if not (0 < self.lr0 <= self.lr1 <= self.lr2):
            raise ValueError("learning rates must satisfy 0 < lr0 <= lr1 <= lr2")
        if not (0 < self.b1 < self.b2):
            raise ValueError("bands must satisfy 0 < b1 < b2")
        mode_id(self.residual_mode)

    @property
    def param_dim(self) -> int:
        return 10 if self.optimize_focal else 9


@dataclass(frozen=True)
class AlignmentReport:
    """aligner.py:80-108."""

    initial_median_px: float
    final_median_px: float
    learning_rate: float
    loss_trace: np.ndarray
    rotation_delta_deg: np.ndarray
    translation_delta: np.ndarray
    dropped_pairs: int
    degenerate_correspondences: int

    def to_dict(self) -> dict:
        return {
            "initial_median_px": self.initial_median_px,
            "final_median_px": self.final_median_px,
            "learning_rate": self.learning_rate,
            "iterations": int(self.loss_trace.shape[0]),
            "loss_initial": float(self.loss_trace[0]),
            "loss_final": float(self.loss_trace[-1]),
            "loss_trace": [float(x) for x in self.loss_trace],
            "rotation_delta_deg": [float(x) for x in self.rotation_delta_deg],
            "translation_delta": [float(x) for x in self.translation_delta],
            "dropped_pairs": self.dropped_pairs,
            "degenerate_correspondences": self.degenerate_correspondences,
        }


@dataclass(frozen=True)
class LossGradient:
    loss: float
    grad: np.ndarray
    skipped: int


@dataclass(frozen=True)
class ResidualStats:
    degenerate_pairs: int
    degenerate_correspondences: int


@dataclass(frozen=True)
class WeightTable:
    """weighting.py:36-53 (weights flat in match-set order)."""

    weights: np.ndarray
    alpha: float
    avg_density: float


def identity_params(n_frames: int, optimize_focal: bool = False) -> np.ndarray:
    dim = 10 if optimize_focal else 9
    p = np.zeros((n_frames, dim))
    p[:, 0] = 1.0
    p[:, 4] = 1.0
    return p


def select_learning_rate(median_residual: float, cfg: AlignerConfig) -> float:
    if median_residual < 0:
        raise ValueError("median residual must be >= 0")
    if median_residual < cfg.b1:
        return cfg.lr0
    if median_residual > cfg.b2:
        return cfg.lr2
    return cfg.lr1


def _k_inverse(fx, fy, cx, cy):
    """geometry.py:64-71."""
    return np.array([[1.0 / fx, 0.0, -cx / fx], [0.0, 1.0 / fy, -cy / fy], [0.0, 0.0, 1.0]])


def _rot6d_decode(dr):
    """geometry.py:188-207 (host copy for output assembly)."""
    a, b = dr[:3], dr[3:6]
    na = np.linalg.norm(a)
    if na <= 1e-12:
        raise DegenerateRotation6D(f"first column norm {na:.3e} below 1e-12")
    b1 = a / na
    u = b - (b1 @ b) * b1
    nu = np.linalg.norm(u)
    if nu <= 1e-12:
        raise DegenerateRotation6D("columns are parallel; cannot orthonormalize")
    b2 = u / nu
    return np.stack([b1, b2, np.cross(b1, b2)], axis=1)


def _median(e: torch.Tensor) -> float:
    """np.median over the finite entries (mean of the two middle values for even counts)."""
    x = e[torch.isfinite(e)]
    n = x.numel()
    if n == 0:
        return float("nan")
    xs = torch.sort(x).values
    if n % 2:
        return float(xs[n // 2].item())
    a, b = xs[n // 2 - 1: n // 2 + 1].tolist()
    return float(np.mean([a, b]))


class DeviceProblem:
    """aligner.py:_Problem (:143-278) with every array resident on the GPU.

    R (n,3,3), t (n,3), Kinv (n,3,3) are the (canonical-gauge) cameras; pairs are given as
    pair_ij (P,2), offsets (P+1) and the stacked correspondences xy_i, xy_j (K,2).
    """

    def __init__(self, R, t, Kinv, pair_ij, offsets, xy_i, xy_j, mode: int, optimize_focal: bool, gauge: int,
                 device="cuda"):
        dev = torch.device(device)
        f64 = dict(device=dev, dtype=torch.float64)
        self.n = int(np.shape(R)[0])
        self.P = int(np.shape(pair_ij)[0])
        self.dim = 10 if optimize_focal else 9
        self.mode, self.gauge = int(mode), int(gauge)
        pair_ij = np.ascontiguousarray(pair_ij, dtype=np.int32).reshape(-1, 2)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.K = int(offsets[-1]) if offsets.size else 0
        # CSR of (pair, role) entries per frame, ascending pair order (the reference's accumulation order)
        ent = np.stack([2 * np.arange(self.P), 2 * np.arange(self.P) + 1], 1).reshape(-1).astype(np.int32)
        fr = pair_ij.reshape(-1)
        order = np.argsort(fr, kind="stable")
        fptr = np.zeros(self.n + 1, dtype=np.int32)
        np.add.at(fptr, fr + 1, 1)
        fptr = np.cumsum(fptr).astype(np.int32)
        self.t_ = dict(
            pair_ij=torch.as_tensor(pair_ij, device=dev), offsets=torch.as_tensor(offsets, device=dev),
            xy_i=torch.as_tensor(np.ascontiguousarray(xy_i, dtype=np.float64).reshape(-1, 2), **f64),
            xy_j=torch.as_tensor(np.ascontiguousarray(xy_j, dtype=np.float64).reshape(-1, 2), **f64),
            w=torch.ones(max(self.K, 1), **f64),
            frame_ptr=torch.as_tensor(fptr, device=dev), frame_ent=torch.as_tensor(ent[order], device=dev),
            base_R=torch.as_tensor(np.ascontiguousarray(R, dtype=np.float64).reshape(-1, 9), **f64),
            base_t=torch.as_tensor(np.ascontiguousarray(t, dtype=np.float64).reshape(-1, 3), **f64),
            base_Kinv=torch.as_tensor(np.ascontiguousarray(Kinv, dtype=np.float64).reshape(-1, 9), **f64),
            params=torch.as_tensor(identity_params(self.n, optimize_focal), **f64),
            adam_m=torch.zeros(self.n, self.dim, **f64), adam_v=torch.zeros(self.n, self.dim, **f64),
            Rs=torch.empty(self.n, 9, **f64), ts=torch.empty(self.n, 3, **f64), Kinv=torch.empty(self.n, 9, **f64),
            geom=torch.empty(max(self.P, 1), 32, **f64), payload=torch.empty(max(self.P, 1), 32, **f64),
            scalars=torch.zeros(4 + 3 * max(1, -(-self.P // 64)), **f64),
            status=torch.zeros(2, device=dev, dtype=torch.int32),
        )
        self.device = dev
        self.pb = ops.GaProblem(self.n, self.P, self.dim, self.mode, self.gauge,
                                *[self.t_[k].data_ptr() for k in (
                                    "pair_ij", "offsets", "xy_i", "xy_j", "w", "frame_ptr", "frame_ent", "base_R",
                                    "base_t", "base_Kinv", "params", "adam_m", "adam_v", "Rs", "ts", "Kinv",
                                    "geom", "payload", "scalars", "status")])

    # -- state ---------------------------------------------------------------------------------
    def set_params(self, params):
        self.t_["params"].copy_(torch.as_tensor(np.asarray(params, dtype=np.float64).reshape(self.n, self.dim)))
        self._clear_status()
        ops.ga_decode(self.pb)
        self._check_status()

    def params(self) -> np.ndarray:
        return self.t_["params"].cpu().numpy()

    def set_weights(self, w):
        w = torch.as_tensor(w, dtype=torch.float64)
        if w.numel() != self.K:
            raise ValueError("weight table size does not match the match set")
        if self.K:
            self.t_["w"][: self.K].copy_(w.reshape(-1))

    def _clear_status(self):
        # the device only ever sets status bits (atomicOr): clear them before each call that can
        # raise, so one failure does not stick to every later call on valid inputs
        self.t_["status"][0].zero_()

    def _check_status(self):
        st = int(self.t_["status"][0].item())
        if st & 1:
            raise DegenerateRotation6D("a 6D rotation encoding cannot be orthonormalized")
        if st & 2:
            raise ZeroTotalWeight("no correspondence carries positive weight")

    # -- evaluation (aligner.py:189-278) ----------------------------------------------------------
    def residuals_device(self):
        e = torch.empty(max(self.K, 1), device=self.device, dtype=torch.float64)
        dp = torch.zeros(max(self.P, 1), device=self.device, dtype=torch.int32)
        nd = torch.zeros(max(self.P, 1), device=self.device, dtype=torch.int32)
        ops.ga_residuals(self.pb, e, dp, nd)
        return e[: self.K], dp[: self.P], nd[: self.P]

    def residuals(self):
        e, dp, nd = self.residuals_device()
        return e.cpu().numpy(), ResidualStats(int(dp.sum().item()), int(nd.sum().item()))

    def loss_and_gradient(self) -> LossGradient:
        grad = torch.empty(self.n, self.dim, device=self.device, dtype=torch.float64)
        self._clear_status()
        ops.ga_loss_grad(self.pb, grad)
        self._check_status()
        num, den, sk, _ = self.t_["scalars"][:4].tolist()
        return LossGradient(num / den, grad.cpu().numpy(), int(sk))

    def adaptive_weights(self, e: torch.Tensor, alpha: float):
        return adaptive_weights_device(e, alpha)

    def adam(self, t0: int, iters: int, lr: float, bc1, bc2, trace, skipped, use_graph=True):
        ops.ga_adam(self.pb, t0, iters, lr, bc1, bc2, trace, skipped, use_graph)


def adaptive_weights_device(e: torch.Tensor, alpha: float):
    """weighting.py:56-109 on the device: (w tensor, avg_density) for residuals e (NaN = degenerate)."""
    edges = torch.as_tensor(np.linspace(CLIP_RANGE[0], CLIP_RANGE[1], N_BINS + 1), device=e.device)
    w = torch.empty_like(e)
    counts = torch.empty(N_BINS, device=e.device, dtype=torch.int64)
    stats = torch.empty(2 + N_BINS, device=e.device, dtype=torch.float64)
    ops.ga_adaptive_weights(e.contiguous(), edges, alpha, w, counts, stats)
    avg, nfin = stats[:2].tolist()
    if nfin == 0:
        raise EmptyResiduals("no finite residuals to histogram")
    return w, avg


# ------------------------------------------------------------------------------------------------
# array-level driver (used by the duck-typed API below, the tests and the GA bench)

def align_arrays(R, t, intr, pair_ij, offsets, xy_i, xy_j, cfg: AlignerConfig | None = None, conf=None,
                 weights=None, use_graph: bool = True):
    """aligner.py:348-443 on arrays.  intr: (n, >=4) rows (fx, fy, cx, cy, ...).

    Returns dict(out_R, out_t, out_f, loss_trace, report=[median0, median1, lr, dropped, skipped],
    rot_delta, trans_delta, params).
    """
    cfg = cfg or AlignerConfig()
    R = np.asarray(R, dtype=np.float64).reshape(-1, 3, 3)
    t = np.asarray(t, dtype=np.float64).reshape(-1, 3)
    intr = np.asarray(intr, dtype=np.float64)
    n = R.shape[0]
    offsets = np.asarray(offsets, dtype=np.int64)
    pair_ij = np.asarray(pair_ij, dtype=np.int32).reshape(-1, 2)
    counts = np.diff(offsets)
    live = counts > 0
    dropped = int((~live).sum())
    xy_i = np.asarray(xy_i, dtype=np.float64).reshape(-1, 2)
    xy_j = np.asarray(xy_j, dtype=np.float64).reshape(-1, 2)
    if dropped:  # empty pairs own no correspondences: only the pair list and offsets change
        pair_ij = pair_ij[live]
        offsets = np.concatenate([[0], np.cumsum(counts[live])]).astype(np.int64)
    total = int(offsets[-1])
    if len(pair_ij) < 1 or total < MIN_TOTAL_CORRESPONDENCES:
        raise InsufficientCorrespondences(
            f"need >= 1 pair and >= {MIN_TOTAL_CORRESPONDENCES} correspondences, got {len(pair_ij)} pairs / {total}")
    if not (0 <= cfg.gauge_frame < n):
        raise ValueError(f"gauge frame {cfg.gauge_frame} outside rig of {n}")
    if weights is not None:
        weights = np.asarray(weights, dtype=np.float64).reshape(-1)
        if weights.shape[0] != total:
            raise ValueError("weight table size does not match the match set")
    if conf is not None:
        conf = np.asarray(conf, dtype=np.float64).reshape(-1)

    # canonical gauge: origin at the camera centroid (aligner.py:374-383)
    centroid = np.stack([-R[f].T @ t[f] for f in range(n)]).mean(axis=0)
    t_c = np.stack([t[f] + R[f] @ centroid for f in range(n)])
    Kinv = np.stack([_k_inverse(*intr[f, :4]) for f in range(n)])
    prob = DeviceProblem(R, t_c, Kinv, pair_ij, offsets, xy_i, xy_j, mode_id(cfg.residual_mode),
                         cfg.optimize_focal, cfg.gauge_frame)
    ops.ga_decode(prob.pb)
    e0, _, _ = prob.residuals_device()
    if not bool(torch.isfinite(e0).any().item()):
        raise EmptyResiduals("every correspondence is degenerate at the input cameras")

    def make_w(e):
        if cfg.weight_mode == "uniform":
            return torch.ones_like(e)
        if cfg.weight_mode == "confidence":
            if conf is None:
                raise MissingConfidence("match set carries no confidences")
            return torch.as_tensor(conf, device=e.device)
        if cfg.weight_mode == "adaptive":
            return prob.adaptive_weights(e, cfg.alpha)[0]
        raise ValueError(f"unknown weight mode {cfg.weight_mode!r}")

    w = torch.as_tensor(weights, device=prob.device) if weights is not None else make_w(e0)
    if float(w.sum().item()) <= 0:
        raise ZeroTotalWeight("total correspondence weight is zero")
    prob.set_weights(w)
    median0 = _median(e0)
    lr = select_learning_rate(median0, cfg)

    T = cfg.iterations
    its = np.arange(1, T + 1)
    bc1 = torch.as_tensor(np.array([1.0 - ADAM_BETA1 ** int(k) for k in its]), device=prob.device)
    bc2 = torch.as_tensor(np.array([1.0 - ADAM_BETA2 ** int(k) for k in its]), device=prob.device)
    trace = torch.empty(T, device=prob.device, dtype=torch.float64)
    skipped = torch.zeros(1, device=prob.device, dtype=torch.float64)
    seg = cfg.reweight_every if cfg.reweight_every > 0 else T
    t0 = 0
    prob._clear_status()  # bits accumulate over the segments below and are checked once after them
    while t0 < T:
        if t0 > 0:  # aligner.py:405-407: re-weight at t = 1 + k * reweight_every
            e_now, _, _ = prob.residuals_device()
            prob.set_weights(make_w(e_now))
        k = min(seg, T - t0)
        prob.adam(t0, k, lr, bc1, bc2, trace, skipped, use_graph)
        t0 += k
    prob._check_status()
    params = prob.params()
    e1, _, _ = prob.residuals_device()
    median1 = _median(e1)

    out_R, out_t, out_f = R.copy(), t.copy(), intr[:, :2].copy()
    rot_d = np.zeros(n)
    tr_d = np.zeros(n)
    for f in range(n):
        if f == cfg.gauge_frame:
            continue
        dR = _rot6d_decode(params[f, :6])
        Rc = dR @ R[f]
        out_R[f] = Rc
        out_t[f] = (t_c[f] + params[f, 6:9]) - Rc @ centroid
        if cfg.optimize_focal:
            s = float(np.exp(params[f, 9]))
            out_f[f] = (intr[f, 0] * s, intr[f, 1] * s)
        rot_d[f] = float(np.degrees(np.arccos(np.clip((np.trace(dR) - 1.0) / 2.0, -1.0, 1.0))))
        tr_d[f] = float(np.linalg.norm(params[f, 6:9]))
    return dict(out_R=out_R, out_t=out_t, out_f=out_f, loss_trace=trace.cpu().numpy(),
                report=np.array([median0, median1, lr, dropped, float(skipped.item())]), rot_delta=rot_d,
                trans_delta=tr_d, params=params)


# ------------------------------------------------------------------------------------------------
# duck-typed public API (aligner.py:285-443)

def _rig_arrays(rig):
    frames = list(rig.frames)
    R = np.stack([np.asarray(f.pose.R, dtype=np.float64) for f in frames])
    t = np.stack([np.asarray(f.pose.t, dtype=np.float64) for f in frames])
    intr = np.array([[f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy] for f in frames],
                    dtype=np.float64)
    return R, t, intr


def _match_arrays(matches):
    pairs = list(matches.pairs)
    pair_ij = np.array([[p.frame_i, p.frame_j] for p in pairs], dtype=np.int32).reshape(-1, 2)
    cnt = [int(np.shape(p.xy_i)[0]) for p in pairs]
    offsets = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    xy_i = np.concatenate([np.asarray(p.xy_i, dtype=np.float64).reshape(-1, 2) for p in pairs]) if pairs else \
        np.zeros((0, 2))
    xy_j = np.concatenate([np.asarray(p.xy_j, dtype=np.float64).reshape(-1, 2) for p in pairs]) if pairs else \
        np.zeros((0, 2))
    conf = None
    # the reference checks confidences only on the live (non-empty) pairs align() keeps
    # (aligner.py:358-360, weighting.py:108-111): an empty pair without confidences is fine
    live = [p for p, c in zip(pairs, cnt) if c > 0]
    if live and all(getattr(p, "confidence", None) is not None for p in live):
        conf = np.concatenate([np.asarray(p.confidence, dtype=np.float64).reshape(-1) if c > 0 else np.zeros(0)
                               for p, c in zip(pairs, cnt)])
    return pair_ij, offsets, xy_i, xy_j, conf


def _weights_of(weights):
    return None if weights is None else np.asarray(getattr(weights, "weights", weights), dtype=np.float64)


def align(rig, matches, cfg: AlignerConfig | None = None, weights=None):
    """aligner.py:348-443: refine every camera but the gauge frame -> (refined rig, AlignmentReport)."""
    cfg = cfg or AlignerConfig()
    R, t, intr = _rig_arrays(rig)
    pair_ij, offsets, xy_i, xy_j, conf = _match_arrays(matches)
    out = align_arrays(R, t, intr, pair_ij, offsets, xy_i, xy_j, cfg, conf=conf, weights=_weights_of(weights))
    frames = []
    for f, frame in enumerate(rig.frames):
        if f == cfg.gauge_frame:
            frames.append(frame)
            continue
        pose = type(frame.pose)(out["out_R"][f], out["out_t"][f])
        intrinsics = frame.intrinsics
        if cfg.optimize_focal:
            intrinsics = intrinsics.scaled_focal(out["params"][f, 9])
        frames.append(dataclasses.replace(frame, pose=pose, intrinsics=intrinsics))
    refined = type(rig)(tuple(frames))
    rep = out["report"]
    report = AlignmentReport(
        initial_median_px=float(rep[0]), final_median_px=float(rep[1]), learning_rate=float(rep[2]),
        loss_trace=out["loss_trace"], rotation_delta_deg=out["rot_delta"], translation_delta=out["trans_delta"],
        dropped_pairs=int(rep[3]), degenerate_correspondences=int(rep[4]))
    return refined, report


def _problem(rig, matches, cfg: AlignerConfig):
    R, t, intr = _rig_arrays(rig)
    pair_ij, offsets, xy_i, xy_j, _ = _match_arrays(matches)
    Kinv = np.stack([_k_inverse(*x) for x in intr])
    return DeviceProblem(R, t, Kinv, pair_ij, offsets, xy_i, xy_j, mode_id(cfg.residual_mode), cfg.optimize_focal,
                         cfg.gauge_frame)


def epipolar_residuals(rig, matches, mode: str = "geometric"):
    """aligner.py:285-290: residuals of every correspondence at the given cameras (NaN = degenerate)."""
    cfg = AlignerConfig(residual_mode=mode)
    prob = _problem(rig, matches, cfg)
    ops.ga_decode(prob.pb)
    return prob.residuals()


def _weighted_mean(e, w):
    valid = np.isfinite(e)
    wsum = float(w[valid].sum())
    if wsum <= 0:
        raise ZeroTotalWeight("total weight of valid correspondences is zero")
    return float((w[valid] * e[valid]).sum() / wsum)


def weighted_epipolar_loss(rig, matches, weights, mode: str = "geometric") -> float:
    """aligner.py:293-305."""
    e, _ = epipolar_residuals(rig, matches, mode)
    w = _weights_of(weights)
    if w.shape[0] != e.shape[0]:
        raise ValueError("weight table size does not match the match set")
    return _weighted_mean(e, w)


def loss_at(rig, matches, weights, params, cfg: AlignerConfig | None = None) -> float:
    """aligner.py:308-318."""
    cfg = cfg or AlignerConfig()
    prob = _problem(rig, matches, cfg)
    prob.set_params(params)
    e, _ = prob.residuals()
    return _weighted_mean(e, _weights_of(weights))


def loss_gradient(rig, matches, weights, params=None, cfg: AlignerConfig | None = None) -> LossGradient:
    """aligner.py:321-334: analytic gradient; the gauge block is exactly zero."""
    cfg = cfg or AlignerConfig()
    prob = _problem(rig, matches, cfg)
    if params is None:
        params = identity_params(prob.n, cfg.optimize_focal)
    prob.set_params(params)
    prob.set_weights(_weights_of(weights))
    return prob.loss_and_gradient()


def adaptive_weights(residuals, alpha: float = DEFAULT_ALPHA) -> WeightTable:
    """weighting.py:94-109 on the device (histogram + density ratio)."""
    e = torch.as_tensor(np.asarray(residuals, dtype=np.float64).reshape(-1), device="cuda")
    w, avg = adaptive_weights_device(e, alpha)
    return WeightTable(w.cpu().numpy(), float(alpha), float(avg))


__all__ = ["AlignerConfig", "AlignmentReport", "LossGradient", "ResidualStats", "WeightTable", "DeviceProblem",
           "align", "align_arrays", "epipolar_residuals", "weighted_epipolar_loss", "loss_at", "loss_gradient",
           "adaptive_weights", "adaptive_weights_device", "identity_params", "select_learning_rate", "mode_id"]
