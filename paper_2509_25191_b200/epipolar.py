"""Drop-in epipolar kernel implementation for the reference's GA aligner.

Mirrors the reference module interface `epialign.kernels` / `_kernels_cy`
(pkg/src/epialign/kernels.py:12-43, _kernels_cy.pyx:12-116): the constants,
`IMPL`, `pair_residuals(F, xy_i, xy_j, mode)` and
`pair_accumulate(F, xy_i, xy_j, w, mode)` with identical argument meaning,
return types and degenerate / dead-zone semantics.  The per-pair functions take
host numpy arrays like the reference; the batched `pairs_residuals` /
`pairs_accumulate` evaluate every image pair of an alignment step in one launch
(the reference loops over pairs on a host thread pool, aligner.py:190-278).
"""
from __future__ import annotations

import numpy as np
import torch

from . import ops

LINE_NORMAL_EPS = 1e-12
GRAD_DEADZONE = 1e-9
MODE_ALGEBRAIC = 0
MODE_GEOMETRIC = 1
IMPL = "cuda"


def _dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).cuda()


def pairs_residuals(Fs, offsets, xy_i, xy_j, mode: int):
    """All pairs at once (torch CUDA tensors): -> (e [K], n_deg [P])."""
    return ops.epipolar_residuals(Fs, offsets, xy_i, xy_j, mode)


def pairs_accumulate(Fs, offsets, xy_i, xy_j, w, mode: int):
    """All pairs at once: -> (loss_sum [P], weight_sum [P], G [P,3,3], n_skipped [P])."""
    out, sk = ops.epipolar_accumulate(Fs, offsets, xy_i, xy_j, w, mode)
    return out[:, 0], out[:, 1], out[:, 2:].reshape(-1, 3, 3), sk


def pair_residuals(F, xy_i, xy_j, mode):
    """Residuals of one pair; NaN marks degenerate geometric lines. -> (e (k,), n_degenerate)."""
    k = np.shape(xy_i)[0]
    e, nd = pairs_residuals(_dev(np.reshape(F, (1, 3, 3))), _dev([0, k], torch.int64), _dev(xy_i), _dev(xy_j),
                            int(mode))
    return e.cpu().numpy(), int(nd.item())


def pair_accumulate(F, xy_i, xy_j, w, mode):
    """Weighted residual sum and its gradient w.r.t. F for one pair.
    -> (loss_sum, weight_sum, G (3,3), n_skipped)."""
    k = np.shape(xy_i)[0]
    l, ws, G, sk = pairs_accumulate(_dev(np.reshape(F, (1, 3, 3))), _dev([0, k], torch.int64), _dev(xy_i),
                                    _dev(xy_j), _dev(w), int(mode))
    return float(l.item()), float(ws.item()), G[0].cpu().numpy(), int(sk.item())
