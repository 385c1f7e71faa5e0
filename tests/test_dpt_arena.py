"""The DPT heads' buffer arena (heads.DPTHeadDevice.prepare) on CPU, with the vx ops replaced by stand-ins
that propagate per-frame values from what each call reads to what it writes (interior only for
zero-bordered outputs, as the kernels do). Over a multi-chunk call:
  * every zero-bordered input a 3x3 conv reads has a zero border (the re-zeroing of buffers that share
    memory), and
  * the outputs equal those of the same call with separate, unshared buffers (the standalone path): a
    buffer overwritten while a later call still had to read it would change what that call reads.
The plan must also cover every buffer forward_chunk asks for (_pad raises otherwise). The GPU tests check
the same layout numerically with the real kernels."""
import types

import pytest
import torch

from paper_2509_25191_b200 import heads as heads_mod
from paper_2509_25191_b200.aggregator import DeviceWeights
from paper_2509_25191_b200.config import vggt_small
from paper_2509_25191_b200.weights import make_state_dict


class _Ops:
    def __init__(self):
        self.t = 0
        self.bad_borders = []

    def _tick(self):
        self.t += 1
        return 1e-3 * self.t

    @staticmethod
    def _frame_mean(x, F):
        return x.float().reshape(F, -1).mean(1)

    @staticmethod
    def _write(o, F, pad, v):
        tgt = o[:, 1:-1, 1:-1] if pad else o
        tgt.copy_(v.view(F, *([1] * (tgt.dim() - 1))).expand_as(tgt))

    def layernorm_tokens(self, x, start, w, b, eps, out=None, out_dtype=torch.bfloat16):
        F, T, C = x.shape
        v = self._frame_mean(x[:, start:], F) + self._tick()
        return v.view(F, 1, 1).expand(F, T - start, C).reshape(F * (T - start), C).to(out_dtype)

    def gemm_spatial(self, a, w, bias, F, H, W, conv3x3=False, out1=None, out1_pad=False, out2=None, out2_pad=False,
                     relu=False, pos=None, res1=None, res1_pad=False, res2=None, res2_pad=False, subsample2=False,
                     shuffle=1, head=None):
        if conv3x3:
            x = a.reshape(F, H + 2, W + 2, -1)
            if not bool((x[:, 0] == 0).all() and (x[:, -1] == 0).all() and (x[:, :, 0] == 0).all()
                        and (x[:, :, -1] == 0).all()):
                self.bad_borders.append((self.t, tuple(x.shape)))
            v = self._frame_mean(x[:, 1:-1, 1:-1], F)
        else:
            v = self._frame_mean(a, F)
        for r, k in ((res1, 0.37), (res2, 0.21)):
            if r is not None:
                v = v + k * self._frame_mean(r, F)
        v = v + self._tick()
        if head is not None:
            pred, conf = head[3], head[4]
            pred.copy_(v.view(F, 1, 1, 1).expand_as(pred))
            conf.copy_(v.view(F, 1, 1).expand_as(conf))
        for o, pad in ((out1, out1_pad), (out2, out2_pad)):
            if o is not None:
                self._write(o, F, pad, 0.5 * v if o is out2 else v)

    def upsample_bilinear(self, x, size, add=None, out=None, out_pad=False):
        F = x.shape[0]
        H, W = size
        if out is None:
            out = torch.empty(F, H, W, x.shape[3], dtype=x.dtype)
        self._write(out, F, out_pad, self._frame_mean(x, F) + self._tick())
        return out


def _run(prepared: bool, views: int, chunk: int):
    cfg = vggt_small()
    W = DeviceWeights(make_state_dict(cfg, 0), cfg, "cpu")
    head = heads_mod.DPTHeadDevice(W, "depth_head.", "exp")
    N, D, H = cfg.tokens_per_frame, 2 * cfg.embed_dim, cfg.img_size
    g = torch.Generator().manual_seed(0)
    kept = {i: torch.randn(views, N, D, generator=g).bfloat16() for i in cfg.kept_layers}
    pred, conf = torch.empty(views, H, H, 1), torch.empty(views, H, H)
    if prepared:
        head.prepare(min(views, chunk), "cpu")
    head(kept, pred, conf, chunk)
    if prepared:
        assert head._prepared  # __call__ leaves prepared buffers to the caller (VGGT.forward releases them)
        head.release()
    assert not head._bufs
    return pred, conf


@pytest.mark.parametrize("views,chunk", [(7, 3), (3, 3), (5, 2)])
def test_dpt_arena_liveness_and_borders(monkeypatch, views, chunk):
    results = {}
    for prepared in (False, True):
        ops = _Ops()
        monkeypatch.setattr(heads_mod, "ops", types.SimpleNamespace(
            layernorm_tokens=ops.layernorm_tokens, gemm_spatial=ops.gemm_spatial,
            upsample_bilinear=ops.upsample_bilinear))
        results[prepared] = _run(prepared, views, chunk)
        assert not ops.bad_borders, (prepared, ops.bad_borders)
    (pa, ca), (pb, cb) = results[False], results[True]
    assert torch.equal(pa, pb) and torch.equal(ca, cb)
