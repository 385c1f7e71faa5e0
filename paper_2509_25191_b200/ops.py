"""ctypes bindings of the C ABI (`include/vx_api.h`) over torch tensors.

Every function checks shapes/dtypes/devices, passes raw device pointers plus
the current CUDA stream, and raises RuntimeError with `vx_last_error()` on a
non-zero status.  There is no fallback: if `libvx.so` is missing or the device
is not a B200 the import / call fails loudly.
"""
from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import torch

_LIB_PATH = Path(__file__).resolve().parent / "libvx.so"

EPI_BF16, EPI_GELU, EPI_RESID, EPI_QKV, EPI_PATCH, EPI_F32 = range(6)
LF_F32, LF_GELU, LF_SILU_BF16, LF_POSE = range(4)  # vx_linear_f32 epilogues
ATTN_Q_LOG2 = 1  # vx_attention_ex flag: q pre-scaled by log2(e)/sqrt(d)

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f32 = ctypes.c_float


class Epilogue(ctypes.Structure):
    _fields_ = [
        ("bias", _vp), ("out", _vp), ("ldo", _i64),
        ("resid", _vp), ("ldr", _i64), ("gamma", _vp), ("kept", _vp), ("ldk", _i64),
        ("q", _vp), ("k", _vp), ("v", _vp),
        ("qn_w", _vp), ("qn_b", _vp), ("kn_w", _vp), ("kn_b", _vp),
        ("rope_cos", _vp), ("rope_sin", _vp),
        ("embed_dim", _i32), ("head_dim", _i32), ("tokens_total", _i32),
        ("tokens_per_frame", _i32), ("patch_start", _i32), ("grid_w", _i32),
        ("eps", _f32), ("q_scale", _f32), ("col_offset", _i32),
    ]


class Spatial(ctypes.Structure):
    _fields_ = [
        ("conv3x3", _i32), ("F", _i32), ("H", _i32), ("W", _i32), ("subsample2", _i32), ("shuffle", _i32),
        ("relu", _i32), ("pos", _vp), ("res1", _vp), ("res1_pad", _i32), ("res2", _vp), ("res2_pad", _i32),
        ("out1", _vp), ("out1_pad", _i32), ("out2", _vp), ("out2_pad", _i32),
        ("head_w", _vp), ("head_b", _vp), ("head_odim", _i32), ("head_act", _i32),
        ("head_pred", _vp), ("head_conf", _vp),
    ]


class GaProblem(ctypes.Structure):
    """vx_ga_problem (include/vx_api.h)."""
    _fields_ = [
        ("n_frames", _i32), ("n_pairs", _i32), ("dim", _i32), ("mode", _i32), ("gauge", _i32),
        ("pair_ij", _vp), ("offsets", _vp), ("xy_i", _vp), ("xy_j", _vp), ("w", _vp),
        ("frame_ptr", _vp), ("frame_ent", _vp), ("base_R", _vp), ("base_t", _vp), ("base_Kinv", _vp),
        ("params", _vp), ("adam_m", _vp), ("adam_v", _vp), ("Rs", _vp), ("ts", _vp), ("Kinv", _vp),
        ("geom", _vp), ("payload", _vp), ("scalars", _vp), ("status", _vp),
    ]


EXPORTED_SYMBOLS = ("vx_gemm", "vx_attention", "vx_attention_merge", "vx_attention_ex", "vx_layernorm", "vx_layernorm_gather", "vx_patchify",
                    "vx_special_tokens", "vx_dino_tokens", "vx_linear_f32", "vx_adaln_modulate",
                    "vx_upsample_bilinear", "vx_gemm_spatial", "vx_epipolar_residuals",
                    "vx_epipolar_accumulate", "vx_ga_decode", "vx_ga_residuals", "vx_ga_loss_grad",
                    "vx_ga_adam", "vx_ga_adaptive_weights", "vx_matched_points", "vx_unproject_depth",
                    "vx_select_pairs", "vx_pairwise_errors", "vx_num_sms", "vx_launch_count", "vx_last_error", "vx_version")

_lib = None


def load_library(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load libvx.so (no GPU needed) and declare the prototypes."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else _LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: run `python -m paper_2509_25191_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    lib.vx_gemm.argtypes = [_i32, _vp, _i64, _vp, _i64, _i32, _i32, _i32, ctypes.POINTER(Epilogue), _vp]
    lib.vx_attention.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _i64, _i64, _vp]
    lib.vx_attention_merge.argtypes = [_vp, _vp, _vp, _i32, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32,
                                       _i64, _i64, _vp]
    if hasattr(lib, "vx_attention_ex"):  # (absent from builds before it; tools/ A/B older libraries)
        lib.vx_attention_ex.argtypes = [_vp, _vp, _vp, _i32, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _i32, _i32,
                                        _i32, _i64, _i64, _i32, _vp]
    lib.vx_layernorm.argtypes = [_vp, _i32, _i64, _vp, _i32, _i64, _vp, _vp, _i32, _i32, _f32, _vp]
    lib.vx_layernorm_gather.argtypes = [_vp, _i32, _i64, _vp, _i32, _i64, _vp, _vp, _i32, _i32, _f32, _i32, _i32,
                                        _i32, _vp]
    lib.vx_patchify.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp]
    lib.vx_linear_f32.argtypes = [_i32, _vp, _i64, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp, _vp]
    lib.vx_adaln_modulate.argtypes = [_vp, _vp, _vp, _i32, _i32, _f32, _vp]
    lib.vx_special_tokens.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, _vp]
    lib.vx_dino_tokens.argtypes = [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]
    lib.vx_upsample_bilinear.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _i32, _vp]
    lib.vx_gemm_spatial.argtypes = [_vp, _vp, _i32, _i32, _vp, ctypes.POINTER(Spatial), _vp]
    lib.vx_epipolar_residuals.argtypes = [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]
    lib.vx_epipolar_accumulate.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp]
    _pb = ctypes.POINTER(GaProblem)
    _f64 = ctypes.c_double
    lib.vx_ga_decode.argtypes = [_pb, _vp]
    lib.vx_ga_residuals.argtypes = [_pb, _vp, _vp, _vp, _vp]
    lib.vx_ga_loss_grad.argtypes = [_pb, _vp, _vp]
    lib.vx_ga_adam.argtypes = [_pb, _i32, _i32, _f64, _vp, _vp, _vp, _vp, _i32, _vp]
    lib.vx_ga_adaptive_weights.argtypes = [_vp, _i64, _vp, _i32, _f64, _vp, _vp, _vp, _vp]
    lib.vx_matched_points.argtypes = [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _f64,
                                      _vp, _vp, _vp, _vp]
    lib.vx_unproject_depth.argtypes = [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]
    lib.vx_select_pairs.argtypes = [_vp, _i32, _f64, _vp, _vp, _vp]
    lib.vx_pairwise_errors.argtypes = [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]
    lib.vx_last_error.restype = ctypes.c_char_p
    lib.vx_version.restype = ctypes.c_char_p
    lib.vx_launch_count.restype = ctypes.c_uint64
    for name in EXPORTED_SYMBOLS:
        if name in ("vx_last_error", "vx_version", "vx_launch_count") or not hasattr(lib, name):
            continue  # (tests/test_abi.py checks that the product library exports every symbol)
        getattr(lib, name).restype = _i32
    if path is None:
        _lib = lib
    return lib


def use_library(path: os.PathLike) -> ctypes.CDLL:
    """Bind every op of this module to another build of the library (tools/: A/B runs against a
    `-DVX_DIAG` build from build.build_diag); the product path never calls this."""
    global _lib
    _lib = load_library(path)
    return _lib


# number of vx C-ABI calls issued by this process
launch_count = 0


def kernel_launches() -> int:
    """Kernels libvx has launched in this process (bench.py's gpu_launches; vx_launch_count)."""
    load_library()
    return int(_lib.vx_launch_count())


def _check(status: int, what: str):
    global launch_count
    launch_count += 1
    if status != 0:
        msg = _lib.vx_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({status}): {msg}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _req(t, dtype, name):
    if not t.is_cuda:
        raise RuntimeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")


def _rowmajor(t, name):
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name}: expected a 2-D row-major view, got shape {tuple(t.shape)} "
                         f"strides {t.stride()}")
    return t.stride(0)


# ---------------------------------------------------------------------------
def gemm(a: torch.Tensor, w: torch.Tensor, epi: int = EPI_BF16, bias=None, out=None, resid=None,
         gamma=None, kept=None, qkv=None, qk_norm=None, rope=None, head_dim=0, tokens_total=0,
         tokens_per_frame=1, patch_start=0, grid_w=1, eps=1e-5, q_scale=0.0, embed_dim=0, col_offset=0):
    """D = a @ w.T with the given fused epilogue (see include/vx_api.h). EPI_QKV: q_scale != 0
    multiplies q before its bf16 store (Q_LOG2_SCALE(d) for attention(..., q_log2=True)); w (and bias)
    may be the row slice [col_offset, col_offset + N) of the [3C, C] qkv weight, with embed_dim = C."""
    load_library()
    _req(a, torch.bfloat16, "a")
    _req(w, torch.bfloat16, "w")
    lda = _rowmajor(a, "a")
    ldw = _rowmajor(w, "w")
    M, K = a.shape
    N = w.shape[0]
    if w.shape[1] != K:
        raise ValueError(f"gemm: K mismatch {a.shape} x {w.shape}")
    ep = Epilogue()
    if bias is not None:
        _req(bias, torch.float32, "bias")
        ep.bias = bias.data_ptr()
    if epi in (EPI_BF16, EPI_GELU, EPI_F32):
        want = torch.float32 if epi == EPI_F32 else torch.bfloat16
        if out is None:
            out = torch.empty(M, N, device=a.device, dtype=want)
        _req(out, want, "out")
        ep.out = out.data_ptr()
        ep.ldo = _rowmajor(out, "out")
    if epi in (EPI_RESID, EPI_PATCH):
        _req(resid, torch.float32, "resid")
        ep.resid = resid.data_ptr()
        ep.ldr = _rowmajor(resid, "resid")
    if epi == EPI_RESID:
        _req(gamma, torch.float32, "gamma")
        ep.gamma = gamma.data_ptr()
        if kept is not None:
            _req(kept, torch.bfloat16, "kept")
            ep.kept = kept.data_ptr()
            ep.ldk = _rowmajor(kept, "kept")
    if epi == EPI_QKV:
        q, k, v = qkv
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            _req(t, torch.bfloat16, nm)
            if not t.is_contiguous():
                raise ValueError(f"{nm} must be contiguous [H, T, d]")
        ep.q, ep.k, ep.v = q.data_ptr(), k.data_ptr(), v.data_ptr()
        if qk_norm is not None:
            qw, qb, kw, kb = qk_norm
            ep.qn_w, ep.qn_b, ep.kn_w, ep.kn_b = (t.data_ptr() for t in (qw, qb, kw, kb))
        if rope is not None:
            ep.rope_cos, ep.rope_sin = rope[0].data_ptr(), rope[1].data_ptr()
        ep.embed_dim = embed_dim or N // 3
        ep.col_offset = col_offset
        ep.head_dim = head_dim
        ep.tokens_total = tokens_total
        ep.q_scale = q_scale
    ep.tokens_per_frame = tokens_per_frame
    ep.patch_start = patch_start
    ep.grid_w = grid_w
    ep.eps = eps
    _check(_lib.vx_gemm(epi, _ptr(a), lda, _ptr(w), ldw, M, N, K, ctypes.byref(ep), _stream()), "vx_gemm")
    return out


def Q_LOG2_SCALE(head_dim: int) -> float:
    """q scale that puts the attention scores in log2 units (gemm q_scale for attention q_log2=True)."""
    return 1.4426950408889634 / math.sqrt(head_dim)


def attention(q, k, v, out, nseq: int, Lq: int, Lk: int, lse=None, q_log2: bool = False):
    """Flash attention over q [H, Tq, d], k/v [H, Tk, d] -> out [Tq', H*d] (bf16). q_log2: q already
    holds q * Q_LOG2_SCALE(d) (the qkv epilogue's q_scale); the result means the same."""
    load_library()
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _req(t, torch.bfloat16, nm)
    H, Tq, D = q.shape
    Tk = k.shape[1]
    if k.shape != v.shape or k.shape[0] != H or k.shape[2] != D:
        raise ValueError("attention: q/k/v shape mismatch")
    if not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
        raise ValueError("attention: q/k/v must be contiguous")
    ldo = _rowmajor(out, "out")
    if lse is not None:
        _req(lse, torch.float32, "lse")
    if q_log2:
        _check(_lib.vx_attention_ex(_ptr(q), _ptr(k), _ptr(v), 0, None, 0, _ptr(lse), _ptr(out), ldo, D, H, nseq, Lq,
                                    Lk, Tq, Tk, ATTN_Q_LOG2, _stream()), "vx_attention_ex")
    else:
        _check(_lib.vx_attention(_ptr(q), _ptr(k), _ptr(v), _ptr(out), ldo, _ptr(lse), D, H, nseq, Lq, Lk,
                                 Tq, Tk, _stream()), "vx_attention")
    return out


def attention_merge(q, k, v, mode: int, o_acc, lse_acc, out=None, nseq: int = 1, Lq: int = 0, Lk: int = 0,
                    q_log2: bool = False):
    """One ring step with the fused LSE merge (vx_attention_merge): mode 1 first / 2 merge / 3 final (-> out)."""
    load_library()
    for t, nm in ((q, "q"), (k, "k"), (v, "v")):
        _req(t, torch.bfloat16, nm)
        if not t.is_contiguous():
            raise ValueError(f"attention_merge: {nm} must be contiguous")
    _req(o_acc, torch.float32, "o_acc")
    _req(lse_acc, torch.float32, "lse_acc")
    H, Tq, D = q.shape
    Tk = k.shape[1]
    ld_acc = _rowmajor(o_acc, "o_acc")
    ldo = 0
    if mode == 3:
        _req(out, torch.bfloat16, "out")
        ldo = _rowmajor(out, "out")
    if q_log2:
        _check(_lib.vx_attention_ex(_ptr(q), _ptr(k), _ptr(v), mode, _ptr(o_acc), ld_acc, _ptr(lse_acc),
                                    _ptr(out) if mode == 3 else None, ldo, D, H, nseq, Lq or Tq, Lk or Tk, Tq, Tk,
                                    ATTN_Q_LOG2, _stream()), "vx_attention_ex")
    else:
        _check(_lib.vx_attention_merge(_ptr(q), _ptr(k), _ptr(v), mode, _ptr(o_acc), ld_acc, _ptr(lse_acc),
                                       _ptr(out) if mode == 3 else None, ldo, D, H, nseq, Lq or Tq, Lk or Tk, Tq, Tk,
                                       _stream()), "vx_attention_merge")


def layernorm(x, w, b, eps, out=None, out_dtype=torch.bfloat16):
    load_library()
    if not x.is_cuda:
        raise RuntimeError("layernorm: CUDA tensor required")
    ldx = _rowmajor(x, "x")
    rows, cols = x.shape
    if out is None:
        out = torch.empty(rows, cols, device=x.device, dtype=out_dtype)
    ldy = _rowmajor(out, "out")
    code = {torch.float32: 0, torch.bfloat16: 1}
    _check(_lib.vx_layernorm(_ptr(x), code[x.dtype], ldx, _ptr(out), code[out.dtype], ldy, _ptr(w), _ptr(b),
                             rows, cols, eps, _stream()), "vx_layernorm")
    return out


def layernorm_tokens(x, start: int, w, b, eps, out=None, out_dtype=torch.bfloat16):
    """LayerNorm of x[:, start:, :] for x [F, T, C] contiguous, written as [F*(T-start), C] (no gather copy)."""
    load_library()
    if not x.is_cuda or not x.is_contiguous() or x.dim() != 3:
        raise RuntimeError("layernorm_tokens: contiguous CUDA [F, T, C] required")
    F_, T, C = x.shape
    rows = F_ * (T - start)
    if out is None:
        out = torch.empty(rows, C, device=x.device, dtype=out_dtype)
    ldy = _rowmajor(out, "out")
    code = {torch.float32: 0, torch.bfloat16: 1}
    _check(_lib.vx_layernorm_gather(_ptr(x), code[x.dtype], C, _ptr(out), code[out.dtype], ldy, _ptr(w), _ptr(b),
                                    rows, C, eps, T - start, T, start, _stream()), "vx_layernorm_gather")
    return out


def patchify(images, patch: int, kpad: int, out=None):
    load_library()
    _req(images, torch.float32, "images")
    images = images.contiguous()
    S, C, H, W = images.shape
    P = (H // patch) * (W // patch)
    if out is None:
        out = torch.empty(S * P, kpad, device=images.device, dtype=torch.bfloat16)
    _check(_lib.vx_patchify(_ptr(images), _ptr(out), S, H, W, patch, kpad, _stream()), "vx_patchify")
    return out


def special_tokens(x, tokens, S, tpf):
    load_library()
    _req(x, torch.float32, "x")
    _req(tokens, torch.float32, "tokens")
    ntok, C = tokens.shape[-2], tokens.shape[-1]
    _check(_lib.vx_special_tokens(_ptr(x), _ptr(tokens.contiguous()), S, tpf, ntok, C, _stream()),
           "vx_special_tokens")
    return x


def linear_f32(x, w, bias, epi: int = LF_F32, out=None, prev=None, act_out=None):
    """fp32 out = epi(x @ w.T + bias) (vx_linear_f32).  x (M, K) or one broadcast row (1, K) with
    `rows`; LF_SILU_BF16 writes bf16; LF_POSE (N = 9) writes pred = prev + delta to `out` and
    activate_pose(pred) to `act_out`."""
    load_library()
    _req(x, torch.float32, "x")
    _req(w, torch.float32, "w")
    ldw = _rowmajor(w, "w")
    N, K = w.shape
    if x.dim() != 2 or x.shape[1] != K or (x.stride(1) != 1 and K > 1):
        raise ValueError(f"linear_f32: x must be (M, {K}) row-major, got {tuple(x.shape)} strides {x.stride()}")
    M = x.shape[0]
    ldx = x.stride(0) if M > 1 else K  # stride 0: one row broadcast to all M (expand)
    if bias is not None:
        _req(bias, torch.float32, "bias")
    want = torch.bfloat16 if epi == LF_SILU_BF16 else torch.float32
    if out is None:
        out = torch.empty(M, N, device=x.device, dtype=want)
    _req(out, want, "out")
    ldo = _rowmajor(out, "out")
    if epi == LF_POSE:
        if act_out is None or prev is not None and (prev.shape != out.shape or not prev.is_contiguous()):
            raise ValueError("linear_f32: pose epilogue needs act_out and a (M, 9) prev like out")
        _req(act_out, torch.float32, "act_out")
        if act_out.shape != out.shape or not (out.is_contiguous() and act_out.is_contiguous()):
            raise ValueError("linear_f32: pose outputs must be contiguous (M, 9)")
    _check(_lib.vx_linear_f32(epi, _ptr(x), ldx, _ptr(w), ldw, _ptr(bias), M, N, K, _ptr(out), ldo, _ptr(prev),
                              _ptr(act_out), _stream()), "vx_linear_f32")
    return out


def adaln_modulate(tok, mod, eps: float, out=None):
    """gate * (LN_noaffine(tok) * (1 + scale) + shift) + tok, mod = [shift | scale | gate] (vx_adaln_modulate)."""
    load_library()
    _req(tok, torch.float32, "tok")
    _req(mod, torch.float32, "mod")
    S, D = tok.shape
    if not (tok.is_contiguous() and mod.is_contiguous()) or tuple(mod.shape) != (S, 3 * D):
        raise ValueError("adaln_modulate: contiguous tok (S, D) and mod (S, 3D) required")
    if out is None:
        out = torch.empty_like(tok)
    _check(_lib.vx_adaln_modulate(_ptr(tok), _ptr(mod), _ptr(out), S, D, eps, _stream()), "vx_adaln_modulate")
    return out


def dino_tokens(x, cls, reg, pos, S: int, tpf: int):
    """DINOv2 cls / register tokens and position embedding on the patch-embedded stream x [S*tpf, C] fp32."""
    load_library()
    for t, nm in ((x, "x"), (cls, "cls"), (reg, "reg"), (pos, "pos")):
        _req(t, torch.float32, nm)
        if not t.is_contiguous():
            raise ValueError(f"dino_tokens: {nm} must be contiguous")
    C = x.shape[-1]
    nreg = reg.numel() // C
    if pos.numel() != (tpf - nreg) * C:
        raise ValueError("dino_tokens: pos must be [1 + patches, C]")
    _check(_lib.vx_dino_tokens(_ptr(x), _ptr(cls), _ptr(reg), _ptr(pos), S, tpf, nreg, C, _stream()),
           "vx_dino_tokens")
    return x


def upsample_bilinear(x: torch.Tensor, size, add=None, out=None, out_pad: bool = False):
    """NHWC bf16 [F, h, w, C] -> [F, H, W, C] (or the interior of a zero-bordered
    [F, H+2, W+2, C] buffer when out_pad), align_corners=True, + optional [H, W, C] add."""
    load_library()
    _req(x, torch.bfloat16, "x")
    if not x.is_contiguous():
        raise ValueError("upsample_bilinear: x must be contiguous NHWC")
    F_, h, w, C = x.shape
    H, W = size
    if out is None:
        shape = (F_, H + 2, W + 2, C) if out_pad else (F_, H, W, C)
        out = (torch.zeros if out_pad else torch.empty)(shape, device=x.device, dtype=torch.bfloat16)
    if add is not None:
        _req(add, torch.bfloat16, "add")
        if tuple(add.shape) != (H, W, C) or not add.is_contiguous():
            raise ValueError("upsample_bilinear: add must be contiguous [H, W, C]")
    _check(_lib.vx_upsample_bilinear(_ptr(x), F_, h, w, C, _ptr(out), H, W, _ptr(add), int(out_pad), _stream()),
           "vx_upsample_bilinear")
    return out


def gemm_spatial(a, w, bias, F: int, H: int, W: int, conv3x3=False, out1=None, out1_pad=False, out2=None,
                 out2_pad=False, relu=False, pos=None, res1=None, res1_pad=False, res2=None, res2_pad=False,
                 subsample2=False, shuffle=1, head=None):
    """DPT spatial GEMM (see include/vx_api.h vx_gemm_spatial).

    a: bf16 rows [F*(H+2)*(W+2), Cin] (conv3x3, zero-padded NHWC) or [F*H*W, K];
    w: bf16 [N, K] (conv3x3: K = 9*Cin ordered (ky, kx, cin)).
    head = (w_fp32 [odim, 32], b_fp32, act, pred [F,H,W,odim-1], conf [F,H,W]) fuses the output head.
    """
    load_library()
    _req(a, torch.bfloat16, "a")
    _req(w, torch.bfloat16, "w")
    if not (a.is_contiguous() and w.is_contiguous()):
        raise ValueError("gemm_spatial: a and w must be contiguous")
    N, K = w.shape
    sp = Spatial()
    sp.conv3x3, sp.F, sp.H, sp.W = int(conv3x3), F, H, W
    sp.subsample2, sp.shuffle, sp.relu = int(subsample2), shuffle, int(relu)
    for name, t in (("pos", pos), ("res1", res1), ("res2", res2), ("out1", out1), ("out2", out2)):
        if t is not None:
            _req(t, torch.bfloat16, name)
            if not t.is_contiguous():
                raise ValueError(f"gemm_spatial: {name} must be contiguous")
            setattr(sp, name, t.data_ptr())
    sp.res1_pad, sp.res2_pad, sp.out1_pad, sp.out2_pad = int(res1_pad), int(res2_pad), int(out1_pad), int(out2_pad)
    if head is not None:
        hw, hb, act, pred, conf = head
        for t, nm in ((hw, "head_w"), (hb, "head_b"), (pred, "head_pred"), (conf, "head_conf")):
            _req(t, torch.float32, nm)
        sp.head_w, sp.head_b, sp.head_pred, sp.head_conf = hw.data_ptr(), hb.data_ptr(), pred.data_ptr(), conf.data_ptr()
        sp.head_odim, sp.head_act = hw.shape[0], act
    if bias is not None:
        _req(bias, torch.float32, "bias")
    _check(_lib.vx_gemm_spatial(_ptr(a), _ptr(w), N, K, _ptr(bias), ctypes.byref(sp), _stream()), "vx_gemm_spatial")
    return out1


def epipolar_residuals(F, offsets, xy_i, xy_j, mode: int):
    """Batched pair_residuals: F [P,3,3] f64, offsets [P+1] int64, xy [K,2] f64 -> (e [K], n_deg [P])."""
    load_library()
    for t, nm, dt in ((F, "F", torch.float64), (offsets, "offsets", torch.int64), (xy_i, "xy_i", torch.float64),
                      (xy_j, "xy_j", torch.float64)):
        _req(t, dt, nm)
        if not t.is_contiguous():
            raise ValueError(f"{nm} must be contiguous")
    P = F.shape[0]
    e = torch.empty(xy_i.shape[0], device=F.device, dtype=torch.float64)
    nd = torch.empty(P, device=F.device, dtype=torch.int32)
    _check(_lib.vx_epipolar_residuals(_ptr(F), _ptr(offsets), _ptr(xy_i), _ptr(xy_j), P, mode, _ptr(e), _ptr(nd),
                                      _stream()), "vx_epipolar_residuals")
    return e, nd


def epipolar_accumulate(F, offsets, xy_i, xy_j, w, mode: int):
    """Batched pair_accumulate -> (out [P, 11] = loss, wsum, G row-major; n_skipped [P])."""
    load_library()
    for t, nm, dt in ((F, "F", torch.float64), (offsets, "offsets", torch.int64), (xy_i, "xy_i", torch.float64),
                      (xy_j, "xy_j", torch.float64), (w, "w", torch.float64)):
        _req(t, dt, nm)
        if not t.is_contiguous():
            raise ValueError(f"{nm} must be contiguous")
    P = F.shape[0]
    out = torch.empty(P, 11, device=F.device, dtype=torch.float64)
    sk = torch.empty(P, device=F.device, dtype=torch.int32)
    _check(_lib.vx_epipolar_accumulate(_ptr(F), _ptr(offsets), _ptr(xy_i), _ptr(xy_j), _ptr(w), P, mode, _ptr(out),
                                       _ptr(sk), _stream()), "vx_epipolar_accumulate")
    return out, sk


# ---------------------------------------------------------------------------
# Global-Alignment optimiser (ga.cu); the problem struct is built by paper_2509_25191_b200.ga


def ga_decode(pb: GaProblem):
    load_library()
    _check(_lib.vx_ga_decode(ctypes.byref(pb), _stream()), "vx_ga_decode")


def ga_residuals(pb: GaProblem, e, deg_pair, n_deg):
    load_library()
    _check(_lib.vx_ga_residuals(ctypes.byref(pb), _ptr(e), _ptr(deg_pair), _ptr(n_deg), _stream()),
           "vx_ga_residuals")


def ga_loss_grad(pb: GaProblem, grad):
    load_library()
    _check(_lib.vx_ga_loss_grad(ctypes.byref(pb), _ptr(grad), _stream()), "vx_ga_loss_grad")


def ga_adam(pb: GaProblem, t0: int, iters: int, lr: float, bc1, bc2, trace, skipped, use_graph: bool = True):
    load_library()
    _check(_lib.vx_ga_adam(ctypes.byref(pb), t0, iters, float(lr), _ptr(bc1), _ptr(bc2), _ptr(trace), _ptr(skipped),
                           int(use_graph), _stream()), "vx_ga_adam")


def ga_adaptive_weights(e, edges, alpha: float, w, counts, stats):
    load_library()
    for t, nm, dt in ((e, "e", torch.float64), (edges, "edges", torch.float64), (w, "w", torch.float64),
                      (counts, "counts", torch.int64), (stats, "stats", torch.float64)):
        _req(t, dt, nm)
    _check(_lib.vx_ga_adaptive_weights(_ptr(e), e.numel(), _ptr(edges), edges.numel() - 1, float(alpha), _ptr(w),
                                       _ptr(counts), _ptr(stats), _stream()), "vx_ga_adaptive_weights")


# ---------------------------------------------------------------------------
# scene-level consumers (scene.cu); paper_2509_25191_b200.scene builds the arguments


def matched_points(depth, map_offset, map_hw, slot, R, t, Kinv, pair_ij, offsets, xy_i, xy_j, w, threshold: float):
    """-> (points [K, 6], gap [K], state int8 [K]) per correspondence."""
    load_library()
    K = xy_i.shape[0]
    dev = xy_i.device
    points = torch.empty(K, 6, device=dev, dtype=torch.float64)
    gap = torch.empty(K, device=dev, dtype=torch.float64)
    state = torch.empty(K, device=dev, dtype=torch.int8)
    if depth.dtype not in (torch.float32, torch.float64):
        raise TypeError("depth maps must be float32 or float64")
    _check(_lib.vx_matched_points(_ptr(depth), int(depth.dtype == torch.float32), _ptr(map_offset), _ptr(map_hw),
                                  _ptr(slot), _ptr(R), _ptr(t), _ptr(Kinv), _ptr(pair_ij), _ptr(offsets),
                                  pair_ij.shape[0], _ptr(xy_i), _ptr(xy_j), _ptr(w), float(threshold), _ptr(points),
                                  _ptr(gap), _ptr(state), _stream()), "vx_matched_points")
    return points, gap, state


def unproject_depth(depth, extrinsic, intrinsic, out=None):
    """depth fp32 [S, H, W], extrinsic [S, 3, 4], intrinsic [S, 3, 3] -> world points fp32 [S, H, W, 3]."""
    load_library()
    for x, nm in ((depth, "depth"), (extrinsic, "extrinsic"), (intrinsic, "intrinsic")):
        _req(x, torch.float32, nm)
        if not x.is_contiguous():
            raise ValueError(f"{nm} must be contiguous")
    S, H, W = depth.shape
    if out is None:
        out = torch.empty(S, H, W, 3, device=depth.device, dtype=torch.float32)
    _check(_lib.vx_unproject_depth(_ptr(depth), S, H, W, _ptr(extrinsic), _ptr(intrinsic), _ptr(out), _stream()),
           "vx_unproject_depth")
    return out


def select_pairs(R, threshold_deg: float):
    """R fp64 [n, 9] -> (flag int8 [n(n-1)/2], angle fp64 [n(n-1)/2]) in upper-triangle order."""
    load_library()
    n = R.shape[0]
    m = n * (n - 1) // 2
    flag = torch.zeros(max(m, 1), device=R.device, dtype=torch.int8)
    angle = torch.empty(max(m, 1), device=R.device, dtype=torch.float64)
    _check(_lib.vx_select_pairs(_ptr(R), n, float(threshold_deg), _ptr(flag), _ptr(angle), _stream()),
           "vx_select_pairs")
    return flag[:m], angle[:m]


def pairwise_errors(Rp, tp, Rg, tg, gt_of, order_invariant: bool):
    load_library()
    n = Rp.shape[0]
    m = n * (n - 1) // 2 * (2 if order_invariant else 1)
    dev = Rp.device
    rre = torch.empty(max(m, 1), device=dev, dtype=torch.float64)
    rte = torch.empty(max(m, 1), device=dev, dtype=torch.float64)
    flag = torch.empty(max(m, 1), device=dev, dtype=torch.uint8)
    _check(_lib.vx_pairwise_errors(_ptr(Rp), _ptr(tp), _ptr(Rg), _ptr(tg), _ptr(gt_of), n, int(order_invariant),
                                   _ptr(rre), _ptr(rte), _ptr(flag), _stream()), "vx_pairwise_errors")
    return rre[:m], rte[:m], flag[:m]
