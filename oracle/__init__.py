"""CPU fp64 oracle for fused neighborhood attention — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2403_04690_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``na_oracle.c`` (see its header for the
definition and the PAPER.md passages it follows); this module only compiles
that file with gcc and marshals arguments through ctypes.

Parity pins (tests/test_oracle_pins.py, all ``-m "not gpu"``):
  * window rule            — brute-force "most centred in-bounds window" enumeration
                             and SPEC examples
  * full window, dil 1      — dense softmax attention, Eq. 1
  * causal full window      — dense lower-triangular attention
  * kernel size 1           — O = V, linear projection
  * dilation                — composition over residue classes
  * gradients               — central finite differences + torch autograd
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "na_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

F64, F32, F16, BF16 = 0, 1, 2, 3


class Problem(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("extent", ctypes.c_int32 * 3),
        ("kernel_size", ctypes.c_int32 * 3),
        ("dilation", ctypes.c_int32 * 3),
        ("is_causal", ctypes.c_int32 * 3),
        ("scale", ctypes.c_double),
    ]


def make_problem(batch, heads, extent, head_dim, kernel_size, dilation=None, is_causal=None,
                 scale=0.0) -> Problem:
    r = len(extent)
    dilation = dilation or [1] * r
    is_causal = is_causal or [0] * r
    pad = lambda xs, f: list(xs) + [f] * (3 - len(xs))
    return Problem(r, batch, heads, head_dim,
                   (ctypes.c_int32 * 3)(*pad(extent, 1)),
                   (ctypes.c_int32 * 3)(*pad(kernel_size, 1)),
                   (ctypes.c_int32 * 3)(*pad(dilation, 1)),
                   (ctypes.c_int32 * 3)(*pad([int(bool(c)) for c in is_causal], 0)),
                   float(scale))


def build(force: bool = False) -> str:
    """Compile liboracle.so (host code only: gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "na_oracle.h"))):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            P = ctypes.POINTER(Problem)
            vp, dp, i64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64
            L.nar_check.argtypes = [P]
            L.nar_axis_window.argtypes = [ctypes.c_int] * 5 + [ctypes.POINTER(ctypes.c_int)] * 2
            L.nar_contains.argtypes = [P, i64, i64]
            L.nar_fwd.argtypes = [P, ctypes.c_int, vp, vp, vp, dp, dp]
            L.nar_fwd_tokens.argtypes = [P, ctypes.c_int, vp, vp, vp, i64, vp, dp, dp]
            L.nar_bwd.argtypes = [P, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, dp, dp, dp]
            L.nar_bwd_gather.argtypes = [P, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, dp, dp, dp]
            L.nar_bwd_tokens.argtypes = [P, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, i64, vp, dp, dp,
                                         dp]
            _lib = L
    return _lib


# ---------------------------------------------------------------- marshalling

def _as_host(x):
    """Return (contiguous host buffer object, dtype code).  Accepts numpy arrays
    or CPU torch tensors (fp64/fp32/fp16/bf16).  bf16/fp16 are passed as raw
    16-bit patterns and upcast exactly inside the C code."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().contiguous()
            if x.device.type != "cpu":
                x = x.cpu()
            code = {torch.float64: F64, torch.float32: F32, torch.float16: F16,
                    torch.bfloat16: BF16}[x.dtype]
            return x, code, x.data_ptr()
    except ImportError:  # pragma: no cover
        pass
    x = np.ascontiguousarray(x)
    code = {np.dtype(np.float64): F64, np.dtype(np.float32): F32, np.dtype(np.float16): F16}[x.dtype]
    return x, code, x.ctypes.data


def _prep(q, k, v, *more):
    bufs = [_as_host(t) for t in (q, k, v) + more]
    codes = {b[1] for b in bufs}
    if len(codes) != 1:
        raise TypeError("oracle inputs must share one dtype")
    return bufs, codes.pop()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def check(p: Problem) -> int:
    return lib().nar_check(ctypes.byref(p))


def axis_window(L, k, dil, causal, x):
    f, l = ctypes.c_int(), ctypes.c_int()
    n = lib().nar_axis_window(L, k, dil, int(causal), x, ctypes.byref(f), ctypes.byref(l))
    return f.value, l.value, n


def contains(p: Problem, x: int, y: int) -> bool:
    return bool(lib().nar_contains(ctypes.byref(p), x, y))


def _tokens(p):
    n = 1
    for a in range(p.rank):
        n *= p.extent[a]
    return n


def fwd(p: Problem, q, k, v):
    """Full forward.  Returns (O [B,H,N,D] fp64, LSE [B,H,N] fp64) as numpy."""
    (bq, bk, bv), code = _prep(q, k, v)
    N, BH, D = _tokens(p), p.batch * p.heads, p.head_dim
    o = np.empty((BH * N * D,), np.float64)
    lse = np.empty((BH * N,), np.float64)
    rc = lib().nar_fwd(ctypes.byref(p), code, bq[2], bk[2], bv[2], _ptr(o), _ptr(lse))
    if rc:
        raise ValueError(f"oracle rejected problem (code {rc})")
    return o.reshape(p.batch, p.heads, N, D), lse.reshape(p.batch, p.heads, N)


def fwd_tokens(p: Problem, q, k, v, tokens):
    (bq, bk, bv), code = _prep(q, k, v)
    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
    o = np.empty((len(t), p.head_dim), np.float64)
    lse = np.empty((len(t),), np.float64)
    rc = lib().nar_fwd_tokens(ctypes.byref(p), code, bq[2], bk[2], bv[2], len(t), t.ctypes.data,
                              _ptr(o), _ptr(lse))
    if rc:
        raise ValueError(f"oracle rejected problem (code {rc})")
    return o, lse


def bwd(p: Problem, q, k, v, d_o, stored_o: bool = False):
    """Full backward.  Returns (dQ, dK, dV), each [B,H,N,D] fp64.

    stored_o=False: the exact gradient.  stored_o=True: the softmax-Jacobian
    term D_x = <dO_x, O_x> uses O as the method stores it -- the oracle's own
    fp64 O rounded to the inputs' dtype (reading R12)."""
    (bq, bk, bv, bo), code = _prep(q, k, v, d_o)
    N, BH, D = _tokens(p), p.batch * p.heads, p.head_dim
    outs = [np.empty((BH * N * D,), np.float64) for _ in range(3)]
    rc = lib().nar_bwd(ctypes.byref(p), code, code if stored_o else F64, bq[2], bk[2], bv[2], bo[2],
                       *map(_ptr, outs))
    if rc:
        raise ValueError(f"oracle rejected problem (code {rc})")
    return tuple(o.reshape(p.batch, p.heads, N, D) for o in outs)


def bwd_gather(p: Problem, q, k, v, d_o, stored_o: bool = False):
    """Full backward in gather form (parallel over tokens; for whole-slice
    checks of large problems).  Same result as bwd() up to fp64 summation
    order; returns (dQ, dK, dV), each [B,H,N,D] fp64."""
    (bq, bk, bv, bo), code = _prep(q, k, v, d_o)
    N, BH, D = _tokens(p), p.batch * p.heads, p.head_dim
    outs = [np.empty((BH * N * D,), np.float64) for _ in range(3)]
    rc = lib().nar_bwd_gather(ctypes.byref(p), code, code if stored_o else F64, bq[2], bk[2], bv[2],
                              bo[2], *map(_ptr, outs))
    if rc:
        raise ValueError(f"oracle rejected problem (code {rc})")
    return tuple(o.reshape(p.batch, p.heads, N, D) for o in outs)


def fwd_full_tokens(p: Problem, q, k, v):
    """Full forward via the token form (parallel over tokens rather than
    slices); returns (O [B,H,N,D], LSE [B,H,N])."""
    N, BH, D = _tokens(p), p.batch * p.heads, p.head_dim
    o, lse = fwd_tokens(p, q, k, v, np.arange(BH * N, dtype=np.int64))
    return o.reshape(p.batch, p.heads, N, D), lse.reshape(p.batch, p.heads, N)


def bwd_tokens(p: Problem, q, k, v, d_o, tokens, stored_o: bool = False):
    (bq, bk, bv, bo), code = _prep(q, k, v, d_o)
    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
    outs = [np.empty((len(t), p.head_dim), np.float64) for _ in range(3)]
    rc = lib().nar_bwd_tokens(ctypes.byref(p), code, code if stored_o else F64, bq[2], bk[2], bv[2],
                              bo[2], len(t),
                              t.ctypes.data, *map(_ptr, outs))
    if rc:
        raise ValueError(f"oracle rejected problem (code {rc})")
    return tuple(outs)


def num_threads() -> int:
    return lib().nar_num_threads()
