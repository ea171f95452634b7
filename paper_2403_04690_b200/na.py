"""ctypes binding of include/na.h — argument marshalling only.

Every step of the computation runs in libna.so's CUDA kernels.  Tensors are
torch CUDA tensors indexed [B, H, X0 (, X1 (, X2)), D]; a non-contiguous
layout (e.g. a heads-last [B, X..., H, D] tensor viewed with permute) is
passed to the ABI as element strides, so all tensors of one call must share
q's strides (outputs are allocated with them).  LSE is always a contiguous
fp32 [B, H, X...] tensor.  The call is enqueued on torch's current CUDA
stream.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libna.so")

NA_F32, NA_F16, NA_BF16 = 0, 1, 2
NA_IMPL_AUTO, NA_IMPL_SIMT, NA_IMPL_TC = 0, 1, 2
_DTYPES = {torch.float32: NA_F32, torch.float16: NA_F16, torch.bfloat16: NA_BF16}
_IMPLS = {"auto": NA_IMPL_AUTO, "simt": NA_IMPL_SIMT, "tc": NA_IMPL_TC}


class Problem(ctypes.Structure):
    """Mirror of ``na_problem`` (include/na.h)."""
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("extent", ctypes.c_int32 * 3),
        ("kernel_size", ctypes.c_int32 * 3),
        ("dilation", ctypes.c_int32 * 3),
        ("is_causal", ctypes.c_int32 * 3),
        ("scale", ctypes.c_float),
        ("dtype", ctypes.c_int32),
        ("impl", ctypes.c_int32),
        ("strides", ctypes.c_void_p),
    ]


class NAError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{status_string(status)} ({status}): {detail}")
        self.status = status


_lib = None

EXPORTS = ("na_validate", "na_fwd", "na_bwd", "na_bwd_workspace_size", "na_selected_impl",
           "na_bf16_precise",
           "na_status_string", "na_last_error", "na_last_launch_count", "na_profile_enable",
           "na_profile_collect", "na_kernel_name", "na_plan_candidates", "na_tune",
           "na_get_plan_choice", "na_set_plan_choice")


def lib():
    """Load libna.so (must have been built in-tree; raises if missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() or "
                              "python -m paper_2403_04690_b200.build (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER(Problem)
        vp = ctypes.c_void_p
        L.na_validate.argtypes = [P]
        L.na_validate.restype = ctypes.c_int
        L.na_fwd.argtypes = [P, vp, vp, vp, vp, vp, vp]
        L.na_fwd.restype = ctypes.c_int
        L.na_bwd.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
        L.na_bwd.restype = ctypes.c_int
        L.na_bwd_workspace_size.argtypes = [P]
        L.na_bwd_workspace_size.restype = ctypes.c_size_t
        L.na_selected_impl.argtypes = [P]
        L.na_selected_impl.restype = ctypes.c_int
        L.na_bf16_precise.argtypes = [P]
        L.na_bf16_precise.restype = ctypes.c_int
        L.na_status_string.argtypes = [ctypes.c_int]
        L.na_status_string.restype = ctypes.c_char_p
        L.na_last_error.argtypes = []
        L.na_last_error.restype = ctypes.c_char_p
        L.na_last_launch_count.argtypes = []
        L.na_last_launch_count.restype = ctypes.c_int
        L.na_profile_enable.argtypes = [ctypes.c_int]
        L.na_profile_enable.restype = None
        L.na_profile_collect.argtypes = [ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_float), ctypes.c_int]
        L.na_profile_collect.restype = ctypes.c_int
        L.na_kernel_name.argtypes = [ctypes.c_int]
        L.na_kernel_name.restype = ctypes.c_char_p
        I3 = ctypes.c_int32 * 3
        L.na_plan_candidates.argtypes = [P]
        L.na_plan_candidates.restype = ctypes.c_int
        L.na_tune.argtypes = [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, I3]
        L.na_tune.restype = ctypes.c_int
        L.na_get_plan_choice.argtypes = [P, I3]
        L.na_get_plan_choice.restype = ctypes.c_int
        L.na_set_plan_choice.argtypes = [P, I3]
        L.na_set_plan_choice.restype = ctypes.c_int
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().na_status_string(s).decode()


def _check(status: int):
    if status != 0:
        raise NAError(status, lib().na_last_error().decode())


def make_problem(batch, heads, extent, head_dim, kernel_size, dilation=None, is_causal=None,
                 scale=None, dtype=torch.float16, impl="auto") -> Problem:
    r = len(extent)
    if isinstance(kernel_size, int):
        kernel_size = [kernel_size] * r
    dilation = [dilation] * r if isinstance(dilation, int) else (dilation or [1] * r)
    is_causal = [is_causal] * r if isinstance(is_causal, bool) else (is_causal or [False] * r)
    pad = lambda xs, f: [int(x) for x in xs] + [f] * (3 - len(xs))
    A = ctypes.c_int32 * 3
    return Problem(r, batch, heads, head_dim, A(*pad(extent, 1)), A(*pad(kernel_size, 1)),
                   A(*pad(dilation, 1)), A(*pad([bool(c) for c in is_causal], 0)),
                   float(scale) if scale else 0.0, _DTYPES[dtype], _IMPLS[impl], None)


def _problem_from(q: torch.Tensor, kernel_size, dilation, is_causal, scale, impl) -> Problem:
    if q.dim() < 4 or q.dim() > 6:
        raise ValueError("expected [B, H, X0 (, X1 (, X2)), D]")
    B, H, *ext, D = q.shape
    p = make_problem(B, H, ext, D, kernel_size, dilation, is_causal, scale, q.dtype, impl)
    if not q.is_contiguous():  # na_problem.strides: [B, H, X0, X1, X2, D] in elements
        sB, sH, *sX, sD = q.stride()
        p._strides = (ctypes.c_int64 * 6)(sB, sH, *(list(sX) + [0] * (3 - len(sX))), sD)
        p.strides = ctypes.cast(p._strides, ctypes.c_void_p)
    return p


def _like(q: torch.Tensor) -> torch.Tensor:
    """An output with q's shape, dtype, device and strides."""
    return torch.empty_like(q) if q.is_contiguous() else \
        torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device):
    """The current torch stream of `device` (the tensors' device, which the
    caller has made current with torch.cuda.device)."""
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _need_lse(lse: torch.Tensor, q: torch.Tensor):
    if lse.device != q.device or lse.dtype != torch.float32 or lse.shape != q.shape[:-1] or \
            not lse.is_contiguous():
        raise ValueError(f"lse must be a contiguous fp32 tensor of shape {tuple(q.shape[:-1])} "
                         f"on {q.device}")


def _need_cuda(q: torch.Tensor):
    if q.device.type != "cuda":
        raise ValueError("libna runs on CUDA tensors only (there is no CPU path)")


def _need(t: torch.Tensor, like: torch.Tensor, name: str):
    if t.device != like.device or t.dtype != like.dtype or t.shape != like.shape or \
            t.stride() != like.stride():
        raise ValueError(f"{name} must be a {like.dtype} tensor of shape {tuple(like.shape)} "
                         f"and strides {like.stride()} (q's) on {like.device}")


def na_validate(p: Problem) -> int:
    return lib().na_validate(ctypes.byref(p))


def na_selected_impl(p: Problem) -> int:
    return lib().na_selected_impl(ctypes.byref(p))


def na_bf16_precise(p: Problem) -> int:
    """1: the error-compensated bf16 kernel variant runs for p (R13)."""
    return lib().na_bf16_precise(ctypes.byref(p))


def na_bwd_workspace_size(p: Problem) -> int:
    return lib().na_bwd_workspace_size(ctypes.byref(p))


def last_launch_count() -> int:
    return lib().na_last_launch_count()


def profile_enable(on: bool = True):
    """Bracket every launch of this thread with CUDA events (benchmarking)."""
    lib().na_profile_enable(1 if on else 0)


def profile_collect(max_entries: int = 4096):
    """[(kernel name, device ms), ...] for the launches since the last collect."""
    ids = (ctypes.c_int * max_entries)()
    ms = (ctypes.c_float * max_entries)()
    n = lib().na_profile_collect(ids, ms, max_entries)
    return [(lib().na_kernel_name(ids[i]).decode(), float(ms[i])) for i in range(min(n, max_entries))]


def na_fwd(q, k, v, kernel_size, dilation=None, is_causal=None, scale=None, impl="auto",
           out=None, lse=None, return_lse=True):
    """Fused NA forward.  Returns (O, LSE) (LSE fp32 [B,H,X...]) or O.
    Enqueued on the current stream of q's device."""
    p = _problem_from(q, kernel_size, dilation, is_causal, scale, impl)
    _need_cuda(q)
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _need(t, q, n)
    with torch.cuda.device(q.device):
        o = _like(q) if out is None else out
        _need(o, q, "out")
        if return_lse:
            if lse is None:
                lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
            _need_lse(lse, q)
        _check(lib().na_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                            _ptr(lse) if return_lse else None, _stream(q.device)))
    return (o, lse) if return_lse else o


def na_bwd(q, k, v, o, d_o, lse, kernel_size, dilation=None, is_causal=None, scale=None,
           impl="auto", dq=None, dk=None, dv=None, workspace=None):
    """Fused NA backward.  Returns (dQ, dK, dV).  Enqueued on the current
    stream of q's device."""
    p = _problem_from(q, kernel_size, dilation, is_causal, scale, impl)
    _need_cuda(q)
    for t, n in ((k, "k"), (v, "v"), (o, "o"), (d_o, "d_o")):
        _need(t, q, n)
    _need_lse(lse, q)
    with torch.cuda.device(q.device):
        dq = _like(q) if dq is None else dq
        dk = _like(q) if dk is None else dk
        dv = _like(q) if dv is None else dv
        for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
            _need(t, q, n)
        need = na_bwd_workspace_size(p)
        if workspace is None:
            workspace = torch.empty((max(need, 16) + 3) // 4, dtype=torch.float32, device=q.device)
        if workspace.device != q.device or not workspace.is_contiguous():
            raise ValueError(f"workspace must be a contiguous tensor on {q.device}")
        _check(lib().na_bwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(d_o),
                            _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(workspace),
                            workspace.numel() * workspace.element_size(), _stream(q.device)))
    return dq, dk, dv


def na_plan_candidates(p: Problem) -> int:
    """How many tile plans na_tune would measure for `p` (1: nothing to tune)."""
    return lib().na_plan_candidates(ctypes.byref(p))


def na_get_plan_choice(p: Problem):
    c = (ctypes.c_int32 * 3)()
    _check(lib().na_get_plan_choice(ctypes.byref(p), c))
    return tuple(c)


def na_set_plan_choice(p: Problem, choice):
    _check(lib().na_set_plan_choice(ctypes.byref(p), (ctypes.c_int32 * 3)(*choice)))


def na_tune(q, k, v, d_o, kernel_size, dilation=None, is_causal=None, scale=None):
    """Measure the planner's candidate tile plans for this problem (forward,
    dK/dV and dQ separately) on scratch outputs and keep the fastest for later
    calls with the same geometry.  Returns the picks (fwd, dkdv, dq)."""
    p = _problem_from(q, kernel_size, dilation, is_causal, scale, "auto")
    _need_cuda(q)
    for t, n in ((k, "k"), (v, "v"), (d_o, "d_o")):
        _need(t, q, n)
    o, dq, dk, dv = (_like(q) for _ in range(4))
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
    ws = torch.empty((max(na_bwd_workspace_size(p), 16) + 3) // 4, dtype=torch.float32, device=q.device)
    c = (ctypes.c_int32 * 3)()
    with torch.cuda.device(q.device):
        _check(lib().na_tune(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                             _ptr(d_o), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel() * 4,
                             _stream(q.device), c))
    return tuple(c)
