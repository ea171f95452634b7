"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every entry point include/na.h declares, and validates problems exactly as
documented (SPEC S:62-70 constraint list, readings R2/R6)."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from paper_2403_04690_b200 import build as na_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def na():
    na_build.build()
    import paper_2403_04690_b200 as pkg
    pkg.lib()
    return pkg


def header_functions():
    text = open(os.path.join(ROOT, "include", "na.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(na_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(na):
    names = header_functions()
    assert {"na_fwd", "na_bwd", "na_validate", "na_bwd_workspace_size"} <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", na.na.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (na_[a-z_]+)\b", out))
    assert set(names) <= exported, set(names) - exported
    L = na.lib()
    for n in names:
        assert hasattr(L, n)


def test_library_is_sm100a(na):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", na.na.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def P(na, **kw):
    base = dict(batch=1, heads=1, extent=[16], head_dim=64, kernel_size=[3])
    base.update(kw)
    return na.make_problem(**base)


@pytest.mark.parametrize("kw,status", [
    (dict(), 0),
    (dict(extent=[5], kernel_size=[3]), 0),
    (dict(extent=[5], kernel_size=[4]), 5),                     # S:69 even window
    (dict(extent=[8], kernel_size=[5], dilation=[2]), 7),       # S:70 exceeds class
    (dict(extent=[8], kernel_size=[4], is_causal=[True]), 0),   # even k ok when causal
    (dict(extent=[8], kernel_size=[3], dilation=[0]), 6),
    (dict(extent=[8], kernel_size=[0]), 4),
    (dict(head_dim=12), 9),
    (dict(head_dim=264), 9),
    (dict(head_dim=12, dtype=torch.float32), 0),
    (dict(extent=[4, 4, 4, 4], kernel_size=[3, 3, 3, 3]), 2),
    (dict(batch=0), 3),
    (dict(extent=[0], kernel_size=[1]), 3),
    (dict(extent=[9, 9], kernel_size=[3, 9], dilation=[1, 2]), 7),
])
def test_validation_codes(na, kw, status):
    if len(kw.get("extent", [1])) > 3:
        p = P(na)
        p.rank = 4
    else:
        p = P(na, **kw)
    assert na.na_validate(p) == status
    if status:
        assert na.lib().na_last_error().decode()


def test_layout_and_impl_codes(na):
    def strided(st, **kw):
        p = P(na, **kw)
        p._arr = (ctypes.c_int64 * 6)(*st)
        p.strides = ctypes.cast(p._arr, ctypes.c_void_p)
        return na.na_validate(p)
    assert strided(range(6)) == 11                                  # head_dim stride != 1
    assert strided([16 * 64 * 2, 64, 2 * 64, 0, 0, 1], heads=2) == 0  # heads-last [B, X, H, D]
    assert strided([0, 64, 64, 0, 0, 1]) == 11                       # a stride < 1
    assert strided([1024, 68, 136, 0, 0, 1], heads=2) == 10         # 136 B rows: not 16-B multiples
    assert strided([4096, 64, 256, 5, 0, 1], extent=[16]) == 0       # X1/X2 ignored beyond rank
    # the binding passes a non-contiguous tensor's strides
    x = torch.empty(2, 16, 4, 64, dtype=torch.float16).permute(0, 2, 1, 3)
    p = na.na._problem_from(x, [3], None, None, None, "auto")
    assert list(p._strides) == [16 * 4 * 64, 64, 4 * 64, 0, 0, 1]
    assert na.na_validate(p) == 0
    p = P(na)
    p.impl = 7
    assert na.na_validate(p) == 14


def test_workspace_size(na):
    # max(SIMT D vector BH*N*4, tensor-core row-vector layout BH*nres*2*plane*4)
    # where plane = prod over axes of ceil(L/dil), innermost padded to 4 (na.h).
    p = P(na, batch=2, heads=3, extent=[7, 5], kernel_size=[3, 3])
    assert na.na_bwd_workspace_size(p) == 2 * 3 * 1 * 2 * (7 * 8) * 4
    p = P(na, batch=1, heads=2, extent=[9], kernel_size=[3], dilation=[2])
    assert na.na_bwd_workspace_size(p) == 2 * 2 * 2 * 8 * 4       # classes of 5 and 4 -> 8
    p = P(na, batch=1, heads=1, extent=[64], kernel_size=[3])
    assert na.na_bwd_workspace_size(p) == 2 * 64 * 4
    assert na.na_bwd_workspace_size(P(na, kernel_size=[4])) == 0


def test_fp32_selects_simt(na):
    assert na.na_selected_impl(P(na, dtype=torch.float32)) == na.NA_IMPL_SIMT
    assert na.na_selected_impl(P(na, dtype=torch.float32, impl="tc")) == -1
    assert na.na_selected_impl(P(na, kernel_size=[4])) == -1


def test_bf16_variant_rule(na):
    """DESIGN.md R13: the error-compensated bf16 variant runs iff some window
    holds < 128 keys (product of k over the non-causal axes)."""
    bf = torch.bfloat16
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[300], kernel_size=[127])) == 1
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[300], kernel_size=[129])) == 0
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[300], kernel_size=[255], is_causal=[1])) == 1
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[128, 128], kernel_size=[13, 13],
                                dilation=[2, 2])) == 0                      # config D
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[40, 40], kernel_size=[11, 11])) == 1
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[16, 40, 40], kernel_size=[7, 7, 7],
                                is_causal=[1, 0, 0])) == 1                  # 49 keys at t = 0
    assert na.na_bf16_precise(P(na, dtype=bf, extent=[16, 40, 40], kernel_size=[3, 7, 7])) == 0
    assert na.na_bf16_precise(P(na, extent=[300], kernel_size=[7])) == 0     # fp16
    assert na.na_bf16_precise(P(na, dtype=bf, kernel_size=[4])) == -1       # invalid


def test_no_silent_fallback_for_16bit(na):
    """A 16-bit problem the tensor-core path cannot run is refused under AUTO
    (NA_ERR_IMPL before any launch) and runs on the CUDA cores only when asked."""
    L = na.lib()
    p = P(na, extent=[200], kernel_size=[3], dilation=[9])  # dilation > 8: outside TMA strides
    assert na.na_selected_impl(p) == -1
    assert L.na_fwd(ctypes.byref(p), 16, 16, 16, 16, None, None) == 14  # NA_ERR_IMPL
    assert b"NA_IMPL_SIMT" in L.na_last_error()
    p = P(na, extent=[200], kernel_size=[3], dilation=[9], impl="simt")
    assert na.na_selected_impl(p) == na.NA_IMPL_SIMT
    assert na.na_selected_impl(P(na)) == na.NA_IMPL_TC


def test_fwd_rejects_before_launch(na):
    """Validation errors are returned synchronously with no launch (no GPU here)."""
    L = na.lib()
    p = P(na, kernel_size=[4])
    assert L.na_fwd(ctypes.byref(p), None, None, None, None, None, None) == 5
    p = P(na)
    assert L.na_fwd(ctypes.byref(p), None, None, None, None, None, None) == 1
    fake = ctypes.c_void_p(0x1008)
    assert L.na_fwd(ctypes.byref(p), fake, fake, fake, fake, None, None) == 10
    ok = ctypes.c_void_p(0x1000)
    assert L.na_bwd(ctypes.byref(p), ok, ok, ok, ok, ok, ok, ok, ok, ok, None, 0, None) == 12


def test_status_strings(na):
    for s in range(15):
        assert na.status_string(s)


def test_plan_choice_host_api(na):
    """Tile-plan tuning API (host side, no GPU): candidate counts, pick
    round-trip, range checks."""
    p1 = na.make_problem(1, 2, [300], 64, [7], dtype=torch.float16)
    assert na.na_plan_candidates(p1) == 1            # rank 1: one plan
    p32 = na.make_problem(1, 2, [16, 16], 16, [3, 3], dtype=torch.float32)
    assert na.na_plan_candidates(p32) == 1           # SIMT path: nothing to tune
    p3 = na.make_problem(1, 2, [16, 64, 64], 64, [7, 7, 7], is_causal=[True, False, False],
                         dtype=torch.float16)
    n = na.na_plan_candidates(p3)
    assert 1 < n <= 4
    assert na.na_get_plan_choice(p3) == (0, 0, 0)    # the model's plan by default
    na.na_set_plan_choice(p3, (n - 1, 0, 1))
    assert na.na_get_plan_choice(p3) == (n - 1, 0, 1)
    with pytest.raises(na.NAError):
        na.na_set_plan_choice(p3, (n, 0, 0))
    na.na_set_plan_choice(p3, (0, 0, 0))
    bad = na.make_problem(1, 2, [8], 64, [9], dtype=torch.float16)  # window exceeds extent
    assert na.na_plan_candidates(bad) == -1
