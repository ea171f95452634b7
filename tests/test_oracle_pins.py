"""Pins the CPU oracle (oracle/na_oracle.c) to things other than itself.

Every pin is something PAPER.md (P:line) or mathematics fixes, or a SPEC.md
worked example (tests/golden/spec_examples.json):

* window rule  — brute-force enumeration of all in-bounds k-windows of a
  residue class, choosing the most centred one (Fig. 2 caption, P:110-120:
  "only attempts to center the query"); causal = the k nearest predecessors
  (P:117-118); dilation = residue classes.
* full window, dilation 1, non-causal == dense softmax attention (Eq. 1,
  P:135-140; "matches it when equal to input size").
* causal full window == dense lower-triangular attention.
* kernel size 1 == linear projection, O = V.
* dilation == composition over residue-class sub-problems.
* DiNAT-style 56x56, k=7, dilation 8: every window is its whole 7x7 class
  (closed form: dense attention inside each class).
* gradients == central finite differences of the oracle's own forward, and
  == torch autograd of dense masked attention whose mask comes from the
  brute-force predicate above (not from the oracle).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


# ----------------------------------------------------------- brute force

def brute_axis_keys(L, k, dil, causal, x):
    """Key coordinates on one axis, by enumeration (independent of the oracle)."""
    r = x % dil
    members = list(range(r, L, dil))          # the residue class of x
    xc = members.index(x)
    n = len(members)
    if causal:
        sel = [j for j in range(n) if j <= xc and xc - j < k]
    else:
        best = None
        for s in range(0, n - k + 1):         # every in-bounds window of k members
            if not (s <= xc <= s + k - 1):
                continue
            off = abs((s + (k - 1) / 2) - xc)  # distance of the query from the centre
            if best is None or off < best[0]:
                best = (off, s)
        sel = list(range(best[1], best[1] + k))
    return [members[j] for j in sel]


def brute_mask(extent, kernel, dil, causal):
    """Dense [N, N] boolean neighborhood mask from brute_axis_keys."""
    per_axis = [[set(brute_axis_keys(extent[a], kernel[a], dil[a], causal[a], x))
                 for x in range(extent[a])] for a in range(len(extent))]
    coords = list(itertools.product(*[range(e) for e in extent]))
    N = len(coords)
    m = np.zeros((N, N), dtype=bool)
    for i, cx in enumerate(coords):
        for j, cy in enumerate(coords):
            m[i, j] = all(cy[a] in per_axis[a][cx[a]] for a in range(len(extent)))
    return m


def dense_masked_attention(q, k, v, mask, scale):
    """torch fp64 reference: softmax(scale QK^T masked) V over [BH, N, D]."""
    s = scale * q @ k.transpose(-1, -2)
    s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    return torch.softmax(s, dim=-1) @ v, lse


def rand(shape, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float64)


def problem_inputs(extent, D, B=1, H=2, seed=0, with_do=False):
    shape = (B, H, *extent, D)
    ts = [rand(shape, seed + i) for i in range(4 if with_do else 3)]
    return ts


# ----------------------------------------------------------- window rule

@pytest.mark.parametrize("causal", [0, 1])
def test_axis_window_matches_brute_force(causal):
    n = 0
    for L in range(1, 20):
        for dil in range(1, 6):
            for k in range(1, L // dil + 1):
                if not causal and k % 2 == 0:
                    continue
                for x in range(L):
                    keys = brute_axis_keys(L, k, dil, causal, x)
                    first, last, cnt = oracle.axis_window(L, k, dil, causal, x)
                    assert (first, last, cnt) == (keys[0], keys[-1], len(keys)), (L, k, dil, x)
                    n += 1
    assert n > 2500


def test_spec_window_start_examples():
    for e in GOLDEN["window_start"]:
        first, last, cnt = oracle.axis_window(e["extent"], e["window"], 1, int(e["causal"]), e["i"])
        assert (first, cnt) == (e["start"], e["size"]), e["cite"]


def test_spec_contains_examples():
    for e in GOLDEN["contains"]:
        p = oracle.make_problem(1, 1, e["extent"], 4, e["kernel"], e["dilation"], e["causal"])
        flat = lambda c: int(np.ravel_multi_index(c, e["extent"]))
        assert oracle.contains(p, flat(e["q"]), flat(e["c"])) == e["result"], e["cite"]


def test_spec_inverse_neighborhood_examples():
    for e in GOLDEN["inverse_neighborhood"]:
        p = oracle.make_problem(1, 1, [e["extent"]], 4, [e["window"]])
        qs = [x for x in range(e["extent"]) if oracle.contains(p, x, e["c"])]
        assert qs == e["queries"], e["cite"]


def test_spec_halo_examples():
    for e in GOLDEN["halo_range"]:
        ws = [oracle.axis_window(e["extent"], e["window"], 1, int(e["causal"]), x)
              for x in range(e["q_lo"], e["q_hi"] + 1)]
        assert (min(w[0] for w in ws), max(w[1] for w in ws)) == (e["lo"], e["hi"]), e["cite"]


def test_spec_partition_examples():
    for e in GOLDEN["partition_dilated"]:
        classes = sorted({tuple(brute_axis_keys(e["extent"], len(range(r, e["extent"], e["dilation"])),
                                                e["dilation"], 1, x))
                          for r in range(e["dilation"])
                          for x in [list(range(r, e["extent"], e["dilation"]))[-1]]})
        assert [list(c) for c in classes] == e["classes"], e["cite"]
        # the oracle's full-class window reproduces the same classes
        for cls in e["classes"]:
            f, l, n = oracle.axis_window(e["extent"], len(cls), e["dilation"], 0, cls[0])
            assert list(range(f, l + 1, e["dilation"])) == cls


def test_spec_validate_examples():
    codes = {"even_window": 4, "window_exceeds": 6}
    for e in GOLDEN["validate"]:
        p = oracle.make_problem(1, 1, e["extent"], 4, e["kernel"], e["dilation"], e["causal"])
        rc = oracle.check(p)
        assert (rc == 0) == e["ok"], e["cite"]
        if not e["ok"]:
            assert rc == codes[e["error"]], e["cite"]


def test_contains_matches_brute_mask_multi_axis():
    for extent, kernel, dil, causal in [([6, 7], [3, 5], [2, 1], [0, 1]),
                                        ([4, 5, 6], [3, 2, 3], [1, 2, 1], [0, 1, 0]),
                                        ([9], [3], [3], [1])]:
        p = oracle.make_problem(1, 1, extent, 4, kernel, dil, causal)
        m = brute_mask(extent, kernel, dil, causal)
        N = m.shape[0]
        got = np.array([[oracle.contains(p, x, y) for y in range(N)] for x in range(N)])
        assert (got == m).all()
        assert m.diagonal().all()                      # self always in N(x)


def test_na_differs_from_sliding_window_at_edges():
    """NA shifts the window inward; SWA masks out-of-bounds keys."""
    first, last, n = oracle.axis_window(7, 3, 1, 0, 0)
    assert (first, last, n) == (0, 2, 3)               # SWA would give {0, 1}
    first, last, n = oracle.axis_window(7, 3, 1, 0, 6)
    assert (first, last, n) == (4, 6, 3)               # SWA would give {5, 6}


# ----------------------------------------------------------- forward pins

@pytest.mark.parametrize("extent", [[9], [5, 7], [3, 3, 5]])
def test_full_window_is_self_attention(extent):
    """k = input size, dilation 1 -> Eq. 1 exactly."""
    D = 8
    q, k, v = problem_inputs(extent, D, seed=10)
    p = oracle.make_problem(1, 2, extent, D, extent)
    o, lse = oracle.fwd(p, q, k, v)
    N = int(np.prod(extent))
    qf, kf, vf = (t.reshape(2, N, D) for t in (q, k, v))
    ref = torch.softmax(qf @ kf.transpose(-1, -2) / math.sqrt(D), dim=-1) @ vf
    ref_lse = torch.logsumexp(qf @ kf.transpose(-1, -2) / math.sqrt(D), dim=-1)
    np.testing.assert_allclose(o.reshape(2, N, D), ref.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse.reshape(2, N), ref_lse.numpy(), rtol=0, atol=1e-12)


def test_causal_full_window_is_causal_attention():
    """causal full window = dense causal attention (library SDPA)."""
    L, D = 11, 8
    q, k, v = problem_inputs([L], D, seed=20)
    p = oracle.make_problem(1, 2, [L], D, [L], [1], [1])
    o, _ = oracle.fwd(p, q, k, v)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.reshape(1, 2, L, D), k.reshape(1, 2, L, D), v.reshape(1, 2, L, D), is_causal=True)
    np.testing.assert_allclose(o, ref.numpy(), rtol=0, atol=1e-12)


def test_kernel_one_is_linear_projection():
    """window size 1 == linear projection: O = V bitwise, LSE = s_xx."""
    extent, D = [4, 5], 6
    q, k, v = problem_inputs(extent, D, seed=30)
    p = oracle.make_problem(1, 2, extent, D, [1, 1], [2, 1], [0, 1], scale=0.3)
    o, lse = oracle.fwd(p, q, k, v)
    assert np.array_equal(o, v.reshape(1, 2, 20, D).numpy())
    np.testing.assert_allclose(lse, 0.3 * (q * k).sum(-1).reshape(1, 2, 20).numpy(), atol=1e-13)


@pytest.mark.parametrize("case", [
    ([16], [3], [4], [0]),
    ([15], [3], [4], [1]),               # ragged classes: 4,4,4,3
    ([8, 9], [3, 3], [2, 3], [0, 0]),
    ([6, 7, 5], [3, 3, 1], [2, 2, 1], [1, 0, 0]),
])
def test_dilation_is_residue_class_composition(case):
    """dilated NA == non-dilated NA on every residue class, bitwise."""
    extent, kernel, dil, causal = case
    D = 4
    q, k, v = problem_inputs(extent, D, seed=40)
    p = oracle.make_problem(1, 2, extent, D, kernel, dil, causal)
    o, lse = oracle.fwd(p, q, k, v)
    o = o.reshape(1, 2, *extent, D)
    lse = lse.reshape(1, 2, *extent)
    for res in itertools.product(*[range(d) for d in dil]):
        sl = tuple(slice(r, None, d) for r, d in zip(res, dil))
        sub = [t[(slice(None), slice(None)) + sl].contiguous() for t in (q, k, v)]
        sub_ext = list(sub[0].shape[2:-1])
        ps = oracle.make_problem(1, 2, sub_ext, D, kernel, None, causal)
        os_, ls_ = oracle.fwd(ps, *sub)
        assert np.array_equal(o[(slice(None), slice(None)) + sl], os_.reshape(1, 2, *sub_ext, D))
        assert np.array_equal(lse[(slice(None), slice(None)) + sl], ls_.reshape(1, 2, *sub_ext))


def test_dinat_class_is_whole_window():
    """Config C with dilation 8: 56 = 8 x 7, k = 7 -> each window is its whole
    7x7 residue class, so the result is dense attention inside each class."""
    D = 8
    q, k, v = problem_inputs([56, 56], D, B=1, H=1, seed=50)
    p = oracle.make_problem(1, 1, [56, 56], D, [7, 7], [8, 8])
    o, lse = oracle.fwd(p, q, k, v)
    o = o.reshape(56, 56, D)
    for ry, rx in [(0, 0), (3, 5), (7, 7)]:
        cls = lambda t: t[0, 0, ry::8, rx::8].reshape(49, D)
        ref = torch.softmax(cls(q) @ cls(k).T / math.sqrt(D), -1) @ cls(v)
        np.testing.assert_allclose(o[ry::8, rx::8].reshape(49, D), ref.numpy(), atol=1e-12)


CASES = [
    ([7], [3], [1], [0]),
    ([9], [3], [2], [1]),
    ([10], [4], [1], [1]),
    ([5, 6], [3, 3], [1, 2], [0, 1]),
    ([3, 4, 5], [3, 3, 3], [1, 1, 1], [1, 0, 0]),
    ([4, 4, 6], [1, 3, 3], [1, 1, 2], [0, 0, 0]),
]


@pytest.mark.parametrize("case", CASES)
def test_forward_and_backward_match_dense_autograd(case):
    """Oracle == torch autograd through dense masked attention, mask from the
    brute-force predicate (no oracle code involved in the reference)."""
    extent, kernel, dil, causal = case
    D, B, H = 5, 1, 2
    q, k, v, do = problem_inputs(extent, D, B, H, seed=60, with_do=True)
    p = oracle.make_problem(B, H, extent, D, kernel, dil, causal, scale=0.37)
    o, lse = oracle.fwd(p, q, k, v)
    dq, dk, dv = oracle.bwd(p, q, k, v, do)
    N = int(np.prod(extent))
    mask = torch.from_numpy(brute_mask(extent, kernel, dil, causal))
    qf, kf, vf = (t.reshape(B * H, N, D).clone().requires_grad_(True) for t in (q, k, v))
    ref, ref_lse = dense_masked_attention(qf, kf, vf, mask, 0.37)
    ref.backward(do.reshape(B * H, N, D))
    tol = dict(rtol=0, atol=1e-12)
    np.testing.assert_allclose(o.reshape(B * H, N, D), ref.detach().numpy(), **tol)
    np.testing.assert_allclose(lse.reshape(B * H, N), ref_lse.detach().numpy(), **tol)
    np.testing.assert_allclose(dq.reshape(B * H, N, D), qf.grad.numpy(), **tol)
    np.testing.assert_allclose(dk.reshape(B * H, N, D), kf.grad.numpy(), **tol)
    np.testing.assert_allclose(dv.reshape(B * H, N, D), vf.grad.numpy(), **tol)


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("case", CASES[:4])
def test_stored_output_backward_matches_dense_formula(case, dt):
    """Reading R12: with stored_o the softmax-Jacobian term uses O as the method
    stores it (fp64 -> fp32 -> the inputs' 16-bit dtype, round to nearest
    even).  Reference: torch fp64 dense masked attention, torch's own dtype
    conversion of O, and the textbook gradient formulas (no oracle code)."""
    extent, kernel, dil, causal = case
    D, B, H = 6, 1, 2
    q, k, v, do = (t.to(dt) for t in problem_inputs(extent, D, B, H, seed=80, with_do=True))
    p = oracle.make_problem(B, H, extent, D, kernel, dil, causal, scale=0.41)
    dq, dk, dv = oracle.bwd(p, q, k, v, do, stored_o=True)
    N = int(np.prod(extent))
    mask = torch.from_numpy(brute_mask(extent, kernel, dil, causal))
    qf, kf, vf, dof = (t.double().reshape(B * H, N, D) for t in (q, k, v, do))
    s = (0.41 * qf @ kf.transpose(-1, -2)).masked_fill(~mask, float("-inf"))
    P = torch.softmax(s, dim=-1)
    o_stored = (P @ vf).float().to(dt).double()
    Dx = (dof * o_stored).sum(-1, keepdim=True)
    dS = P * (dof @ vf.transpose(-1, -2) - Dx)
    tol = dict(rtol=0, atol=1e-12)
    np.testing.assert_allclose(dq.reshape(B * H, N, D), (0.41 * dS @ kf).numpy(), **tol)
    np.testing.assert_allclose(dk.reshape(B * H, N, D), (0.41 * dS.transpose(-1, -2) @ qf).numpy(), **tol)
    np.testing.assert_allclose(dv.reshape(B * H, N, D), (P.transpose(-1, -2) @ dof).numpy(), **tol)
    # and the stored O differs from the exact one: the term is not a no-op
    ex = oracle.bwd(p, q, k, v, do)[0]
    assert np.abs(ex - dq).max() > 0


@pytest.mark.parametrize("case", CASES[:4])
def test_backward_matches_finite_differences(case):
    """Central differences (h = 1e-5) of L = <dO, O> through the oracle's own
    forward; relative error <= 1e-6."""
    extent, kernel, dil, causal = case
    D = 3
    q, k, v, do = problem_inputs(extent, D, 1, 1, seed=70, with_do=True)
    p = oracle.make_problem(1, 1, extent, D, kernel, dil, causal)
    grads = oracle.bwd(p, q, k, v, do)
    h = 1e-5
    loss = lambda qq, kk, vv: float((oracle.fwd(p, qq, kk, vv)[0].reshape(do.shape) * do.numpy()).sum())
    rng = np.random.default_rng(0)
    for which, g in enumerate(grads):
        flat_g = g.reshape(-1)
        for idx in rng.choice(flat_g.size, size=min(12, flat_g.size), replace=False):
            args = [q.clone(), k.clone(), v.clone()]
            args[which].view(-1)[idx] += h
            lp = loss(*args)
            args[which].view(-1)[idx] -= 2 * h
            lm = loss(*args)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - flat_g[idx]) <= 1e-6 * max(1.0, abs(fd)), (which, idx, fd, flat_g[idx])


def test_zero_output_grad_gives_zero_grads():
    q, k, v = problem_inputs([6, 5], 4, seed=80)
    p = oracle.make_problem(1, 2, [6, 5], 4, [3, 3])
    for g in oracle.bwd(p, q, k, v, torch.zeros_like(q)):
        assert not g.any()


def test_kernel_one_gradients():
    """k = 1: dV = dO, dQ = dK = 0."""
    q, k, v, do = problem_inputs([7], 4, seed=90, with_do=True)
    p = oracle.make_problem(1, 2, [7], 4, [1])
    dq, dk, dv = oracle.bwd(p, q, k, v, do)
    assert np.array_equal(dv, do.reshape(1, 2, 7, 4).numpy())
    assert not dq.any() and not dk.any()


@pytest.mark.parametrize("case", CASES)
def test_token_forms_equal_full_forms(case):
    """Gather (per-token) and scatter (full) forms of the oracle agree."""
    extent, kernel, dil, causal = case
    D, B, H = 4, 2, 1
    q, k, v, do = problem_inputs(extent, D, B, H, seed=100, with_do=True)
    p = oracle.make_problem(B, H, extent, D, kernel, dil, causal)
    o, lse = oracle.fwd(p, q, k, v)
    dq, dk, dv = oracle.bwd(p, q, k, v, do)
    N = int(np.prod(extent))
    toks = np.arange(B * H * N)
    ot, lt = oracle.fwd_tokens(p, q, k, v, toks)
    dqt, dkt, dvt = oracle.bwd_tokens(p, q, k, v, do, toks)
    for full, tok in [(o, ot), (dq, dqt), (dk, dkt), (dv, dvt)]:
        np.testing.assert_allclose(full.reshape(-1, D), tok, rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse.reshape(-1), lt, rtol=0, atol=1e-13)


@pytest.mark.parametrize("stored", [False, True])
@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("case", CASES)
def test_gather_and_token_forms_equal_scatter_form_16bit(case, dt, stored):
    """The per-token (bwd_tokens) and whole-problem gather (bwd_gather) forms
    of the backward equal the scatter form (bwd) on 16-bit inputs, with the
    exact D_x and with the stored-O D_x of reading R12 -- the scatter form
    with stored_o is itself pinned to torch's dense formula above
    (test_stored_output_backward_matches_dense_formula), so every form the
    GPU parity tests use is pinned."""
    extent, kernel, dil, causal = case
    D, B, H = 8, 1, 2
    q, k, v, do = (t.to(dt) for t in problem_inputs(extent, D, B, H, seed=101, with_do=True))
    p = oracle.make_problem(B, H, extent, D, kernel, dil, causal)
    full = oracle.bwd(p, q, k, v, do, stored_o=stored)
    N = int(np.prod(extent))
    toks = np.arange(B * H * N)
    tok = oracle.bwd_tokens(p, q, k, v, do, toks, stored_o=stored)
    gat = oracle.bwd_gather(p, q, k, v, do, stored_o=stored)
    for f, t, g in zip(full, tok, gat):
        np.testing.assert_allclose(f.reshape(-1, D), t, rtol=0, atol=1e-12)
        np.testing.assert_allclose(f, g, rtol=0, atol=1e-12)
    o, lse = oracle.fwd(p, q, k, v)
    of, lf = oracle.fwd_full_tokens(p, q, k, v)
    np.testing.assert_allclose(o, of, rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse, lf, rtol=0, atol=1e-13)
    if stored:  # the stored-O term is not a no-op on these inputs
        exact = oracle.bwd(p, q, k, v, do, stored_o=False)
        assert np.abs(exact[0] - full[0]).max() > 0


def test_half_inputs_are_upcast_exactly():
    """fp16 / bf16 inputs give the same result as their exact fp64 upcast."""
    q, k, v = problem_inputs([9], 8, seed=110)
    p = oracle.make_problem(1, 2, [9], 8, [3])
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        qh, kh, vh = (t.to(dt) for t in (q, k, v))
        a = oracle.fwd(p, qh, kh, vh)
        b = oracle.fwd(p, qh.double(), kh.double(), vh.double())
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
