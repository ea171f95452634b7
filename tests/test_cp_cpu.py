"""Context parallelism (paper_2403_04690_b200/cp.py) on
CPU: world sizes 2 and 4 over gloo, halo rows exchanged point to point, the
per-slab compute done by the fp64 oracle (no GPU here).  The owned rows of
O, LSE, dQ, dK, dV gathered from the ranks equal the single-process oracle
result on the whole problem -- which checks the halo width, the slab
windows (border clamping, residue classes, causal axes) and the exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import na_synth
import oracle

CASES = [
    # extent, kernel, dilation, causal
    ([40], [7], [2], [0]),
    ([37], [5], [1], [1]),
    ([24, 10], [5, 3], [2, 1], [0, 1]),
    ([13, 6, 7], [3, 3, 5], [1, 2, 1], [1, 0, 0]),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_fns(cfg):
    D = cfg.head_dim

    def prob(t):
        B, H, *ext = t.shape[:-1]
        return oracle.make_problem(B, H, ext, D, list(cfg.kernel_size), list(cfg.dilation),
                                   [int(c) for c in cfg.is_causal])

    def fwd(q, k, v, **kw):
        o, lse = oracle.fwd(prob(q), q, k, v)
        return torch.from_numpy(o).view(q.shape), torch.from_numpy(lse).view(q.shape[:-1])

    def bwd(q, k, v, o, do, lse, **kw):
        return tuple(torch.from_numpy(g).view(q.shape) for g in oracle.bwd(prob(q), q, k, v, do))

    return fwd, bwd


def _worker(rank, world, port, out_dir, case_idx):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_04690_b200.cp import ContextParallel
    ext, ker, dil, cau = CASES[case_idx]
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=4, batch=1, heads=2, dtype=torch.float64)
    q, k, v, do = na_synth.make_inputs(cfg)
    fwd, bwd = _oracle_fns(cfg)
    cp = ContextParallel(ext, ker, dil, [bool(c) for c in cau], fwd_fn=fwd, bwd_fn=bwd)
    o, lse, ctx = cp.forward(*(cp.own_rows(t) for t in (q, k, v)))
    dq, dk, dv = cp.backward(ctx, cp.own_rows(do))
    outs = {}
    for name, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
        parts = [None] * world
        dist.all_gather_object(parts, t.contiguous())
        outs[name] = parts
    if rank == 0:
        torch.save(outs, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case_idx", range(len(CASES)))
def test_context_parallel_matches_whole_problem(tmp_path, world, case_idx):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case_idx), nprocs=world, join=True)
    res = torch.load(tmp_path / "res.pt")
    ext, ker, dil, cau = CASES[case_idx]
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=4, batch=1, heads=2, dtype=torch.float64)
    q, k, v, do = na_synth.make_inputs(cfg)
    p = oracle.make_problem(1, 2, ext, 4, ker, dil, cau)
    ro, rlse = oracle.fwd(p, q, k, v)
    rdq, rdk, rdv = oracle.bwd(p, q, k, v, do)
    shp = tuple(q.shape)
    ref = {"o": ro.reshape(shp), "lse": rlse.reshape(shp[:-1]), "dq": rdq.reshape(shp),
           "dk": rdk.reshape(shp), "dv": rdv.reshape(shp)}
    for name, parts in res.items():
        got = torch.cat(parts, dim=2).numpy()
        np.testing.assert_allclose(got, ref[name], rtol=0, atol=1e-12, err_msg=name)


def test_split_halo_and_ranges():
    from paper_2403_04690_b200.cp import make_split
    s = make_split([16384], [255], [1], 8)
    assert [s.own(g) for g in range(8)] == [(g * 2048, (g + 1) * 2048) for g in range(8)]
    assert s.slab(0) == (0, 2048 + 255) and s.slab(7) == (7 * 2048 - 255, 16384)
    s = make_split([16, 64, 64], [7, 7, 7], [1, 1, 1], 4)
    assert s.halo == 7 and s.slab(1) == (0, 15)
