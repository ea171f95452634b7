"""Multi-process (gloo, world sizes 2 and 4, CPU) coverage of the N>1 path.

The hot path shards batch x heads with no data-path collective (DESIGN.md
§8): of a config's BH = B*H slices, rank g of G owns the
flattened range [g*BH/G, (g+1)*BH/G) (bench.shard_range) and seeds each
slice by its global index, so the union of the ranks' work is bitwise the
single-process computation of the SAME problem at every G (strong split).
Timings are combined with a max over ranks, per-rank parity rows with an
all_gather (bench.gather_rows).  The per-rank "kernel" here is the CPU
oracle (no GPU in CI)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import na_synth
import oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CFG = na_synth.small_config([40], [7], [2], [1], head_dim=8, batch=2, heads=4)
BH = CFG.batch * CFG.heads


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    bh0, bh1 = bench.shard_range(rank, world, BH)
    n = bh1 - bh0
    q, k, v = na_synth.make_inputs(CFG, bh_range=(bh0, bh1), with_do=False)
    p = oracle.make_problem(1, n, list(CFG.extent), CFG.head_dim, list(CFG.kernel_size),
                            list(CFG.dilation), list(CFG.is_causal))
    o, lse = oracle.fwd(p, q, k, v)
    o_t = torch.from_numpy(o.reshape(n, -1))
    parts = [torch.empty_like(o_t) for _ in range(world)]
    dist.all_gather(parts, o_t)
    slowest = bench.reduce_max(float(rank + 1), world, device="cpu")
    rows = bench.gather_rows([float(rank), float(bh0), float(bh1)], world, device="cpu")
    if rank == 0:
        torch.save({"parts": parts, "slowest": slowest, "rows": rows}, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bxh_strong_split_is_bitwise_the_single_process_result(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = torch.load(tmp_path / "res.pt")
    assert res["slowest"] == float(world)
    # the ranks' ranges tile [0, BH) in order, each of BH / world slices
    assert [r[0] for r in res["rows"]] == [float(g) for g in range(world)]
    assert [(r[1], r[2]) for r in res["rows"]] == [(g * BH / world, (g + 1) * BH / world) for g in range(world)]
    # single process over all BH global slices: the same problem at every G
    q, k, v = na_synth.make_inputs(CFG, bh_range=(0, BH), with_do=False)
    p = oracle.make_problem(1, BH, list(CFG.extent), CFG.head_dim, list(CFG.kernel_size),
                            list(CFG.dilation), list(CFG.is_causal))
    o, _ = oracle.fwd(p, q, k, v)
    full = torch.from_numpy(o.reshape(BH, -1))
    assert torch.equal(torch.cat(res["parts"]), full)


def test_shard_range_covers_every_config_at_every_world():
    import bench
    for name, cfg in na_synth.CONFIGS.items():
        bh = cfg.batch * cfg.heads
        for world in (1, 2, 4, 8):
            rs = [bench.shard_range(g, world, bh) for g in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == bh
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            if name != "A":  # A has one slice; every other config splits evenly
                assert all(r[1] - r[0] == bh // world for r in rs)


def test_slice_seeding_independent_of_range():
    """A slice's values depend only on its global index, not on the range asked."""
    a = na_synth.slice_tensor(CFG, "q", 1, 3)
    b = na_synth.slice_tensor(CFG, "q", 0, 4)
    assert torch.equal(a, b[1:3])
