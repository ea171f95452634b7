"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 path.

The hot path shards batch x heads with no data-path collective (DESIGN.md
§8): rank r owns global (b,h) slices [r*BH, (r+1)*BH) and seeds each slice by
its global index, so the union of the ranks' work is bitwise the
single-process computation.  Timings are combined with a max over ranks.
The per-rank "kernel" here is the CPU oracle (no GPU in CI)."""
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


CFG = na_synth.small_config([40], [7], [2], [1], head_dim=8, batch=2, heads=2)
BH_PER_RANK = 2


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rng = bench.shard_range(rank, BH_PER_RANK)
    q, k, v = na_synth.make_inputs(CFG, bh_range=rng, with_do=False)
    p = oracle.make_problem(1, BH_PER_RANK, list(CFG.extent), CFG.head_dim, list(CFG.kernel_size),
                            list(CFG.dilation), list(CFG.is_causal))
    o, lse = oracle.fwd(p, q, k, v)
    o_t = torch.from_numpy(o.reshape(BH_PER_RANK, -1))
    parts = [torch.empty_like(o_t) for _ in range(world)]
    dist.all_gather(parts, o_t)
    slowest = bench.reduce_max(float(rank + 1), world, device="cpu")
    if rank == 0:
        torch.save({"parts": parts, "slowest": slowest}, os.path.join(out_dir, "res.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_bxh_sharding_is_bitwise_the_single_process_result(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = torch.load(tmp_path / "res.pt")
    assert res["slowest"] == float(world)
    # single process over all world * BH_PER_RANK global slices
    n = world * BH_PER_RANK
    q, k, v = na_synth.make_inputs(CFG, bh_range=(0, n), with_do=False)
    p = oracle.make_problem(1, n, list(CFG.extent), CFG.head_dim, list(CFG.kernel_size),
                            list(CFG.dilation), list(CFG.is_causal))
    o, _ = oracle.fwd(p, q, k, v)
    full = torch.from_numpy(o.reshape(n, -1))
    assert torch.equal(torch.cat(res["parts"]), full)


def test_slice_seeding_independent_of_range():
    """A slice's values depend only on its global index, not on the range asked."""
    a = na_synth.slice_tensor(CFG, "q", 1, 3)
    b = na_synth.slice_tensor(CFG, "q", 0, 4)
    assert torch.equal(a, b[1:3])
