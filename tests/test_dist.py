"""N > 1 control flow on CPU: world-size-2 gloo process group (SURVEY §4
"CI without GPUs").  Each rank plans its row block (host-only planner), the
plan is checked byte for byte against the oracle partitioner of that shard,
the shard's C is computed by the fp64 oracle as a stand-in for the GPU kernel,
the blocks are all-gathered with the product's all_gather_rows, and the
stitched C must equal the unsharded oracle result exactly.  Max/sum-over-ranks
reductions (bench timing) are checked too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2506_15174_b200 import escs, shard, synth
        A = synth.magnitude_pruned(m, 300, 0.9, 77)
        B = synth.dense_b(300, 32, 78)
        S, pl = shard.plan_shard(A, 32, world, rank, ufi=4, T=16, host_only=1)
        r0, r1 = shard.shard_rows(m, world, rank)
        assert S.m == r1 - r0
        got = pl.export()
        ref = oracle.partition(S.m, S.k, S.rowptr, S.colidx, 4, 16, bCols=32)
        assert got["header"] == ref["header"]
        for name in oracle.PLAN_ARRAYS:
            assert np.array_equal(got[name], ref[name]), name
        C_local = torch.from_numpy(oracle.spmm(S.m, S.k, S.rowptr, S.colidx, S.vals, B))
        C = shard.all_gather_rows(C_local, m, world)
        full = oracle.spmm(A.m, A.k, A.rowptr, A.colidx, A.vals, B)
        assert np.array_equal(C.numpy(), full)
        mx = shard.max_over_ranks([float(rank + 1), -float(rank)])
        sm = shard.sum_over_ranks([float(S.nnz)])
        assert mx == [float(world), 0.0]
        assert sm == [float(A.nnz)]
        results[rank] = True
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [64, 101])     # even and uneven row blocks
def test_rowblock_sharding_gloo_world2(m):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert dict(results) == {0: True, 1: True}


def test_shard_bounds_cover_rows():
    from paper_2506_15174_b200 import shard
    for m in (1, 7, 131072):
        for world in (1, 2, 4, 8):
            blocks = [shard.shard_rows(m, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_partition_problems_lpt():
    from paper_2506_15174_b200 import shard, synth
    costs = [p.flops for p in synth.transformer_suite()]
    for world in (1, 2, 4, 8):
        parts = shard.partition_problems(costs, world)
        flat = sorted(i for part in parts for i in part)
        assert flat == list(range(len(costs)))          # every problem exactly once
        loads = [sum(costs[i] for i in part) for part in parts]
        # LPT bound: max load <= mean + largest single cost
        assert max(loads) <= sum(costs) / world + max(costs)
        assert parts == shard.partition_problems(costs, world)   # deterministic
