"""Row-block sharding of A across ranks (north_star: "row-block
sharding of A across the 8 GPUs of one box, with B replicated and no
collective on the hot path except an optional NCCL all-gather of C").

Rank r of G owns rows [r*m/G, (r+1)*m/G) of A and C; it plans its own shard
(panels are shard-relative), B is replicated, and C blocks are independent.
The optional all-gather of C uses torch.distributed (NCCL on GPUs, gloo in the
CPU tests).  This module is plumbing only: no arithmetic of the method.
"""
from __future__ import annotations

from . import synth


def shard_rows(m: int, world: int, rank: int):
    """Rows [r0, r1) owned by `rank`."""
    return synth.shard_bounds(m, world, rank)


def shard_matrix(A: "synth.CSR", world: int, rank: int) -> "synth.CSR":
    r0, r1 = shard_rows(A.m, world, rank)
    return synth.row_block(A, r0, r1) if world > 1 else A


def plan_shard(A: "synth.CSR", bcols: int, world: int, rank: int, **params):
    """escs plan of this rank's row block (host-only when params say so)."""
    from . import escs
    S = shard_matrix(A, world, rank)
    params = {k: v for k, v in params.items() if v}
    if params:
        return S, escs.escs_plan_ex(S.m, S.k, S.nnz, S.rowptr, S.colidx, bcols, **params)
    return S, escs.escs_plan(S.m, S.k, S.nnz, S.rowptr, S.colidx, bcols)


def partition_problems(costs, world: int):
    """Independent problems (a layer suite) over ranks: longest-processing-
    time-first greedy on the given costs (e.g. flops), deterministic (ties by
    index, then lowest rank).  Returns one list of problem indices per rank,
    each in ascending order."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(x) for x in out]


def all_gather_rows(C_local, m: int, world: int, group=None):
    """Optional all-gather of the C row blocks into the full m x n C on every
    rank.  Row blocks may differ by one row; they are padded to the largest
    block for all_gather_into_tensor and trimmed afterwards."""
    import torch
    import torch.distributed as dist
    n = C_local.shape[1]
    blocks = [shard_rows(m, world, r) for r in range(world)]
    rows_max = max(r1 - r0 for r0, r1 in blocks)
    buf = torch.zeros((rows_max, n), dtype=C_local.dtype, device=C_local.device)
    buf[:C_local.shape[0]] = C_local
    out = torch.empty((world * rows_max, n), dtype=C_local.dtype, device=C_local.device)
    try:
        dist.all_gather_into_tensor(out, buf, group=group)
    except (RuntimeError, NotImplementedError):   # backends without the fused form (gloo + CUDA)
        dist.all_gather(list(out.split(rows_max)), buf, group=group)
    parts = [out[r * rows_max:r * rows_max + (r1 - r0)] for r, (r0, r1) in enumerate(blocks)]
    return torch.cat(parts, 0)


def max_over_ranks(values, device=None):
    """Element-wise MAX over ranks (device-side times: the straggler decides)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


class FusedGather:
    """Full m x n C in symmetric memory on every rank, for the SpMM fused
    with its all-gather (SURVEY §8(e) "optional NCCL all-gather of C", NEXT
    row f1): rank r's escs kernel stores each finished C row straight into
    every rank's C over NVLink (peer pointers, or one NVLS multicast store
    when the switch supports it), so there is no separate collective and the
    transfer overlaps the SpMM tile by tile.

    run() = symmetric-memory barrier (peers are done reading the previous C)
    -> escs_spmm_scatter -> barrier (all rows landed).  Plumbing only."""

    def __init__(self, m: int, n: int, group=None, multicast: bool = True):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.m, self.n = m, n
        dev = torch.device("cuda", torch.cuda.current_device())
        self.C = symm.empty((m, n), dtype=torch.float32, device=dev)
        self.handle = symm.rendezvous(self.C, self.group)
        off = self.C.storage_offset()
        self.peers = [self.handle.get_buffer(r, (m, n), torch.float32, off)
                      for r in range(self.world)]
        self.mc_ptr = None
        if multicast and self.world > 1 and self.handle.has_multicast_support():
            self.mc_ptr = self.handle.multicast_ptr + 4 * off
        self.r0, self.r1 = shard_rows(m, self.world, self.rank)

    @property
    def mode(self) -> str:
        return "multicast" if self.mc_ptr is not None else "p2p"

    def run(self, plan, vals, B, stream=None) -> None:
        from . import escs
        self.handle.barrier(channel=0)
        if self.mc_ptr is not None:
            escs.escs_spmm_scatter(plan, vals, B, [self.mc_ptr], self.r0, stream, multicast=True)
        else:
            escs.escs_spmm_scatter(plan, vals, B, self.peers, self.r0, stream)
        self.handle.barrier(channel=0)
