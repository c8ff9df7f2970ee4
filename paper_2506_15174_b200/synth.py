"""Seeded synthetic inputs for the ESC SpMM hot path (arXiv 2506.15174).

This module is shared by the oracle side (tests) and the CUDA side (tests,
bench) and therefore holds NONE of the method's arithmetic: it only draws
sparsity patterns, values and dense B matrices.  Recipes follow SURVEY.md
§8(d) and are restated in DESIGN.md ("Input recipe").

All generators use numpy's PCG64 (``np.random.default_rng(seed)``) and return
plain numpy arrays: CSR ``rowptr``/``colidx`` int32, ``vals`` fp32 and row-major
fp32 ``B``.  The paper's workload is DLMC, which is not available
offline; these are magnitude-pruned stand-ins with the same shapes and
sparsities.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CSR", "Problem", "magnitude_pruned", "power_law", "uniform_large", "dense_b",
    "dyadic_twin", "transformer_suite", "resnet_suite", "suite", "config", "SPARSITIES",
    "TRANSFORMER_SHAPES", "RESNET_SHAPES", "RESNET50_ALL_SHAPES", "BCOLS", "resnet50_full_suite",
]

SPARSITIES = (0.70, 0.80, 0.90, 0.95, 0.98)
TRANSFORMER_SHAPES = ((512, 512), (2048, 512), (512, 2048))        # P:664 "most common sizes"
RESNET_SHAPES = ((256, 2304), (512, 4608), (2048, 512))             # im2col M x (C*kh*kw)
# all 21 distinct ResNet-50 conv/fc GEMM shapes (M = out channels, K = in*kh*kw;
# the paper's "21 different sizes"; SURVEY §8(d) C3 extended suite)
RESNET50_ALL_SHAPES = ((64, 147), (64, 64), (64, 576), (256, 64), (64, 256), (128, 256),
                       (128, 1152), (512, 128), (512, 256), (128, 512), (256, 512),
                       (256, 2304), (1024, 256), (1024, 512), (256, 1024), (512, 1024),
                       (512, 4608), (2048, 512), (2048, 1024), (512, 2048), (1000, 2048))
BCOLS = (32, 64, 128)


@dataclass
class CSR:
    m: int
    k: int
    rowptr: np.ndarray      # int32[m+1]
    colidx: np.ndarray      # int32[nnz], strictly increasing per row
    vals: np.ndarray        # float32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def dense(self) -> np.ndarray:
        """Dense fp32 image (tiny cases / cuBLAS baseline only)."""
        D = np.zeros((self.m, self.k), np.float32)
        rows = np.repeat(np.arange(self.m), np.diff(self.rowptr))
        D[rows, self.colidx] = self.vals
        return D


@dataclass
class Problem:
    name: str
    A: CSR
    B: np.ndarray           # float32[k, bCols], row-major
    meta: dict = field(default_factory=dict)

    @property
    def bcols(self) -> int:
        return int(self.B.shape[1])

    @property
    def flops(self) -> int:
        """Metric numerator: 2*nnz*bCols (BASELINE.json metric)."""
        return 2 * self.A.nnz * self.bcols

    @property
    def bytes_comp(self) -> int:
        """Compulsory bytes: CSR A once, B once, C once."""
        A = self.A
        return 8 * A.nnz + 4 * (A.m + 1) + 4 * A.k * self.bcols + 4 * A.m * self.bcols


def _csr_from_sorted_linear(lin: np.ndarray, m: int, k: int, vals: np.ndarray) -> CSR:
    rows = (lin // k).astype(np.int64)
    cols = (lin % k).astype(np.int32)
    counts = np.bincount(rows, minlength=m)
    rowptr = np.zeros(m + 1, np.int64)
    np.cumsum(counts, out=rowptr[1:])
    if rowptr[-1] >= 2 ** 31:
        raise ValueError("nnz exceeds int32")
    return CSR(m, k, rowptr.astype(np.int32), cols, vals.astype(np.float32))


def nnz_for(m: int, k: int, s: float) -> int:
    """nnz = round((1-s)*m*k) (512x512 at 0.7 -> 78,643)."""
    return int(round((1.0 - s) * m * k))


def magnitude_pruned(m: int, k: int, s: float, seed: int) -> CSR:
    """Dense N(0,1) fp32, keep the nnz largest |w| (ties: row-major index)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((m, k), dtype=np.float32).ravel()
    nnz = nnz_for(m, k, s)
    order = np.argsort(-np.abs(w), kind="stable")[:nnz]
    lin = np.sort(order)
    return _csr_from_sorted_linear(lin, m, k, w[lin])


def _tail_values(rng, n: int, s: float) -> np.ndarray:
    """Random sign x |N(0,1)| conditioned on |w| > Phi^-1(1-(1-s)/2): what
    magnitude pruning of an iid Gaussian leaves behind."""
    from scipy.special import ndtri
    d = 1.0 - s
    u = 1.0 - rng.random(n)                    # (0, 1]
    mag = -ndtri(0.5 * d * u)                  # = Phi^-1(1 - d/2 * u)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return (sign * mag).astype(np.float32)


def _rows_to_csr(m, k, lens, rng, s) -> CSR:
    rowptr = np.zeros(m + 1, np.int64)
    np.cumsum(lens, out=rowptr[1:])
    nnz = int(rowptr[-1])
    if nnz >= 2 ** 31:
        raise ValueError("nnz exceeds int32")
    colidx = np.empty(nnz, np.int32)
    for i in range(m):
        L = int(lens[i])
        if L == 0:
            continue
        if L == k:
            c = np.arange(k, dtype=np.int32)
        else:
            c = np.sort(rng.choice(k, L, replace=False)).astype(np.int32)
        colidx[rowptr[i]:rowptr[i + 1]] = c
    vals = _tail_values(rng, nnz, s)
    return CSR(m, k, rowptr.astype(np.int32), colidx, vals)


def power_law(m: int, k: int, s: float, seed: int) -> CSR:
    """C4: row lengths L_rank = min(k, max(1, floor(c/(rank+1)))), c by
    bisection so sum L <= nnz, remainder +1 round-robin from rank 0 skipping
    full rows; rows permuted by a seeded permutation; columns uniform without
    replacement per row; tail-Gaussian values."""
    rng = np.random.default_rng(seed)
    nnz = nnz_for(m, k, s)
    ranks = np.arange(1, m + 1, dtype=np.float64)

    def lens_for(c):
        return np.minimum(k, np.maximum(1, np.floor(c / ranks))).astype(np.int64)

    lo, hi = 0.0, float(k) * m
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if lens_for(mid).sum() <= nnz:
            lo = mid
        else:
            hi = mid
    L = lens_for(lo)
    rem = nnz - int(L.sum())
    while rem > 0:
        for r in range(m):
            if rem == 0:
                break
            if L[r] < k:
                L[r] += 1
                rem -= 1
    perm = rng.permutation(m)
    lens = np.empty(m, np.int64)
    lens[perm] = L
    return _rows_to_csr(m, k, lens, rng, s)


def uniform_large(m: int, k: int, s: float, seed: int) -> CSR:
    """C5: exactly nnz positions spread uniformly over m*k.  Row counts are
    Binomial(k, 1-s) adjusted by +-1 on uniformly chosen rows to the exact
    total (m*k = 2^34 is beyond numpy's multivariate-hypergeometric), then
    columns uniform without replacement per row; tail-Gaussian values."""
    rng = np.random.default_rng(seed)
    nnz = nnz_for(m, k, s)
    lens = rng.binomial(k, 1.0 - s, size=m).astype(np.int64)
    diff = nnz - int(lens.sum())
    while diff != 0:
        rows = rng.integers(0, m, size=abs(diff))
        step = 1 if diff > 0 else -1
        np.add.at(lens, rows, step)
        np.clip(lens, 0, k, out=lens)
        diff = nnz - int(lens.sum())
    return _rows_to_csr(m, k, lens, rng, s)


def dense_b(k: int, n: int, seed: int) -> np.ndarray:
    """B ~ U[-1, 1) fp32, row-major k x n."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(k, n)).astype(np.float32)


def dyadic_twin(A: CSR, n: int, seed: int):
    """Same pattern, A values in {+-0.5, +-1, +-2}, B integers in [-8, 8]:
    every product and partial sum is an exact multiple of 0.5 below 2^23, so
    any summation order gives the same fp32 result."""
    rng = np.random.default_rng(seed)
    vals = rng.choice(np.array([-2.0, -1.0, -0.5, 0.5, 1.0, 2.0], np.float32), A.nnz)
    B = rng.integers(-8, 9, size=(A.k, n)).astype(np.float32)
    return CSR(A.m, A.k, A.rowptr, A.colidx, vals.astype(np.float32)), B


# ------------------------------------------------------------------ configs

def _shape_seed(shape_idx: int, s_idx: int) -> int:
    return 1000 + 10 * shape_idx + s_idx


def _suite(shapes, shape_base, bcols=BCOLS, sparsities=SPARSITIES):
    out = []
    for si, (m, k) in enumerate(shapes):
        for pi, s in enumerate(sparsities):
            seed = _shape_seed(shape_base + si, pi)
            A = magnitude_pruned(m, k, s, seed)
            for n in bcols:
                out.append(Problem(f"{m}x{k}@{int(round(s * 100))}%/b{n}", A,
                                   dense_b(k, n, seed + 5000 + n),
                                   {"m": m, "k": k, "s": s, "bcols": n, "seed": seed}))
    return out


def transformer_suite(bcols=BCOLS, sparsities=SPARSITIES):
    """configs[1]: {512x512, 2048x512, 512x2048} x 70..98% x bCols 32/64/128."""
    return _suite(TRANSFORMER_SHAPES, 0, bcols, sparsities)


def resnet_suite(bcols=BCOLS, sparsities=SPARSITIES):
    """configs[2]: ResNet-50 im2col {256x2304, 512x4608, 2048x512}."""
    return _suite(RESNET_SHAPES, 3, bcols, sparsities)


def resnet50_full_suite(bcols=BCOLS, sparsities=SPARSITIES):
    """Extended configs[2]: every ResNet-50 layer shape (21) x sparsities x bCols."""
    return _suite(RESNET50_ALL_SHAPES, 100, bcols, sparsities)


def suite(bcols=BCOLS, sparsities=SPARSITIES):
    return transformer_suite(bcols, sparsities) + resnet_suite(bcols, sparsities)


def config(name: str) -> Problem:
    """Single named configs: c1, c4, c5."""
    if name == "c1":
        A = magnitude_pruned(256, 256, 0.90, 1)
        return Problem("c1:256x256@90%/b32", A, dense_b(256, 32, 2), {"s": 0.9})
    if name == "c4":
        A = power_law(16384, 16384, 0.99, 16384)
        return Problem("c4:powerlaw16384@99%/b128", A, dense_b(16384, 128, 16385), {"s": 0.99})
    if name == "c5":
        A = uniform_large(131072, 131072, 0.995, 131072)
        return Problem("c5:131072@99.5%/b128", A, dense_b(131072, 128, 131073), {"s": 0.995})
    raise KeyError(name)


def row_block(A: CSR, r0: int, r1: int) -> CSR:
    """Rows [r0, r1) of A as their own CSR (row-block sharding)."""
    a, b = int(A.rowptr[r0]), int(A.rowptr[r1])
    return CSR(r1 - r0, A.k, (A.rowptr[r0:r1 + 1] - a).astype(np.int32),
               A.colidx[a:b].copy(), A.vals[a:b].copy())


def shard_bounds(m: int, world: int, rank: int):
    """Rank r owns rows [r*m/G, (r+1)*m/G)."""
    return (rank * m) // world, ((rank + 1) * m) // world


def random_csr(m: int, k: int, nnz: int, seed: int, empty_rows=(), dense_rows=()) -> CSR:
    """Small edge-case generator: uniform pattern with forced empty/dense rows."""
    rng = np.random.default_rng(seed)
    lin = np.sort(rng.choice(m * k, size=min(nnz, m * k), replace=False)) if m * k else np.zeros(0, np.int64)
    D = np.zeros((m, k), bool)
    D.ravel()[lin] = True
    for r in empty_rows:
        D[r, :] = False
    for r in dense_rows:
        D[r, :] = True
    lin = np.flatnonzero(D.ravel())
    vals = rng.uniform(-1, 1, lin.size).astype(np.float32)
    vals[vals == 0] = 0.5
    return _csr_from_sorted_linear(lin, m, k, vals)
