"""GPU parity of the staged record walk (escs_params.staged = 2: B rows of a
CTA's column range staged in shared memory by TMA bulk copies, the column
ranges' partials combined in the kernel -- or by a second launch when the
grid cannot be co-resident) against the fp64 oracle.

C: bit-exact on dyadic twins (G1, every partial sum exact, so any summation
order gives the oracle's value) and within G2 (max rel err 1e-4,
north_star) on real values; bitwise reproducible across calls and graph
replays (the combine sums in range order; its counters self-reset).
"""
import os

import numpy as np
import pytest

import oracle
from paper_2506_15174_b200 import synth

from test_gpu_parity import check_exact, check_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def run_staged(torch, A, B, **params):
    from paper_2506_15174_b200 import escs
    n = B.shape[1]
    pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, n, packed=1, staged=2, **params)
    dv = torch.from_numpy(A.vals).cuda() if A.nnz else torch.zeros(1, device="cuda")
    dB = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    pk = escs.escs_pack(pl, dv)
    C = torch.full((A.m, n), float("nan"), device="cuda")
    escs.escs_spmm_packed(pl, pk, dB, C)
    torch.cuda.synchronize()
    return C.cpu().numpy(), pl, pk, dB


def both(torch, A, n, seed, **params):
    """Real values within G2, then the dyadic twin bit-exact, same parameters."""
    B = synth.dense_b(A.k, n, seed)
    C, pl, _, _ = run_staged(torch, A, B, **params)
    check_tol(A, B, C)
    Ad, Bd = synth.dyadic_twin(A, n, seed + 1)
    Cd, _, _, _ = run_staged(torch, Ad, Bd, **params)
    check_exact(Ad, Bd, Cd)
    return pl.info


@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("ufi", [1, 2, 3, 4, 6, 8])
def test_staged_ufi_bcols(torch_cuda, ufi, n):
    A = synth.magnitude_pruned(384, 1536, 0.7, 100 + ufi)
    info = both(torch_cuda, A, n, 7, ufi=ufi)
    assert info["staged"] == 1 and info["h"] == ufi


@pytest.mark.parametrize("ufi,W,npw,ns", [(1, 16, 4, 9), (2, 8, 2, 4), (3, 16, 2, 5), (4, 6, 1, 11),
                                          (8, 16, 1, 37), (4, 16, 2, 37), (6, 8, 1, 13), (2, 3, 4, 5)])
def test_staged_tiles_ragged(torch_cuda, ufi, W, npw, ns):
    """Ragged m (not a multiple of UFi nor of the row block), odd k, explicit
    tiles incl. one range (no combine) and many ranges."""
    A = synth.magnitude_pruned(437, 1291, 0.75, 31)
    info = both(torch_cuda, A, 128, 9, ufi=ufi, st_warps=W, st_npw=npw, st_nsplit=ns)
    assert (info["st_warps"], info["st_npw"], info["st_nsplit"]) == (W, npw, ns)


@pytest.mark.parametrize("ufi", [1, 4, 8])
def test_staged_single_range(torch_cuda, ufi):
    """One column range (st_nsplit = 1): each CTA writes C directly."""
    A = synth.magnitude_pruned(1000, 200, 0.7, 41)
    info = both(torch_cuda, A, 128, 21, ufi=ufi, st_warps=8, st_nsplit=1)
    assert info["st_nsplit"] == 1 and info["st_launches"] == 1


def test_staged_f8_lane_map(torch_cuda):
    A = synth.magnitude_pruned(512, 2048, 0.7, 5)
    info = both(torch_cuda, A, 128, 3, ufi=4, colf=8)
    assert info["colf"] == 8


def test_staged_two_launch_fallback(torch_cuda, monkeypatch):
    """ESCS_ST_COOP=0: the ranges' partials are summed by a second launch."""
    monkeypatch.setenv("ESCS_ST_COOP", "0")
    A = synth.magnitude_pruned(512, 4608, 0.7, 17)
    info = both(torch_cuda, A, 128, 5, ufi=8, st_warps=16, st_nsplit=37)
    assert info["st_launches"] == 2


def test_staged_more_ctas_than_sms(torch_cuda):
    """A grid larger than one wave (not co-resident): the two-launch combine."""
    A = synth.magnitude_pruned(2048, 1024, 0.8, 19)
    info = both(torch_cuda, A, 64, 11, ufi=2, st_warps=4, st_npw=1, st_nsplit=8)
    assert info["st_ctas"] > 148


def test_staged_degenerate(torch_cuda):
    cases = [synth.CSR(5, 9, np.zeros(6, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32)),
             synth.magnitude_pruned(1, 50, 0.5, 1), synth.magnitude_pruned(40, 1, 0.5, 2),
             synth.magnitude_pruned(17, 33, 0.0, 3), synth.random_csr(64, 300, 900, 4, empty_rows=(0, 5, 63),
                                                                     dense_rows=(7,))]
    for A in cases:
        for ufi in (1, 3, 8):
            both(torch_cuda, A, 32, 13, ufi=ufi)


def test_staged_powerlaw(torch_cuda):
    A = synth.power_law(1024, 2048, 0.95, 23)
    both(torch_cuda, A, 128, 15, ufi=4, st_warps=8)


def test_staged_deterministic_and_graph_replay(torch_cuda):
    """Bitwise equal across repeated calls and CUDA-graph replays (the
    in-kernel combine's counters reset themselves)."""
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    A = synth.magnitude_pruned(512, 4608, 0.7, 29)
    B = synth.dense_b(A.k, 128, 31)
    C0, pl, pk, dB = run_staged(torch, A, B, ufi=8, st_warps=16, st_nsplit=37)
    assert pl.info["st_launches"] == 1 and pl.info["st_nsplit"] == 37
    C = torch.empty(A.m, 128, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            escs.escs_spmm_packed(pl, pk, dB, C, stream=s)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), C0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(4):
            escs.escs_spmm_packed(pl, pk, dB, C, stream=s)
    for _ in range(3):
        C.fill_(float("nan"))
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), C0)


def test_staged_probe_runs(torch_cuda):
    torch = torch_cuda
    from paper_2506_15174_b200 import escs
    A = synth.magnitude_pruned(512, 2048, 0.7, 37)
    B = synth.dense_b(A.k, 128, 1)
    _, pl, pk, dB = run_staged(torch, A, B, ufi=4)
    info = pl.info
    sink = torch.full((info["st_ctas"] * 32 * info["st_warps"],), float("nan"), device="cuda")
    escs.escs_gather_probe_packed(pl, pk, dB, sink)
    torch.cuda.synchronize()
    assert torch.isfinite(sink).all()


def test_staged_autotuned_suite_layers(torch_cuda):
    """The plan-time tuner with staged = 2 (staged plans only) and with the
    default (both walks) on the 70% layers the staged walk targets."""
    probs = [p for p in synth.suite(sparsities=(0.7,)) if p.bcols in (64, 128)][:6]
    for p in probs:
        for st in (2, 0):
            from paper_2506_15174_b200 import escs
            A = p.A
            pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, p.bcols, packed=1, autotune=1, staged=st)
            if st == 2:
                assert pl.info["staged"] == 1
            dv = torch_cuda.from_numpy(A.vals).cuda()
            pk = escs.escs_pack(pl, dv)
            C = torch_cuda.empty(A.m, p.bcols, device="cuda")
            escs.escs_spmm_packed(pl, pk, torch_cuda.from_numpy(p.B).cuda(), C)
            torch_cuda.cuda.synchronize()
            check_tol(A, p.B, C.cpu().numpy())


def test_tuning_cache_reuses_parameters(torch_cuda, monkeypatch):
    """A second matrix of the same class (shape, nnz, bCols, request) is planned
    with the first one's tuned parameters (autotuned = 2), and is exact."""
    from paper_2506_15174_b200 import escs
    monkeypatch.delenv("ESCS_TUNE_CACHE", raising=False)
    A1 = synth.magnitude_pruned(389, 771, 0.8, 501)   # a shape no other test tunes
    A2 = synth.magnitude_pruned(389, 771, 0.8, 502)
    assert A1.nnz == A2.nnz
    p1 = escs.escs_plan_ex(A1.m, A1.k, A1.nnz, A1.rowptr, A1.colidx, 64, packed=1, autotune=1, tile_order=1)
    p2 = escs.escs_plan_ex(A2.m, A2.k, A2.nnz, A2.rowptr, A2.colidx, 64, packed=1, autotune=1, tile_order=1)
    i1, i2 = p1.info, p2.info
    assert i1["autotuned"] == 1 and i2["autotuned"] == 2
    for key in ("h", "T", "cta_warps", "ufk", "colf", "staged", "st_nsplit"):
        assert i1[key] == i2[key], key
    Ad, Bd = synth.dyadic_twin(A2, 64, 3)
    dv = torch_cuda.from_numpy(Ad.vals).cuda()
    pk = escs.escs_pack(p2, dv)
    C = torch_cuda.empty(A2.m, 64, device="cuda")
    escs.escs_spmm_packed(p2, pk, torch_cuda.from_numpy(Bd).cuda(), C)
    torch_cuda.cuda.synchronize()
    check_exact(Ad, Bd, C.cpu().numpy())


def test_tuning_cache_file_across_processes(torch_cuda, tmp_path):
    """ESCS_TUNE_CACHE_FILE: a second process plans with the first one's tuned
    parameters (autotuned = 2) -- the same plans under a profiler."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2506_15174_b200 import escs, synth\n"
            "A = synth.magnitude_pruned(256, 512, 0.8, 9)\n"
            "pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, autotune=1)\n"
            "i = pl.info; print(i['autotuned'], i['h'], i['T'], i['cta_warps'], i['ufk'], i['colf'])\n") % root
    env = dict(os.environ, ESCS_TUNE_CACHE_FILE=str(tmp_path / "tune.txt"))
    out = [subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
           .stdout.split() for _ in range(2)]
    assert out[0][0] == "1" and out[1][0] == "2"
    assert out[0][1:] == out[1][1:]


@pytest.mark.parametrize("cv", [-2, -1, 25, 100])
def test_explicit_carveout_exact(torch_cuda, cv):
    """escs_params.carveout only changes the L1 / shared split of the launches:
    the result is bitwise the same as the automatic carveout's."""
    from paper_2506_15174_b200 import escs
    A = synth.magnitude_pruned(512, 1024, 0.8, 77)
    Ad, Bd = synth.dyadic_twin(A, 64, 5)
    outs = []
    for c in (0, cv):
        pl = escs.escs_plan_ex(A.m, A.k, A.nnz, A.rowptr, A.colidx, 64, packed=1, carveout=c, T=40, cta_warps=4)
        exp_cv = {0: None, -2: 0, -1: -1}.get(c, c)
        if exp_cv is not None:
            assert pl.info["carveout"] == exp_cv
        pk = escs.escs_pack(pl, torch_cuda.from_numpy(Ad.vals).cuda())
        C = torch_cuda.empty(A.m, 64, device="cuda")
        escs.escs_spmm_packed(pl, pk, torch_cuda.from_numpy(Bd).cuda(), C)
        torch_cuda.cuda.synchronize()
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    check_exact(Ad, Bd, outs[1])
