"""kkt::update: the factor after an active-set change
equals a fresh factorization of the updated Newton system (kkt_solver.hpp:
152-161). The GPU takes the reference's refactorization path; the reference
build (oracle/_ref, kkt_update.cpp) takes its hyperbolic-Householder
low-rank path for the small ranks used here. Bars: the reference's own
update-vs-refactor tolerance (test_kkt_update.cpp:127-241, 1e-8) on the
solution, KKT residual as the parity suite."""
import numpy as np
import pytest

from pyoracle import RefOracle, ref_available

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqOCPBatch, EqRhsBatch, kkt_residual, rel_error

pytestmark = pytest.mark.gpu


def newton_system(base, D, E, sig):
    """Stage Hessians augmented as synth.qpalm_sequence (qpalm.cpp:184-221)."""
    N = base.N
    DS = D * sig[:, :N, :, None]
    R = base.R + np.einsum("bjki,bjkl->bjil", DS, D)
    S = base.S + np.einsum("bjki,bjkl->bjil", DS, E[:, :N])
    ES = E * sig[..., None]
    Q = base.Q + np.einsum("bjki,bjkl->bjil", ES, E)
    return EqOCPBatch(base.A, base.B, R, S, Q, base.f, base.r, base.q, base.x_init)


@pytest.mark.skipif(not ref_available(), reason="reference build not available")
@pytest.mark.parametrize("changes", [[(5, 3), (20, 7), (41, 0)], [(0, 2), (63, 5), (64, 1)]])
def test_update_matches_reference_low_rank_update(changes):
    base = synth.generate(4, seed=2, batch=1, N=64)
    D, E, sig = synth.qpalm_data(base, seed=2, iters=1)
    sig0 = sig[0]
    sig1 = sig0.copy()
    for j, i in changes:  # a few active-set changes (rank < rho * nx per column)
        sig1[0, j, i] *= 10.0
    p_old, p_new = newton_system(base, D, E, sig0), newton_system(base, D, E, sig1)
    ds = sig1 - sig0
    N = base.N
    ref, rc, rep = RefOracle().update_solve(p_old, p_new, 16, D[0], E[0, :N], E[0, N], ds[0, :N], ds[0, N])
    assert rc == 0 and rep[0] > 0  # the reference updated columns (low-rank path)
    f = kkt.factor(p_old, kkt.FactorOptions(P=16))
    f2, report = kkt.update(f, p_new, E[:, :N], D, E[:, N], ds[:, :N], ds[:, N])
    assert report["columns_refactored"][0] == rep[0] + rep[1]
    sol = kkt.solve(f2, p_new, EqRhsBatch.of_problem(p_new))
    assert rel_error(sol, ref).max() <= 1e-8
    res_gpu = kkt_residual(p_new, EqRhsBatch.of_problem(p_new), sol).max()
    res_ref = kkt_residual(p_new, EqRhsBatch.of_problem(p_new), ref).max()
    assert res_gpu <= max(1e-10, 4 * res_ref)


def test_update_without_change_keeps_factor():
    base = synth.generate(4, seed=3, batch=1, N=32)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1)
    p = newton_system(base, D, E, sig[0])
    f = kkt.factor(p, kkt.FactorOptions(P=8))
    N = base.N
    f2, report = kkt.update(f, p, E[:, :N], D, E[:, N], np.zeros((1, N, 24)), np.zeros((1, 24)))
    assert f2 is f and report["columns_refactored"] == [0] and not report["schur_refactored"]
