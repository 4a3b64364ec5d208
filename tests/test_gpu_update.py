"""kkt::update on the GPU (kkt_update.cpp:372-477): the
low-rank hyperbolic-Householder column update (update.cu) for columns whose
update rank is below rho nx, refactorization above it (or on a breakdown),
then the Schur complement / CR factor re-formed.

Checked against the reference's own kkt::update (oracle/_ref builds
kkt_update.cpp): the per-instance UpdateReport column counts equal the
reference's, and the solution of the updated factor matches the reference's
updated factor within its own update-vs-refactor bar (test_kkt_update.cpp:
127-241: 1e-8); the updated GPU factor's blocks match a fresh factorization
of the new problem, and kkt::solve with other right-hand sides agrees."""
import numpy as np
import pytest

from pyoracle import Oracle, RefOracle, ref_available

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


def _changed(sig0, changes, factor=10.0):
    sig1 = sig0.copy()
    for (b, j, i, fac) in changes:
        sig1[b, j, i] = sig0[b, j, i] * fac if fac != 0 else 0.0
    return sig1


def _run(base, D, E, sig0, sig1, P):
    N = base.N
    p_old, p_new = newton_system(base, D, E, sig0), newton_system(base, D, E, sig1)
    ds = sig1 - sig0
    f = kkt.factor(p_old, kkt.FactorOptions(P=P))
    f2, report = kkt.update(f, p_new, E[:, :N], D, E[:, N], ds[:, :N], ds[:, N])
    return p_old, p_new, ds, f2, report


# (b, stage j, row i, factor): multiply sigma (10 = more weight, 0.1 = less,
# 0 = row leaves the active set: a negative dSigma, hyperbolic rotations)
LOW_RANK = [
    [(0, 5, 3, 10.0), (0, 20, 7, 10.0), (0, 41, 0, 10.0)],
    [(0, 0, 2, 10.0), (0, 63, 5, 0.1), (0, 64, 1, 10.0)],  # stage 0 and the terminal rows
    [(0, 10, 4, 0.0), (0, 11, 9, 0.0), (0, 30, 2, 0.3)],    # down-dates
]


@pytest.mark.skipif(not ref_available(), reason="reference build not available")
@pytest.mark.parametrize("changes", LOW_RANK)
def test_low_rank_update_matches_reference(changes):
    base = synth.generate(4, seed=2, batch=1, N=64)
    D, E, sig = synth.qpalm_data(base, seed=2, iters=1)
    sig0 = sig[0]
    sig1 = _changed(sig0, changes)
    p_old, p_new, ds, f2, report = _run(base, D, E, sig0, sig1, 16)
    N = base.N
    ref, rc, rep = RefOracle().update_solve(p_old, p_new, 16, D[0], E[0, :N], E[0, N], ds[0, :N], ds[0, N])
    assert rc == 0 and rep[0] > 0  # the reference took its low-rank path
    assert report["columns_updated"][0] == rep[0]
    assert report["columns_refactored"][0] == rep[1]
    sol = kkt.solve(f2, p_new, EqRhsBatch.of_problem(p_new))
    assert rel_error(sol, ref).max() <= 1e-8
    res_gpu = kkt_residual(p_new, EqRhsBatch.of_problem(p_new), sol).max()
    res_ref = kkt_residual(p_new, EqRhsBatch.of_problem(p_new), ref).max()
    assert res_gpu <= max(1e-10, 4 * res_ref)


@pytest.mark.parametrize("changes", LOW_RANK)
def test_updated_blocks_equal_fresh_factor(changes):
    base = synth.generate(4, seed=2, batch=1, N=64)
    D, E, sig = synth.qpalm_data(base, seed=2, iters=1)
    sig1 = _changed(sig[0], changes)
    _, p_new, _, f2, report = _run(base, D, E, sig[0], sig1, 16)
    assert sum(report["columns_updated"]) > 0
    fresh = kkt.factor(p_new, kkt.FactorOptions(P=16)).materialize(0)
    got = f2.materialize(0)
    for k in ("LH", "LB", "Acl", "LA", "T", "Mfwd", "Mbwd", "W", "schur_diag", "schur_sub", "cr_L"):
        scale = max(1.0, np.abs(fresh[k]).max())
        assert np.abs(got[k] - fresh[k]).max() <= 1e-8 * scale, k


@pytest.mark.skipif(not ref_available(), reason="reference build not available")
def test_high_rank_column_is_refactored_like_the_reference():
    base = synth.generate(4, seed=4, batch=1, N=64)
    D, E, sig = synth.qpalm_data(base, seed=4, iters=1)
    # 9 rows of stage 5 (column 1's stages) change: rank 9 >= rho nx = 8
    changes = [(0, 5, i, 10.0) for i in range(9)] + [(0, 40, 1, 10.0)]
    sig1 = _changed(sig[0], changes)
    p_old, p_new, ds, f2, report = _run(base, D, E, sig[0], sig1, 16)
    N = base.N
    ref, rc, rep = RefOracle().update_solve(p_old, p_new, 16, D[0], E[0, :N], E[0, N], ds[0, :N], ds[0, N])
    assert rc == 0
    assert (report["columns_updated"][0], report["columns_refactored"][0]) == (rep[0], rep[1])
    assert rep[1] >= 1
    sol = kkt.solve(f2, p_new, EqRhsBatch.of_problem(p_new))
    assert rel_error(sol, ref).max() <= 1e-8


def test_batch_of_instances_mixed_paths():
    base = synth.generate(4, seed=5, batch=3, N=64)
    D, E, sig = synth.qpalm_data(base, seed=5, iters=1)
    changes = [(0, 3, 1, 10.0), (0, 50, 2, 0.0),                        # instance 0: updates
               (1, 7, 0, 5.0)] + [(1, 20, i, 10.0) for i in range(12)]  # 1: update + refactor
    # instance 2: unchanged
    sig1 = _changed(sig[0], changes)
    _, p_new, _, f2, report = _run(base, D, E, sig[0], sig1, 16)
    assert report["columns_updated"][0] == 2 and report["columns_refactored"][0] == 0
    assert report["columns_updated"][1] == 1 and report["columns_refactored"][1] == 1
    assert report["columns_updated"][2] == 0 and not report["schur_refactored"][2]
    sol = kkt.solve(f2, p_new, EqRhsBatch.of_problem(p_new))
    ref, rc, _ = Oracle().solve_problem(p_new, 16)
    assert rc == 0
    assert rel_error(sol, ref).max() <= 1e-8


def test_successive_updates_track_fresh_factor():
    # an active-set sequence like the QPALM inner loop: update after update
    base = synth.generate(4, seed=6, batch=2, N=64)
    D, E, sig = synth.qpalm_data(base, seed=6, iters=1)
    N = base.N
    rng = np.random.default_rng(7)
    sig_cur = sig[0].copy()
    f = kkt.factor(newton_system(base, D, E, sig_cur), kkt.FactorOptions(P=16))
    for _ in range(4):
        sig_new = sig_cur.copy()
        for b in range(2):
            for _ in range(3):
                j, i = rng.integers(0, N + 1), rng.integers(0, 24)
                sig_new[b, j, i] *= rng.choice([0.1, 10.0])
        ds = sig_new - sig_cur
        p_new = newton_system(base, D, E, sig_new)
        f, _ = kkt.update(f, p_new, E[:, :N], D, E[:, N], ds[:, :N], ds[:, N])
        sig_cur = sig_new
    sol = kkt.solve(f, p_new, EqRhsBatch.of_problem(p_new))
    ref = kkt.solve_problem(p_new, kkt.FactorOptions(P=16))
    assert rel_error(sol, ref).max() <= 1e-8
    rhs2 = EqRhsBatch(rng.standard_normal(ref.u.shape), rng.standard_normal((2, N + 1, base.nx)),
                      rng.standard_normal(ref.lam.shape))
    s2 = kkt.solve(f, p_new, rhs2)
    r2 = kkt.solve(kkt.factor(p_new, kkt.FactorOptions(P=16)), p_new, rhs2)
    assert rel_error(s2, r2).max() <= 1e-8


def test_update_without_change_keeps_factor():
    base = synth.generate(4, seed=3, batch=1, N=32)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1)
    p = newton_system(base, D, E, sig[0])
    f = kkt.factor(p, kkt.FactorOptions(P=8))
    N = base.N
    before = f.materialize(0)
    f2, report = kkt.update(f, p, E[:, :N], D, E[:, N], np.zeros((1, N, 24)), np.zeros((1, 24)))
    assert f2 is f and report["columns_refactored"] == [0] and report["schur_refactored"] == [False]
    after = f.materialize(0)
    for k in before:
        assert np.array_equal(before[k], after[k]), k


def test_update_other_shape_device_arrays():
    # config-1 stage shape (nx 20, nu 10, P 16), ny 6 rows, CUDA tensors
    import torch
    base = synth.generate(1, seed=8, batch=2, N=64)
    rng = np.random.default_rng(9)
    ny, N = 6, base.N
    D = rng.standard_normal((2, N, ny, base.nu))
    E = rng.standard_normal((2, N + 1, ny, base.nx))
    sig0 = 10.0 ** rng.uniform(-1, 2, (2, N + 1, ny))
    sig1 = _changed(sig0, [(0, 9, 2, 10.0), (1, 33, 5, 0.0), (1, 34, 1, 3.0)])
    p_old, p_new = newton_system(base, D, E, sig0), newton_system(base, D, E, sig1)
    ds = sig1 - sig0

    def dev(p):
        d = EqOCPBatch.__new__(EqOCPBatch)
        for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
            setattr(d, k, torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda())
        return d

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    f = kkt.factor(dev(p_old), kkt.FactorOptions(P=16))
    f2, report = kkt.update(f, dev(p_new), t(E[:, :N]), t(D), t(E[:, N]), t(ds[:, :N]), t(ds[:, N]))
    assert report["columns_updated"] == [1, 1]  # stages 33 and 34 share column 9
    sol = kkt.solve(f2, p_new, EqRhsBatch.of_problem(p_new))
    ref = kkt.solve_problem(p_new, kkt.FactorOptions(P=16))
    assert rel_error(sol, ref).max() <= 1e-8
