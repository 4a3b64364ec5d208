"""CPU tests: the C oracle restatement is pinned against the reference's own
outputs (golden fixtures from the reference build, and the reference library
itself where it was built), plus the model/property checks of the
reference's test suite that do not need a GPU."""
import numpy as np
import pytest

import golden_util
from pyoracle import Oracle, RefOracle, ref_available

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.mark.parametrize("name", golden_util.names())
def test_oracle_matches_reference_golden(oracle, name):
    p, P, ref_sol, z = golden_util.load(name)
    sol, rc, st = oracle.solve_problem(p, P)
    assert rc == 0
    assert rel_error(sol, ref_sol).max() <= 1e-12
    res = kkt_residual(p, EqRhsBatch.of_problem(p), sol).max(axis=1)
    # the oracle's residual is at the reference's own level
    assert np.all(res <= np.maximum(1e-12, 10 * z["residual"]))


@pytest.mark.parametrize("name", [n for n in golden_util.names() if n.startswith("kat_")])
def test_oracle_factor_blocks_match_reference(oracle, name):
    p, P, _, z = golden_util.load(name)
    fb, rc, _ = oracle.factor_blocks(p, P)
    assert rc == 0
    for k in ("LH", "LB", "Acl", "LA", "T", "Mfwd", "Mbwd", "W", "schur_diag", "schur_sub"):
        ref = z["fb_" + k]
        assert np.abs(fb[k] - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), k


def test_fma_counts_match_reference_counter(oracle):
    # SURVEY §8d algorithmic FLOPs: 2 x reference FMA counter
    assert oracle.fma_counts(64, 10, 5, 4) == (329660, 79580)
    assert oracle.fma_counts(128, 20, 10, 16) == (5242400, 596640)
    assert oracle.fma_counts(4096, 12, 4, 256) == (29816352, 6571520)
    assert oracle.fma_counts(256, 16, 8, 16) == (5335808, 791168)


@pytest.mark.skipif(not ref_available(), reason="reference build not available")
def test_oracle_vs_reference_library_all_configs(oracle):
    ref = RefOracle()
    for cfg, N in [(0, None), (1, 48), (2, 512), (3, 32), (4, 64)]:
        p = synth.generate(cfg, seed=3, batch=2, N=N)
        P = synth.CONFIGS[cfg].P
        a, rc, _ = oracle.solve_problem(p, P)
        b, res, rc2, _ = ref.solve_problem(p, P)
        assert rc == rc2 == 0
        assert rel_error(a, b).max() <= 1e-12


def test_zero_rhs_gives_zero_solution(oracle):
    # test_kkt.cpp:114-121
    p = synth.generate(0, seed=1, batch=1, N=16)
    z = EqRhsBatch.zero(p)
    sol, rc, _ = oracle.solve(p, z, 4)
    assert rc == 0
    assert np.all(sol.u == 0) and np.all(sol.x[:, 1:] == 0)


def test_cross_P_consistency(oracle):
    # test_kkt.cpp:125-131
    p = synth.generate(0, seed=2, batch=1, N=32)
    sols = [oracle.solve_problem(p, P)[0] for P in (1, 2, 4, 8, 16)]
    for s in sols[1:]:
        assert rel_error(s, sols[0]).max() < 1e-12


def test_nu2_kats():
    # test_kkt.cpp:34-39
    assert kkt.nu2(1, 8) == 0 and kkt.nu2(4, 8) == 2
    assert kkt.nu2(0, 8) == 3 and kkt.nu2(6, 8) == 1


def test_oracle_reports_pivot_failure(oracle):
    p = synth.generate(0, seed=0, batch=2, N=16)
    p.R[1, 5] = -np.eye(p.nu) * 10.0  # indefinite stage Hessian in instance 1
    sol, rc, st = oracle.solve_problem(p, 4)
    assert rc == 2
    assert st[0].code == 0 and st[1].code == 2 and st[1].kind == 0


def test_generator_shapes_and_properties():
    p = synth.generate(1, seed=0, batch=2, N=8)
    assert p.A.shape == (2, 8, 20, 20) and p.S.shape == (2, 8, 10, 20)
    rho = np.abs(np.linalg.eigvals(p.A[0])).max(axis=1)
    assert np.allclose(rho, 0.95)
    # SPD stage Hessians
    H = np.block([[p.R[0, 3], p.S[0, 3]], [p.S[0, 3].T, p.Q[0, 3]]])
    assert np.linalg.eigvalsh(H).min() > 0
    # subsets are reproducible on their own
    q = synth.generate(1, seed=0, batch=1, N=8, start=1)
    assert np.array_equal(q.A[0], p.A[1])
