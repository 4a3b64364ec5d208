"""Shape sweep: the runtime-shape and specialised kernels over stage shapes
and horizons the BASELINE configs do not hit -- nx or nu of 1, odd sizes,
sizes straddling the 8-row DMMA tiles (7/8/9, 15/16/17, 33), horizons shorter
than P (every partition but one is padding, `pad_problem`,
`kkt_factor.cpp:30-47`) and N not a multiple of P -- each against the C
oracle (solution rel. error <= 1e-9, KKT residual <= 1e-10, the reference's
`test_kkt.cpp` bars).

The CPU half checks the oracle itself on the same cases (residual only), so
the GPU half compares against a checker that is known to solve them.
"""
import dataclasses

import numpy as np
import pytest

from pyoracle import Oracle

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqOCPBatch, EqRhsBatch, kkt_residual, rel_error

REL_TOL = 1e-9
RES_TOL = 1e-10

# (N, nx, nu, P, batch)
SHAPES = [
    (1, 3, 2, 1, 2), (1, 4, 4, 8, 1), (2, 1, 1, 2, 3), (3, 2, 5, 4, 2),
    (7, 7, 1, 4, 2), (9, 8, 8, 2, 2), (17, 9, 3, 4, 2), (33, 15, 9, 8, 1),
    (21, 16, 8, 16, 2), (40, 17, 7, 8, 1), (12, 24, 8, 4, 1), (10, 33, 5, 2, 1),
    (64, 5, 10, 64, 1), (50, 12, 4, 32, 2), (16, 40, 24, 4, 1), (8, 72, 8, 2, 1),
    (20, 64, 32, 4, 1),
]


def _problem(N, nx, nu, P, batch, seed=5):
    cfg = dataclasses.replace(synth.CONFIGS[0], N=N, nx=nx, nu=nu, P=P, batch=batch)
    cols = [[] for _ in range(9)]
    for i in range(batch):
        for c, v in zip(cols, synth._instance(cfg, N, seed + 1000 * nx + nu, i)[:9]):
            c.append(v)
    return EqOCPBatch(*[np.stack(c) for c in cols])


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.mark.parametrize("N,nx,nu,P,batch", SHAPES)
def test_oracle_solves_shape(oracle, N, nx, nu, P, batch):
    p = _problem(N, nx, nu, P, batch)
    ref, rc, _ = oracle.solve_problem(p, P)
    assert rc == 0
    assert kkt_residual(p, EqRhsBatch.of_problem(p), ref).max() <= RES_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("N,nx,nu,P,batch", SHAPES)
def test_gpu_shape_vs_oracle(oracle, N, nx, nu, P, batch):
    p = _problem(N, nx, nu, P, batch)
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    ref, rc, _ = oracle.solve_problem(p, P)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL
    assert np.array_equal(sol.x[:, 0], p.x_init)


@pytest.mark.gpu
@pytest.mark.parametrize("N,nx,nu,P", [(9, 96, 8, 4), (9, 84, 1, 16), (9, 87, 1, 1)])
def test_gpu_shape_beyond_envelope_is_rejected(N, nx, nu, P):
    """Shapes whose blocks exceed the kernels' shared memory fail up front
    with CYQ_INVALID_ARG (ValueError), as the reference's std::invalid_argument
    for bad options -- never a CUDA launch error."""
    p = _problem(N, nx, nu, P, 1)
    with pytest.raises(ValueError, match="too large"):
        kkt.solve_problem(p, kkt.FactorOptions(P=P))


@pytest.mark.gpu
@pytest.mark.parametrize("N,nx,nu,P,batch", SHAPES[::2] + [(16, 40, 8, 4, 1)])
def test_gpu_factor_solve_new_rhs_shape_vs_oracle(oracle, N, nx, nu, P, batch):
    """kkt::factor once, kkt::solve with an independent rhs (the forward
    sweep kernel) -- kkt_solve.cpp:23-309 -- on the same shape sweep."""
    p = _problem(N, nx, nu, P, batch)
    f = kkt.factor(p, kkt.FactorOptions(P=P))
    rng = np.random.default_rng(N * 100 + nx)
    rhs = EqRhsBatch(rng.standard_normal((batch, N, nu)), rng.standard_normal((batch, N + 1, nx)),
                     rng.standard_normal((batch, N, nx)))
    sol = kkt.solve(f, p, rhs)
    ref, rc, _ = oracle.solve(p, rhs, P)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, rhs, sol).max() <= RES_TOL
