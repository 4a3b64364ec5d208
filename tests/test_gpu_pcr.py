"""FactorOptions::tail = pcr on the GPU: cyclic reduction
down to min(P, vlen) Schur blocks, then parallel cyclic reduction of that
tail (block_tridiag.cpp:364-486 pcr_factor / PCRFactor::resolve, the tail
hand-off of kkt_factor.cpp:214-247 and kkt_solve.cpp:149-179), inside the
fused Schur kernel (schur_fused.cu; the 8-CTA cluster variant for a single
long horizon).

Checked against the reference's own pcr tail (oracle/_ref, set_tail("pcr"))
and its golden fixtures tests/golden/tail_pcr_*: solution rel. error <= 1e-9,
KKT residual <= 1e-10; and against the GPU's cr1 path within the
reference's own pcr-vs-cr1 bar (test_kkt.cpp:152-156: 1e-10).
"""
import numpy as np
import pytest

import golden_util
from pyoracle import RefOracle, ref_available

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9
RES_TOL = 1e-10


@pytest.mark.parametrize("name", [n for n in golden_util.names() if n.startswith("tail_pcr")])
def test_pcr_goldens(name):
    p, P, ref_sol, z = golden_util.load(name)
    opts = kkt.FactorOptions(P=P, tail="pcr", vlen=int(z["vlen"]))
    sol = kkt.solve_problem(p, opts)
    assert rel_error(sol, ref_sol).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL
    # the pcr path is a different algorithm from cr1: close, not the same bits
    cr1 = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    assert rel_error(sol, cr1).max() <= 1e-10
    assert any(not np.array_equal(getattr(sol, k), getattr(cr1, k)) for k in ("u", "x", "lam"))


# (cfg, N, batch, P, vlen): tails of 2..P blocks, all-PCR (vlen >= P), the
# cluster kernel (config 2 shape, one instance, P >= 64), every fused nx
CASES = [(1, 64, 3, 16, 2), (1, 64, 3, 16, 4), (1, 64, 2, 16, 16), (1, 64, 2, 16, 64),
         (4, 64, 2, 8, 4), (0, 64, 1, 4, 4), (0, 64, 1, 4, 2), (2, 1024, 1, 64, 8),
         (2, 4096, 1, 256, 8), (2, 4096, 1, 256, 64), (1, 128, 70, 16, 8)]


@pytest.mark.skipif(not ref_available(), reason="reference build unavailable")
@pytest.mark.parametrize("cfg,N,batch,P,vlen", CASES)
def test_pcr_vs_reference(cfg, N, batch, P, vlen):
    p = synth.generate(cfg, seed=41, batch=batch, N=N)
    ref = RefOracle()
    ref.set_tail("pcr")
    try:
        rsol, res, rc, _ = ref.solve_problem(p, P, vlen=vlen)
    finally:
        ref.set_tail("cr1")
    assert rc == 0
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P, tail="pcr", vlen=vlen))
    assert rel_error(sol, rsol).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL


@pytest.mark.parametrize("cfg,N,P,vlen", [(1, 64, 16, 4), (2, 4096, 256, 8), (1, 64, 16, 16)])
def test_pcr_factor_then_solve(cfg, N, P, vlen):
    # kkt::factor with the pcr tail, then kkt::solve (the resolve over the
    # stored PCR factor) with the problem's rhs and an independent one
    p = synth.generate(cfg, seed=42, batch=2 if cfg != 2 else 1, N=N)
    opts = kkt.FactorOptions(P=P, tail="pcr", vlen=vlen)
    f = kkt.factor(p, opts)
    s1 = kkt.solve(f, p, EqRhsBatch.of_problem(p))
    s2 = kkt.solve_problem(p, opts)
    assert rel_error(s1, s2).max() <= 1e-13
    rng = np.random.default_rng(8)
    rhs = EqRhsBatch.of_problem(p)
    rhs2 = EqRhsBatch(rng.standard_normal(rhs.ru.shape), rng.standard_normal(rhs.qx.shape),
                      rng.standard_normal(rhs.fd.shape))
    s3 = kkt.solve(f, p, rhs2)
    s4 = kkt.solve(kkt.factor(p, kkt.FactorOptions(P=P)), p, rhs2)
    assert rel_error(s3, s4).max() <= 1e-10
    z = kkt.solve(f, p, EqRhsBatch.zero(p))
    assert np.all(z.u == 0.0) and np.all(z.x[:, 1:] == 0.0) and np.all(z.lam == 0.0)


def test_pcr_pivot_failure_reported():
    # a negative-definite stage Hessian fails in the Riccati panel first;
    # the per-instance status and the other instances are unaffected
    p = synth.generate(1, seed=43, batch=3, N=32)
    p.R[1, 3] = -50.0 * np.eye(p.nu)
    sol, rc, st = kkt.solve_problem(p, kkt.FactorOptions(P=16, tail="pcr", vlen=4),
                                    raise_on_error=False)
    assert rc == 2 and st[1].code == 2 and st[0].code == 0 and st[2].code == 0
    good = kkt.solve_problem(p.subset([0, 2]), kkt.FactorOptions(P=16, tail="pcr", vlen=4))
    assert rel_error(sol.__class__(sol.u[[0, 2]], sol.x[[0, 2]], sol.lam[[0, 2]]), good).max() <= 1e-13
