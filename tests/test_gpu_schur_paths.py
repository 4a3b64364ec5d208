"""GPU parity of both Schur/CR implementations: the fused one-CTA-per-instance
kernel (schur_fused.cu, the default for batches >= 64) and the per-level
batch-wide kernels (schur_tiles.cu + schur_cr.cu, small batches), forced with
the context option `schur` ("auto" = fused, "levels"). Same bars as test_gpu_parity.py: solution rel. error
<= 1e-9 against the reference's golden outputs / the C oracle, KKT residual
<= 1e-10 (config 4: the scale-aware bound of test_gpu_parity.py).
"""
import numpy as np
import pytest

import golden_util
from pyoracle import Oracle

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9
RES_TOL = 1e-10
FUSED_NX = (10, 12, 16, 20)


@pytest.fixture
def schur_mode(request):
    with kkt.Context.default().options(schur="auto" if request.param == "fused" else request.param):
        yield request.param


GOLDEN_FUSED = [n for n in golden_util.names()
                if not n.startswith("kat_n16_nx3") and not n.startswith("kat_n8")
                and not n.startswith("kat_n5") and not n.startswith("kat_n13")]


@pytest.mark.parametrize("schur_mode", ["fused", "levels"], indirect=True)
@pytest.mark.parametrize("name", GOLDEN_FUSED)
def test_golden_both_schur_paths(schur_mode, name):
    p, P, ref_sol, z = golden_util.load(name)
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    assert rel_error(sol, ref_sol).max() <= REL_TOL
    res = kkt_residual(p, EqRhsBatch.of_problem(p), sol).max(axis=1)
    bound = np.maximum(RES_TOL, 4 * z["residual"]) if "qpalm" in name else RES_TOL
    assert np.all(res <= bound), f"residual {res.max():.3e}"


@pytest.mark.parametrize("schur_mode", ["fused"], indirect=True)
def test_fused_factor_then_solve(schur_mode):
    # kkt::solve over a stored factor: the solve-only branch of the fused
    # kernel (bwd_neg from the stored T, CR solve from the stored Linv/U/Y)
    oracle = Oracle()
    p = synth.generate(1, seed=21, batch=3, N=32)
    f = kkt.factor(p, kkt.FactorOptions(P=16))
    rhs = EqRhsBatch.of_problem(p)
    s1 = kkt.solve(f, p, rhs)
    s2 = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    assert rel_error(s1, s2).max() <= 1e-13
    rng = np.random.default_rng(3)
    rhs2 = EqRhsBatch(rng.standard_normal(rhs.ru.shape), rng.standard_normal(rhs.qx.shape),
                      rng.standard_normal(rhs.fd.shape))
    s3 = kkt.solve(f, p, rhs2)
    ref, rc, _ = oracle.solve(p, rhs2, 16)
    assert rc == 0
    assert rel_error(s3, ref).max() <= REL_TOL
    z = kkt.solve(f, p, EqRhsBatch.zero(p))
    assert np.all(z.u == 0.0) and np.all(z.x[:, 1:] == 0.0) and np.all(z.lam == 0.0)


@pytest.mark.parametrize("schur_mode", ["fused"], indirect=True)
@pytest.mark.parametrize("P", [1, 2, 4, 8, 32])
def test_fused_cross_P(schur_mode, P):
    # every CR depth, including P = 1 (base only) and P = 2 (one level)
    p = synth.generate(1, seed=22, batch=2, N=64)
    s = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    ref, rc, _ = Oracle().solve_problem(p, P)
    assert rc == 0
    assert rel_error(s, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), s).max() <= RES_TOL


def test_default_selection_large_batch_matches_oracle():
    # batch >= 64 selects the fused kernel without any override
    assert kkt.Context.default().get_option("schur") == 0
    p = synth.generate(1, seed=23, batch=64, N=32)
    s = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    ref, rc, _ = Oracle().solve_problem(p, 16)
    assert rc == 0
    assert rel_error(s, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), s).max() <= RES_TOL


@pytest.mark.parametrize("schur_mode", ["fused", "levels"], indirect=True)
def test_schur_paths_bitwise_deterministic(schur_mode):
    p = synth.generate(4, seed=24, batch=2, N=32)
    a = kkt.solve_problem(p, kkt.FactorOptions(P=8))
    b = kkt.solve_problem(p, kkt.FactorOptions(P=8))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(a, k), getattr(b, k))


@pytest.mark.parametrize("P", [64, 256, 512])
def test_cluster_schur_single_long_horizon(P):
    # one instance: the CR tree runs on a cluster of 8 CTAs (DSMEM solve
    # vectors, cluster barriers); must match the single-CTA kernel and the
    # C oracle
    N = 16 * P
    p = synth.generate(2, seed=31, batch=1, N=N)
    s_cl = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    with kkt.Context.default().options(schur_cluster=0):
        s_one = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    assert rel_error(s_cl, s_one).max() <= 1e-12
    ref, rc, _ = Oracle().solve_problem(p, P)
    assert rc == 0
    assert rel_error(s_cl, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), s_cl).max() <= RES_TOL
    # kkt::solve over the stored factor (solve-only branch on the cluster)
    f = kkt.factor(p, kkt.FactorOptions(P=P))
    s2 = kkt.solve(f, p, EqRhsBatch.of_problem(p))
    assert rel_error(s2, s_cl).max() <= 1e-13


@pytest.fixture(params=["warp", "two_warp"])
def riccati_mode(request):
    with kkt.Context.default().options(panel=request.param):
        yield request.param


@pytest.mark.parametrize("name", ["cfg0_N64_b1_P4", "cfg2_N512_b1_P128", "cfg1_N40_b3_P16",
                                  "cfg4_N64_b2_P16", "kat_n64_nx16_P4"])
def test_both_warp_panels_match_reference(riccati_mode, name):
    # single-warp panel (batches) and the two-warp producer/consumer panel
    # (the default for latency-bound launches of <= 2 chains per SM)
    p, P, ref_sol, z = golden_util.load(name)
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    assert rel_error(sol, ref_sol).max() <= REL_TOL
    res = kkt_residual(p, EqRhsBatch.of_problem(p), sol).max(axis=1)
    assert np.all(res <= RES_TOL)


def test_tmem_panel_variant_matches_oracle():
    # opt-in variant of the config-1 warp panel with W in tensor memory
    # (tcgen05.st / tcgen05.ld, 4 chains per CTA); a batch large enough for
    # the batched (non producer/consumer) path
    p = synth.generate(1, seed=8, batch=24, N=128)
    with kkt.Context.default().options(panel="warp_tmem"):
        sol = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    ref, rc, _ = Oracle().solve_problem(p, 16)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL
