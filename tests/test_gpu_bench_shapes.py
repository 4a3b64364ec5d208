"""GPU parity of exactly the kernel instantiations bench.py times, at the
BASELINE shapes and batch sizes that select them (VERDICT r1 "test what the
bench times"):

  config 1, batch > 4 x SMs   -> schur_fused_kernel<20, 2, 1> (2-warp CTAs)
  config 3, N = 512           -> riccati_cta_kernel<32, 64, 16>, schur_big,
                                 backsub_tile at 16 stages per column
  config 4, N = 256, fused    -> riccati_warp_kernel<8, 16, 1, 24> (Newton
                                 assembly fused into the panel)

Bars as in test_gpu_parity.py: solution rel. error <= 1e-9 against the C
oracle / the reference's golden outputs, KKT residual <= 1e-10 (config 4:
<= max(1e-10, 4 x the reference's own residual on the same system).
"""
import numpy as np
import pytest

import golden_util
from pyoracle import Oracle

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch, EqRhsBatch, EqSolutionBatch, kkt_residual, rel_error

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9
RES_TOL = 1e-10


def _dev(p):
    import torch
    d = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(d, k, torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda())
    return d


def _host(sol):
    return EqSolutionBatch(*[getattr(sol, k).cpu().numpy() for k in ("u", "x", "lam")])


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.fixture(scope="module")
def cfg1_big():
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    # one more instance than the 4-warp CTA slots: the default selection
    # takes the 2-warp fused Schur kernel, as the config-1 bench does
    return synth.generate(1, seed=17, batch=4 * sms + 8)


def test_config1_two_warp_schur_full_batch_vs_oracle(oracle, cfg1_big):
    p = cfg1_big
    ctx = kkt.Context.default()
    assert ctx.get_option("schur_warps") == 0  # automatic choice
    sol = _host(kkt.solve_problem(_dev(p), kkt.FactorOptions(P=16)))
    ref, rc, _ = oracle.solve_problem(p, 16)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL
    # forcing the 2-warp CTAs gives the same bits as the default choice
    with ctx.options(schur_warps=2):
        forced = _host(kkt.solve_problem(_dev(p), kkt.FactorOptions(P=16)))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(forced, k), getattr(sol, k))


@pytest.mark.parametrize("nx,nu", [(10, 5), (12, 4), (16, 8), (20, 10)])
def test_schur_two_vs_four_warps_each_nx(oracle, nx, nu):
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS[1], N=64, nx=nx, nu=nu, P=16, batch=64)
    cols = [[] for _ in range(9)]
    for i in range(cfg.batch):
        for c, v in zip(cols, synth._instance(cfg, cfg.N, 40 + nx, i)[:9]):
            c.append(v)
    p = EqOCPBatch(*[np.stack(c) for c in cols])
    ctx = kkt.Context.default()
    sols = {}
    for nw in (2, 4):
        with ctx.options(schur_warps=nw):
            sols[nw] = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    ref, rc, _ = oracle.solve_problem(p, 16)
    assert rc == 0
    for nw, s in sols.items():
        assert rel_error(s, ref).max() <= REL_TOL, nw
        assert kkt_residual(p, EqRhsBatch.of_problem(p), s).max() <= RES_TOL, nw
    # the CTA width changes the warp -> block assignment, not the arithmetic
    assert rel_error(sols[2], sols[4]).max() <= 1e-14


def test_config3_full_horizon_vs_oracle(oracle):
    # 16 stages per partition column (the bench's N = 512), two instances
    p = synth.generate(3, seed=23, batch=2)
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=32))
    ref, rc, _ = oracle.solve_problem(p, 32)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL


def test_config3_full_horizon_factor_solve_vs_oracle(oracle):
    # kkt::factor + kkt::solve with an independent rhs at the bench shape
    p = synth.generate(3, seed=24, batch=1)
    f = kkt.factor(p, kkt.FactorOptions(P=32))
    rng = np.random.default_rng(5)
    rhs = EqRhsBatch.of_problem(p)
    rhs2 = EqRhsBatch(rng.standard_normal(rhs.ru.shape), rng.standard_normal(rhs.qx.shape),
                      rng.standard_normal(rhs.fd.shape))
    s = kkt.solve(f, p, rhs2)
    ref, rc, _ = oracle.solve(p, rhs2, 32)
    assert rc == 0
    assert rel_error(s, ref).max() <= REL_TOL


@pytest.mark.parametrize("it", [0, 19])
def test_config4_fused_newton_N256_matches_reference(it):
    # golden: the reference's solution of iteration `it` of the config-4
    # Newton sequence at the bench horizon N = 256 (make_golden.py
    # --bench-shapes); here the GPU assembles it inside the panel kernel
    import torch
    p_ref, P, ref_sol, z = golden_util.load(f"cfg4_qpalm_N256_b1_P16_it{it}")
    base = synth.generate(4, seed=0, batch=1)
    D, E, sig = synth.qpalm_data(base, seed=0, iters=it + 1)
    ctx = kkt.Context.default()
    ctx.profile(True)
    ctx.profile_read(reset=True)
    sol = kkt.solve_newton(_dev(base), torch.from_numpy(D).cuda(), torch.from_numpy(E).cuda(),
                           torch.from_numpy(np.ascontiguousarray(sig[it])).cuda(),
                           kkt.FactorOptions(P=P), ctx=ctx)
    kern = ctx.profile_read(reset=True)
    ctx.profile(False)
    assert kern["augment"][1] == 0, "fused path expected (no assembly kernel)"
    host = _host(sol)
    assert rel_error(host, ref_sol).max() <= REL_TOL
    res = kkt_residual(p_ref, EqRhsBatch.of_problem(p_ref), host).max(axis=1)
    assert np.all(res <= np.maximum(RES_TOL, 4 * z["residual"]))


def test_config4_fused_newton_full_batch_vs_unfused():
    # the bench's 512-instance batch through the fused kernel against the
    # two-kernel path (assembly kernel + plain panel) on the same systems
    import torch
    base = synth.generate(4, seed=3, batch=512, N=64)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1)
    args = (_dev(base), torch.from_numpy(D).cuda(), torch.from_numpy(E).cuda(),
            torch.from_numpy(np.ascontiguousarray(sig[0])).cuda(), kkt.FactorOptions(P=16))
    ctx = kkt.Context.default()
    fused = _host(kkt.solve_newton(*args, ctx=ctx))
    with ctx.options(fused_augment=0):
        two = _host(kkt.solve_newton(*args, ctx=ctx))
    assert rel_error(fused, two).max() <= 1e-10


def test_config3_tma_staging_variant_matches_oracle(oracle):
    # opt-in CTA panel staging [B A] with TMA bulk copies (cp.async.bulk,
    # mbarrier complete_tx): same results as the cp.async default
    p = synth.generate(3, seed=25, batch=2)
    ctx = kkt.Context.default()
    with ctx.options(panel="cta_tma"):
        sol = kkt.solve_problem(p, kkt.FactorOptions(P=32))
    ref, rc, _ = oracle.solve_problem(p, 32)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    base = kkt.solve_problem(p, kkt.FactorOptions(P=32))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(sol, k), getattr(base, k))


def test_config3_pivot_failure_reported_by_the_pivot_warp():
    # the CTA panel's pivot warp owns every pivot check: an indefinite R at one
    # stage of one instance is reported for that instance, chain and stage only
    p = synth.generate(3, seed=31, batch=3, N=64)
    P, n = 4, 16                # 16 stages per chain
    j = 37                      # Partition::stage_of: stage n c - s -> chain 3, position 11
    c, spos = -(-j // n), n * -(-j // n) - j
    p.R[1, j] = -5.0 * np.eye(p.nu)
    sol, rc, st = kkt.solve_problem(p, kkt.FactorOptions(P=P), raise_on_error=False)
    assert rc == 2
    assert [s.code != 0 for s in st] == [False, True, False]
    assert (st[1].column_or_level, st[1].stage) == (c, spos) == (3, 11) and 0 <= st[1].pivot < p.nu
    good = p.subset([0, 2])
    ref = kkt.solve_problem(good, kkt.FactorOptions(P=P))
    got = sol.__class__(sol.u[[0, 2]], sol.x[[0, 2]], sol.lam[[0, 2]])
    assert rel_error(got, ref).max() < 1e-13
