"""GPU parity tests: the sm_100a path (through the C ABI) against the
reference's golden outputs and the C oracle, on the reference's own test
properties:
  solution rel. error <= 1e-9 (||z_gpu - z_ref||_inf / max(1, ||z_ref||_inf))
  KKT residual (kkt_residual_eq, absolute inf-norm) <= 1e-10, except config 4
  whose Hessians reach 1e5 and where the reference itself exceeds 1e-10
  (BASELINE.md §4): there the scale-aware residual r / (max||H||*||z|| +
  ||rhs||) <= 1e-16 and r <= max(1e-10, 4 x the oracle's residual).
"""
import numpy as np
import pytest

import golden_util
from pyoracle import Oracle

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch, EqRhsBatch, kkt_residual, rel_error, residual_scale

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9
RES_TOL = 1e-10


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.mark.parametrize("name", golden_util.names())
def test_golden_reference_outputs(name):
    p, P, ref_sol, z = golden_util.load(name)
    tail = str(z["tail"]) if "tail" in z else "cr1"  # pcr / pcg fixtures: reference tails
    vlen = int(z["vlen"]) if "vlen" in z else 4
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P, tail=tail, vlen=vlen))
    err = rel_error(sol, ref_sol)
    assert err.max() <= REL_TOL, f"rel err {err.max():.3e}"
    res = kkt_residual(p, EqRhsBatch.of_problem(p), sol).max(axis=1)
    bound = np.maximum(RES_TOL, 4 * z["residual"]) if "qpalm" in name else RES_TOL
    assert np.all(res <= bound), f"residual {res.max():.3e}"
    assert np.array_equal(sol.x[:, 0], p.x_init)


@pytest.mark.parametrize("cfg,N,batch", [(0, None, 1), (1, None, 6), (2, None, 1),
                                         (3, 64, 2), (4, None, 3), (1, 40, 3)])
def test_configs_vs_oracle(oracle, cfg, N, batch):
    p = synth.generate(cfg, seed=11, batch=batch, N=N)
    P = synth.CONFIGS[cfg].P
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=P))
    ref, rc, _ = oracle.solve_problem(p, P)
    assert rc == 0
    assert rel_error(sol, ref).max() <= REL_TOL
    assert kkt_residual(p, EqRhsBatch.of_problem(p), sol).max() <= RES_TOL


def test_config4_newton_sequence(oracle):
    base = synth.generate(4, seed=5, batch=2, N=64)
    for p in synth.qpalm_sequence(base, seed=5, iters=3):
        sol = kkt.solve_problem(p, kkt.FactorOptions(P=16))
        ref, rc, _ = oracle.solve_problem(p, 16)
        assert rc == 0
        assert rel_error(sol, ref).max() <= REL_TOL
        rhs = EqRhsBatch.of_problem(p)
        r_gpu = kkt_residual(p, rhs, sol).max(axis=1)
        r_ref = kkt_residual(p, rhs, ref).max(axis=1)
        # Hessians reach ~1e5 here and the reference itself exceeds the
        # absolute 1e-10 bar: scale-aware residual
        # (SURVEY §7 hard part 6) plus the raw residual within a small
        # multiple of the oracle's own on the same instance.
        scale = residual_scale(p, rhs, sol)
        assert np.all(r_gpu / scale <= 1e-16)
        assert np.all(r_gpu <= np.maximum(RES_TOL, 4 * r_ref))


def test_zero_rhs_gives_exact_zero():
    # test_kkt.cpp:114-121
    p = synth.generate(0, seed=4, batch=2, N=16)
    f = kkt.factor(p, kkt.FactorOptions(P=4))
    s = kkt.solve(f, p, EqRhsBatch.zero(p))
    assert np.all(s.u == 0.0) and np.all(s.x[:, 1:] == 0.0) and np.all(s.lam == 0.0)


def test_factor_then_solve_matches_solve_problem(oracle):
    p = synth.generate(1, seed=6, batch=3, N=32)
    f = kkt.factor(p, kkt.FactorOptions(P=16))
    rhs = EqRhsBatch.of_problem(p)
    s1 = kkt.solve(f, p, rhs)
    s2 = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    assert rel_error(s1, s2).max() <= 1e-13
    # a different rhs with the same factor
    rng = np.random.default_rng(0)
    rhs2 = EqRhsBatch(rng.standard_normal(rhs.ru.shape), rng.standard_normal(rhs.qx.shape),
                      rng.standard_normal(rhs.fd.shape))
    s3 = kkt.solve(f, p, rhs2)
    ref, rc, _ = oracle.solve(p, rhs2, 16)
    assert rel_error(s3, ref).max() <= REL_TOL


def test_cross_P_consistency_and_determinism():
    # test_kkt.cpp:125-139
    p = synth.generate(0, seed=8, batch=2, N=64)
    sols = [kkt.solve_problem(p, kkt.FactorOptions(P=P)) for P in (1, 2, 4, 8, 16, 64)]
    for s in sols[1:]:
        assert rel_error(s, sols[0]).max() < 1e-8
    a = kkt.solve_problem(p, kkt.FactorOptions(P=4))
    b = kkt.solve_problem(p, kkt.FactorOptions(P=4))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(a, k), getattr(b, k))


def test_factor_blocks_match_oracle(oracle):
    # block-level parity on the reference's public Factor members
    for cfg, N, P in [(0, 64, 4), (1, 32, 16), (4, 32, 8)]:
        p = synth.generate(cfg, seed=9, batch=1, N=N)
        f = kkt.factor(p, kkt.FactorOptions(P=P))
        got = f.materialize(0)
        ref, rc, _ = oracle.factor_blocks(p, P)
        assert rc == 0
        for k in ("LH", "LB", "Acl", "LA"):
            scale = max(1.0, np.abs(ref[k]).max())
            assert np.abs(got[k] - ref[k]).max() <= 1e-11 * scale, k


def test_pivot_failure_is_per_instance():
    p = synth.generate(0, seed=0, batch=3, N=16)
    p.R[1, 5] = -10.0 * np.eye(p.nu)
    with pytest.raises(kkt.FactorizeError) as ei:
        kkt.solve_problem(p, kkt.FactorOptions(P=4))
    bad = ei.value.status
    assert [s.instance for s in bad] == [1]
    sol, rc, st = kkt.solve_problem(p, kkt.FactorOptions(P=4), raise_on_error=False)
    assert rc == 2 and st[0].code == 0 and st[2].code == 0
    good = p.subset([0, 2])
    ref = kkt.solve_problem(good, kkt.FactorOptions(P=4))
    assert rel_error(sol.__class__(sol.u[[0, 2]], sol.x[[0, 2]], sol.lam[[0, 2]]), ref).max() < 1e-13


def test_device_resident_inputs_match_host():
    import torch
    p = synth.generate(1, seed=12, batch=4, N=32)
    host = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    dev = kkt.EqOCPBatch.__new__(kkt.EqOCPBatch)
    for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
        setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
    sd = kkt.solve_problem(dev, kkt.FactorOptions(P=16))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(sd, k).cpu().numpy(), getattr(host, k))


def test_split_device_batch_matches_unsplit():
    # option split=2: a device batch as two halves on two streams (capi
    # split_device_pipeline) -- bit-identical to the single-stream launch
    import torch
    p = synth.generate(1, seed=13, batch=300, N=32)
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
    b = kkt.solve_problem(dev, kkt.FactorOptions(P=8))
    with kkt.Context.default().options(split=2):
        a = kkt.solve_problem(dev, kkt.FactorOptions(P=8))
    for k in ("u", "x", "lam"):
        assert torch.equal(getattr(a, k), getattr(b, k))
