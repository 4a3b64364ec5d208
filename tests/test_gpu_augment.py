"""Newton-system assembly on the GPU (cyq_augment_hessians_batch, restating
qpalm::assemble_newton, qpalm.cpp:167-225, equality part) for BASELINE
config 4: the augmented Hessians match the host construction of
synth.qpalm_sequence to 1e-13 (relative), and solving the GPU-augmented
Newton systems reproduces the reference's golden outputs for the same
systems (tests/golden/cfg4_qpalm_*) and the C oracle."""
import numpy as np
import pytest

import golden_util
from pyoracle import Oracle

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch, EqRhsBatch, kkt_residual, rel_error

pytestmark = pytest.mark.gpu


def _dev(p):
    import torch
    d = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(d, k, torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda())
    return d


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("gamma_inv", [0.0, 0.25])
def test_augmented_hessians_match_host(gamma_inv):
    base = synth.generate(4, seed=7, batch=3, N=32)
    D, E, sig = synth.qpalm_data(base, seed=7, iters=3)
    seq = list(synth.qpalm_sequence(base, seed=7, iters=3))
    pd = _dev(base)
    for it in range(3):
        out = kkt.augment_hessians(pd, _t(D), _t(E), _t(sig[it]), gamma_inv=gamma_inv)
        R = seq[it].R + gamma_inv * np.eye(base.nu)
        Q = seq[it].Q + gamma_inv * np.eye(base.nx)
        Q[:, 0] -= gamma_inv * np.eye(base.nx)  # gamma^-1 I for stages j >= 1 only
        for got, ref in ((out.R, R), (out.S, seq[it].S), (out.Q, Q)):
            g = got.cpu().numpy()
            assert np.abs(g - ref).max() <= 1e-13 * np.abs(ref).max()
        for k in ("A", "B", "f", "r", "q", "x_init"):
            assert getattr(out, k) is getattr(pd, k)


@pytest.mark.parametrize("it", [0, 1])
def test_gpu_newton_systems_reproduce_reference(it):
    # the golden fixtures cfg4_qpalm_N64_b2_P16_it{0,1} hold the reference's
    # solutions of the host-assembled Newton systems of make_golden.py
    # (base = config 4 at N = 64, batch 2, seed 0; qpalm_sequence seed 0)
    p_ref, P, ref_sol, z = golden_util.load(f"cfg4_qpalm_N64_b2_P16_it{it}")
    base = synth.generate(4, seed=0, batch=2, N=64)
    for k in ("A", "B", "f", "r", "q", "x_init"):
        assert np.array_equal(getattr(base, k), getattr(p_ref, k))
    D, E, sig = synth.qpalm_data(base, seed=0, iters=it + 1)
    aug = kkt.augment_hessians(_dev(base), _t(D), _t(E), _t(sig[it]))
    for k in ("R", "S", "Q"):
        g, r = getattr(aug, k).cpu().numpy(), getattr(p_ref, k)
        assert np.abs(g - r).max() <= 1e-13 * np.abs(r).max()
    sol = kkt.solve_problem(aug, kkt.FactorOptions(P=P))
    host = kkt.EqSolutionBatch(*[getattr(sol, k).cpu().numpy() for k in ("u", "x", "lam")])
    assert rel_error(host, ref_sol).max() <= 1e-9
    rhs = EqRhsBatch.of_problem(p_ref)
    res = kkt_residual(p_ref, rhs, host).max(axis=1)
    assert np.all(res <= np.maximum(1e-10, 4 * z["residual"]))


def test_twenty_iteration_loop_matches_oracle():
    base = synth.generate(4, seed=9, batch=2, N=32)
    D, E, sig = synth.qpalm_data(base, seed=9, iters=20)
    pd, Dd, Ed = _dev(base), _t(D), _t(E)
    seq = list(synth.qpalm_sequence(base, seed=9, iters=20))
    orc = Oracle()
    out = None
    for it in (0, 7, 19):
        out = kkt.augment_hessians(pd, Dd, Ed, _t(sig[it]), out=out)
        sol = kkt.solve_problem(out, kkt.FactorOptions(P=16))
        host = kkt.EqSolutionBatch(*[getattr(sol, k).cpu().numpy() for k in ("u", "x", "lam")])
        ref, rc, _ = orc.solve_problem(seq[it], 16)
        assert rc == 0
        assert rel_error(host, ref).max() <= 1e-9


def _host(sol):
    return kkt.EqSolutionBatch(*[getattr(sol, k).cpu().numpy() for k in ("u", "x", "lam")])


@pytest.mark.parametrize("gamma_inv", [0.0, 0.25])
def test_fused_newton_matches_assembly_kernel_path(gamma_inv):
    # kkt.solve_newton fuses the assembly into the stage-panel loads at the
    # config-4 stage shape; it must agree with assembly kernel + solve_problem
    base = synth.generate(4, seed=11, batch=3, N=32)
    D, E, sig = synth.qpalm_data(base, seed=11, iters=2)
    pd, Dd, Ed = _dev(base), _t(D), _t(E)
    ctx = kkt.Context.default()
    for it in range(2):
        ctx.profile(True)
        ctx.profile_read(reset=True)
        fused = kkt.solve_newton(pd, Dd, Ed, _t(sig[it]), kkt.FactorOptions(P=16), gamma_inv=gamma_inv)
        kern = ctx.profile_read(reset=True)
        ctx.profile(False)
        assert kern["augment"][1] == 0  # no separate assembly kernel ran
        aug = kkt.augment_hessians(pd, Dd, Ed, _t(sig[it]), gamma_inv=gamma_inv)
        two = kkt.solve_problem(aug, kkt.FactorOptions(P=16))
        hf, h2 = _host(fused), _host(two)
        assert rel_error(hf, h2).max() <= 1e-12
        p_aug = EqOCPBatch(*[getattr(aug, k).cpu().numpy() for k in OCP_FIELDS])
        rhs = EqRhsBatch.of_problem(p_aug)
        res_f = kkt_residual(p_aug, rhs, hf).max(axis=1)
        res_2 = kkt_residual(p_aug, rhs, h2).max(axis=1)
        assert np.all(res_f <= np.maximum(1e-10, 4 * res_2))


@pytest.mark.parametrize("it", [0, 1])
def test_fused_newton_reproduces_reference(it):
    p_ref, P, ref_sol, z = golden_util.load(f"cfg4_qpalm_N64_b2_P16_it{it}")
    base = synth.generate(4, seed=0, batch=2, N=64)
    D, E, sig = synth.qpalm_data(base, seed=0, iters=it + 1)
    sol = kkt.solve_newton(_dev(base), _t(D), _t(E), _t(sig[it]), kkt.FactorOptions(P=P))
    host = _host(sol)
    assert rel_error(host, ref_sol).max() <= 1e-9
    res = kkt_residual(p_ref, EqRhsBatch.of_problem(p_ref), host).max(axis=1)
    assert np.all(res <= np.maximum(1e-10, 4 * z["residual"]))


def test_newton_other_shape_uses_assembly_kernel():
    # no fused variant for the config-1 stage shape: assembly kernel + pipeline
    base = synth.generate(1, seed=5, batch=2, N=32)
    D, E, sig = synth.qpalm_data(base, seed=5, iters=1, ny=12)
    pd = _dev(base)
    got = _host(kkt.solve_newton(pd, _t(D), _t(E), _t(sig[0]), kkt.FactorOptions(P=8)))
    aug = kkt.augment_hessians(pd, _t(D), _t(E), _t(sig[0]))
    ref = _host(kkt.solve_problem(aug, kkt.FactorOptions(P=8)))
    for k in ("u", "x", "lam"):
        assert np.array_equal(getattr(got, k), getattr(ref, k))


def test_fused_newton_P_invariance():
    base = synth.generate(4, seed=3, batch=2, N=64)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1)
    pd, Dd, Ed, sd = _dev(base), _t(D), _t(E), _t(sig[0])
    a = _host(kkt.solve_newton(pd, Dd, Ed, sd, kkt.FactorOptions(P=16)))
    b = _host(kkt.solve_newton(pd, Dd, Ed, sd, kkt.FactorOptions(P=4)))
    assert rel_error(a, b).max() <= 1e-8
