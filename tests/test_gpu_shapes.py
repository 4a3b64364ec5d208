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
    # the CTA panel (nx = 64, nu = 32): one stage per chain, N < P (padding
    # chains), N not a multiple of P, a single chain, two stages
    (4, 64, 32, 4, 2), (3, 64, 32, 4, 1), (13, 64, 32, 4, 2), (6, 64, 32, 1, 1), (8, 64, 32, 4, 3),
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


# (N, nx, nu, ny, P): Newton-system assembly kernel (cyq_augment_hessians_batch)
NEWTON_SHAPES = [(5, 3, 1, 1, 2), (6, 1, 1, 5, 1), (9, 17, 9, 33, 4), (7, 40, 24, 64, 2),
                 (12, 8, 8, 8, 8), (10, 20, 10, 24, 4)]


@pytest.mark.gpu
@pytest.mark.parametrize("N,nx,nu,ny,P", NEWTON_SHAPES)
def test_gpu_newton_assembly_shapes(oracle, N, nx, nu, ny, P):
    """qpalm::assemble_newton (qpalm.cpp:184-221) on the GPU for stage shapes
    other than config 4's: Hessians vs the host construction, and the
    Newton solve vs the oracle on the host-assembled system."""
    import torch

    base = _problem(N, nx, nu, P, 2)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1, ny=ny)
    ref_p = next(synth.qpalm_sequence(base, seed=3, iters=1, ny=ny))
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
        setattr(dev, k, torch.from_numpy(np.ascontiguousarray(getattr(base, k))).cuda())
    Dd, Ed, sd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (D, E, sig[0]))
    aug = kkt.augment_hessians(dev, Dd, Ed, sd)
    for got, ref in ((aug.R, ref_p.R), (aug.S, ref_p.S), (aug.Q, ref_p.Q)):
        assert np.abs(got.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()
    sol = kkt.solve_newton(dev, Dd, Ed, sd, kkt.FactorOptions(P=P))
    ref, rc, _ = oracle.solve_problem(ref_p, P)
    assert rc == 0
    got = type(ref)(*[a.cpu().numpy() if hasattr(a, "cpu") else a for a in (sol.u, sol.x, sol.lam)])
    assert rel_error(got, ref).max() <= REL_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("nx,nu,ny", [(8, 4, 65), (40, 25, 8)])
def test_gpu_newton_assembly_beyond_envelope_is_rejected(nx, nu, ny):
    import torch

    base = _problem(4, nx, nu, 2, 1)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1, ny=ny)
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
        setattr(dev, k, torch.from_numpy(np.ascontiguousarray(getattr(base, k))).cuda())
    Dd, Ed, sd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (D, E, sig[0]))
    with pytest.raises(ValueError):
        kkt.augment_hessians(dev, Dd, Ed, sd)


@pytest.mark.gpu
def test_gpu_calls_follow_torch_current_stream():
    """Calls with CUDA torch tensors run on torch's current stream: inputs
    written by torch work still queued on that stream (behind a 20 ms sleep)
    are complete when the assembly kernel reads them, and the result is
    complete when torch reads it back on the same stream."""
    import torch

    base = _problem(6, 17, 9, 2, 2)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1, ny=33)
    ref_p = next(synth.qpalm_sequence(base, seed=3, iters=1, ny=33))
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
        setattr(dev, k, torch.from_numpy(np.ascontiguousarray(getattr(base, k))).cuda())
    src = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (D, E, sig[0])]
    dst = [torch.zeros_like(a) for a in src]
    kkt.augment_hessians(dev, *src)  # loads the kernel (a lazy module load synchronizes)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(40_000_000)  # ~20 ms of GPU time ahead of the copies
        for d, a in zip(dst, src):
            d.copy_(a, non_blocking=True)
        aug = kkt.augment_hessians(dev, *dst)
        R = aug.R.cpu()
    assert np.abs(R.numpy() - ref_p.R).max() <= 1e-13 * np.abs(ref_p.R).max()
    assert kkt.Context.default()._cur == s.cuda_stream
