"""QPALM augmented-Lagrangian gradients on the GPU (SURVEY §8f row f2,
qpalm::eval_al_gradients, qpalm.cpp:106-165) against the reference's own
function (oracle/_ref compiles qpalm.cpp): yhat, ru, qx, cres within 1e-12
relative, at the config-4 shape (nx 16, nu 8, ny 24) with a mix of active /
inactive / two-sided bounds, and at other shapes; plus a Newton step built
from them (qpalm.cpp:391-405) through the GPU factor + solve."""
import numpy as np
import pytest

from pyoracle import RefOracle, ref_available

from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch, EqSolutionBatch, rel_error

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="reference build unavailable")]


def _state(p, ny, seed):
    rng = np.random.default_rng(seed)
    b, N, nx, nu = p.batch, p.N, p.nx, p.nu
    D = rng.standard_normal((b, N, ny, nu))
    Cm = rng.standard_normal((b, N + 1, ny, nx))
    lo = rng.uniform(-2, 0, (b, N + 1, ny))
    hi = lo + rng.uniform(0, 3, (b, N + 1, ny))
    lo[..., ::5] = -np.inf  # one-sided rows
    hi[..., 1::7] = np.inf
    u = rng.standard_normal((b, N, nu))
    x = rng.standard_normal((b, N + 1, nx))
    x[:, 0] = p.x_init
    y = rng.standard_normal((b, N + 1, ny))
    sigma = 10.0 ** rng.uniform(-2, 4, (b, N + 1, ny))
    ubar = u + 0.1 * rng.standard_normal(u.shape)
    xbar = x + 0.1 * rng.standard_normal(x.shape)
    return D, Cm, lo, hi, u, x, y, sigma, ubar, xbar


def _dev(p):
    import torch
    d = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(d, k, torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda())
    return d


@pytest.mark.parametrize("cfg,N,batch,ny,nx,nu", [(4, 64, 3, 24, None, None), (4, 256, 2, 24, None, None),
                                                  (1, 32, 2, 7, None, None), (0, 16, 2, 40, 33, 9)])
def test_al_gradients_match_reference(cfg, N, batch, ny, nx, nu):
    import dataclasses
    import torch
    if nx is None:
        p = synth.generate(cfg, seed=61, batch=batch, N=N)
    else:
        c = dataclasses.replace(synth.CONFIGS[cfg], N=N, nx=nx, nu=nu, batch=batch)
        cols = list(zip(*[synth._instance(c, N, 61, i)[:9] for i in range(batch)]))
        p = EqOCPBatch(*[np.stack(v) for v in cols])
    st = _state(p, ny, 62)
    gamma_inv = 1e-7
    ref = RefOracle().al_gradients(p, *st, gamma_inv)
    got = kkt.al_gradients(_dev(p), *[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in st],
                           gamma_inv)
    for k in ("yhat", "ru", "qx", "cres"):
        g = got[k].cpu().numpy()
        scale = max(1.0, np.abs(ref[k]).max())
        assert np.abs(g - ref[k]).max() <= 1e-12 * scale, k


def test_newton_step_from_gradients():
    # qpalm.cpp:391-405: rhs = -(ru, qx, cres) solved with the Newton
    # system's factor; on the GPU: gradients -> rhs -> factor + solve
    import torch
    from pyoracle import Oracle
    p = synth.generate(4, seed=63, batch=2, N=64)
    st = _state(p, 24, 64)
    got = kkt.al_gradients(_dev(p), *[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in st], 1e-7)
    rhs = kkt.newton_rhs(got)
    f = kkt.factor(_dev(p), kkt.FactorOptions(P=16))
    step = kkt.solve(f, _dev(p), rhs)
    hrhs = kkt.EqRhsBatch(*[np.ascontiguousarray(a.cpu().numpy()) for a in (rhs.ru, rhs.qx, rhs.fd)])
    ref, rc, _ = Oracle().solve(p, hrhs, 16)
    assert rc == 0
    host = EqSolutionBatch(*[getattr(step, k).cpu().numpy() for k in ("u", "x", "lam")])
    assert rel_error(host, ref).max() <= 1e-9
