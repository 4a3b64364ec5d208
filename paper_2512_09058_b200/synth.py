"""Seeded synthetic OCP instances for the five BASELINE.json configs.

No public benchmark suite is named by the reference for this path (the
paper's mass-spring set needs Eigen's matrix exponential, unbuildable here),
so these seeded generators with the BASELINE.json shapes and distributions
stand in for it (DESIGN.md §"Inputs"):

  Q_k = M M'/nx + I, R_k = L L'/nu + I  (M, L ~ N(0,1)),  S_k = 0
  A_k ~ N(0,1) rescaled to spectral radius 0.95, B_k ~ N(0, 1/nu)
  q_k, r_k, f_k ~ N(0,1), x0 ~ N(0,1)
  cfg 1: S_k ~ N(0, 0.01) and [R S; S' Q] += 2I
  cfg 3: Q_k, R_k += 2I
  cfg 4: ny = 24 rows D_k (ny x nu), E_k (ny x nx) ~ N(0,1); Newton-system
         Hessians R + D'ΣD, S + D'ΣE, Q + E'ΣE with Σ log-uniform in
         [1e-2, 1e4], ~30% of Σ redrawn per iteration (20 iterations).

Instance i of config c with seed s is drawn from its own stream
numpy.random.default_rng([s, c, i]), so any subset of a batch is
reproducible on its own (parity tests use small subsets of the full batch).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .ocp import EqOCPBatch


@dataclass(frozen=True)
class Config:
    idx: int
    N: int
    nx: int
    nu: int
    P: int
    batch: int
    name: str
    ny: int = 0
    iters: int = 1


CONFIGS = {
    0: Config(0, 64, 10, 5, 4, 1, "single OCP N=64 nx=10 nu=5 P=4"),
    1: Config(1, 128, 20, 10, 16, 1024, "batch 1024 N=128 nx=20 nu=10 P=16"),
    2: Config(2, 4096, 12, 4, 256, 1, "single long-horizon N=4096 nx=12 nu=4 P=256"),
    3: Config(3, 512, 64, 32, 32, 256, "batch 256 N=512 nx=64 nu=32 P=32"),
    # BASELINE.json leaves P open for config 4; P = 16 is recorded in DESIGN.md
    4: Config(4, 256, 16, 8, 16, 512, "QPALM batch 512 N=256 nx=16 nu=8 ny=24 x20", ny=24, iters=20),
}


def _spd(rng, batch, n):
    m = rng.standard_normal((batch, n, n))
    return m @ m.transpose(0, 2, 1) / n + np.eye(n)


def _instance(cfg: Config, N: int, seed: int, i: int):
    nx, nu = cfg.nx, cfg.nu
    rng = np.random.default_rng([seed, cfg.idx, i])
    Q = _spd(rng, N + 1, nx)
    R = _spd(rng, N, nu)
    A = rng.standard_normal((N, nx, nx))
    rho = np.abs(np.linalg.eigvals(A)).max(axis=1)
    A *= (0.95 / rho)[:, None, None]
    B = rng.standard_normal((N, nx, nu)) / np.sqrt(nu)
    S = np.zeros((N, nu, nx))
    if cfg.idx == 1:
        S = rng.standard_normal((N, nu, nx)) * 0.1
        R += 2 * np.eye(nu)
        Q += 2 * np.eye(nx)
    if cfg.idx == 3:
        R += 2 * np.eye(nu)
        Q += 2 * np.eye(nx)
    q = rng.standard_normal((N + 1, nx))
    r = rng.standard_normal((N, nu))
    f = rng.standard_normal((N, nx))
    x0 = rng.standard_normal(nx)
    return A, B, R, S, Q, f, r, q, x0, rng


def generate(cfg_idx: int, seed: int = 0, batch: int | None = None,
             N: int | None = None, start: int = 0) -> EqOCPBatch:
    """Instances start..start+batch-1 of config `cfg_idx` (horizon override
    `N` for reduced-size parity cases). Config 4 returns the base problems
    (before any Newton augmentation; see `qpalm_sequence`)."""
    cfg = CONFIGS[cfg_idx]
    batch = cfg.batch if batch is None else batch
    N = cfg.N if N is None else N
    cols = [[] for _ in range(9)]
    # instances are independent streams: drawn on a thread pool (LAPACK's
    # eigvals for the spectral-radius scaling dominates and releases the
    # GIL), one BLAS thread each; the values do not depend on the pool
    workers = min(batch, os.cpu_count() or 1) if batch * N * cfg.nx ** 3 > 1 << 24 else 1
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits
        with threadpool_limits(1), ThreadPoolExecutor(workers) as ex:
            insts = list(ex.map(lambda i: _instance(cfg, N, seed, i)[:9], range(start, start + batch)))
    else:
        insts = [_instance(cfg, N, seed, i)[:9] for i in range(start, start + batch)]
    for vals in insts:
        for c, v in zip(cols, vals):
            c.append(v)
    return EqOCPBatch(*[np.stack(c) for c in cols])


def qpalm_data(base: EqOCPBatch, seed: int = 0, iters: int = 20, ny: int = 24, start: int = 0):
    """Config 4 inputs of the Newton sequence: D (b, N, ny, nu), E (b, N+1,
    ny, nx) and the iters x (b, N+1, ny) Σ diagonals of `qpalm_sequence`
    (same random streams)."""
    b, N, nx, nu = base.batch, base.N, base.nx, base.nu
    rngs = [np.random.default_rng([seed, 4, start + i, 7]) for i in range(b)]
    D = np.stack([g.standard_normal((N, ny, nu)) for g in rngs])
    E = np.stack([g.standard_normal((N + 1, ny, nx)) for g in rngs])
    logs = np.stack([g.uniform(-2, 4, (N + 1, ny)) for g in rngs])
    sig = []
    for it in range(iters):
        if it > 0:
            for k, g in enumerate(rngs):
                mask = g.random((N + 1, ny)) < 0.3
                logs[k][mask] = g.uniform(-2, 4, int(mask.sum()))
        sig.append(10.0 ** logs)
    return D, E, np.stack(sig)


def qpalm_sequence(base: EqOCPBatch, seed: int = 0, iters: int = 20, ny: int = 24,
                   start: int = 0):
    """Config 4: yields `iters` augmented Newton systems per instance,
    mirroring qpalm::assemble_newton (qpalm.cpp:184-221) without Γ:
    R + D'ΣD, S + D'ΣE, Q + E'ΣE per stage; stage 0 takes the D part (its
    S and Q never enter the factorization), the terminal Q_N takes
    E_N'Σ_N E_N. About 30% of Σ is redrawn log-uniformly in [1e-2, 1e4]
    each iteration (active-set change)."""
    b, N, nx, nu = base.batch, base.N, base.nx, base.nu
    rngs = [np.random.default_rng([seed, 4, start + i, 7]) for i in range(b)]
    D = np.stack([g.standard_normal((N, ny, nu)) for g in rngs])
    E = np.stack([g.standard_normal((N + 1, ny, nx)) for g in rngs])
    logs = np.stack([g.uniform(-2, 4, (N + 1, ny)) for g in rngs])
    for it in range(iters):
        if it > 0:
            for k, g in enumerate(rngs):
                mask = g.random((N + 1, ny)) < 0.3
                logs[k][mask] = g.uniform(-2, 4, int(mask.sum()))
        sig = 10.0 ** logs
        DS = D * sig[:, :N, :, None]
        R = base.R + np.einsum("bjki,bjkl->bjil", DS, D)
        S = base.S + np.einsum("bjki,bjkl->bjil", DS, E[:, :N])
        ES = E * sig[..., None]
        Q = base.Q + np.einsum("bjki,bjkl->bjil", ES, E)
        yield EqOCPBatch(base.A, base.B, R, S, Q, base.f, base.r, base.q, base.x_init)


def line_search_data(batch: int, m: int, seed: int = 0, one_sided: float = 0.05,
                     zero_delta: float = 0.02):
    """Seeded exact-line-search instances with the reference test's
    distributions (test_line_search.cpp:17-31): eta ~ 2 U(0.1, 3), psi'(0+)
    ~ -5 U(0.1, 3) (descent at tau = 0), alpha, delta ~ N(0, 1); plus the
    QPALM cases add_term filters: infinite alpha (one-sided bounds,
    qpalm.cpp:285-296) and delta = 0. Returns alpha, delta (b, m), eta, beta (b,)."""
    rng = np.random.default_rng([seed, 5])
    eta = 2.0 * rng.uniform(0.1, 3.0, batch)
    beta = -5.0 * rng.uniform(0.1, 3.0, batch)
    alpha = rng.standard_normal((batch, m))
    delta = rng.standard_normal((batch, m))
    alpha[rng.random((batch, m)) < one_sided] = np.inf
    delta[rng.random((batch, m)) < zero_delta] = 0.0
    # a descent direction, as QPALM's Newton step is: shift beta by the terms
    # active at tau = 0+ so that psi'(0+) = -5 U(0.1, 3)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = alpha / delta
    keep = (delta != 0) & np.isfinite(t)
    w = np.where(keep, delta * np.abs(delta), 0.0)
    t = np.where(keep, t, 0.0)
    act0 = ((t <= 0) & (w > 0)) | ((t > 0) & (w < 0))
    beta = beta - np.sum(np.where(act0, -t * w, 0.0), axis=1)
    return alpha, delta, eta, beta
