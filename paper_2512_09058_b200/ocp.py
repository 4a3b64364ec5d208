"""Batched OCP data types: the reference's EqOCP / EqRhs / EqSolution
(proj/include/cyqlone/ocp.hpp:24-59) with a leading instance dimension.

Every array is C-contiguous float64, instance-major, stage-major, row-major
per block -- exactly the layout `include/cyqlone_b200.h` documents for the
C ABI, so a batch can be handed to the library (host or device) without any
repacking:

    A[b][N][nx][nx]   B[b][N][nx][nu]   R[b][N][nu][nu]   S[b][N][nu][nx]
    Q[b][N+1][nx][nx] f[b][N][nx]       r[b][N][nu]       q[b][N+1][nx]
    x_init[b][nx]
    rhs:  ru[b][N][nu]  qx[b][N+1][nx]  fd[b][N][nx]
    sol:  u[b][N][nu]   x[b][N+1][nx]   lam[b][N][nx]
"""
from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

OCP_FIELDS = ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init")
RHS_FIELDS = ("ru", "qx", "fd")
SOL_FIELDS = ("u", "x", "lam")


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class EqOCPBatch:
    """Equality-constrained LQ OCPs (ocp.hpp:24-38), batched."""

    A: np.ndarray
    B: np.ndarray
    R: np.ndarray
    S: np.ndarray
    Q: np.ndarray
    f: np.ndarray
    r: np.ndarray
    q: np.ndarray
    x_init: np.ndarray

    def __post_init__(self):
        for fld in fields(self):
            setattr(self, fld.name, _c(getattr(self, fld.name)))
        b, N, nx, _ = self.A.shape
        nu = self.B.shape[3]
        exp = {
            "A": (b, N, nx, nx), "B": (b, N, nx, nu), "R": (b, N, nu, nu),
            "S": (b, N, nu, nx), "Q": (b, N + 1, nx, nx), "f": (b, N, nx),
            "r": (b, N, nu), "q": (b, N + 1, nx), "x_init": (b, nx),
        }
        for k, shp in exp.items():
            if getattr(self, k).shape != shp:
                raise ValueError(f"EqOCPBatch.{k}: shape {getattr(self, k).shape} != {shp}")

    @property
    def batch(self) -> int:
        return self.A.shape[0]

    @property
    def N(self) -> int:
        return self.A.shape[1]

    @property
    def nx(self) -> int:
        return self.A.shape[2]

    @property
    def nu(self) -> int:
        return self.B.shape[3]

    def arrays(self):
        return [getattr(self, k) for k in OCP_FIELDS]

    def subset(self, idx) -> "EqOCPBatch":
        idx = np.atleast_1d(idx)
        return EqOCPBatch(*[getattr(self, k)[idx] for k in OCP_FIELDS])

    def nbytes(self) -> int:
        return sum(a.nbytes for a in self.arrays())


@dataclass
class EqRhsBatch:
    """Right-hand sides (ocp.hpp:45-53), batched."""

    ru: np.ndarray
    qx: np.ndarray
    fd: np.ndarray

    def __post_init__(self):
        for k in RHS_FIELDS:
            setattr(self, k, _c(getattr(self, k)))

    @staticmethod
    def zero(p: EqOCPBatch) -> "EqRhsBatch":
        return EqRhsBatch(np.zeros((p.batch, p.N, p.nu)),
                          np.zeros((p.batch, p.N + 1, p.nx)),
                          np.zeros((p.batch, p.N, p.nx)))

    @staticmethod
    def of_problem(p: EqOCPBatch) -> "EqRhsBatch":
        """EqRhs::of_problem (ocp.cpp:154-174): negated gradients with the
        eliminated initial state folded into ru[0] and fd[0]."""
        ru = -p.r.copy()
        fd = -p.f.copy()
        qx = -p.q.copy()
        qx[:, 0, :] = 0.0
        ru[:, 0, :] -= np.einsum("bij,bj->bi", p.S[:, 0], p.x_init)
        fd[:, 0, :] -= np.einsum("bij,bj->bi", p.A[:, 0], p.x_init)
        return EqRhsBatch(ru, qx, fd)

    def arrays(self):
        return [getattr(self, k) for k in RHS_FIELDS]


@dataclass
class EqSolutionBatch:
    """Solutions (ocp.hpp:55-59), batched; x[:, 0] = x_init."""

    u: np.ndarray
    x: np.ndarray
    lam: np.ndarray

    @staticmethod
    def empty(batch: int, N: int, nx: int, nu: int) -> "EqSolutionBatch":
        return EqSolutionBatch(np.zeros((batch, N, nu)),
                               np.zeros((batch, N + 1, nx)),
                               np.zeros((batch, N, nx)))

    def stacked(self) -> np.ndarray:
        """(batch, ·) stack of (u, x[1..N], lam) -- the parity vector."""
        b = self.u.shape[0]
        return np.concatenate([self.u.reshape(b, -1), self.x[:, 1:].reshape(b, -1),
                               self.lam.reshape(b, -1)], axis=1)

    def arrays(self):
        return [getattr(self, k) for k in SOL_FIELDS]


def rel_error(got: EqSolutionBatch, ref: EqSolutionBatch) -> np.ndarray:
    """Per-instance ||z_gpu - z_ref||_inf / max(1, ||z_ref||_inf) over the
    stacked (u, x[1..N], lam) -- SURVEY §8c parity protocol."""
    g, r = got.stacked(), ref.stacked()
    return np.abs(g - r).max(axis=1) / np.maximum(1.0, np.abs(r).max(axis=1))


def kkt_residual(p: EqOCPBatch, rhs: EqRhsBatch, s: EqSolutionBatch) -> np.ndarray:
    """Vectorised kkt_residual_eq (ocp.cpp:180-230): returns (batch, 4) of
    (stat_u, stat_x, dynamics, terminal) infinity norms."""
    u, x, lam = s.u, s.x, s.lam
    N = p.N
    # stationarity in u: R u + S x (j > 0) + B' lam - ru
    gu = np.einsum("bjik,bjk->bji", p.R, u) + np.einsum("bjki,bjk->bji", p.B, lam) - rhs.ru
    gu[:, 1:] += np.einsum("bjik,bjk->bji", p.S[:, 1:], x[:, 1:N])
    # dynamics: B u + A x (j > 0) - x_next - fd
    c = np.einsum("bjik,bjk->bji", p.B, u) - x[:, 1:] - rhs.fd
    c[:, 1:] += np.einsum("bjik,bjk->bji", p.A[:, 1:], x[:, 1:N])
    # stationarity in x, j = 1..N-1: S' u + Q x + A' lam - lam_prev - qx
    gx = (np.einsum("bjki,bjk->bji", p.S[:, 1:], u[:, 1:])
          + np.einsum("bjik,bjk->bji", p.Q[:, 1:N], x[:, 1:N])
          + np.einsum("bjki,bjk->bji", p.A[:, 1:], lam[:, 1:])
          - lam[:, :N - 1] - rhs.qx[:, 1:N])
    gt = np.einsum("bik,bk->bi", p.Q[:, N], x[:, N]) - lam[:, N - 1] - rhs.qx[:, N]
    out = np.zeros((p.batch, 4))
    out[:, 0] = np.abs(gu).reshape(p.batch, -1).max(axis=1)
    out[:, 1] = np.abs(gx).reshape(p.batch, -1).max(axis=1) if N > 1 else 0.0
    out[:, 2] = np.abs(c).reshape(p.batch, -1).max(axis=1)
    out[:, 3] = np.abs(gt).max(axis=1)
    return out


def residual_scale(p: EqOCPBatch, rhs: EqRhsBatch, s: EqSolutionBatch) -> np.ndarray:
    """Scale for the scale-aware residual (SURVEY §7 hard part 6):
    max_k ||H_k||_inf * ||z||_inf + ||rhs||_inf, per instance."""
    b = p.batch
    hn = np.maximum.reduce([
        np.abs(p.R).sum(-1).max(axis=(1, 2)) + np.abs(p.S).sum(-1).max(axis=(1, 2)),
        np.abs(p.Q).sum(-1).max(axis=(1, 2)) + np.abs(p.S).sum(-2).max(axis=(1, 2)),
        np.abs(p.A).sum(-1).max(axis=(1, 2)) + np.abs(p.B).sum(-1).max(axis=(1, 2)) + 1.0,
    ])
    zn = np.abs(s.stacked()).max(axis=1)
    rn = np.maximum.reduce([np.abs(a).reshape(b, -1).max(axis=1) for a in rhs.arrays()])
    return hn * zn + rn
