"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's dense
structural check of a factorization,
  factor_reconstruction_error (proj/tests/support/dense_ref.cpp:149-286):
build the permuted KKT matrix K (stage-wise u, x, interior multipliers per
partition column, then the P coupling multipliers ordered by increasing
2-adic valuation with index 0 last, dense_ref.cpp:160-172) and the block
lower factor L with signature D (+I on u / x, -I on interior and coupling
multipliers) from the factor blocks, and return ||L D L' - K||_F / ||K||_F.
The reference asserts < 1e-10 (test_kkt.cpp:66-103).

`blocks` holds the reference's public Factor members for one instance, as
paper_2512_09058_b200.kkt.Factor.materialize() / pyoracle.RefOracle.
factor_blocks(cr=True) return them: LH, LB, Acl (n, P, ...), LA, T (P, ...),
cr_L / cr_U / cr_Y (P-1, ...: level l slot mm at P - (P >> l) + mm), cr_Lbase.
The problem must not need padding (N a multiple of P).
"""
from __future__ import annotations

import numpy as np

from paper_2512_09058_b200.kkt import nu2


def _stage_of(c, s, n, Np):
    return (n * c - s) % Np


def factor_reconstruction_error(blocks, p, inst: int, P: int) -> float:
    nx, nu, N = p.nx, p.nu, p.N
    assert N % P == 0, "unpadded problems only"
    n = N // P
    Np = N
    col_sz = n * (nu + nx) + (n - 1) * nx
    dim = P * col_sz + P * nx

    def ubase(c, s):
        return c * col_sz + s * (nu + 2 * nx)

    def xbase(c, s):
        return ubase(c, s) + nu

    def lbase(c, t):
        return xbase(c, t) + nx

    lgP = 0
    while (1 << lgP) < P:
        lgP += 1
    pos = [0] * P
    at = 0
    for lv in range(lgP + 1):
        for i in range(1, P):
            if nu2(i, P) == lv:
                pos[i] = at
                at += 1
    pos[0] = at

    def cbase(i):
        return P * col_sz + pos[i] * nx

    A, B, R, S, Q = (getattr(p, k)[inst] for k in ("A", "B", "R", "S", "Q"))
    K = np.zeros((dim, dim))

    def put(r0, c0, blk, sym=True):
        K[r0:r0 + blk.shape[0], c0:c0 + blk.shape[1]] += blk
        if sym:
            K[c0:c0 + blk.shape[1], r0:r0 + blk.shape[0]] += blk.T

    I = np.eye(nx)
    for c in range(P):
        for s in range(n):
            j = _stage_of(c, s, n, Np)
            xi = j if j != 0 else Np
            Sj = np.zeros((nu, nx)) if j == 0 else S[j]
            K[ubase(c, s):ubase(c, s) + nu, ubase(c, s):ubase(c, s) + nu] = R[j]
            K[xbase(c, s):xbase(c, s) + nx, xbase(c, s):xbase(c, s) + nx] = Q[xi]
            put(ubase(c, s), xbase(c, s), Sj, False)
            K[xbase(c, s):xbase(c, s) + nx, ubase(c, s):ubase(c, s) + nu] = Sj.T
            if s + 1 < n:
                j2 = _stage_of(c, s + 1, n, Np)
                put(lbase(c, s), xbase(c, s), -I)
                put(lbase(c, s), ubase(c, s + 1), B[j2])
                put(lbase(c, s), xbase(c, s + 1), A[j2])
        j = _stage_of(c, 0, n, Np)
        put(cbase(c), ubase(c, 0), B[j])
        if j != 0:
            put(cbase(c), xbase(c, 0), A[j])
        put(cbase(c), xbase((c + 1) % P, n - 1), -I)

    L = np.zeros((dim, dim))
    D = np.ones(dim)
    for c in range(P):
        T = blocks["T"][c]
        for s in range(n):
            LH = blocks["LH"][s, c]
            LR, LS, LQ = LH[:nu, :nu], LH[nu:, :nu], LH[nu:, nu:]
            L[ubase(c, s):ubase(c, s) + nu, ubase(c, s):ubase(c, s) + nu] = LR
            L[xbase(c, s):xbase(c, s) + nx, ubase(c, s):ubase(c, s) + nu] = LS
            L[xbase(c, s):xbase(c, s) + nx, xbase(c, s):xbase(c, s) + nx] = LQ
            LQinvT = np.linalg.inv(LQ.T)
            if s + 1 < n:
                L[lbase(c, s):lbase(c, s) + nx, xbase(c, s):xbase(c, s) + nx] = -LQinvT
                L[lbase(c, s):lbase(c, s) + nx, lbase(c, s):lbase(c, s) + nx] = -LQinvT
                D[lbase(c, s):lbase(c, s) + nx] = -1
                j2 = _stage_of(c, s + 1, n, Np)
                BAt = np.vstack([B[j2].T, (A[j2].T if j2 != 0 else np.zeros((nx, nx)))])
                V = BAt @ LQ
                L[ubase(c, s + 1):ubase(c, s + 1) + nu, lbase(c, s):lbase(c, s) + nx] = V[:nu]
                L[xbase(c, s + 1):xbase(c, s + 1) + nx, lbase(c, s):lbase(c, s) + nx] = V[nu:]
                Acl = blocks["Acl"][s, c]
                L[cbase(c):cbase(c) + nx, xbase(c, s):xbase(c, s) + nx] = Acl @ LQinvT
                L[cbase(c):cbase(c) + nx, lbase(c, s):lbase(c, s) + nx] = Acl @ LQinvT
            else:
                L[cbase(c):cbase(c) + nx, xbase(c, s):xbase(c, s) + nx] = blocks["LA"][c]
                cp = (c - 1 + P) % P
                L[cbase(cp):cbase(cp) + nx, xbase(c, s):xbase(c, s) + nx] = -T
            L[cbase(c):cbase(c) + nx, ubase(c, s):ubase(c, s) + nu] = blocks["LB"][s, c]
    for lv in range(lgP):
        half = (P >> lv) // 2
        for mm in range(half):
            i = (2 * mm + 1) << lv
            a, b = i - (1 << lv), i + (1 << lv)
            slot = P - (P >> lv) + mm
            L[cbase(i):cbase(i) + nx, cbase(i):cbase(i) + nx] = blocks["cr_L"][slot]
            L[cbase(a):cbase(a) + nx, cbase(i):cbase(i) + nx] = blocks["cr_U"][slot]
            if b < P:
                L[cbase(b):cbase(b) + nx, cbase(i):cbase(i) + nx] = blocks["cr_Y"][slot]
    L[cbase(0):cbase(0) + nx, cbase(0):cbase(0) + nx] = blocks["cr_Lbase"]
    for i in range(P):
        D[cbase(i):cbase(i) + nx] = -1
    recon = (L * D) @ L.T
    return float(np.linalg.norm(recon - K) / np.linalg.norm(K))
