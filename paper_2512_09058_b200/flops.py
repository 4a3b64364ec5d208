"""Algorithmic FLOP counts of the KKT factor+solve, per instance.

Closed-form restatement of the reference's own multiply-add counter
(batla::flops, kernels.cpp:8-15): each kernel call of factor
(kkt_factor.cpp:109-247, block_tridiag.cpp:126-238) and solve
(kkt_solve.cpp:23-309) adds the same count the reference adds, so the totals
equal the reference's instrumented counts (pinned in tests/test_flops.py
against the C oracle, itself pinned against the reference build). FLOPs =
2 x FMA. Split by the phases each GPU kernel implements, for the per-kernel
roofline in bench.py.
"""
from __future__ import annotations


def _tri(n):
    return n * (n + 1) // 2


def _potrf(n):
    return n * (n + 1) * (n + 2) // 6


def _trsyrk(n):
    return sum((i + 1) * (n - i) for i in range(n))


def fma_phases(N: int, nx: int, nu: int, P: int) -> dict:
    nux = nx + nu
    Np = P * ((N + P - 1) // P)
    n = Np // P
    # ---- factor_lanes stage loop, per column (kkt_factor.cpp:125-158)
    ric = 0
    for s in range(n):
        if s > 0:
            ric += nx * _tri(nux)          # syrk V V'
        ric += _potrf(nux)                 # potrf
        ric += nx * _tri(nu)               # trsm LB
        ric += nx * nx * nu                # gemm Acl
        if s + 1 < n:
            ric += nx * nux * nx           # gemm hatBA
            ric += nux * _tri(nx)          # trmm V
        else:
            ric += nx * _tri(nx)           # trsm LA
    # ---- Schur contributions (kkt_factor.cpp:163-185)
    mfwd = n * nu * _tri(nx) + nx * _tri(nx)            # syrk LB, syrk LA
    tcoup = _potrf(nx) + _trsyrk(nx) + nx * _tri(nx)    # trtri, trsyrk, trmm W
    assemble = 2 * nx * nx                               # add_scaled x2 per column
    # ---- cyclic reduction factor (block_tridiag.cpp:126-238)
    cr = 0
    size = P
    while size > 1:
        half = size // 2
        for mm in range(half):
            k = 2 * mm + 1
            cr += _potrf(nx) + nx * _tri(nx)             # potrf, trsm U
            if k < size - 1:
                cr += nx * _tri(nx)                      # trsm Y
        for mm in range(half):
            cr += nx * _tri(nx)                          # syrk U
            if mm > 0:
                cr += nx * _tri(nx)                      # syrk Y
            if mm < half - 1:
                cr += nx * nx * nx                       # gemm K
        size = half
    cr += _potrf(nx)                                     # base
    # ---- forward substitution per column (kkt_solve.cpp:72-134)
    fwd = 0
    for s in range(n):
        fwd += _tri(nu) + nx * nu + _tri(nx)
        if s + 1 < n:
            fwd += _tri(nx) + nx + _tri(nx) + nu * nx + nx * nx
    for s in range(n):
        fwd += nx * nu
        if s + 1 < n:
            fwd += nx + _tri(nx) + nx * nx
        else:
            fwd += nx * nx
    bwdneg = _tri(nx)                                    # trmm T x
    # ---- CR forward/backward trsv (mat-vecs `mv` are not counted by the
    # reference, block_tridiag.cpp:18-27)
    crs = 0
    size = P
    while size > 1:
        crs += 2 * (size // 2) * _tri(nx)
        size //= 2
    crs += 2 * _tri(nx)
    # ---- back substitution per column (kkt_solve.cpp:193-266)
    bwd = 0
    for s in range(n):
        bwd += nu * nx
        if s + 1 < n:
            bwd += nx * nx + _tri(nx) + nx
        else:
            bwd += nx * nx + _tri(nx) + nx
    for s in range(n):
        if s + 1 < n:
            bwd += nu * nx + nx * nx + _tri(nx) + nx + _tri(nx) + _tri(nx) + nx
        bwd += _tri(nx) + nu * nx + _tri(nu)
    per = {
        "riccati": P * ric, "mfwd": P * mfwd, "schur_coupling": P * tcoup,
        "assemble": P * assemble, "cr_factor": cr,
        "forward_sweep": P * fwd, "bwd_neg": P * bwdneg, "cr_solve": crs,
        "back_substitution": P * bwd,
    }
    per["factor"] = (per["riccati"] + per["mfwd"] + per["schur_coupling"] + per["assemble"]
                     + per["cr_factor"])
    per["solve"] = per["forward_sweep"] + per["bwd_neg"] + per["cr_solve"] + per["back_substitution"]
    # phases implemented by each GPU kernel of the fused solve_problem path
    per["kernel_riccati_panel"] = per["riccati"] + per["mfwd"] + per["forward_sweep"]
    per["kernel_schur_cr"] = (per["schur_coupling"] + per["assemble"] + per["cr_factor"]
                              + per["bwd_neg"] + per["cr_solve"])
    per["kernel_backsub"] = per["back_substitution"]
    return per


def flops_per_solve(N: int, nx: int, nu: int, P: int) -> float:
    ph = fma_phases(N, nx, nu, P)
    return 2.0 * (ph["factor"] + ph["solve"])


def assembly_flops(N: int, nx: int, nu: int, ny: int) -> float:
    """Newton-system assembly of one instance (qpalm::assemble_newton,
    qpalm.cpp:184-221, equality part), symmetric blocks counted once:
    R_j + D_j' Σ D_j (lower), S_j + D_j' Σ C_j for j < N, Q_j + C_j' Σ C_j
    (lower) for 1 <= j <= N. FLOPs = 2 x FMA (the Σ scaling folded into
    the products, as the GPU kernels do)."""
    fma = N * (ny * _tri(nu) + ny * nu * nx) + N * ny * _tri(nx)
    return 2.0 * fma


def problem_bytes(N: int, nx: int, nu: int) -> int:
    """Compulsory input bytes of one EqOCP as the C ABI reads it (full
    row-major blocks; SURVEY §8d counts packed R, Q)."""
    return 8 * (N * nx * nx + N * nx * nu + N * nu * nu + N * nu * nx + (N + 1) * nx * nx
                + N * nx + N * nu + (N + 1) * nx + nx)


def solution_bytes(N: int, nx: int, nu: int) -> int:
    return 8 * (N * nu + (N + 1) * nx + N * nx)
