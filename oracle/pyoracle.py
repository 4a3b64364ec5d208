"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the CPU checkers.

  Oracle()     -> oracle/liboracle.so      (plain-C restatement, "port")
  RefOracle()  -> oracle/_ref/libcyqref.so (the reference built from its own
                                            sources, "reference")

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product path never does. Both libraries are (re)built with
`make -C oracle` when missing and buildable (the reference only where
/root/reference exists; its .so travels to the GPU box prebuilt).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/proj"

i64 = C.c_int64
dp = C.POINTER(C.c_double)


class Dims(C.Structure):
    _fields_ = [("N", i64), ("nx", i64), ("nu", i64), ("P", i64), ("batch", i64)]


class Ocp(C.Structure):
    _fields_ = [(k, dp) for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init")]


class Rhs(C.Structure):
    _fields_ = [(k, dp) for k in ("ru", "qx", "fd")]


class Sol(C.Structure):
    _fields_ = [(k, dp) for k in ("u", "x", "lam")]


class FactorBlocks(C.Structure):
    _fields_ = [(k, dp) for k in ("LH", "LB", "Acl", "LA", "T", "Mfwd", "Mbwd", "W",
                                  "schur_diag", "schur_sub")]


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("kind", C.c_int32), ("instance", i64),
                ("column_or_level", i64), ("stage", i64), ("pivot", i64)]


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(dp)


def _dims(p, P):
    return Dims(p.N, p.nx, p.nu, P, p.batch)


def _ocp(p):
    return Ocp(*[_p(a) for a in p.arrays()])


def _sol_arrays(p):
    from paper_2512_09058_b200.ocp import EqSolutionBatch
    return EqSolutionBatch.empty(p.batch, p.N, p.nx, p.nu)


def _load(path, target):
    if not os.path.exists(path):
        r = subprocess.run(["make", "-C", HERE, target], capture_output=True, text=True)
        if r.returncode != 0 or not os.path.exists(path):
            raise RuntimeError(f"cannot build {path}: {r.stderr[-2000:]}")
    return C.CDLL(path)


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libcyqref.so")) or os.path.isdir(REF_SRC)


class _Base:
    prefix = ""

    def __init__(self, lib):
        self.lib = lib

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def kkt_residual(self, p, rhs, sol):
        out = np.zeros((p.batch, 4))
        f = self.fn("kkt_residual")
        f.restype = None
        f(C.byref(_dims(p, 1)), C.byref(_ocp(p)), C.byref(Rhs(*[_p(a) for a in rhs.arrays()])),
          C.byref(Sol(*[_p(a) for a in sol.arrays()])), _p(out))
        return out

    def fma_counts(self, N, nx, nu, P):
        out = (C.c_uint64 * 2)()
        f = self.fn("fma_counts")
        f.restype = None
        f(C.byref(Dims(N, nx, nu, P, 1)), out)
        return int(out[0]), int(out[1])


def _ls_arrays(alpha, delta, eta, beta):
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    eta = np.ascontiguousarray(eta, dtype=np.float64).reshape(-1)
    beta = np.ascontiguousarray(beta, dtype=np.float64).reshape(-1)
    return alpha.reshape(len(eta), -1), delta.reshape(len(eta), -1), eta, beta


class Oracle(_Base):
    """The plain-C restatement (oracle/cyq_oracle.c)."""

    prefix = "oc_"

    def __init__(self):
        super().__init__(_load(os.path.join(HERE, "liboracle.so"), "oracle"))
        self.lib.oc_bench_solve_problem.restype = C.c_double

    def solve_problem(self, p, P):
        sol = _sol_arrays(p)
        st = (Status * p.batch)()
        rc = self.lib.oc_solve_problem(C.byref(_dims(p, P)), C.byref(_ocp(p)),
                                       C.byref(Sol(*[_p(a) for a in sol.arrays()])), st)
        return sol, rc, list(st)

    def solve(self, p, rhs, P):
        sol = _sol_arrays(p)
        st = (Status * p.batch)()
        rc = self.lib.oc_solve(C.byref(_dims(p, P)), C.byref(_ocp(p)),
                               C.byref(Rhs(*[_p(a) for a in rhs.arrays()])),
                               C.byref(Sol(*[_p(a) for a in sol.arrays()])), st)
        return sol, rc, list(st)

    def factor_blocks(self, p, P):
        return _factor_blocks(self.lib.oc_factor_export, p, P, None)

    def line_search(self, alpha, delta, eta, beta):
        """tau[b], rc[b] of oc_line_search for a batch (alpha, delta: (b, m))."""
        alpha, delta, eta, beta = _ls_arrays(alpha, delta, eta, beta)
        tau, rc = np.zeros(len(eta)), np.zeros(len(eta), dtype=np.int32)
        t = C.c_double()
        for b in range(len(eta)):
            rc[b] = self.lib.oc_line_search(i64(alpha.shape[1]), _p(alpha[b]), _p(delta[b]),
                                            C.c_double(eta[b]), C.c_double(beta[b]), C.byref(t))
            tau[b] = t.value
        return tau, rc

    def bench_line_search(self, alpha, delta, eta, beta, threads):
        alpha, delta, eta, beta = _ls_arrays(alpha, delta, eta, beta)
        tau = np.zeros(len(eta))
        f = self.lib.oc_bench_line_search
        f.restype = C.c_double
        return f(i64(len(eta)), i64(alpha.shape[1]), _p(alpha), _p(delta), _p(eta), _p(beta),
                 _p(tau), C.c_int(threads))

    def bench(self, p, P, n_solves, threads):
        sol = _sol_arrays(p)
        return self.lib.oc_bench_solve_problem(
            C.byref(_dims(p, P)), C.byref(_ocp(p)), i64(n_solves), C.c_int(threads),
            C.byref(Sol(*[_p(a) for a in sol.arrays()])))


class RefOracle(_Base):
    """The reference's own sources (oracle/_ref/libcyqref.so)."""

    prefix = "ref_"

    def __init__(self):
        super().__init__(_load(os.path.join(HERE, "_ref", "libcyqref.so"), "ref"))
        self.lib.ref_bench_solve_problem.restype = C.c_double

    def set_tail(self, tail: str):
        """FactorOptions::tail of the following calls: cr1 | pcr | pcg."""
        self.lib.ref_set_tail(C.c_int({"cr1": 0, "pcr": 1, "pcg": 2}[tail]))

    def solve_problem(self, p, P, vlen=4, threads=1):
        sol = _sol_arrays(p)
        res = np.zeros(p.batch)
        st = (Status * p.batch)()
        rc = self.lib.ref_solve_problem(C.byref(_dims(p, P)), C.byref(_ocp(p)), i64(vlen),
                                        C.c_int(threads),
                                        C.byref(Sol(*[_p(a) for a in sol.arrays()])),
                                        _p(res), st)
        return sol, res, rc, list(st)

    def solve(self, p, rhs, P, vlen=4):
        sol = _sol_arrays(p)
        st = (Status * p.batch)()
        rc = self.lib.ref_solve(C.byref(_dims(p, P)), C.byref(_ocp(p)),
                                C.byref(Rhs(*[_p(a) for a in rhs.arrays()])), i64(vlen),
                                C.byref(Sol(*[_p(a) for a in sol.arrays()])), st)
        return sol, rc, list(st)

    def factor_blocks(self, p, P, vlen=4, cr=False):
        out, rc, st = _factor_blocks(self.lib.ref_factor_export, p, P, vlen)
        if cr and rc == 0:  # Factor::schur_cr (instance 0)
            nx = p.nx
            for k in ("cr_L", "cr_U", "cr_Y"):
                out[k] = np.zeros((max(P - 1, 0), nx, nx))
            out["cr_Lbase"] = np.zeros((nx, nx))
            st2 = Status()
            rc = self.lib.ref_factor_export_cr(C.byref(_dims(p, P)), C.byref(_ocp(p)), i64(vlen),
                                               *[_p(out[k]) for k in ("cr_L", "cr_U", "cr_Y", "cr_Lbase")],
                                               C.byref(st2))
        return out, rc, st

    def random_eq_ocp(self, N, nx, nu, seed, conditioning=10.0):
        from paper_2512_09058_b200.ocp import EqOCPBatch
        arrs = [np.zeros(s) for s in [(1, N, nx, nx), (1, N, nx, nu), (1, N, nu, nu),
                                      (1, N, nu, nx), (1, N + 1, nx, nx), (1, N, nx),
                                      (1, N, nu), (1, N + 1, nx), (1, nx)]]
        f = self.lib.ref_random_eq_ocp
        f.restype = None
        f(i64(N), i64(nx), i64(nu), C.c_uint64(seed), C.c_double(conditioning),
          *[_p(a) for a in arrs])
        return EqOCPBatch(*arrs)

    def line_search(self, alpha, delta, eta, beta):
        """tau[b], rc[b], iterations[b] of the reference's line_search_exact."""
        alpha, delta, eta, beta = _ls_arrays(alpha, delta, eta, beta)
        tau, rc = np.zeros(len(eta)), np.zeros(len(eta), dtype=np.int32)
        it = np.zeros(len(eta), dtype=np.int64)
        t, n = C.c_double(), i64()
        for b in range(len(eta)):
            rc[b] = self.lib.ref_line_search(i64(alpha.shape[1]), _p(alpha[b]), _p(delta[b]),
                                             C.c_double(eta[b]), C.c_double(beta[b]), C.byref(t),
                                             C.byref(n))
            tau[b], it[b] = t.value, n.value
        return tau, rc, it

    def bench_line_search(self, alpha, delta, eta, beta, threads):
        alpha, delta, eta, beta = _ls_arrays(alpha, delta, eta, beta)
        tau = np.zeros(len(eta))
        f = self.lib.ref_bench_line_search
        f.restype = C.c_double
        return f(i64(len(eta)), i64(alpha.shape[1]), _p(alpha), _p(delta), _p(eta), _p(beta),
                 _p(tau), C.c_int(threads))

    def update_solve(self, p_old, p_new, P, D, C, C_term, ds_stage, ds_term, rho=0.5):
        """kkt::factor(p_old) -> kkt::update -> kkt::solve(of_problem(p_new)) for
        instance 0. D (N, ny, nu), C (N, ny, nx), C_term (ny_term, nx),
        ds_stage (N, ny), ds_term (ny_term,). Returns (sol, rc, report[4])."""
        sol = _sol_arrays(p_new.subset(np.arange(1)) if p_new.batch > 1 else p_new)
        rep = np.zeros(4, dtype=np.int64)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (D, C, C_term, ds_stage, ds_term)]
        ny, ny_t = arrs[0].shape[1], arrs[2].shape[0]
        f = self.lib.ref_update_solve
        rc = f(C_dims(p_old, P), C_ocp(p_old), C_ocp(p_new),
               i64(ny), _p(arrs[0]), _p(arrs[1]), i64(ny_t), _p(arrs[2]), _p(arrs[3]), _p(arrs[4]),
               ctypes_double(rho), C_sol(sol), rep.ctypes.data_as(C_i64p))
        return sol, rc, rep

    def al_gradients(self, p, D, Cm, bl, bu, u, x, y, sigma, ubar, xbar, gamma_inv):
        """The reference's qpalm::eval_al_gradients (qpalm.cpp:106-165) per
        instance; arrays in the C ABI layout (see cyq_al_gradients_batch)."""
        b, N, nx, nu, ny = p.batch, p.N, p.nx, p.nu, D.shape[2]
        out = {"ru": np.zeros((b, N, nu)), "qx": np.zeros((b, N + 1, nx)),
               "yhat": np.zeros((b, N + 1, ny)), "cres": np.zeros((b, N, nx))}
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (D, Cm, bl, bu, u, x, y, sigma, ubar, xbar)]
        rc = self.lib.ref_al_gradients(C.byref(_dims(p, 1)), C.byref(_ocp(p)), i64(ny),
                                       *[_p(a) for a in arrs], C.c_double(gamma_inv),
                                       *[_p(out[k]) for k in ("ru", "qx", "yhat", "cres")])
        if rc != 0:
            raise RuntimeError("reference eval_al_gradients failed")
        return out

    def bench_latency(self, p, P, vlen, workers, reps):
        """Best single-instance factor+solve time (s) of instance 0 with
        FactorOptions{P, vlen, workers} over `reps` repetitions."""
        f = self.lib.ref_bench_latency
        f.restype = C.c_double
        return f(C.byref(_dims(p, P)), C.byref(_ocp(p)), i64(vlen), i64(workers), i64(reps))

    def bench(self, p, P, n_solves, threads, vlen=4):
        return self.lib.ref_bench_solve_problem(C.byref(_dims(p, P)), C.byref(_ocp(p)),
                                                i64(vlen), i64(n_solves), C.c_int(threads))


def C_dims(p, P):
    return C.byref(_dims(p, P))


def C_ocp(p):
    return C.byref(_ocp(p))


def C_sol(sol):
    return C.byref(Sol(*[_p(a) for a in sol.arrays()]))


C_i64p = C.POINTER(C.c_int64)
ctypes_double = C.c_double


def _factor_blocks(fn, p, P, vlen):
    N, nx, nu = p.N, p.nx, p.nu
    nux = nx + nu
    Np = P * ((N + P - 1) // P)
    n = Np // P
    out = {
        "LH": np.zeros((n, P, nux, nux)), "LB": np.zeros((n, P, nx, nu)),
        "Acl": np.zeros((n, P, nx, nx)), "LA": np.zeros((P, nx, nx)),
        "T": np.zeros((P, nx, nx)), "Mfwd": np.zeros((P, nx, nx)),
        "Mbwd": np.zeros((P, nx, nx)), "W": np.zeros((P, nx, nx)),
        "schur_diag": np.zeros((P, nx, nx)), "schur_sub": np.zeros((P, nx, nx)),
    }
    fb = FactorBlocks(*[_p(out[k]) for k, _ in FactorBlocks._fields_])
    st = Status()
    args = [C.byref(_dims(p, P)), C.byref(_ocp(p))]
    if vlen is not None:
        args.append(i64(vlen))
    rc = fn(*args, C.byref(fb), C.byref(st))
    return out, rc, st
