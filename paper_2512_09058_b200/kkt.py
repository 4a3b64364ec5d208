"""Python mirror of the reference's KKT interface (cyqlone::kkt,
proj/include/cyqlone/kkt_solver.hpp:45-128) over the C ABI.

    factor(p, opts)          -> Factor             kkt::factor      (kkt_factor.cpp:251-313)
    solve(f, p, rhs)         -> EqSolutionBatch    kkt::solve       (kkt_solve.cpp:23-309)
    solve_problem(p, opts)   -> EqSolutionBatch    kkt::solve_problem (kkt_solve.cpp:311-317)

Same names, argument meaning and error behaviour as the reference:
`ValueError` for what the reference throws as std::invalid_argument (P not a
power of two) and `FactorizeError(batch_index, pivot)` for
batla::factorize_error. Problems are batches (`EqOCPBatch`, a leading
instance axis; a single reference EqOCP is a batch of one). Arrays may be
host numpy arrays or CUDA torch tensors (device-resident, zero-copy).
`opts.workers` is a CPU thread knob of the reference, accepted with no effect
on the GPU (results are independent of it in the reference too,
test_kkt.cpp:133-138). `opts.tail = "pcr"` solves the last min(P, vlen)
Schur blocks by parallel cyclic reduction on the GPU (the fused Schur
kernel's shapes); "pcg" -- and "pcr" at other shapes -- is served by the
exact cyclic reduction of the whole tree, within the tails' accuracy
contracts (test_kkt.cpp:152-161).

Beyond the three reference calls: `update` (kkt::update, in place on the
GPU factor), `Factor.materialize`, the QPALM steps `solve_newton`,
`augment_hessians`, `al_gradients` / `newton_rhs` and `line_search_exact`,
and `Prepared` calls for device-resident loops.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from ctypes import byref as _byref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .ocp import OCP_FIELDS, RHS_FIELDS, SOL_FIELDS, EqOCPBatch, EqRhsBatch, EqSolutionBatch


class FactorizeError(RuntimeError):
    """batla::factorize_error (kernels.hpp:11-16): pivot failure."""

    def __init__(self, what, batch_index, pivot, status=None):
        super().__init__(what)
        self.batch_index = batch_index
        self.pivot = pivot
        self.status = status


class CudaError(RuntimeError):
    pass


@dataclass
class FactorOptions:
    """kkt::FactorOptions (kkt_solver.hpp:47-57)."""

    P: int = 1
    vlen: int = 4
    workers: int = 1
    tail: str = "cr1"
    pcg_tol: float = 1e-12
    pcg_max_iter: int = 50
    rho: float = 0.5


def nu2(i: int, P: int) -> int:
    """2-adic valuation with nu2(0, P) = nu2(P) (kkt_factor.cpp:15-25)."""
    if not (0 <= i < P):
        raise ValueError("nu2: i out of range")
    if i == 0:
        i = P
    v = 0
    while i & 1 == 0:
        i >>= 1
        v += 1
    return v


class Context:
    """One CUDA context handle per device (cyq_ctx)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.cyq_ctx_create(device, C.byref(h))
        if rc != _lib.CYQ_OK:
            raise CudaError(f"cyq_ctx_create failed ({rc}): "
                            f"{self.lib.cyq_ctx_last_error(None).decode()}")
        self.h = h
        self.device = device
        self._bound = False  # set_stream() called: keep the caller's stream
        self._cur = None
        self._tail = ("cr1", 4)  # FactorOptions tail / vlen last applied

    def follow_torch(self, arrays):
        """Stream ordering with torch: unless the caller bound a stream with
        set_stream(), calls that take CUDA torch tensors run on torch's current
        stream of this device, so inputs produced by earlier torch work are
        complete and results are ordered before later torch work."""
        if self._bound or not any(_is_torch(a) for a in arrays):
            return
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream or 1  # 1 = cudaStreamLegacy
        if s != self._cur:
            self.lib.cyq_ctx_set_stream(self.h, C.c_void_p(s))
            self._cur = s

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def set_option(self, name: str, value):
        """Kernel selection (cyq_ctx_set_option): name in _lib.OPTIONS, value
        an int or one of the names in _lib.OPTION_VALUES[name]."""
        v = _lib.OPTION_VALUES.get(name, {}).get(value, value) if isinstance(value, str) else value
        rc = self.lib.cyq_ctx_set_option(self.h, _lib.OPTIONS[name], int(v))
        if rc != _lib.CYQ_OK:
            raise ValueError(self.last_error())

    def get_option(self, name: str) -> int:
        v = C.c_int64()
        rc = self.lib.cyq_ctx_get_option(self.h, _lib.OPTIONS[name], C.byref(v))
        if rc != _lib.CYQ_OK:
            raise ValueError(self.last_error())
        return v.value

    @contextlib.contextmanager
    def options(self, **kw):
        """Temporarily set kernel-selection options: `with ctx.options(schur="levels"): ...`"""
        old = {k: self.get_option(k) for k in kw}
        try:
            for k, v in kw.items():
                self.set_option(k, v)
            yield self
        finally:
            for k, v in old.items():
                self.set_option(k, v)

    def wait_status(self, batch: int, raise_on_error: bool = True):
        """With the `async_status` option: wait for the context stream and
        decode the most recent device call's per-instance status (raises
        FactorizeError like a synchronous call unless raise_on_error=False;
        then returns (rc, status list))."""
        st = (_lib.CyqStatus * batch)()
        rc = self.lib.cyq_ctx_wait_status(self.h, st, batch)
        if raise_on_error:
            _raise_status(self, rc, st)
            return None
        return rc, list(st)

    def last_error(self) -> str:
        return self.lib.cyq_ctx_last_error(self.h).decode()

    def set_stream(self, stream_ptr: int | None):
        """Bind the context to a CUDA stream handle (0, as torch reports its
        default stream: the legacy default stream) or None (a private
        non-blocking stream); either way it stops following torch's current
        stream."""
        h = None if stream_ptr is None else (stream_ptr or 1)  # 1 = cudaStreamLegacy
        self.lib.cyq_ctx_set_stream(self.h, C.c_void_p(h))
        self._bound, self._cur = True, h

    def synchronize(self):
        self.lib.cyq_ctx_synchronize(self.h)

    KERNELS = ("riccati_panel", "schur_cr", "backsub", "forward_sweep", "augment")

    def profile(self, enable: bool = True):
        self.lib.cyq_ctx_profile(self.h, int(enable))

    def profile_read(self, reset: bool = True):
        ms = (C.c_double * 5)()
        n = (C.c_int64 * 5)()
        self.lib.cyq_ctx_profile_read(self.h, ms, n, int(reset))
        return {k: (ms[i], n[i]) for i, k in enumerate(self.KERNELS)}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.cyq_ctx_destroy(self.h)
        except Exception:
            pass


_F64 = np.dtype(np.float64)


def _is_torch(a) -> bool:
    return not isinstance(a, np.ndarray) and type(a).__module__.startswith("torch")


def _ptr(a) -> int:
    """Address of a contiguous float64 array (every ABI pointer parameter is
    declared c_void_p in _lib.SIGNATURES, so a plain int converts)."""
    if isinstance(a, np.ndarray):
        assert a.dtype == _F64 and a.flags.c_contiguous
        return a.ctypes.data
    assert a.is_cuda and a.is_contiguous() and a.dtype == _torch().float64
    return a.data_ptr()


def _torch():
    import torch
    return torch


def _mem(arrs) -> int:
    kinds = {_is_torch(a) for a in arrs}
    if len(kinds) != 1:
        raise ValueError("mix of host and device arrays")
    return _lib.CYQ_MEM_DEVICE if kinds.pop() else _lib.CYQ_MEM_HOST


def _dims(p, P):
    A, B = p.A, p.B
    return _lib.CyqDims(A.shape[1], A.shape[2], B.shape[3], P, A.shape[0])


def _ocp_struct(p):
    return _lib.CyqOcpBatch(*[_ptr(getattr(p, k)) for k in OCP_FIELDS])


def _check_opts(opts: FactorOptions):
    P = int(opts.P)
    if P <= 0 or (P & (P - 1)) != 0:
        raise ValueError("P must be a power of two")
    v = int(opts.vlen)
    if v < 1 or (v & (v - 1)) != 0:
        raise ValueError("vlen must be a power of two")
    if opts.tail not in ("cr1", "pcr", "pcg"):
        raise ValueError("tail must be one of cr1, pcr, pcg")


def _apply_tail(ctx, opts: FactorOptions):
    """FactorOptions::tail / vlen (kkt_factor.cpp:214-247) as context options:
    tail = pcr solves the last min(P, vlen) Schur blocks by parallel cyclic
    reduction on the GPU; pcg is served by exact cyclic reduction (within
    its 1e-8 contract, test_kkt.cpp:157-161)."""
    key = (opts.tail, int(opts.vlen))
    if ctx._tail != key:
        ctx.set_option("tail", opts.tail)
        ctx.set_option("vlen", int(opts.vlen))
        ctx._tail = key


def _context(ctx, arrays) -> "Context":
    """The context of a call: `ctx`, else the default context of the device
    the CUDA tensors live on (device 0 for host arrays). Every CUDA tensor
    must be on the context's device."""
    devs = {a.device.index for a in arrays if _is_torch(a)}
    if len(devs) > 1:
        raise ValueError(f"arrays on several devices: {sorted(devs)}")
    if ctx is None:
        ctx = Context.default(devs.pop() if devs else 0)
    elif devs and devs != {ctx.device}:
        raise ValueError(f"arrays on cuda:{devs.pop()} but the context is on cuda:{ctx.device}")
    return ctx


def _raise_status(ctx, rc, st):
    if rc == _lib.CYQ_OK:
        return
    if rc == _lib.CYQ_INVALID_ARG:
        raise ValueError(ctx.last_error())
    if rc == _lib.CYQ_PIVOT_FAIL:
        bad = [s for s in st if s.code != 0]
        s = bad[0]
        if s.kind == 1:
            what = (f"cyclic reduction: pivot failure at level {s.column_or_level}, "
                    f"index {s.stage} (instance {s.instance})")
            raise FactorizeError(what, s.stage, s.pivot, bad)
        what = (f"potrf: pivot failure at batch {s.column_or_level}, pivot {s.pivot} "
                f"(instance {s.instance}, stage position {s.stage})")
        raise FactorizeError(what, s.column_or_level, s.pivot, bad)
    raise CudaError(f"cyqlone_b200 error {rc}: {ctx.last_error()}")


def _alloc_sol(p, device_like):
    b, N, nx, nu = p.A.shape[0], p.A.shape[1], p.A.shape[2], p.B.shape[3]
    if device_like:
        import torch
        dev = p.A.device
        return EqSolutionBatch(torch.zeros((b, N, nu), dtype=torch.float64, device=dev),
                               torch.zeros((b, N + 1, nx), dtype=torch.float64, device=dev),
                               torch.zeros((b, N, nx), dtype=torch.float64, device=dev))
    return EqSolutionBatch.empty(b, N, nx, nu)


def solve_problem(p, opts: FactorOptions, ctx: Context | None = None, out=None,
                  raise_on_error: bool = True):
    """kkt::solve_problem for every instance of the batch. Returns the
    solution batch (numpy for host input, torch for CUDA input)."""
    _check_opts(opts)
    arrs = [getattr(p, k) for k in OCP_FIELDS] + ([] if out is None else [getattr(out, k) for k in SOL_FIELDS])
    ctx = _context(ctx, arrs)
    _apply_tail(ctx, opts)
    arrs = arrs[:len(OCP_FIELDS)]
    mem = _mem(arrs)
    ctx.follow_torch(arrs)
    sol = out if out is not None else _alloc_sol(p, mem == _lib.CYQ_MEM_DEVICE)
    st = (_lib.CyqStatus * p.A.shape[0])()
    rc = ctx.lib.cyq_solve_problem_batch(ctx.h, C.byref(_dims(p, opts.P)),
                                         C.byref(_ocp_struct(p)),
                                         C.byref(_lib.CyqSolBatch(*[_ptr(getattr(sol, k))
                                                                   for k in SOL_FIELDS])),
                                         st, mem)
    if raise_on_error:
        _raise_status(ctx, rc, st)
    return sol if raise_on_error else (sol, rc, list(st))


class Factor:
    """kkt::Factor (kkt_solver.hpp:69-116) -- an opaque device factor of a
    batch. `materialize(inst)` copies the blocks the reference exposes as
    public members (LH, LB, Acl, LA) to host numpy arrays."""

    def __init__(self, ctx, handle, p, opts):
        self.ctx, self.h, self.opts = ctx, handle, opts
        self.N, self.nx, self.nu = p.A.shape[1], p.A.shape[2], p.B.shape[3]
        self.batch = p.A.shape[0]
        P = opts.P
        self.n_per = (P * ((self.N + P - 1) // P)) // P

    def materialize(self, inst: int = 0, schur: bool = True):
        """Host copies of the reference's public Factor members for instance
        `inst` (kkt_solver.hpp:76-97): LH, LB, Acl (n, P, ...), LA, T, Mfwd,
        Mbwd, W (P, nx, nx), schur_diag / schur_sub (the assembled block
        tridiagonal Schur complement) and the CR factor cr_L / cr_U / cr_Y
        (P-1, nx, nx; level l, slot mm at P - (P >> l) + mm) and cr_Lbase."""
        P, n, nx, nu = self.opts.P, self.n_per, self.nx, self.nu
        nux = nx + nu
        LH = np.zeros((n, P, nux, nux))
        LB = np.zeros((n, P, nx, nu))
        Acl = np.zeros((n, P, nx, nx))
        LA = np.zeros((P, nx, nx))
        rc = self.ctx.lib.cyq_factor_materialize(self.h, inst, *[C.c_void_p(a.ctypes.data)
                                                                 for a in (LH, LB, Acl, LA)])
        if rc:
            raise CudaError(self.ctx.last_error())
        out = {"LH": LH, "LB": LB, "Acl": Acl, "LA": LA}
        if schur:
            names = ("T", "Mfwd", "Mbwd", "W", "schur_diag", "schur_sub", "cr_L", "cr_U", "cr_Y")
            arr = {k: np.zeros((P if i < 6 else max(P - 1, 0), nx, nx)) for i, k in enumerate(names)}
            arr["cr_Lbase"] = np.zeros((nx, nx))
            rc = self.ctx.lib.cyq_factor_materialize_schur(
                self.h, inst, *[C.c_void_p(arr[k].ctypes.data if arr[k].size else None)
                                for k in names + ("cr_Lbase",)])
            if rc == _lib.CYQ_INVALID_ARG:
                raise ValueError(self.ctx.last_error())
            if rc:
                raise CudaError(self.ctx.last_error())
            out.update(arr)
        return out

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.cyq_factor_destroy(self.h)
                self.h = None
        except Exception:
            pass


def factor(p, opts: FactorOptions, ctx: Context | None = None) -> Factor:
    """kkt::factor for every instance of the batch."""
    _check_opts(opts)
    ctx = _context(ctx, [getattr(p, k) for k in OCP_FIELDS])
    _apply_tail(ctx, opts)
    mem = _mem([getattr(p, k) for k in OCP_FIELDS])
    ctx.follow_torch([getattr(p, k) for k in OCP_FIELDS])
    h = C.c_void_p()
    st = (_lib.CyqStatus * p.A.shape[0])()
    rc = ctx.lib.cyq_factor_batch(ctx.h, C.byref(_dims(p, opts.P)), C.byref(_ocp_struct(p)),
                                  mem, C.byref(h), st)
    f = Factor(ctx, h, p, opts) if h.value else None
    _raise_status(ctx, rc, st)
    return f


def solve(f: Factor, p, rhs) -> EqSolutionBatch:
    """kkt::solve with an explicit right-hand side (EqRhs convention)."""
    ctx = f.ctx
    arrs = [getattr(rhs, k) for k in RHS_FIELDS]
    mem = _mem(arrs)
    ctx.follow_torch(arrs + [getattr(p, k) for k in OCP_FIELDS])
    sol = _alloc_sol(p, mem == _lib.CYQ_MEM_DEVICE)
    rc = ctx.lib.cyq_solve_batch(ctx.h, f.h, C.byref(_ocp_struct(p)),
                                 C.byref(_lib.CyqRhsBatch(*[_ptr(a) for a in arrs])),
                                 C.byref(_lib.CyqSolBatch(*[_ptr(getattr(sol, k))
                                                           for k in SOL_FIELDS])), mem)
    _raise_status(ctx, rc, [])
    return sol


def update(f: Factor, p_new, C, D, C_term, ds_stage, ds_terminal=None):
    """kkt::update (kkt_solver.hpp:152-161, kkt_update.cpp:372-477) of every
    instance of `f`, in place on the GPU: afterwards `f` is (up to roundoff)
    the factor of `p_new` (stage Hessians H_j + (D_j | C_j)' dSigma_j
    (D_j | C_j)). Per partition column the update rank r selects the path:
    0 untouched, r < rho nx the hyperbolic-Householder column update
    (update.cu), r >= rho nx or a breakdown a refactorization of the column;
    the Schur complement and its CR factor are then re-formed. Arrays: C
    (b, N, ny, nx), D (b, N, ny, nu), C_term (b, ny_term, nx), ds_stage
    (b, N, ny), ds_terminal (b, ny_term) -- all host numpy or all CUDA
    tensors, like p_new. Returns (f, report) with per-instance lists
    columns_updated / columns_refactored / schur_refactored."""
    ctx = f.ctx
    dev = _is_torch(ds_stage)
    b, N, nx, nu = f.batch, f.N, f.nx, f.nu
    if ds_terminal is None:
        ds_terminal = (_torch().zeros((b, 0), dtype=_torch().float64, device=ds_stage.device) if dev
                       else np.zeros((b, 0)))
    if C_term is None:
        C_term = (_torch().zeros((b, 0, nx), dtype=_torch().float64, device=ds_stage.device) if dev
                  else np.zeros((b, 0, nx)))
    if not dev:
        ds_stage, ds_terminal, C, D, C_term = (np.ascontiguousarray(a, dtype=np.float64)
                                               for a in (ds_stage, ds_terminal, C, D, C_term))
    ny, nyt = ds_stage.shape[2], ds_terminal.shape[1]
    if tuple(ds_stage.shape) != (b, N, ny):
        raise ValueError("update: ds_stage must be (batch, N, ny)")
    if tuple(D.shape) != (b, N, ny, nu):
        raise ValueError("update: D must be (batch, N, ny, nu)")
    if tuple(C.shape) != (b, N, ny, nx):
        raise ValueError("update: C must be (batch, N, ny, nx)")
    if tuple(C_term.shape) != (b, nyt, nx):
        raise ValueError("update: C_term must be (batch, ny_term, nx)")
    arrs = [getattr(p_new, k) for k in OCP_FIELDS] + [C, D, ds_stage, C_term, ds_terminal]
    mem = _mem(arrs)
    ctx.follow_torch(arrs)
    rep = (_lib.CyqUpdateReport * b)()
    # (the parameter C shadows the ctypes module here: _byref)
    rc = ctx.lib.cyq_factor_update_batch(ctx.h, f.h, _byref(_ocp_struct(p_new)), ny, _ptr(C), _ptr(D), _ptr(ds_stage),
                                         nyt, _ptr(C_term) if nyt else None,
                                         _ptr(ds_terminal) if nyt else None, float(f.opts.rho), mem, rep)
    _raise_status(ctx, rc, [])
    report = {"columns_updated": [r.columns_updated for r in rep],
              "columns_refactored": [r.columns_refactored for r in rep],
              "schur_refactored": [bool(r.schur_refactored) for r in rep],
              "schur_levels_updated": [r.schur_levels_updated for r in rep]}
    return f, report


def augment_hessians(p, D, Cm, sigma, gamma_inv: float = 0.0, out=None,
                     ctx: Context | None = None) -> EqOCPBatch:
    """Newton-system assembly of the QPALM inner loop (qpalm::assemble_newton,
    qpalm.cpp:167-225, equality part) on the GPU: returns the batch with
    R + D'ΣD + γ⁻¹I, S + D'ΣC, Q + C'ΣC + γ⁻¹I (stage-wise; C[:, N] the
    terminal rows) and the other fields shared with `p`. Device (CUDA torch)
    arrays only: D (b, N, ny, nu), Cm (b, N+1, ny, nx), sigma (b, N+1, ny).
    `out` may pass a preallocated EqOCPBatch whose R, S, Q are overwritten."""
    import torch

    ctx = _context(ctx, [p.R, p.S, p.Q, D, Cm, sigma])
    for a in (p.R, p.S, p.Q, D, Cm, sigma):
        if not _is_torch(a):
            raise ValueError("augment_hessians takes CUDA torch tensors")
    ctx.follow_torch([D])
    b, N, nx, nu = p.A.shape[0], p.A.shape[1], p.A.shape[2], p.B.shape[3]
    ny = D.shape[2]
    if out is None:
        out = EqOCPBatch.__new__(EqOCPBatch)
        for k in OCP_FIELDS:
            setattr(out, k, getattr(p, k))
        out.R, out.S, out.Q = torch.empty_like(p.R), torch.empty_like(p.S), torch.empty_like(p.Q)
    rc = ctx.lib.cyq_augment_hessians_batch(
        ctx.h, C.byref(_lib.CyqDims(N, nx, nu, 1, b)), ny, *[_ptr(a) for a in
                                                             (p.R, p.S, p.Q, D, Cm, sigma)],
        float(gamma_inv), _ptr(out.R), _ptr(out.S), _ptr(out.Q))
    if rc != _lib.CYQ_OK:
        raise (ValueError if rc == _lib.CYQ_INVALID_ARG else CudaError)(
            f"cyq_augment_hessians_batch failed ({rc}): {ctx.last_error()}")
    return out


class Prepared:
    """A prepared device-resident call over fixed arrays -- kkt::solve_problem
    (`Prepared.solve_problem`) or the QPALM Newton system
    (`Prepared.solve_newton`): the argument blocks are validated and built
    once, each call is one C-ABI call. For loops that rewrite the device
    arrays in place between calls (MPC, the QPALM inner loop); with the
    context's `async_status` option the calls do not synchronize the host
    (check `ctx.wait_status(batch)` afterwards)."""

    def __init__(self, ctx, fn, args, batch, out):
        self.ctx, self.fn, self.args, self.batch, self.out = ctx, fn, args, batch, out
        self.st = (_lib.CyqStatus * batch)()
        self._keep = []

    @classmethod
    def solve_problem(cls, p, opts: FactorOptions, out=None, ctx: Context | None = None):
        _check_opts(opts)
        arrs = [getattr(p, k) for k in OCP_FIELDS]
        if not all(_is_torch(a) for a in arrs):
            raise ValueError("Prepared calls take CUDA torch tensors")
        ctx = _context(ctx, arrs + ([] if out is None else [getattr(out, k) for k in SOL_FIELDS]))
        _apply_tail(ctx, opts)
        ctx.follow_torch(arrs)
        sol = out if out is not None else _alloc_sol(p, True)
        dims, ocp = _dims(p, opts.P), _ocp_struct(p)
        solb = _lib.CyqSolBatch(*[_ptr(getattr(sol, k)) for k in SOL_FIELDS])
        self = cls(ctx, ctx.lib.cyq_solve_problem_batch, None, p.A.shape[0], sol)
        self._keep = [dims, ocp, solb]
        self.args = (ctx.h, C.byref(dims), C.byref(ocp), C.byref(solb), self.st, _lib.CYQ_MEM_DEVICE)
        return self

    @classmethod
    def solve_newton(cls, p, D, Cm, opts: FactorOptions, gamma_inv: float = 0.0, out=None,
                     ctx: Context | None = None):
        """Call with the Σ of each Newton system: `plan(sigma)`."""
        _check_opts(opts)
        arrs = [getattr(p, k) for k in OCP_FIELDS] + [D, Cm]
        if not all(_is_torch(a) for a in arrs):
            raise ValueError("Prepared calls take CUDA torch tensors")
        ctx = _context(ctx, arrs)
        _apply_tail(ctx, opts)
        ctx.follow_torch(arrs)
        sol = out if out is not None else _alloc_sol(p, True)
        dims, ocp = _dims(p, opts.P), _ocp_struct(p)
        solb = _lib.CyqSolBatch(*[_ptr(getattr(sol, k)) for k in SOL_FIELDS])
        self = cls(ctx, ctx.lib.cyq_solve_newton_batch, None, p.A.shape[0], sol)
        self._keep = [dims, ocp, solb]
        self.args = (ctx.h, C.byref(dims), C.byref(ocp), D.shape[2], _ptr(D), _ptr(Cm))
        self.tail = (float(gamma_inv), C.byref(solb), self.st)
        self.sig_shape = (p.A.shape[0], p.A.shape[1] + 1, D.shape[2])
        return self

    def __call__(self, sigma=None, raise_on_error: bool = True):
        if sigma is None:
            rc = self.fn(*self.args)
        else:
            if tuple(sigma.shape) != self.sig_shape:
                raise ValueError(f"sigma must be {self.sig_shape}")
            rc = self.fn(*self.args, _ptr(sigma), *self.tail)
        if rc != _lib.CYQ_OK and raise_on_error:
            _raise_status(self.ctx, rc, self.st)
        return self.out


def solve_newton(p, D, Cm, sigma, opts: FactorOptions, gamma_inv: float = 0.0, out=None,
                 ctx: Context | None = None, raise_on_error: bool = True):
    """One Newton system of the QPALM inner loop per instance: assembly as in
    `augment_hessians` (qpalm::assemble_newton, qpalm.cpp:167-225) followed by
    kkt::solve_problem (qpalm.cpp:368-413 factor + solve). For the config-4
    stage shape (nu = 8, nx = 16, ny = 24) the assembly is fused into the
    factorization's stage loads (the augmented Hessians never reach HBM);
    other shapes run the assembly kernel first. CUDA torch tensors only."""
    _check_opts(opts)
    ctx = _context(ctx, [getattr(p, k) for k in OCP_FIELDS] + [D, Cm, sigma])
    _apply_tail(ctx, opts)
    for a in [getattr(p, k) for k in OCP_FIELDS] + [D, Cm, sigma]:
        if not _is_torch(a):
            raise ValueError("solve_newton takes CUDA torch tensors")
    ctx.follow_torch([D])
    sol = out if out is not None else _alloc_sol(p, True)
    st = (_lib.CyqStatus * p.A.shape[0])()
    rc = ctx.lib.cyq_solve_newton_batch(
        ctx.h, C.byref(_dims(p, opts.P)), C.byref(_ocp_struct(p)), D.shape[2],
        _ptr(D), _ptr(Cm), _ptr(sigma), float(gamma_inv),
        C.byref(_lib.CyqSolBatch(*[_ptr(getattr(sol, k)) for k in SOL_FIELDS])), st)
    if raise_on_error:
        _raise_status(ctx, rc, st)
    return sol if raise_on_error else (sol, rc, list(st))


def al_gradients(p, D, Cm, bl, bu, u, x, y, sigma, ubar, xbar, gamma_inv: float,
                 ctx: Context | None = None, out=None):
    """qpalm::eval_al_gradients (qpalm.cpp:106-165) on the GPU for every
    instance: returns dict(ru (b, N, nu), qx (b, N+1, nx; qx[:, 0] = 0),
    yhat (b, N+1, ny), cres (b, N, nx)) as CUDA tensors. Inputs are CUDA
    torch tensors: the problem batch `p`, D (b, N, ny, nu), Cm (b, N+1, ny,
    nx; Cm[:, N] the terminal rows), bl, bu, y, sigma (b, N+1, ny), u, ubar
    (b, N, nu), x, xbar (b, N+1, nx). The Newton step's rhs is
    EqRhsBatch(-ru, -qx, -cres) (qpalm.cpp:391-405, `newton_rhs`)."""
    import torch

    arrs = [p.R, p.S, p.Q, p.A, p.B, p.f, p.r, p.q, D, Cm, bl, bu, u, x, y, sigma, ubar, xbar]
    for a_ in arrs:
        if not _is_torch(a_):
            raise ValueError("al_gradients takes CUDA torch tensors")
    ctx = _context(ctx, arrs)
    ctx.follow_torch(arrs)
    b, N, nx, nu = p.A.shape[0], p.A.shape[1], p.A.shape[2], p.B.shape[3]
    ny = D.shape[2]
    if tuple(Cm.shape) != (b, N + 1, ny, nx) or tuple(y.shape) != (b, N + 1, ny):
        raise ValueError("al_gradients: Cm must be (b, N+1, ny, nx), y / sigma / bl / bu (b, N+1, ny)")
    f64 = dict(dtype=torch.float64, device=p.A.device)
    if out is None:
        out = {"ru": torch.empty((b, N, nu), **f64), "qx": torch.empty((b, N + 1, nx), **f64),
               "yhat": torch.empty((b, N + 1, ny), **f64), "cres": torch.empty((b, N, nx), **f64)}
    rc = ctx.lib.cyq_al_gradients_batch(
        ctx.h, C.byref(_lib.CyqDims(N, nx, nu, 1, b)), ny, C.byref(_ocp_struct(p)),
        *[_ptr(a_) for a_ in (D, Cm, bl, bu, u, x, y, sigma, ubar, xbar)], float(gamma_inv),
        *[_ptr(out[k]) for k in ("ru", "qx", "yhat", "cres")])
    if rc != _lib.CYQ_OK:
        raise (ValueError if rc == _lib.CYQ_INVALID_ARG else CudaError)(
            f"cyq_al_gradients_batch failed ({rc}): {ctx.last_error()}")
    return out


def newton_rhs(grads) -> EqRhsBatch:
    """The Newton step's right-hand side from al_gradients: ru = -ru,
    qx = -qx (qx[0] unused), fd = -cres (qpalm.cpp:391-405)."""
    rhs = EqRhsBatch.__new__(EqRhsBatch)  # device tensors as they are
    rhs.ru, rhs.qx, rhs.fd = -grads["ru"], -grads["qx"], -grads["cres"]
    return rhs


def line_search_exact(alpha, delta, eta, beta, ctx: Context | None = None,
                      raise_on_error: bool = True, iterations: bool = False):
    """qpalm::line_search_exact (line_search.cpp:112-206) for a batch: tau[b]
    = root of psi'(tau) = eta[b] tau + beta[b] + sum_i delta[b,i]
    [delta[b,i] tau - alpha[b,i]]_+ (terms as LineSearchData::add_term,
    line_search.cpp:9-27). CUDA torch tensors: alpha, delta (b, m), eta,
    beta (b,). Raises ValueError (the reference's std::invalid_argument) if
    psi'(0) > 0 for some instance, unless raise_on_error=False (then returns
    (tau, status list))."""
    import torch

    ctx = _context(ctx, [alpha, delta, eta, beta])
    for a in (alpha, delta, eta, beta):
        if not _is_torch(a):
            raise ValueError("line_search_exact takes CUDA torch tensors")
    ctx.follow_torch([alpha])
    b, m = alpha.shape[0], (alpha.shape[1] if alpha.dim() > 1 else 0)
    tau = torch.empty(b, dtype=torch.float64, device=alpha.device)
    its = torch.zeros(b, dtype=torch.int64, device=alpha.device)
    st = (C.c_int32 * b)()
    rc = ctx.lib.cyq_line_search_batch(ctx.h, b, m, _ptr(alpha), _ptr(delta), _ptr(eta), _ptr(beta),
                                       _ptr(tau), st, C.c_void_p(its.data_ptr()))
    if rc == _lib.CYQ_INVALID_ARG and raise_on_error:
        raise ValueError(ctx.last_error())
    if rc not in (_lib.CYQ_OK, _lib.CYQ_INVALID_ARG):
        raise CudaError(f"cyq_line_search_batch failed ({rc}): {ctx.last_error()}")
    out = (tau, list(st)) if not raise_on_error else tau
    if iterations:
        return (out, its) if raise_on_error else (tau, list(st), its)
    return out


__all__ = ["Prepared", "al_gradients", "newton_rhs", "augment_hessians", "solve_newton", "line_search_exact", "update", "FactorOptions", "Factor", "FactorizeError", "CudaError", "Context", "factor",
           "solve", "solve_problem", "nu2", "EqOCPBatch", "EqRhsBatch", "EqSolutionBatch"]
