"""The C++ host interface (include/cyqlone_b200/kkt_solver.hpp, ocp.hpp): the
reference's cyqlone::kkt::{factor, solve, solve_problem} signatures over the
sm_100a library, exercised by the C++ driver tests/cpp/test_kkt_host.cpp.

CPU: the library and driver build with g++, export the reference's entry
points, and fail loudly without a GPU (no CPU fallback).
GPU: the driver's property tests (test_kkt.cpp-style) pass, and the driver
reproduces the reference's golden outputs through the single-instance C++
entry point (rel. error <= 1e-9, KKT residual <= 1e-10).
"""
import os
import subprocess

import numpy as np
import pytest

import golden_util
from paper_2512_09058_b200 import build as B
from paper_2512_09058_b200.ocp import EqRhsBatch, EqSolutionBatch, kkt_residual, rel_error

DRIVER = B.HOST_TEST_OUT


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(B.OUT):
        B.build()
    if not (os.path.exists(B.HOST_OUT) and os.path.exists(DRIVER)):
        B.build_host()


def test_driver_links_and_runs():
    r = subprocess.run([DRIVER, "compile-only"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr


def test_host_library_exports_reference_entry_points():
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", B.HOST_OUT], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("cyqlone::kkt::factor(cyqlone::ocp::EqOCP const&, cyqlone::kkt::FactorOptions const&, "
                "cyqlone::kkt::FlopTrace*)",
                "cyqlone::kkt::solve(cyqlone::kkt::Factor const&, cyqlone::ocp::EqOCP const&, "
                "cyqlone::ocp::EqRhs const&)",
                "cyqlone::kkt::solve_problem(cyqlone::ocp::EqOCP const&, cyqlone::kkt::FactorOptions const&, "
                "cyqlone::kkt::Factor*)",
                "cyqlone::ocp::kkt_residual_eq(cyqlone::ocp::EqOCP const&, cyqlone::ocp::EqRhs const&, "
                "cyqlone::ocp::EqSolution const&)",
                "cyqlone::ocp::EqRhs::of_problem(cyqlone::ocp::EqOCP const&)"):
        assert sym in out, sym


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_fails_loudly_without_gpu():
    r = subprocess.run([DRIVER, "selftest"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cpp_property_suite():
    r = subprocess.run([DRIVER, "selftest"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK (0 failures)" in r.stdout


def _write_input(path, p, P):
    hdr = np.array([p.N, p.nx, p.nu, P, p.batch], dtype=np.int64)
    with open(path, "wb") as fh:
        fh.write(hdr.tobytes())
        for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
            fh.write(np.ascontiguousarray(getattr(p, k), dtype=np.float64).tobytes())


GOLDEN_SMALL = [n for n in golden_util.names() if "N4096" not in n]


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLDEN_SMALL)
def test_cpp_entry_point_reproduces_golden(tmp_path, name):
    p, P, ref, z = golden_util.load(name)
    fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
    _write_input(fin, p, P)
    r = subprocess.run([DRIVER, "golden", str(fin), str(fout)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    raw = np.fromfile(fout, dtype=np.float64)
    b, N, nx, nu = p.batch, p.N, p.nx, p.nu
    nu_, nx_ = b * N * nu, b * (N + 1) * nx
    sol = EqSolutionBatch(raw[:nu_].reshape(b, N, nu), raw[nu_:nu_ + nx_].reshape(b, N + 1, nx),
                          raw[nu_ + nx_:].reshape(b, N, nx))
    assert rel_error(sol, ref).max() <= 1e-9
    res = kkt_residual(p, EqRhsBatch.of_problem(p), sol).max(axis=1)
    bound = np.maximum(1e-10, 4 * z["residual"]) if "qpalm" in name else 1e-10
    assert np.all(res <= bound)
