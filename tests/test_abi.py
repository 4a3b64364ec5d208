"""CPU tests of the C ABI boundary: the library loads, exports every entry
point include/cyqlone_b200.h declares, validates arguments like the
reference (std::invalid_argument -> CYQ_INVALID_ARG) and fails loudly (no
CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2512_09058_b200 import _lib, kkt, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cyqlone_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cyq_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (cyq_\w+)", out))
    for name in declared():
        assert name in exported, name
        assert hasattr(lib, name)
    assert set(_lib.SIGNATURES) == set(declared())


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


# The kernels the BASELINE configs run (bench.py / launch lists): every
# stage-panel and Schur/CR kernel must issue FP64 tensor-core DMMAs
LIVE_DMMA_KERNELS = [
    "riccati_warp_kernelILi10ELi20ELi1ELi0ELb0",   # config 1 panel
    "riccati_warp_kernelILi8ELi16ELi1ELi24ELb0",   # config 4 panel (fused Newton assembly)
    "riccati_pc_kernelILi5ELi10",                  # config 0 panel
    "riccati_pc_kernelILi4ELi12",                  # config 2 panel
    "riccati_cta_kernelILi32ELi64ELi16ELb0",       # config 3 panel
    "riccati_cta_kernelILi32ELi64ELi16ELb1",       # config 3 panel, TMA-staged variant
    "schur_fused_kernelILi20ELi2ELi1",             # config 1 Schur/CR (batch > 4 x SMs)
    "schur_fused_kernelILi20ELi4ELi1",
    "schur_fused_kernelILi16ELi4ELi1",             # config 4 Schur/CR
    "schur_fused_kernelILi12ELi16ELi8",            # config 2 Schur/CR (8-CTA cluster)
    "schur_fused_kernelILi10ELi16ELi1",            # config 0 Schur/CR
    "schur_big_kernelILi64ELi16",                  # config 3 Schur/CR
    "riccati_panel_kernel_t",                      # generic panel (other shapes)
]


def test_kernels_use_dmma():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    funcs = out.split("Function : ")[1:]
    for tag in LIVE_DMMA_KERNELS:
        hits = [f for f in funcs if tag in f.split("\n", 1)[0]]
        assert hits, f"kernel {tag} not in the library"
        assert all("DMMA" in f for f in hits), f"{tag}: no DMMA in its SASS"


def test_version_string():
    assert b"sm_100a" in _lib.load().cyq_version()


def test_invalid_P_raises_value_error_before_touching_device():
    p = synth.generate(0, seed=0, batch=1, N=8)
    with pytest.raises(ValueError):
        kkt.solve_problem(p, kkt.FactorOptions(P=3))
    with pytest.raises(ValueError):
        kkt.solve_problem(p, kkt.FactorOptions(P=4, vlen=3))


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.cyq_ctx_create(0, C.byref(h)) == _lib.CYQ_NO_DEVICE
    p = synth.generate(0, seed=0, batch=1, N=8)
    with pytest.raises(kkt.CudaError):
        kkt.solve_problem(p, kkt.FactorOptions(P=4))


def test_tma_variant_issues_bulk_copies():
    # the TMA-staged CTA panel carries UBLKCP (cp.async.bulk) in its SASS
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    funcs = {f.split("\n", 1)[0]: f for f in out.split("Function : ")[1:]}
    tma = [f for k, f in funcs.items() if "riccati_cta_kernelILi32ELi64ELi16ELb1" in k]
    assert tma and "UBLKCP" in tma[0]
