"""The GPU factor's public blocks (kkt::Factor members, kkt_solver.hpp:76-97)
materialized to the host -- LH, LB, Acl, LA, T, sc_Mfwd, sc_Mbwd, sc_W, the
assembled Schur complement and its CR factor (schur_cr: L, U, Y per level,
L_base) -- against the reference's own factor (oracle/_ref) block by block,
and the reference's structural check factor_reconstruction_error
(dense_ref.cpp:149-286, numpy port tests/dense_ref.py, pinned on the CPU by
test_dense_ref.py) on the GPU blocks: < 1e-10 as test_kkt.cpp:66-103."""
import numpy as np
import pytest

from dense_ref import factor_reconstruction_error
from pyoracle import RefOracle, ref_available

from paper_2512_09058_b200 import kkt, synth

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="reference build unavailable")]

KEYS = ("LH", "LB", "Acl", "LA", "T", "Mfwd", "Mbwd", "W", "schur_diag", "schur_sub",
        "cr_L", "cr_U", "cr_Y", "cr_Lbase")


# fused Schur kernel (nx 10 / 12 / 16 / 20; CTA and cluster variants) and the
# CTA-level kernel for tile-aligned blocks (nx 32 / 64)
@pytest.mark.parametrize("cfg,N,P,nx,nu", [(0, 64, 4, None, None), (1, 32, 16, None, None),
                                           (2, 512, 64, None, None), (4, 32, 8, None, None),
                                           (0, 32, 4, 32, 8), (3, 64, 8, None, None), (1, 64, 1, None, None)])
def test_factor_blocks_match_reference(cfg, N, P, nx, nu):
    import dataclasses
    if nx is None:
        p = synth.generate(cfg, seed=51, batch=1, N=N)
    else:
        c = dataclasses.replace(synth.CONFIGS[cfg], N=N, nx=nx, nu=nu, P=P, batch=1)
        vals = synth._instance(c, N, 51, 0)[:9]
        p = kkt.EqOCPBatch(*[v[None] for v in vals])
    f = kkt.factor(p, kkt.FactorOptions(P=P))
    got = f.materialize(0)
    ref, rc, _ = RefOracle().factor_blocks(p, P, cr=True)
    assert rc == 0
    for k in KEYS:
        if ref[k].size == 0:  # P = 1: no CR levels
            assert got[k].size == 0, k
            continue
        scale = max(1.0, np.abs(ref[k]).max())
        assert np.abs(got[k] - ref[k]).max() <= 1e-11 * scale, k
    assert factor_reconstruction_error(got, p, 0, P) < 1e-10


def test_materialize_instances_of_a_batch():
    p = synth.generate(1, seed=52, batch=5, N=32)
    f = kkt.factor(p, kkt.FactorOptions(P=16))
    for inst in (0, 3):
        got = f.materialize(inst)
        assert factor_reconstruction_error(got, p, inst, 16) < 1e-10


def test_materialize_schur_unavailable_path_raises():
    # the per-level / scalar Schur kernels (unusual nx) keep no persistent
    # Schur blocks: a clear ValueError, the Riccati blocks still come back
    import dataclasses
    c = dataclasses.replace(synth.CONFIGS[0], N=16, nx=5, nu=3, P=4, batch=1)
    p = kkt.EqOCPBatch(*[v[None] for v in synth._instance(c, 16, 3, 0)[:9]])
    f = kkt.factor(p, kkt.FactorOptions(P=4))
    with pytest.raises(ValueError, match="materialize_schur"):
        f.materialize(0)
    assert f.materialize(0, schur=False)["LH"].shape == (4, 4, 8, 8)
