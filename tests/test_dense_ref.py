"""CPU pin of the numpy factor_reconstruction_error port (tests/dense_ref.py,
proj/tests/support/dense_ref.cpp:149-286): the reference's own factor
(oracle/_ref, every public Factor member including the CR factor) must
reconstruct the permuted KKT matrix to < 1e-10, as test_kkt.cpp:66-103
asserts; a perturbed block must not."""
import numpy as np
import pytest

from dense_ref import factor_reconstruction_error
from pyoracle import RefOracle, ref_available

from paper_2512_09058_b200 import synth

pytestmark = pytest.mark.skipif(not ref_available(), reason="reference build unavailable")


@pytest.mark.parametrize("N,nx,nu,P", [(16, 3, 2, 1), (16, 3, 2, 2), (16, 3, 2, 4), (16, 3, 2, 8),
                                       (16, 4, 2, 4), (32, 10, 5, 4), (32, 12, 4, 16)])
def test_reference_factor_reconstructs(N, nx, nu, P):
    ref = RefOracle()
    p = ref.random_eq_ocp(N, nx, nu, 100 + P + nx)
    fb, rc, _ = ref.factor_blocks(p, P, cr=True)
    assert rc == 0
    assert factor_reconstruction_error(fb, p, 0, P) < 1e-10
    bad = dict(fb)
    bad["cr_Lbase"] = fb["cr_Lbase"] * (1 + 1e-6)
    assert factor_reconstruction_error(bad, p, 0, P) > 1e-9


def test_reference_factor_reconstructs_baseline_shape():
    ref = RefOracle()
    p = synth.generate(1, seed=2, batch=1, N=32)
    fb, rc, _ = ref.factor_blocks(p, 16, cr=True)
    assert rc == 0
    assert factor_reconstruction_error(fb, p, 0, 16) < 1e-10
