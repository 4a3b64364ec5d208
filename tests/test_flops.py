"""The closed-form FLOP model used by bench.py equals the reference's own
instrumented multiply-add counter (through the C oracle, whose counts are
pinned to the reference build in test_oracle.py)."""
import pytest
from pyoracle import Oracle

from paper_2512_09058_b200.flops import flops_per_solve, fma_phases

SHAPES = [(64, 10, 5, 4), (128, 20, 10, 16), (4096, 12, 4, 256), (256, 16, 8, 16),
          (512, 64, 32, 32), (13, 3, 2, 4), (16, 3, 2, 1), (5, 2, 1, 4), (40, 20, 10, 16)]


@pytest.mark.parametrize("shape", SHAPES)
def test_closed_form_equals_counter(shape):
    ph = fma_phases(*shape)
    assert (ph["factor"], ph["solve"]) == Oracle().fma_counts(*shape)
    k = ph["kernel_riccati_panel"] + ph["kernel_schur_cr"] + ph["kernel_backsub"]
    assert k == ph["factor"] + ph["solve"]


def test_survey_mflop_per_solve():
    # cfg0 0.818, cfg1 11.68, cfg2 72.78, cfg3 1375.6 MFLOP
    assert round(flops_per_solve(64, 10, 5, 4) / 1e6, 3) == 0.818
    assert round(flops_per_solve(128, 20, 10, 16) / 1e6, 2) == 11.68
    assert round(flops_per_solve(4096, 12, 4, 256) / 1e6, 2) == 72.78
    assert round(flops_per_solve(512, 64, 32, 32) / 1e6, 1) == 1375.6
