import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np
from pyoracle import Oracle
from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqRhsBatch, kkt_residual, rel_error, residual_scale
base = synth.generate(4, seed=5, batch=2, N=64)
for p in synth.qpalm_sequence(base, seed=5, iters=3):
    sol = kkt.solve_problem(p, kkt.FactorOptions(P=16))
    ref, rc, _ = Oracle().solve_problem(p, 16)
    rhs = EqRhsBatch.of_problem(p)
    rg = kkt_residual(p, rhs, sol).max(axis=1); rr = kkt_residual(p, rhs, ref).max(axis=1)
    sc = residual_scale(p, rhs, sol)
    print('rel', rel_error(sol, ref), 'gpu', rg, 'ref', rr, 'scaled gpu', rg/sc, 'scaled ref', rr/sc)
