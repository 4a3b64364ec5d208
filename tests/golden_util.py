"""Loads the golden fixtures of tests/golden/ (made by make_golden.py from
the reference build); regenerates large inputs from their seeds."""
import glob
import os

import numpy as np

from paper_2512_09058_b200 import synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch, EqSolutionBatch

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(name):
    z = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    if "in_A" in z:
        p = EqOCPBatch(*[z["in_" + k] for k in OCP_FIELDS])
    else:
        cfg, seed, start = int(z["regen_cfg"]), int(z["regen_seed"]), int(z["regen_start"])
        N, b = int(z["regen_N"]), int(z["regen_batch"])
        p = synth.generate(cfg, seed=seed, batch=b, N=N, start=start)
        if "regen_iter" in z:
            it = int(z["regen_iter"])
            for k, q in enumerate(synth.qpalm_sequence(p, seed=seed, iters=it + 1, start=start)):
                if k == it:
                    p = q
    chk = np.array([float(np.sum(a)) for a in p.arrays()])
    assert np.allclose(chk, z["checksum"], rtol=1e-12, atol=1e-9), f"{name}: input drift"
    sol = EqSolutionBatch(z["u"], z["x"], z["lam"])
    return p, int(z["P"]), sol, z
