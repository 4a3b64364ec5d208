import sys
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np, torch
from test_gpu_shapes import _problem
from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import EqOCPBatch
for (N, nx, nu, ny, P) in [(9, 17, 9, 33, 4), (5, 17, 9, 33, 4), (9, 17, 9, 32, 4), (7, 40, 24, 64, 2), (7, 40, 24, 8, 2), (7, 8, 8, 64, 2)]:
    base = _problem(N, nx, nu, P, 2)
    D, E, sig = synth.qpalm_data(base, seed=3, iters=1, ny=ny)
    ref_p = next(synth.qpalm_sequence(base, seed=3, iters=1, ny=ny))
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init"):
        setattr(dev, k, torch.from_numpy(np.ascontiguousarray(getattr(base, k))).cuda())
    Dd, Ed, sd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (D, E, sig[0]))
    try:
        aug = kkt.augment_hessians(dev, Dd, Ed, sd); torch.cuda.synchronize()
        errs = [float(np.abs(g.cpu().numpy() - r).max() / np.abs(r).max()) for g, r in ((aug.R, ref_p.R), (aug.S, ref_p.S), (aug.Q, ref_p.Q))]
        zero = [float(np.abs(g.cpu().numpy()).max()) for g in (aug.R, aug.S, aug.Q)]
        print(N, nx, nu, ny, "rel", ["%.1e" % e for e in errs], "maxabs", ["%.1e" % z for z in zero], flush=True)
    except Exception as e:
        print(N, nx, nu, ny, "EXC", str(e)[:120], flush=True)
