"""Small driver for ncu captures: solve_problem on a reduced batch of a
BASELINE config (config 4: one fused Newton system), device-resident inputs (python tools/prof_run.py CFG BATCH REPS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = synth.CONFIGS[cfg]
p = synth.generate(cfg, seed=0, batch=batch)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
if cfg == 4:  # QPALM Newton system: assembly fused into the panel
    D, E, sig = (torch.from_numpy(a).cuda()
                 for a in synth.qpalm_data(p, seed=0, iters=1, ny=c.ny))
    for _ in range(reps):
        s = kkt.solve_newton(dev, D, E, sig[0], kkt.FactorOptions(P=c.P))
else:
    for _ in range(reps):
        s = kkt.solve_problem(dev, kkt.FactorOptions(P=c.P))
torch.cuda.synchronize()
print("ok", float(s.u.abs().max()))
