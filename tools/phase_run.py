"""Per-stage phase clocks of chain 0 of the stage panel (CYQ_OPT_PHASE_PROF),
printed to stderr by the library.   python tools/phase_run.py CFG BATCH"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c = synth.CONFIGS[cfg]
p = synth.generate(cfg, seed=0, batch=batch)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
ctx = kkt.Context(0)
def run():
    try:
        kkt.solve_problem(dev, kkt.FactorOptions(P=c.P), ctx=ctx)
    except kkt.FactorizeError as e:  # elimination builds (tools/variant_build.sh) break the numbers
        print("ignored:", e)


run()
with ctx.options(phase_prof=1):
    run()
torch.cuda.synchronize()
