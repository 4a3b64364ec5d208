"""Per-kernel device time of one configuration (CUDA events around each
launch, averaged over REPS device-resident solve_problem calls).
    python tools/kernel_time.py CFG BATCH [REPS]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

cfg = int(sys.argv[1])
batch = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = synth.CONFIGS[cfg]
p = synth.generate(cfg, seed=0, batch=batch)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = kkt.Context(0)
ctx.set_stream(stream.cuda_stream)
opts = kkt.FactorOptions(P=c.P)
sol = kkt.solve_problem(dev, opts, ctx=ctx)
ctx.profile(True)
ctx.profile_read(reset=True)
for _ in range(reps):
    kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
kern = ctx.profile_read(reset=True)
print(json.dumps({"lib": os.environ.get("CYQ_LIB", "default"), "config": cfg, "batch": batch,
                  "ms": {k: v[0] / reps for k, v in kern.items() if v[1]}}))
