"""CYQ_OPT_SPLIT (device-resident batch as K parts on two streams) at config 3:
    python tools/split_check.py    -> ms per step for K = 1, 2, 4 (measured 30.98 / 30.94 / 30.92: neutral,
the 219 KB panel CTAs leave no room for another kernel's CTAs on their SM)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_09058_b200 import kkt, synth
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch
c = synth.CONFIGS[3]
p = synth.generate(3, seed=0, batch=256)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
ctx = kkt.Context(0); ctx.set_stream(stream.cuda_stream)
opts = kkt.FactorOptions(P=c.P)
for split in (1, 2, 4):
    with ctx.options(split=split):
        sol = kkt.solve_problem(dev, opts, ctx=ctx)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
        e1.record(stream); torch.cuda.synchronize()
        print("split", split, "ms/step", e0.elapsed_time(e1) / 5)
