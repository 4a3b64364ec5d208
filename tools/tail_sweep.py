"""Single-instance latency of the Schur tail variants (FactorOptions::tail =
cr1 / pcr with vlen = tail blocks), device-resident, Prepared calls with async
status and graph replay, CUDA events.   python tools/tail_sweep.py [CFG]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = synth.CONFIGS[cfg]
p = synth.generate(cfg, seed=0, batch=1)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = kkt.Context(0)
ctx.set_stream(stream.cuda_stream)
ctx.set_option("async_status", 1)
ref = kkt.solve_problem(dev, kkt.FactorOptions(P=c.P), ctx=ctx)
for tail, vlen in [("cr1", 4)] + [("pcr", v) for v in (2, 4, 8, 16, 32, 64, 128, 256) if v <= c.P]:
    opts = kkt.FactorOptions(P=c.P, tail=tail, vlen=vlen)
    plan = kkt.Prepared.solve_problem(dev, opts, ctx=ctx)
    for _ in range(20):
        plan()
    ctx.profile(True)
    ctx.profile_read(reset=True)
    for _ in range(50):
        plan()
    kern = ctx.profile_read(reset=True)
    ctx.profile(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(400):
        plan()
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.wait_status(1)
    err = max(float((getattr(plan.out, k) - getattr(ref, k)).abs().max()) for k in ("u", "x", "lam"))
    print(json.dumps({"config": cfg, "tail": tail, "vlen": vlen, "latency_ms": e0.elapsed_time(e1) / 400,
                      "schur_ms": kern["schur_cr"][0] / 50, "max_abs_diff_vs_cr1": err}), flush=True)
