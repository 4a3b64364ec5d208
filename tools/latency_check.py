"""Latency sanity check of repeated device calls (graph replay, async
status): results after each replay and event vs wall-clock timing.
    python tools/latency_check.py CFG [STEPS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
c = synth.CONFIGS[cfg]
p = synth.generate(cfg, seed=0, batch=1)
dev = EqOCPBatch.__new__(EqOCPBatch)
for k in OCP_FIELDS:
    setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = kkt.Context(0)
ctx.set_stream(stream.cuda_stream)
opts = kkt.FactorOptions(P=c.P)
sol = kkt._alloc_sol(dev, True)
ref = kkt.solve_problem(dev, opts, ctx=ctx)
torch.cuda.synchronize()
for mode in [dict(async_status=0, graphs=0), dict(async_status=1, graphs=0), dict(async_status=0, graphs=1),
             dict(async_status=1, graphs=1)]:
    with ctx.options(**mode):
        for _ in range(3):
            kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
        torch.cuda.synchronize()
        for k in ("u", "x", "lam"):
            getattr(sol, k).zero_()
        kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
        torch.cuda.synchronize()
        same = all(torch.equal(getattr(sol, k), getattr(ref, k)) for k in ("u", "x", "lam"))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(steps):
            kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(mode, f"solve_problem event {e0.elapsed_time(e1) / steps * 1e3:.1f} us",
              f"wall {(t1 - t0) / steps * 1e6:.1f} us", flush=True)
        plan = kkt.Prepared.solve_problem(dev, opts, out=sol, ctx=ctx)
        plan()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(steps):
            plan()
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ctx.wait_status(1)
        print(mode, "replay result identical:", same, f"Prepared event {e0.elapsed_time(e1) / steps * 1e3:.1f} us",
              f"wall {(t1 - t0) / steps * 1e6:.1f} us", flush=True)
