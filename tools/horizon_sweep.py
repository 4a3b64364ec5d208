"""Single-instance latency of kkt::solve_problem versus horizon length at the
BASELINE config-2 stage shape (nx = 12, nu = 4), P = N / 16 partitions (16
stages per partition column, so the cyclic-reduction tree deepens by one
level per doubling of N). Device-resident inputs, CUDA events, median of
`reps` runs; one JSON line per N plus a summary (ms per doubling).

    python tools/horizon_sweep.py [reps] > profiles/horizon_sweep_r01.jsonl
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402
from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ctx = kkt.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
rows = []
for N in (256, 512, 1024, 2048, 4096, 8192, 16384):
    P = N // 16
    p = synth.generate(2, seed=0, batch=1, N=N)
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(dev, k, torch.from_numpy(getattr(p, k)).cuda())
    opts = kkt.FactorOptions(P=P)
    sol = kkt._alloc_sol(dev, True)
    for _ in range(5):
        kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
    torch.cuda.synchronize()
    ts = []
    ctx.profile(True)
    ctx.profile_read(reset=True)
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        kkt.solve_problem(dev, opts, ctx=ctx, out=sol)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    kern = ctx.profile_read(reset=True)
    ctx.profile(False)
    row = {"N": N, "P": P, "cr_levels": P.bit_length() - 1, "ms_median": statistics.median(ts),
           "ms_min": min(ts),
           "kernel_ms": {k: round(v[0] / reps, 4) for k, v in kern.items() if v[1]}}
    rows.append(row)
    print(json.dumps(row), flush=True)
steps = [b["ms_median"] - a["ms_median"] for a, b in zip(rows, rows[1:])]
print(json.dumps({"summary": "latency vs horizon at nx=12 nu=4, P=N/16",
                  "ms_added_per_doubling": [round(x, 4) for x in steps],
                  "ratio_N16384_over_N256": rows[-1]["ms_median"] / rows[0]["ms_median"],
                  "N_ratio": 64}))
