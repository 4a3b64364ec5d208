"""Measurement of the batched exact line search at the
config-4 QPALM size: 512 instances x m = 2 ny (N+1) = 12336 terms (lower and
upper side of each of the ny = 24 rows of the N + 1 = 257 stages,
qpalm.cpp:285-296), seeded synthetic terms (synth.line_search_data).

    python tools/linesearch_bench.py [--batch 512] [--m 12336] [--reps 20]

Prints one JSON line: GPU line searches/s (device-resident inputs, CUDA
events), the HBM roofline of the kernel (algorithmic bytes: alpha + delta
read once, the (t, w) scratch written once, eta / beta / tau), probes per
instance, and the reference's CPU line_search_exact on all host cores
(oracle/_ref, the CPU baseline)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_09058_b200 import kkt, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--m", type=int, default=2 * 24 * 257)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    a = ap.parse_args()
    alpha, delta, eta, beta = synth.line_search_data(a.batch, a.m, seed=0)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (alpha, delta, eta, beta)]
    (tau, its) = kkt.line_search_exact(*dev, iterations=True)
    for _ in range(3):
        kkt.line_search_exact(*dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = kkt.Context.default()
    ctx.profile(True)
    ctx.profile_read(reset=True)
    e0.record()
    for _ in range(a.reps):
        kkt.line_search_exact(*dev)
    e1.record()
    torch.cuda.synchronize()
    ms_call = e0.elapsed_time(e1) / a.reps
    k_ms = ctx.profile_read(reset=True)["augment"][0] / a.reps  # slot 4: the line-search kernel
    ctx.profile(False)
    B, m = a.batch, a.m
    algo_bytes = B * m * 8 * 2 + B * m * 16 + B * 8 * 3
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    line = {"metric": "exact line searches per sec (FP64)", "workload":
            f"{B} instances x {m} terms (config-4 QPALM size), seeded synthetic",
            "value": B / (k_ms * 1e-3), "unit": "line searches/s", "kernel_ms": k_ms,
            "call_ms": ms_call, "probes_per_instance_mean": float(its.float().mean()),
            "probes_per_instance_max": int(its.max()),
            "roofline": {"bound": "hbm", "algo_bytes": algo_bytes,
                         "achieved_gbs": algo_bytes / (k_ms * 1e-3) / 1e9, "peak_gbs": hbm,
                         "frac": (algo_bytes / (k_ms * 1e-3) / 1e9 / hbm) if hbm else None}}
    try:
        from pyoracle import RefOracle, ref_available
        if ref_available():
            ref = RefOracle()
            tr, rc, it = ref.line_search(alpha[:8], delta[:8], eta[:8], beta[:8])
            got = tau[:8].cpu().numpy()
            line["parity_vs_reference_max_rel"] = float(np.max(np.abs(got - tr) / np.maximum(1, np.abs(tr))))
            threads = os.cpu_count() or 1
            n = 0
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < a.cpu_seconds:
                ref.bench_line_search(alpha[:64], delta[:64], eta[:64], beta[:64], threads)
                n += 64
            t = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": n / t, "unit": "line searches/s", "cores": threads,
                                    "kind": "reference",
                                    "sample": f"{n} line_search_exact over 64 cycled instances in {t:.1f} s"}
    except Exception as e:  # reference build absent on this host
        line["cpu_baseline"] = {"unavailable": str(e)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
