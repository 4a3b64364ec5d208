"""Benchmark of the B200 KKT factor+solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = kkt::solve_problem (factor + solve with EqRhs::of_problem) of a
batch of independent OCP instances -- BASELINE config 1 by default: 1024
instances, N=128, nx=20, nu=10, P=16, FP64, seeded synthetic data from
paper_2512_09058_b200/synth.py (no public suite exists for this path).

`value`  : solves/s with inputs resident in HBM (device pointers through the
           C ABI), CUDA events on the launching stream, max over ranks.
`e2e`    : the same through the public API with pinned HOST buffers: every
           step copies the problem batch H2D and the solution D2H.
`roofline`: dominant kernel (riccati_panel_kernel), algorithmic FP64 FLOPs
           per launch (reference FMA counter restated in flops.py) / its
           CUDA-event duration, against the measured FP64 DMMA peak.
`cpu_baseline`: the reference's own factor+solve built from its sources
           (oracle/_ref, "reference"; the C restatement "port" if absent) on
           a bounded sample, all host cores, rank 0 at N=1 only.
Multi-GPU (torchrun): each rank solves its own 1024-instance shard (weak
scaling, no collective on the data path); value = all instances / max time.
`--impl reference` times the reference's CPU factor+solve on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2512_09058_b200 import shard, synth  # noqa: E402
from paper_2512_09058_b200.flops import (assembly_flops, fma_phases, flops_per_solve, problem_bytes,  # noqa: E402
                                         solution_bytes)

METRIC = ("OCP KKT factor+solve per sec (FP64) and achieved fraction of FP64 roofline")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        self.lines = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return self

        def reader():
            for line in self.proc.stdout:
                self.lines.append(line)

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        # the timed region starts once the sampler is live (nvidia-smi can take
        # a second to initialise; a short run would otherwise see no sample)
        t0 = time.time()
        while not self.lines and time.time() - t0 < 10 and self.proc.poll() is None:
            time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        # at least two samples after the timed region ended
        n0, t0 = len(self.lines), time.time()
        while len(self.lines) < n0 + 2 and time.time() - t0 < 3 and self.proc.poll() is None:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=5)
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as fh:
            d = json.loads(fh.readline())
        return float(d["dmma_tflops"]), "measured (tools/fp64_peak.cu, DMMA m8n8k4 f64 burst)"
    except Exception:
        return 37.0, "fallback: B200 FP64 tensor datasheet ~37 TFLOP/s"


def ncu_traffic(kernel_tag, cfg_idx, batch):
    """DRAM bytes per launch of a kernel from the committed `ncu --set full`
    summary (profiles/ncu_r01_<tag>[_cfgK].json, tools/ncu_summary.py) -- only
    for the workload it was captured on (config 1: 1024 instances, config 4:
    512 instances, one Newton system)."""
    name = {(1, 1024): kernel_tag, (4, 512): f"{kernel_tag}_cfg4"}.get((cfg_idx, batch))
    path = os.path.join(ROOT, "profiles", f"ncu_r01_{name}.json")
    if name is None or not os.path.exists(path):
        return None, None
    with open(path) as fh:
        d = json.load(fh)
    return d.get("dram_bytes"), f"profiles/ncu_r01_{name}.json ({d.get('report')})"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


_CAL = {}


def cpu_reference_rate(p, P, target_s, impl_kind=None, threads=None):
    """Reference CPU factor+solve throughput on a bounded sample (solves/s);
    the sample size is calibrated once to ~target_s seconds."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle  # CPU checker / baseline only

    threads = threads or os.cpu_count() or 1
    kind = impl_kind
    try:
        if kind in (None, "reference"):
            orc = pyoracle.RefOracle()
            kind = "reference"
            run = lambda n: orc.bench(p, P, n, threads, vlen=4)  # noqa: E731
        else:
            raise RuntimeError
    except Exception:
        orc = pyoracle.Oracle()
        kind = "port"
        run = lambda n: orc.bench(p, P, n, threads)  # noqa: E731
    key = (id(p), kind, threads)
    if key not in _CAL:
        # two-stage calibration: the first short run includes thread start-up
        n0 = max(4 * threads, 64)
        t0 = run(n0)
        if t0 <= 0:
            raise RuntimeError("CPU baseline failed")
        n1 = max(n0, int(n0 * min(2.0, target_s / 4) / max(t0, 1e-6)))
        t1 = run(n1)
        _CAL[key] = max(n1, int(n1 * target_s / max(t1, 1e-6)))
    n = _CAL[key]
    t = run(n)
    if t <= 0:
        raise RuntimeError("CPU baseline failed")
    return n / t, kind, threads, n, t


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    sample = synth.generate(args.config, seed=args.seed, batch=min(64, cfg.batch))
    rates = []
    args.cpu_seconds = min(args.cpu_seconds, 8.0)
    for i in range(args.warmup + args.steps):
        rate, kind, threads, n, t = cpu_reference_rate(sample, cfg.P, args.cpu_seconds)
        if i >= args.warmup:
            rates.append((rate, n, t))
    value = statistics.median(r[0] for r in rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.batch / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, cfg),
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": kind,
                         "sample": f"{rates[0][1]} factor+solve of {sample.batch} cycled "
                                   f"config-{cfg.idx} instances per step (~{args.cpu_seconds:.0f} s)"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, cfg):
    d = {"workload": f"config {cfg.idx}: {cfg.name}", "batch_per_gpu": cfg.batch,
         "N": cfg.N, "nx": cfg.nx, "nu": cfg.nu, "P": cfg.P, "seed": args.seed,
         "parallelism": f"instance-sharded x{args.gpus}",
         "l2": "inputs larger than L2 (no flush)"}
    if cfg.iters > 1:
        d.update({"newton_iters_per_step": cfg.iters, "ny": cfg.ny,
                  "step": "per iteration: GPU Newton-system assembly + factor + solve"})
    return d


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_09058_b200 import kkt
    from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch

    cfg = synth.CONFIGS[args.config]
    B = cfg.batch
    t0 = time.time()
    p, _ = shard.generate_shard(args.config, args.seed, rank, ws, per_rank=B)  # weak scaling
    log(f"[rank {rank}] generated {B} instances ({p.nbytes() / 1e9:.2f} GB) in "
        f"{time.time() - t0:.1f}s")
    opts = kkt.FactorOptions(P=cfg.P)
    stream = torch.cuda.current_stream()
    ctx = kkt.Context(local)
    ctx.set_stream(stream.cuda_stream)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return shard.max_over_ranks(x, device="cuda")

    # ---- device-resident inputs -----------------------------------------
    # config 4 (QPALM Newton systems): one step = `iters` successive
    # refactorizations per instance, each = GPU Newton-system assembly
    # (qpalm::assemble_newton, Σ of that iteration) + factor + solve; D, C and
    # the whole Σ sequence are resident like the problem data.
    iters = cfg.iters
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(dev, k, torch.from_numpy(getattr(p, k)).to("cuda"))
    if iters > 1:
        Dh, Eh, sigh = synth.qpalm_data(p, seed=args.seed, iters=iters, ny=cfg.ny,
                                        start=rank * B)
        Dd, Ed, sigd = (torch.from_numpy(a).to("cuda") for a in (Dh, Eh, sigh))

    def one_step(src, out):
        if iters == 1:
            kkt.solve_problem(src, opts, ctx=ctx, out=out)
            return
        # each Newton system: assembly fused into the factorization's stage
        # loads (kkt.solve_newton), factor + solve
        for it in range(iters):
            kkt.solve_newton(src, Dd, Ed, sigd[it], opts, ctx=ctx, out=out)

    sol = kkt._alloc_sol(dev, True)
    for _ in range(args.warmup):
        one_step(dev, sol)
    barrier()
    ctx.profile(True)
    ctx.profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            one_step(dev, sol)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    kern = ctx.profile_read(reset=True)
    ctx.profile(False)
    ms = max_over_ranks(ms)
    value = ws * B * iters / (ms * 1e-3)

    # ---- end to end: pinned host buffers, H2D + D2H inside the timed region
    pin = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(pin, k, torch.from_numpy(getattr(p, k)).pin_memory().numpy())
    hsol = kkt.EqSolutionBatch(*[torch.zeros(getattr(sol, k).shape, dtype=torch.float64)
                                 .pin_memory().numpy() for k in ("u", "x", "lam")])
    h2d_extra = 0
    if iters == 1:
        def e2e_step():
            kkt.solve_problem(pin, opts, ctx=ctx, out=hsol)
    else:
        # host problem, D, C and Σ sequence pinned; H2D inside the step, every
        # iteration's solution copied back to the host
        pins = [torch.from_numpy(a).pin_memory() for a in (Dh, Eh, sigh)]
        h2d_extra = sum(t.numel() * 8 for t in pins)
        dsol = kkt._alloc_sol(dev, True)
        hsols = [torch.zeros(dsol.u.shape, dtype=torch.float64).pin_memory() for _ in range(3)]

        def e2e_step():
            for k in OCP_FIELDS:
                getattr(dev, k).copy_(torch.from_numpy(getattr(pin, k)), non_blocking=True)
            for dst, src in zip((Dd, Ed, sigd), pins):
                dst.copy_(src, non_blocking=True)
            for it in range(iters):
                kkt.solve_newton(dev, Dd, Ed, sigd[it], opts, ctx=ctx, out=dsol)
                for h, d in zip((hsol.u, hsol.x, hsol.lam), (dsol.u, dsol.x, dsol.lam)):
                    torch.from_numpy(h).copy_(d, non_blocking=True)
    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    e2e = ws * B * iters / (ms_e2e * 1e-3)
    # spot parity of this run's result against the device run
    assert np.array_equal(hsol.u[:4], sol.u[:4].cpu().numpy())

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel --------------------------------
    ph = fma_phases(cfg.N, cfg.nx, cfg.nu, cfg.P)
    k_ms, k_n = kern["riccati_panel"]
    k_avg = k_ms / max(k_n, 1)  # one stage-panel launch per step
    aug_fl = assembly_flops(cfg.N, cfg.nx, cfg.nu, cfg.ny) if iters > 1 else 0.0
    k_flops = (2.0 * ph["kernel_riccati_panel"] + aug_fl) * B  # config 4: assembly fused in
    peak, peak_src = fp64_peak()
    achieved = k_flops / (k_avg * 1e-3) / 1e12
    step_ms_k = sum(v[0] for v in kern.values()) / max(args.steps, 1)
    shares = {k: round(v[0] / max(sum(x[0] for x in kern.values()), 1e-9), 4)
              for k, v in kern.items() if v[1]}
    hbm, hbm_src = hbm_peak()
    traffic, traffic_src = ncu_traffic("riccati", cfg.idx, B)
    # the other two kernels against their own bounds (algorithmic bytes:
    # DESIGN.md §6; the CR/Schur kernel is latency-bound, reported in FLOP/s)
    kms = {k: v[0] / max(v[1], 1) for k, v in kern.items() if v[1]}
    n_per = (cfg.N + cfg.P - 1) // cfg.P
    chains = B * cfg.P
    fac_bytes = chains * n_per * (-(-(cfg.nx + cfg.nu) // 8) * (-(-(cfg.nx + cfg.nu) // 8) + 1) // 2
                                  + -(-(cfg.nx + 1) // 8) * -(-(cfg.nx + cfg.nu) // 8)) * 512
    back_bytes = fac_bytes + B * cfg.N * (cfg.nx * cfg.nx + cfg.nx * cfg.nu) * 8 \
        + solution_bytes(cfg.N, cfg.nx, cfg.nu) * B
    kernel_rooflines = {}
    if "backsub" in kms:
        kernel_rooflines["backsub"] = {
            "bound": "hbm", "unit": "GB/s", "algo_bytes": back_bytes,
            "achieved": back_bytes / (kms["backsub"] * 1e-3) / 1e9, "peak": hbm,
            "frac": back_bytes / (kms["backsub"] * 1e-3) / 1e9 / hbm}
    if "schur_cr" in kms:
        sf = 2.0 * ph["kernel_schur_cr"] * B
        kernel_rooflines["schur_cr"] = {
            "bound": "latency (CR tree depth)", "unit": "TFLOP/s", "algo_flops": sf,
            "achieved": sf / (kms["schur_cr"] * 1e-3) / 1e12, "peak": peak,
            "frac": sf / (kms["schur_cr"] * 1e-3) / 1e12 / peak}
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config generators, synth.py)",
        "config": config_dict(args, cfg),
        "e2e": {"value": e2e, "unit": "solves/s",
                "h2d_bytes_per_step": problem_bytes(cfg.N, cfg.nx, cfg.nu) * B + h2d_extra,
                "d2h_bytes_per_step": solution_bytes(cfg.N, cfg.nx, cfg.nu) * B * iters,
                "ms_per_step": ms_e2e},
        "roofline": {"bound": "tensor", "kernel": "riccati_panel_kernel",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "flops_per_launch": k_flops, "launch_ms": k_avg},
        "step_roofline": {
            "flops_per_step": (flops_per_solve(cfg.N, cfg.nx, cfg.nu, cfg.P) + aug_fl) * B * iters,
            "tflops": (flops_per_solve(cfg.N, cfg.nx, cfg.nu, cfg.P) + aug_fl) * B * iters
            / (ms * 1e-3) / 1e12,
            "frac_fp64": (flops_per_solve(cfg.N, cfg.nx, cfg.nu, cfg.P) + aug_fl) * B * iters
            / (ms * 1e-3) / 1e12 / peak,
            "compulsory_bytes": (problem_bytes(cfg.N, cfg.nx, cfg.nu)
                                 + solution_bytes(cfg.N, cfg.nx, cfg.nu)) * B,
            "hbm_gbs_peak": hbm, "hbm_source": hbm_src},
        "kernel_rooflines": kernel_rooflines,
        "kernel_shares": shares, "kernel_ms_per_step": {k: v[0] / max(args.steps, 1)
                                                        for k, v in kern.items() if v[1]},
        "kernel_sum_ms_per_step": step_ms_k,
        "gpu_launches": int(sum(v[1] for v in kern.values())),
        "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_cpu:
        sample = p.subset(np.arange(min(64, B)))
        if iters > 1:  # CPU reference on iteration 0's Newton systems (assembly not timed)
            sample = next(synth.qpalm_sequence(sample, seed=args.seed, iters=1, ny=cfg.ny))
        rate, kind, threads, n, t = cpu_reference_rate(sample, cfg.P, args.cpu_seconds)
        line["cpu_baseline"] = {
            "value": rate, "unit": "solves/s", "cores": threads, "kind": kind,
            "sample": f"{n} factor+solve over 64 cycled config-{cfg.idx} instances in {t:.1f} s"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
