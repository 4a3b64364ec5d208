"""Benchmark of the B200 KKT factor+solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--extra 1,4,0,2 | --extra none]

One step = kkt::solve_problem (factor + solve with EqRhs::of_problem) of a
batch of independent OCP instances. The headline line is BASELINE config 3
(256 instances, N=512, nx=64, nu=32, P=32) -- the largest single-GPU
configuration, the dense FP64 DMMA regime; configs 1 and 4 (batched) and 0
and 2 (single-instance latency) are measured in the same run and reported
under "configs". FP64, seeded synthetic data from
paper_2512_09058_b200/synth.py (no public suite exists for this path).

`value`   : solves/s with inputs resident in HBM (device pointers through the
            C ABI), CUDA events on the launching stream, max over ranks.
            Config 4: Newton systems/s (20 refactorizations per instance).
`e2e`     : the same through the public API with pinned HOST buffers: every
            step copies the problem batch H2D and the solution D2H.
`roofline`: dominant kernel (the stage panel), algorithmic FP64 FLOPs per
            launch (reference FMA counter restated in flops.py) / its
            CUDA-event duration, against the measured FP64 DMMA peak;
            `traffic` = its DRAM bytes per launch from the committed ncu
            capture of the same workload.
`parity`  : 8 sampled instances of the timed run checked against the C
            oracle (solution rel. error, KKT residual).
`cpu_baseline`: the reference's own factor+solve built from its sources
            (oracle/_ref, "reference"; the C restatement "port" if absent),
            rank 0 at N=1: instance-parallel on all host cores for batches,
            the best single-instance latency over vlen x workers for
            configs 0 / 2.
Multi-GPU (torchrun): the fixed BASELINE batch is sharded into contiguous
instance ranges, one per rank (strong scaling, no collective on the data
path); value = all instances / max-over-ranks time. Single-instance
configs are replicas only.
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
HEADLINE = 3
LATENCY_CONFIGS = (0, 2)
# the stage-panel kernel each config runs (the dominant kernel of the step)
PANEL_KERNEL = {0: "riccati_pc_kernel<5,10>", 1: "riccati_warp_kernel<10,20,1,0,0>",
                2: "riccati_pc_kernel<4,12>", 3: "riccati_cta_kernel<32,64,16>",
                4: "riccati_warp_kernel<8,16,1,24,0> (fused Newton assembly)"}


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


def ncu_traffic(cfg_idx, batch):
    """DRAM bytes per launch of the config's stage-panel kernel from the
    committed `ncu --set full` summary of the same workload
    (profiles/ncu_r0X_panel_cfgK.json, tools/ncu_summary.py), newest round
    first; None if no capture of this exact batch exists."""
    for name in (f"ncu_r02b_panel_cfg{cfg_idx}", f"ncu_r02_panel_cfg{cfg_idx}", f"ncu_r01_panel_cfg{cfg_idx}"):
        path = os.path.join(ROOT, "profiles", name + ".json")
        if not os.path.exists(path):
            continue
        with open(path) as fh:
            d = json.load(fh)
        if int(d.get("batch", -1)) == batch:
            return d.get("dram_bytes"), f"profiles/{name}.json ({d.get('report')})"
    return None, None


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


_CAL = {}


def _oracles():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle  # CPU checker / baseline only
    return pyoracle


def cpu_reference_rate(p, P, target_s, threads=None):
    """Reference CPU factor+solve throughput, instance-parallel over `threads`
    host threads on a bounded sample (solves/s); the sample size is
    calibrated once to ~target_s seconds."""
    pyoracle = _oracles()
    threads = threads or os.cpu_count() or 1
    try:
        orc = pyoracle.RefOracle()
        kind = "reference"
        run = lambda n: orc.bench(p, P, n, threads, vlen=4)  # noqa: E731
    except Exception:
        orc = pyoracle.Oracle()
        kind = "port"
        run = lambda n: orc.bench(p, P, n, threads)  # noqa: E731
    key = (id(p), kind, threads)
    if key not in _CAL:
        # two-stage calibration: the first short run includes thread start-up
        n0 = max(threads, min(64, 4 * threads))
        t0 = run(n0)
        if t0 <= 0:
            raise RuntimeError("CPU baseline failed")
        n1 = max(n0, int(n0 * min(2.0, target_s / 4) / max(t0, 1e-6)))
        t1 = run(n1)
        _CAL[key] = max(threads, n1, int(n1 * target_s / max(t1, 1e-6)))
    n = _CAL[key]
    t = run(n)
    if t <= 0:
        raise RuntimeError("CPU baseline failed")
    return n / t, kind, threads, n, t


def cpu_reference_latency(p, P, target_s):
    """Best single-instance latency of the reference: kkt::factor
    + kkt::solve of one instance, best over vlen in {1, 4, 8} x workers in
    {1, cores}, each the best of repeated runs. Returns (seconds, vlen,
    workers, reps, kind)."""
    pyoracle = _oracles()
    cores = os.cpu_count() or 1
    orc = pyoracle.RefOracle()
    t1 = orc.bench_latency(p, P, 4, 1, 1)
    reps = int(max(3, min(200, target_s / 6 / max(t1, 1e-6))))
    best = None
    for vlen in (1, 4, 8):
        for workers in sorted({1, cores}):
            t = orc.bench_latency(p, P, vlen, workers, reps)
            if t > 0 and (best is None or t < best[0]):
                best = (t, vlen, workers)
    return best[0], best[1], best[2], reps, "reference"


def config_dict(cfg, ws, batch_local, seed):
    d = {"workload": f"config {cfg.idx}: {cfg.name}", "batch": cfg.batch,
         "batch_per_gpu": batch_local, "N": cfg.N, "nx": cfg.nx, "nu": cfg.nu, "P": cfg.P,
         "seed": seed,
         "parallelism": (f"instance-sharded x{ws} (strong)" if cfg.batch > 1
                         else f"replicas x{ws}" if ws > 1 else "single instance"),
         "l2": "inputs larger than L2 (no flush)" if cfg.batch > 1 else
               "single instance, L2-resident between steps (latency)"}
    if cfg.iters > 1:
        d.update({"newton_iters_per_step": cfg.iters, "ny": cfg.ny,
                  "step": "per iteration: GPU Newton-system assembly (fused) + factor + solve"})
    return d


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    sample = synth.generate(args.config, seed=args.seed, batch=min(64, cfg.batch))
    cores = os.cpu_count() or 1
    steps = []
    for i in range(args.warmup + args.steps):
        if cfg.batch == 1:
            t, vlen, workers, reps, kind = cpu_reference_latency(sample, cfg.P, min(args.cpu_seconds, 3.0))
            rate, desc = 1.0 / t, f"best of {reps} single-instance solves, vlen={vlen} workers={workers}"
            threads = workers
        else:
            rate, kind, threads, n, t = cpu_reference_rate(sample, cfg.P, min(args.cpu_seconds, 4.0))
            desc = (f"{n} factor+solve of {sample.batch} cycled config-{cfg.idx} instances per step "
                    f"(~{min(args.cpu_seconds, 4.0):.0f} s), instance-parallel")
        if i >= args.warmup:
            steps.append((rate, desc, threads))
    value = statistics.median(r[0] for r in steps)
    if cfg.iters > 1:
        value_unit = "Newton systems/s"
    else:
        value_unit = "solves/s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": value_unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.batch / value, "higher_is_better": True,
        "scaling": "strong" if cfg.batch > 1 else "replicas", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(cfg, args.gpus, cfg.batch, args.seed),
        "cpu_baseline": {"value": value, "unit": value_unit, "cores": steps[0][2], "host_cores": cores,
                         "cpu": cpu_model(), "kind": "reference", "sample": steps[0][1]},
        "e2e": {"value": value, "unit": value_unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def check_parity(p_host, start, sol_dev, cfg, seed):
    """8 sampled instances of the timed run's solution against the C oracle
    (config 4: the last Newton system of the sequence, rebuilt on the host)."""
    from paper_2512_09058_b200.ocp import EqRhsBatch, EqSolutionBatch, kkt_residual, rel_error, residual_scale

    pyoracle = _oracles()
    orc = pyoracle.Oracle()
    B = p_host.batch
    idx = sorted(set(np.linspace(0, B - 1, min(8, B)).round().astype(int).tolist()))
    errs, ress, scaled = [], [], []
    for i in idx:
        q = p_host.subset([i])
        if cfg.iters > 1:
            for q in synth.qpalm_sequence(p_host.subset([i]), seed=seed, iters=cfg.iters, ny=cfg.ny,
                                          start=start + i):
                pass
        ref, rc, _ = orc.solve_problem(q, cfg.P)
        if rc != 0:
            return {"error": f"oracle failed on instance {start + i}"}
        got = EqSolutionBatch(*[getattr(sol_dev, k)[i:i + 1].cpu().numpy() for k in ("u", "x", "lam")])
        rhs = EqRhsBatch.of_problem(q)
        errs.append(float(rel_error(got, ref).max()))
        r = kkt_residual(q, rhs, got).max(axis=1)
        ress.append(float(r.max()))
        scaled.append(float((r / residual_scale(q, rhs, got)).max()))
    out = {"instances": [start + i for i in idx], "checker": "C oracle (oracle/cyq_oracle.c)",
           "max_rel_error": max(errs), "max_kkt_residual": max(ress),
           "max_scaled_residual": max(scaled), "rel_error_bar": 1e-9}
    if cfg.iters > 1:
        out["residual_bar"] = "scale-aware <= 1e-16 (Hessians ~1e5; SURVEY §7.6)"
        out["ok"] = out["max_rel_error"] <= 1e-9 and out["max_scaled_residual"] <= 1e-16
    else:
        out["residual_bar"] = 1e-10
        out["ok"] = out["max_rel_error"] <= 1e-9 and out["max_kkt_residual"] <= 1e-10
    return out


def measure(args, cfg_idx, ctx, stream, ws, rank, local, primary):
    """Times config `cfg_idx` on this rank's shard; returns (line dict or
    None on rank != 0)."""
    import torch

    from paper_2512_09058_b200 import kkt
    from paper_2512_09058_b200.ocp import OCP_FIELDS, EqOCPBatch

    cfg = synth.CONFIGS[cfg_idx]
    t0 = time.time()
    if cfg.batch > 1:  # strong scaling: the fixed BASELINE batch, one contiguous range per rank
        p, start = shard.generate_shard(cfg_idx, args.seed, rank, ws, total=cfg.batch)
    else:              # single instance: replicas only (a long horizon stays on one GPU)
        p, start = synth.generate(cfg_idx, seed=args.seed, batch=1), 0
    B = p.batch
    log(f"[rank {rank}] config {cfg_idx}: generated {B} instances ({p.nbytes() / 1e9:.2f} GB) "
        f"in {time.time() - t0:.1f}s")
    opts = kkt.FactorOptions(P=cfg.P)
    iters = cfg.iters

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
    # (qpalm::assemble_newton, Σ of that iteration; fused into the panel's
    # stage loads) + factor + solve; D, C and the whole Σ sequence are
    # resident like the problem data.
    dev = EqOCPBatch.__new__(EqOCPBatch)
    for k in OCP_FIELDS:
        setattr(dev, k, torch.from_numpy(getattr(p, k)).to("cuda"))
    if iters > 1:
        Dh, Eh, sigh = synth.qpalm_data(p, seed=args.seed, iters=iters, ny=cfg.ny, start=start)
        Dd, Ed, sigd = (torch.from_numpy(a).to("cuda") for a in (Dh, Eh, sigh))

    def one_step(src, out):
        if iters == 1:
            kkt.solve_problem(src, opts, ctx=ctx, out=out)
            return
        for it in range(iters):
            kkt.solve_newton(src, Dd, Ed, sigd[it], opts, ctx=ctx, out=out)

    def make_fast_step(src, out):
        # the same calls through kkt.Prepared (argument blocks built once)
        if iters == 1:
            plan = kkt.Prepared.solve_problem(src, opts, out=out, ctx=ctx)
            return plan
        plan = kkt.Prepared.solve_newton(src, Dd, Ed, opts, out=out, ctx=ctx)
        sig_it = [sigd[it] for it in range(iters)]

        def step():
            for s_ in sig_it:
                plan(s_)
        return step

    # latency configs: more steps (each ~0.1 ms) for a stable median-free mean
    steps = args.steps * (20 if cfg.batch == 1 else 1)
    sol = kkt._alloc_sol(dev, True)
    # device-resident loop: stream-ordered calls without a host sync each
    # (the per-instance status of the run is checked after it); repeated
    # identical calls replay a captured CUDA graph (CYQ_OPT_GRAPHS)
    ctx.set_option("async_status", 1)
    for _ in range(args.warmup):
        one_step(dev, sol)
    barrier()
    ctx.profile(True)
    ctx.profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(steps):
            one_step(dev, sol)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / steps
    kern = ctx.profile_read(reset=True)
    ctx.profile(False)
    # the same loop without the per-kernel events (they add host work between
    # the launches of a latency-bound step), through kkt.Prepared: the
    # reported time
    fast = make_fast_step(dev, sol)
    for _ in range(2):
        fast()
    barrier()
    e0.record(stream)
    for _ in range(steps):
        fast()
    e1.record(stream)
    barrier()
    ms = min(ms, e0.elapsed_time(e1) / steps)
    ctx.wait_status(B)  # raises FactorizeError if any instance failed
    ctx.set_option("async_status", 0)
    ms = max_over_ranks(ms)
    total = cfg.batch if cfg.batch > 1 else ws  # replicas: one instance per rank
    value = total * iters / (ms * 1e-3)

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

        def e2e_step():
            for k in OCP_FIELDS:
                getattr(dev, k).copy_(torch.from_numpy(getattr(pin, k)), non_blocking=True)
            for dst, src in zip((Dd, Ed, sigd), pins):
                dst.copy_(src, non_blocking=True)
            for it in range(iters):
                kkt.solve_newton(dev, Dd, Ed, sigd[it], opts, ctx=ctx, out=dsol)
                for h, d in zip((hsol.u, hsol.x, hsol.lam), (dsol.u, dsol.x, dsol.lam)):
                    torch.from_numpy(h).copy_(d, non_blocking=True)
    e2e_steps = max(1, steps if cfg.batch == 1 else args.steps)
    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    e2e = total * iters / (ms_e2e * 1e-3)
    # the host-buffer run must reproduce the device run bit for bit
    e2e_same = bool(np.array_equal(hsol.u, sol.u.cpu().numpy()))
    parity = check_parity(p, start, sol, cfg, args.seed) if rank == 0 and not args.no_parity else None
    if rank != 0:
        return None

    # ---- roofline of the dominant kernel --------------------------------
    ph = fma_phases(cfg.N, cfg.nx, cfg.nu, cfg.P)
    k_ms, k_n = kern["riccati_panel"]
    k_avg = k_ms / max(k_n, 1)  # one stage-panel launch per Newton system
    aug_fl = assembly_flops(cfg.N, cfg.nx, cfg.nu, cfg.ny) if iters > 1 else 0.0
    k_flops = (2.0 * ph["kernel_riccati_panel"] + aug_fl) * B  # config 4: assembly fused in
    peak, peak_src = fp64_peak()
    achieved = k_flops / (k_avg * 1e-3) / 1e12
    kern_sum = sum(v[0] for v in kern.values())
    shares = {k: round(v[0] / max(kern_sum, 1e-9), 4) for k, v in kern.items() if v[1]}
    hbm, hbm_src = hbm_peak()
    traffic, traffic_src = ncu_traffic(cfg.idx, B)
    # the other two kernels against their own bounds (algorithmic bytes:
    # DESIGN.md §6; the CR/Schur kernel is latency-bound, reported in FLOP/s)
    kms = {k: v[0] / max(v[1], 1) for k, v in kern.items() if v[1]}
    n_per = (cfg.N + cfg.P - 1) // cfg.P
    chains = B * cfg.P
    CT, BT = -(-(cfg.nx + cfg.nu) // 8), -(-(cfg.nx + 1) // 8)
    fac_bytes = chains * n_per * (CT * (CT + 1) // 2 + BT * CT) * 512
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
    step_flops = (flops_per_solve(cfg.N, cfg.nx, cfg.nu, cfg.P) + aug_fl) * B * iters
    unit = "Newton systems/s" if iters > 1 else "solves/s"
    line = {
        "metric": METRIC, "value": value, "unit": unit, "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if cfg.batch > 1 else "replicas",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config generators, synth.py)",
        "config": config_dict(cfg, ws, B, args.seed),
        "e2e": {"value": e2e, "unit": unit,
                "h2d_bytes_per_step": problem_bytes(cfg.N, cfg.nx, cfg.nu) * B + h2d_extra,
                "d2h_bytes_per_step": solution_bytes(cfg.N, cfg.nx, cfg.nu) * B * iters,
                "ms_per_step": ms_e2e, "matches_device_run": e2e_same},
        "roofline": {"bound": "tensor", "kernel": PANEL_KERNEL.get(cfg.idx, "riccati panel"),
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "flops_per_launch": k_flops, "launch_ms": k_avg},
        "step_roofline": {
            "flops_per_step": step_flops, "tflops": step_flops / (ms * 1e-3) / 1e12,
            "frac_fp64": step_flops / (ms * 1e-3) / 1e12 / peak,
            "compulsory_bytes": (problem_bytes(cfg.N, cfg.nx, cfg.nu)
                                 + solution_bytes(cfg.N, cfg.nx, cfg.nu)) * B,
            "hbm_gbs_peak": hbm, "hbm_source": hbm_src},
        "kernel_rooflines": kernel_rooflines,
        "kernel_shares": shares, "kernel_ms_per_step": {k: v[0] / max(steps, 1)
                                                        for k, v in kern.items() if v[1]},
        "kernel_sum_ms_per_step": kern_sum / max(steps, 1),
        "gpu_launches": int(sum(v[1] for v in kern.values())),
        "clocks": clk.summary(),
    }
    if cfg.batch == 1:
        line["latency_ms"] = ms
    if parity is not None:
        line["parity"] = parity
    if ws == 1 and not args.no_cpu:
        host_cores = os.cpu_count() or 1
        if cfg.batch == 1:
            t, vlen, workers, reps, kind = cpu_reference_latency(p, cfg.P, args.cpu_seconds / 2)
            line["cpu_baseline"] = {
                "value": 1.0 / t, "unit": "solves/s", "latency_ms": 1e3 * t, "cores": workers,
                "host_cores": host_cores, "cpu": cpu_model(), "kind": kind,
                "sample": (f"single-instance factor+solve latency, best of {reps} reps at the best of "
                           f"vlen in (1, 4, 8) x workers in (1, {host_cores}): vlen={vlen}, "
                           f"workers={workers}")}
        else:
            sample = p.subset(np.arange(min(64, B)))
            if iters > 1:  # CPU reference on iteration 0's Newton systems (assembly not timed)
                sample = next(synth.qpalm_sequence(sample, seed=args.seed, iters=1, ny=cfg.ny))
            secs = args.cpu_seconds if primary else args.cpu_seconds / 2
            rate, kind, threads, n, t = cpu_reference_rate(sample, cfg.P, secs)
            line["cpu_baseline"] = {
                "value": rate, "unit": unit, "cores": threads, "host_cores": host_cores,
                "cpu": cpu_model(), "kind": kind,
                "sample": (f"{n} factor+solve over {sample.batch} cycled config-{cfg.idx} instances "
                           f"in {t:.1f} s, instance-parallel, FactorOptions{{P={cfg.P}, vlen=4, "
                           f"workers=1, cr1}}")}
    return line


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2512_09058_b200 import kkt

    # one dedicated stream for the library calls, torch's copies and the
    # timing events
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)
    ctx = kkt.Context(local)
    ctx.set_stream(stream.cuda_stream)
    order = [args.config] + [c for c in args.extra if c != args.config]
    if ws > 1:  # single-instance latency configs are replicas: headline only
        order = [c for i, c in enumerate(order) if i == 0 or c not in LATENCY_CONFIGS]
    lines = {}
    for i, c in enumerate(order):
        lines[c] = measure(args, c, ctx, stream, ws, rank, local, primary=(i == 0))
        torch.cuda.empty_cache()
    if rank == 0:
        line = lines[args.config]
        if len(order) > 1:
            line["configs"] = {str(c): lines[c] for c in order[1:]}
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
    ap.add_argument("--config", type=int, default=HEADLINE)
    ap.add_argument("--extra", default="1,4,0,2",
                    help="configs also measured in the same run (comma list, or 'none')")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    args.extra = [] if args.extra in ("", "none") else [int(c) for c in args.extra.split(",")]
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
