"""Compact summary of an `ncu --set full` capture for profiles/ (committed):
duration, DRAM bytes, throughput, occupancy, issue, pipe utilisation, stall
breakdown and the hottest source lines.

    python tools/ncu_summary.py REPORT KERNEL_REGEX OUT_PREFIX [--algo-flops F] [--algo-bytes B]

writes OUT_PREFIX.json (machine-readable; bench.py reads `dram_bytes` as the
roofline `traffic`) and OUT_PREFIX.txt (human-readable, with the top lines).
"""
import argparse
import csv
import io
import json
import subprocess
import sys

RAW_KEYS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dynamic": "launch__shared_mem_per_block_dynamic",
    "dmma_pipe_pct": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dfma_thread_inst": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
}


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def raw_metrics(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        raise SystemExit(f"no kernel matching {kern} in {rep}")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    res = {"kernel": d.get("Kernel Name", "")}
    for k, m in RAW_KEYS.items():
        if m in d:
            v = _num(d[m])
            unit = u.get(m, "")
            if v is not None and unit in ("Kbyte", "Mbyte", "Gbyte", "byte"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
            if v is not None and unit in ("usecond", "msecond", "nsecond", "us", "ms", "ns"):
                v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}[unit]
            res[k] = v
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): _num(v)
              for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in
                          sorted(stalls.items(), key=lambda kv: -(kv[1] or 0)) if v and v / tot > 0.01}
    if res.get("dram_read_bytes") is not None and res.get("dram_write_bytes") is not None:
        res["dram_bytes"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    return res


def top_lines(rep, kern, n=15):
    out = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, kern,
                          str(n)], capture_output=True, text=True).stdout
    return out.strip().splitlines()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("out")
    ap.add_argument("--algo-flops", type=float, default=None)
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    ap.add_argument("--batch", type=int, default=None, help="instances of the captured launch")
    ap.add_argument("--config", type=int, default=None, help="BASELINE config of the capture")
    a = ap.parse_args()
    res = raw_metrics(a.report, a.kernel)
    res["report"] = a.report.split("/")[-1]
    res["note"] = a.note
    if a.batch is not None:
        res["batch"] = a.batch
    if a.config is not None:
        res["config"] = a.config
    if a.algo_flops and res.get("duration_ns"):
        res["algo_flops"] = a.algo_flops
        res["algo_tflops_under_ncu"] = a.algo_flops / res["duration_ns"] / 1e3
    if a.algo_bytes:
        res["algo_bytes"] = a.algo_bytes
        if res.get("dram_bytes"):
            res["dram_over_algo_bytes"] = res["dram_bytes"] / a.algo_bytes
    lines = top_lines(a.report, a.kernel)
    with open(a.out + ".json", "w") as fh:
        json.dump(res, fh, indent=1)
    with open(a.out + ".txt", "w") as fh:
        fh.write(f"# {res['kernel']}\n# {a.note}\n")
        for k, v in res.items():
            if k not in ("kernel", "stall_share"):
                fh.write(f"{k:28s} {v}\n")
        fh.write("stall share: " + json.dumps(res["stall_share"]) + "\n\n")
        fh.write("hottest source lines (warp-stall samples):\n")
        fh.write("\n".join(lines) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
