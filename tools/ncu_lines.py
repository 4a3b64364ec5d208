"""Top source lines by warp-stall samples from an ncu report
(ncu -i REP -k regex:K --page source --csv --print-source cuda,sass).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ex = int((d.get("Instructions Executed", "0") or "0").replace(",", ""))
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, {"samples": 0, "exec": 0, "src": r[1][:70], "stalls": {}})
    a["samples"] += s
    a["exec"] += ex
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                a["stalls"][k] = a["stalls"].get(k, 0) + int(v or 0)
            except ValueError:
                pass
tot = sum(a["samples"] for a in agg.values()) or 1
print(f"total samples {tot}")
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(a["stalls"].items(), key=lambda kv: -kv[1])[:3]
    sts = " ".join(f"{k[6:]}={v}" for k, v in st if v)
    print(f"{100 * a['samples'] / tot:5.1f}% {f}:{ln:<4d} exec={a['exec']:<10d} {a['src']:<70s} {sts}")
