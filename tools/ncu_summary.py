"""Summarise ncu output (run HERE, no GPU needed) into profiles/<tag>_*.{json,csv}.

  python tools/ncu_summary.py <tag> [--bytes-per-launch N]

Reads gpurun_out/launches_<tag>.csv (gpu__time_duration per launch) and
gpurun_out/prof_<tag>.ncu-rep (--set full of the top kernel)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
alg = None
if "--bytes-per-launch" in sys.argv:
    alg = float(sys.argv[sys.argv.index("--bytes-per-launch") + 1])
out = {"tag": tag}

lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lp):
    txt = open(lp).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(txt)))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
            per[r["Kernel Name"].split("(")[0]].append(v)
    tot = sum(sum(v) for v in per.values())
    out["launch_list"] = {k: {"launches": len(v), "total_us": round(sum(v), 2), "mean_us": round(sum(v) / len(v), 3),
                              "share": round(sum(v) / tot, 4)} for k, v in per.items()}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        f.write("kernel,launch,us\n")
        for k, v in per.items():
            for i, x in enumerate(v):
                f.write(f"{k},{i},{x:.3f}\n")

rp = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
if os.path.exists(rp):
    raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
            "nvlrx__bytes.sum", "nvltx__bytes.sum", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
            "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second"]
    idx = {h: i for i, h in enumerate(hdr)}
    launches = []
    for d in data:
        rec = {}
        for w in want:
            for h, i in idx.items():
                if h == w or (w.startswith("nvl") and h.startswith(w.split(".")[0])):
                    rec[h] = d[i] + (f" {units[i]}" if units[i] else "")
        launches.append(rec)
    out["full"] = launches

    def num(x):
        v, *u = x.split()
        v = float(v.replace(",", ""))
        u = u[0] if u else ""
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    try:
        tr = [num(l["dram__bytes_read.sum"]) + num(l["dram__bytes_write.sum"]) for l in launches]
        out["traffic_bytes_per_launch"] = sum(tr) / len(tr)
        name = launches[0]["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].strip()
        out["kernel"] = name
        if alg:
            out["algorithmic_bytes_per_launch"] = alg
            out["traffic_over_algorithmic"] = out["traffic_bytes_per_launch"] / alg
    except Exception as e:
        out["traffic_error"] = repr(e)
    src = subprocess.run(["ncu", "-i", rp, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    with open(os.path.join(ROOT, "profiles", f"{tag}_source.csv"), "w") as f:
        f.write(src)
    det = subprocess.run(["ncu", "-i", rp, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(ROOT, "profiles", f"{tag}_details.txt"), "w") as f:
        f.write(det)

with open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "full"}, indent=1))
