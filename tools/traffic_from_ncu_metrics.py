"""Per-launch traffic of one kernel from an `ncu --metrics ... --csv` log (run HERE, no GPU):
writes profiles/traffic_<kernel>_<config>_m<m>.json, the file bench.py reads into
roofline.traffic.  For the NVLink-bound XOR encode the traffic is the NVLink receive user
bytes (nvlrx__bytes_data_user.sum); the DRAM bytes and protocol totals ride along.

  python tools/traffic_from_ncu_metrics.py <csv> <kernel-substring> <config> <m> <algorithmic-bytes> <source-note>
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, ksub, config, m, alg, note = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), float(sys.argv[5]), sys.argv[6]
txt = open(path).read()
txt = txt[txt.index('"ID"'):]
per = defaultdict(dict)
for r in csv.DictReader(io.StringIO(txt)):
    if ksub not in r["Kernel Name"]:
        continue
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3,
             "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
    per[(r["ID"], r["Device"])][r["Metric Name"]] = v * scale
launches = list(per.values())
mean = {k: sum(l[k] for l in launches) / len(launches) for k in launches[0]}
kernel = ksub
out = {"kernel": kernel, "config": config, "m": m, "launches": len(launches),
       "metric": "nvlrx__bytes_data_user.sum" if "nvlrx__bytes_data_user.sum" in mean else "dram__bytes_read.sum + dram__bytes_write.sum",
       "bytes_per_launch": mean.get("nvlrx__bytes_data_user.sum", mean.get("dram__bytes_read.sum", 0) + mean.get("dram__bytes_write.sum", 0)),
       "algorithmic_bytes_per_launch": alg,
       "nvlrx_bytes_with_protocol": mean.get("nvlrx__bytes.sum"), "nvltx_bytes": mean.get("nvltx__bytes.sum"),
       "dram_bytes_per_launch": mean.get("dram__bytes_read.sum", 0) + mean.get("dram__bytes_write.sum", 0),
       "ncu_ns_per_launch_serialised": mean.get("gpu__time_duration.sum"),
       "per_launch": launches, "source": note}
out["traffic_over_algorithmic"] = out["bytes_per_launch"] / alg if alg else None
dst = os.path.join(ROOT, "profiles", f"traffic_{kernel}_{config}_m{m}.json")
json.dump(out, open(dst, "w"), indent=1)
print(dst, json.dumps({k: v for k, v in out.items() if k != "per_launch"}))
