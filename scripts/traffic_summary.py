"""ncu per-launch DRAM traffic (scripts/gpu_ncu_traffic.sh CSV) -> JSON:
python scripts/traffic_summary.py gpurun_out/traffic_TAG.csv profiles/traffic_WORKLOAD.json WORKLOAD CODE
Kernel classes as bench.py names them; only the step's launches (the conv
path's forward NTT writes MAC tiles: k_ntt_fwd_*<2>)."""
import csv
import json
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else None
code = sys.argv[4] if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
per = {}
for r in rows[1:]:
    d = per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
classes = {"ntt_fwd": r"k_ntt_fwd_dp_s\d<2[,>]|k_ntt_fwd_s\d<2[,>]|k_ntt_fwd_cols<2[,>]", "mac_fold": r"k_mac_imma|k_mac_fold|k_mac_tc",
           "intt_scatter": r"k_intt_scatter|k_intt_rows", "fc_inv": r"k_fc_inv"}
out = {"source": src, "workload": workload, "code": code, "method": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
       "dram__bytes_write.sum, bench.py --profile --steps 1 --warmup 1 (cold-cache, serialised)"}
for cl, pat in classes.items():
    ls = [d for d in per.values() if re.search(pat, d["name"])]
    if not ls:
        continue
    dram = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls]
    t = [d.get("gpu__time_duration.sum", 0) for d in ls]
    unit = 1.0
    out[cl] = {"launches": len(ls), "mean_dram_bytes_per_launch": sum(dram) / len(ls),
               "mean_duration_ns": sum(t) / len(ls)}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
