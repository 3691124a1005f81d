"""Aggregate an ncu report's SASS instruction counts and stall samples by
CUDA source line: python scripts/ncu_lines.py REP [TOP]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg = {}
fname = "?"
cur = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None:
        continue
    if row[0].strip().isdigit():
        cur = (fname, int(row[0]), row[1].strip()[:70])
    if len(row) > 7 and row[2].startswith("0x") and cur is not None:
        d = dict(zip(hdr[2:], row[2:]))
        a = agg.setdefault(cur, [0, 0])
        try:
            a[0] += int(d.get("Instructions Executed", "0") or 0)
            a[1] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*v[0]/tot_i:5.1f}% inst {100*v[1]/tot_s:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
