"""Aggregate an ncu report's SASS instruction counts by opcode:
python scripts/ncu_opcodes.py REP [TOP]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
ii = hdr.index("Instructions Executed")
agg = {}
for r in rows:
    if len(r) > ii and r[0].startswith("0x"):
        op = r[1].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        try:
            agg[o] = agg.get(o, 0) + int(r[ii] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print("total", tot)
for o, n in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{o:10s} {n:12d} {100 * n / tot:5.1f}%")
