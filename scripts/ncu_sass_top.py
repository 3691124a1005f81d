"""Executed-instruction totals per SASS opcode and per source line range
(scratch tool).  python scripts/ncu_sass_top.py REP"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = {n: i for i, n in enumerate(rows[1])}
ops = collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        ie = float(r[h["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    op = r[h["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    ops[o.split(".")[0]] += ie
    tot += ie
print(f"total {tot:.3e}")
for o, c in ops.most_common(30):
    print(f"{c / tot:6.3f} {o}")
