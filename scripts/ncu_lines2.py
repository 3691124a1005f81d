"""Per-source-line instruction and stall totals from an ncu report
(--page source --print-source cuda,sass).  python scripts/ncu_lines2.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {n: i for i, n in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        ie = float(r[hdr["Instructions Executed"]] or 0)
        st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    k = (fname, int(r[0]))
    a = agg.setdefault(k, [0.0, 0.0, r[1][:90]])
    a[0] += ie
    a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti:.3e}")
for k, (ie, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ie / ti:5.3f} inst {st / ts:5.3f} stall {k[0]}:{k[1]}  {src.strip()}")
