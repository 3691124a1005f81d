"""Brief of one ncu --set full report (scratch tool): duration, issue,
occupancy, pipes, DRAM, top stall reasons, and the source lines with the
most stall samples.  python scripts/ncu_brief.py REPORT.ncu-rep"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
m = dict(zip(h, v))
def g(k):
    return m.get(k, "?")
print("kernel", g("Kernel Name")[:60], "dur_us", float(g("gpu__time_duration.sum")) / 1e3)
for k in ["sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum", "l1tex__t_sectors.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
          "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size"]:
    if k in m:
        print(" ", k, m[k])
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(val)) for k, val in m.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and val.replace(".", "").isdigit()]
tot = sum(x for _, x in st) or 1
print("  stalls:", ", ".join(f"{k} {x / tot:.2f}" for k, x in sorted(st, key=lambda t: -t[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if srows:
    hh = srows[0]
    try:
        il, ic = hh.index("# Address") if "# Address" in hh else None, None
    except Exception:
        il = None
    cols = {n: i for i, n in enumerate(hh)}
    key = next((n for n in hh if n.startswith("Warp Stall Sampling (All")), None)
    if key:
        lines = []
        for r in srows[1:]:
            try:
                lines.append((float(r[cols[key]]), r[cols.get("#", 0)], r[cols.get("Source", 1)][:110]))
            except Exception:
                pass
        tot = sum(x for x, _, _ in lines) or 1
        for x, ln, sc in sorted(lines, reverse=True)[:14]:
            print(f"  {x / tot:5.2f} L{ln}: {sc.strip()}")
