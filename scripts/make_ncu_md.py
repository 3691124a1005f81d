"""profiles/r02_ncu.md from the on-box ncu briefs (scripts/gpu_ncu_all.sh TAG):
python scripts/make_ncu_md.py TAG"""
import glob
import re
import sys

tag = sys.argv[1]
rows = []
for f in sorted(glob.glob(f"/root/repo/gpurun_out/brief_prof_*_{tag}.txt")):
    t = open(f).read()
    m = re.search(r"kernel (.*?)\(.*?dur_us ([0-9.]+)", t)
    if not m:
        continue
    name, dur = m.group(1).replace("void ", ""), float(m.group(2)) * 1e3
    def g(k):
        mm = re.search(re.escape(k) + r" ([0-9.]+)", t)
        return float(mm.group(1)) if mm else float("nan")
    st = re.search(r"stalls: (.*)", t)
    stalls = ", ".join(st.group(1).split(", ")[:3]) if st else ""
    rows.append((name, dur, g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                 g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                 g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                 g("smsp__inst_executed.sum") / 1e6, g("launch__registers_per_thread"), stalls))
out = [f"# Round 2: `ncu --set full` of every step kernel class ({tag})", "",
       "One capture per kernel (`scripts/gpu_ncu_all.sh " + tag + "`, `bench.py --profile`, the",
       "second launch of each instance: config-4 layers 1 / 9 / 15 and the FC, config-5 for the",
       "`N = 32768` kernels); cold-cache and serialised, so durations are not the step's; the",
       "briefs (incl. opcode mixes and the hottest source lines) are summarised on the GPU box",
       "by `scripts/ncu_brief.py`, `ncu_opcodes.py`, `ncu_lines2.py`.", "",
       "| kernel | µs | issue % | warps active % | FP64 pipe % | ALU % | warp-instr (M) | regs | top stalls |",
       "|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| `{r[0]}` | {r[1]:.1f} | {r[2]:.1f} | {r[3]:.1f} | {r[4]:.1f} | {r[5]:.1f} | {r[6]:.2f} | {r[7]:.0f} | {r[8]} |")
open("/root/repo/profiles/r02_ncu.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
