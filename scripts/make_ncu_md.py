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
READING = """
Reading (round 2, final state):
* The FP64 step kernels (forward NTT, K4, full inverse) run their FP64 pipe at
  43-58 % with 50-60 % of issue slots busy; DADD + DFMA + DMUL are 52-58 % of
  their instructions, the hottest source lines are the two FMA-magic quotient
  lines of `dp_mulmod` / `dp_reduce`.  The remaining stalls are global-load
  latency (`long_scoreboard` 0.17-0.23: the forward NTT's input vectors, K4's
  phi1 and fold rows), FP64 dependency chains (`wait` 0.12-0.20) and FP64 pipe
  contention (`math_pipe_throttle` 0.09-0.18, `not_selected` 0.12-0.19) --
  i.e. they sit between latency- and pipe-bound, not on address arithmetic.
* The config-5 row writer is issue-bound (77 % issue, 75 % SM throughput):
  each output word costs the FP64 mask encoding (enc_dp) and a
  canonicalisation; it writes 848 MB per launch at 0.62 of the HBM roof.
* The K = 16 int8 `mma.sync` MAC (TMA-staged) now waits on its operand tile
  (`long_scoreboard` 0.31: one TMA unit per CTA, 5 CTAs/SM); the K = 32 / 64
  instances are bound by the IMMA pipe in bursts (`math_pipe_throttle`
  0.15-0.21) and their 13-accumulator dependency chains (`wait` 0.22-0.28) at
  23 % warp occupancy (122-128 registers).  IMMA is 10 % of the K = 16
  instance's instructions; the byte-diagonal recombination (IMAD / IADD3) is
  half of them.
* The tcgen05 MAC (config 5, `k_mac_tc<1, 1>`, TMA-staged) reaches 74 % SM
  throughput with only 21 % of issue slots busy: the tensor pipe carries the
  work, the CUDA cores wait on TMEM loads and the operand mbarrier
  (`long_scoreboard` 0.60); a third of its instructions are the
  recombination's wide multiply-adds (`madw`).
* Shared-memory bank conflicts: K4 s = 8 0.22 and the full inverse 0.22
  conflicts per wavefront (the padded GS passes), the forward NTT 0.03.
"""
out = [f"# Round 2: `ncu --set full` of every step kernel class ({tag})", "",
       "One capture per kernel (`scripts/gpu_ncu_r02l.sh " + tag + "`, `bench.py --profile`, the",
       "second launch of each instance: config-4 layers 1 / 9 / 15 and the FC, config-5 for the",
       "`N = 32768` kernels, `scripts/ntt_one.py` for the full inverse NTT); cold-cache and serialised, so durations are not the step's; the",
       "briefs (incl. opcode mixes and the hottest source lines) are summarised on the GPU box",
       "by `scripts/ncu_brief.py`, `ncu_opcodes.py`, `ncu_lines2.py`.", "",
       "| kernel | µs | issue % | warps active % | FP64 pipe % | ALU % | warp-instr (M) | regs | top stalls |",
       "|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| `{r[0]}` | {r[1]:.1f} | {r[2]:.1f} | {r[3]:.1f} | {r[4]:.1f} | {r[5]:.1f} | {r[6]:.2f} | {r[7]:.0f} | {r[8]} |")
out += READING.rstrip("\n").split("\n")
open("/root/repo/profiles/r02_ncu.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
