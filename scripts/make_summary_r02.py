"""Write profiles/r02_summary.md (+ copies of the bench lines and launch list)
from one evidence refresh (scripts/gpu_round2_evidence.sh TAG):
python scripts/make_summary_r02.py TAG "code-state sentence"."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

tag, state = sys.argv[1], sys.argv[2]
G, P = "/root/repo/gpurun_out/", "/root/repo/profiles/"
for src, dst in [(f"bench_{tag}.json", "bench_r02.json"), (f"bench_cfg5_{tag}.json", "bench_cfg5_r02.json"),
                 (f"bench_ref_{tag}.json", "bench_ref_r02.json"), (f"launches_{tag}.csv", "launches_r02.csv")]:
    shutil.copy(G + src, P + dst)
rows = [r for r in csv.reader(l for l in open(P + "launches_r02.csv") if l.startswith('"'))]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        a = agg[r[ki].split("(")[0]]
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
# the step's kernels: everything launched by he_conv_ex / he_fc_ex in the step
# (the FC's forward transform shares k_ntt_fwd_dp16_s1 with the NTT limbs/s
#  measurement of the same run, so it is left out of the table)
step_pat = ("k_intt_scatter", "k_intt_rows", "k_ntt_fwd_dp_s1<2", "k_ntt_fwd_cols<2", "k_mac_imma",
            "k_fc_inv")
step = [k for k in agg if any(k.startswith(x) or x in k for x in step_pat)]
tot = sum(agg[k][1] for k in step)
tab = "\n".join(f"| `{k}` | {agg[k][0]} | {agg[k][1]/1e3:.1f} | {agg[k][1]/tot:.3f} |"
                for k in sorted(step, key=lambda k: -agg[k][1]))
d = json.load(open(P + "bench_r02.json"))
d5 = json.load(open(P + "bench_cfg5_r02.json"))
dr = json.load(open(P + "bench_ref_r02.json"))
ra, st = d["roofline_all"], d["stages_ms_per_step"]
pl = "\n".join(f"| {r['layer']} | {r['s']} | {r['c_o']} | {1e3*r['ntt_ms']:.1f} | {1e3*r['mac_ms']:.1f} | "
               f"{1e3*r['intt_ms']:.1f} |" for r in d["per_layer"])
def rl(k):
    v = ra[k]
    extra = f"{v.get('dfma_pipe_frac', 0):.3f}" if "dfma_pipe_frac" in v else "--"
    alt = v.get("alu_frac", v.get("hbm_frac"))
    tr = v.get("traffic")
    return (f"| {k} | {v['bound']} | {v['achieved']:.1f} {v['unit']} | {v['peak']:.1f} | **{v['frac']:.3f}** | "
            f"{alt:.3f} | {extra} | {v['algorithmic_bytes_per_launch']/1e6:.1f} | "
            f"{(tr or 0)/1e6:.1f} |")
ntt = "\n".join(f"| {r['N']} | {r['forward']['limbs_per_s']/1e6:.2f} M ({r['forward']['frac_u1_fp64_roof']:.2f}) | "
                f"{r['inverse']['limbs_per_s']/1e6:.2f} M ({r['inverse']['frac_u1_fp64_roof']:.2f}) |"
                for r in d["ntt"]["sizes"])
cpu = d["cpu_baseline"]
st1 = cpu.get("single_thread", {})
mi_ = d5.get("multi_image") or {}
txt = f"""# Round 2 evidence (B200, sm_100a) -- `{tag}`

Code state: {state}

## Headline (`profiles/bench_r02.json`: `python bench.py --steps 20 --warmup 5`)

Config 4 (plain-20: 19 conv + FC 64→100, N = 16384, L = 6, B = 32; CUDA graph,
six layer streams): **{d['ms_per_step']:.3f} ms/step = {d['value']:.4g} ct×pt evals/s
= {1000*d['ms_per_plain20_image']:.1f} µs per plain-20 image** (round 1: 2.266 ms,
1.154e7).  Payload-only step {d['payload_only']['ms_per_step']:.3f} ms.  e2e (host
buffers, 50-bit wire): {d['e2e']['ms_per_step']:.2f} ms ({100*d['e2e']['pcie']['frac']:.0f} % of the PCIe H2D
copy roof of the same bytes).  Clocks {d['clocks']['sm_mhz']:.0f}/{d['clocks']['sm_max_mhz']:.0f} MHz,
throttle reasons {d['clocks']['reasons'] or 'none'}.

Sequential analysis pass {d['sequential_ms_per_step']:.3f} ms: forward NTT {st['ntt_fwd']:.3f}, MAC
{st['mac_fold']:.3f}, INTT + scatter + mask {st['intt_scatter']:.3f}, FC {st['fc_ntt_fwd']+st['fc_inv']:.3f}, gaps
{st['gaps']:.3f} ms (round 1: 0.807 / 1.077 / 1.039).

## Roofline (`roofline_all`, achieved = algorithmic work ÷ live CUDA-event kernel time)

| kernel | bound | achieved | peak | frac | other-bound frac | DFMA-pipe frac | alg. MB/launch | DRAM MB/launch (ncu) |
|---|---|---|---|---|---|---|---|---|
{rl('ntt_fwd')}
{rl('mac_fold')}
{rl('intt_scatter')}

Dominant kernel: `{d['roofline']['kernel']}`, frac {d['roofline']['frac']:.3f} (round 1: mac_fold 0.254).
MAC arithmetic roof: {ra['mac_fold'].get('alu_peak_source')}.  DRAM traffic from
`profiles/traffic_plain20.json` (same workload's ncu pass).

## Per layer (sequential pass, µs)

| layer | s | c_o | NTT | MAC | INTT+scatter |
|---|---|---|---|---|---|
{pl}

## NTT limbs/s (`ntt.sizes`; fraction of the U1 FP64 butterfly roof)

| N | forward | inverse |
|---|---|---|
{ntt}

## Config 5 (`profiles/bench_cfg5_r02.json`, `--workload cfg5`: N = 32768, L = 12, 256 images)

{d5['ms_per_step']:.3f} ms/step = {d5['value']:.4g} evals/s; MAC {d5['config']['mac']}; fracs:
NTT {d5['roofline_all']['ntt_fwd']['frac']:.3f}, MAC {d5['roofline_all']['mac_fold']['frac']:.3f}
({d5['roofline_all']['mac_fold']['bound']}), INTT {d5['roofline_all']['intt_scatter']['frac']:.3f}.
Multi-image packing (R31, s = 64, {mi_.get('images_per_ciphertext')} images per ciphertext):
{mi_.get('ms_per_step', 0):.3f} ms for the 256 images against {mi_.get('one_image_per_ct', {}).get('ms_per_step', 0):.3f} ms,
c0 and c0^r bytes per image {mi_.get('c0_bytes_per_image', 0)/1e3:.0f} KB vs {mi_.get('c0_bytes_per_image_one_per_ct', 0)/1e3:.0f} KB.

## CPU baselines (host of the GPU box: {cpu.get('cpu_model')}, {cpu['cores']} cores)

* Oracle (sparse-direct definition), all cores: {cpu['value']:.4g} evals/s ({cpu['sample']}).
* Oracle, one thread: {st1.get('value', 0):.4g} evals/s, {st1.get('s_per_image', 0):.2f} s per plain-20 image.
* CPU textbook-NTT path (`oracle/cpu_ntt_baseline.c`), all cores: {cpu.get('ntt_path', {}).get('value', 0):.4g} evals/s;
  one thread: {st1.get('ntt_path', {}).get('value', 0):.4g} evals/s.  For 3×3 filters the sparse-direct
  definition is the faster CPU method.
* `--impl reference` (the oracle as the reference arm, 1 image per step): {dr['value']:.4g} evals/s.

## Launch list (`profiles/launches_r02.csv`; ncu gpu__time_duration of `bench.py --profile --steps 1 --warmup 1`; cold-cache, serialised; step kernels)

| kernel | launches | total µs | share |
|---|---|---|---|
{tab}
"""
open(P + "r02_summary.md", "w").write(txt)
print(txt[:400])
