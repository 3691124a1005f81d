"""Write profiles/r01_TAG_summary.md from the bench line, launch list and
config-5 line of one evidence refresh:
python scripts/make_summary.py TAG "code-state sentence" [traffic-csv-tag]"""
import collections
import csv
import json
import sys

tag, state = sys.argv[1], sys.argv[2]
ttag = sys.argv[3] if len(sys.argv) > 3 else tag
P = "/root/repo/profiles/"
rows = [r for r in csv.reader(open(P + f"launches_r01_{tag}.csv")) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        a = agg[r[ki].split("(")[0]]
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
step = [k for k in agg if any(x in k for x in ("k_intt_scatter", "k_ntt_fwd_dp_s1<2>",
                                                "k_ntt_fwd_cols<2>", "k_mac_imma", "k_fc_inv"))]
tot = sum(agg[k][1] for k in step)
tab = "\n".join(f"| `{k}` | {agg[k][0]} | {agg[k][1]/1e3:.1f} | {agg[k][1]/tot:.3f} |"
                for k in sorted(step, key=lambda k: -agg[k][1]))
share = lambda s: sum(agg[k][1] for k in step if s in k) / tot
d = json.load(open(P + f"bench_r01_{tag}.json"))
e5 = json.load(open(P + f"bench_cfg5_r01_{tag}.json"))
ra, st, s5 = d["roofline_all"], d["stages_ms_per_step"], e5["stages_ms_per_step"]
pc = d["e2e"]["pcie"]
txt = f"""# Round 1, {tag} evidence (B200, sm_100a) -- latest

Code state: {state}

**Bench** (`profiles/bench_r01_{tag}.json`, `python bench.py --steps 10
--warmup 3`): **{d['ms_per_step']:.3f} ms/step = {d['value']:.4g} ct×pt evals/s**
(config 4: 19 conv + FC, N = 16384, L = 6, B = 32; CUDA graph, {d['config']['streams']}
streams, layer jobs overlapped; {1000*d['ms_per_plain20_image']:.1f} µs per plain-20 image; MAC:
{d['config']['mac']}).  Payload-only step {d['payload_only']['ms_per_step']:.3f} ms.
Sequential analysis pass {d['sequential_ms_per_step']:.3f} ms: NTT {st['ntt_fwd']:.3f}, MAC
{st['mac_fold']:.3f}, INTT+scatter {st['intt_scatter']:.3f}, FC {st['fc_ntt_fwd']+st['fc_inv']:.3f}, gaps
{st['gaps']:.3f} ms.  NTT limbs/s at N = 16384: forward {d['ntt']['limbs_per_s']/1e6:.2f} M
({100*d['ntt']['frac']:.0f} % of the FP64 roof), inverse {d['ntt']['inverse_limbs_per_s']/1e6:.2f} M ({100*d['ntt']['inverse_frac']:.0f} %).
e2e (host buffers, 50-bit wire, device φ1): {d['e2e']['ms_per_step']:.2f} ms; the H2D copy of the
same bytes alone {pc['h2d_only_ms']:.2f} ms ({pc['h2d_gbs']:.1f} GB/s) → {100*pc['frac']:.0f} % of the PCIe H2D roof.
Sparse c0 upload + one-limb payload: {d['e2e']['sparse_upload_modswitch']['ms_per_step']:.2f} ms.
Client per step: {d['client']['ms_per_step']:.2f} ms; encrypted plain-20 chain: {d['chain']['ms_per_step']:.2f} ms per 32
images.  Ablation: unfolded {d['ablation']['unfolded_conv_ms_per_step']:.1f} ms vs folded
{d['ablation']['folded_conv_ms_per_step_sequential']:.2f} ms ({d['ablation']['fold_speedup']:.1f}×).  CPU oracle: {d['cpu_baseline']['value']:.4g} evals/s on
{d['cpu_baseline']['cores']} cores (GPU/CPU {d['value']/d['cpu_baseline']['value']:.0f}×); `--impl reference`:
`profiles/bench_ref_r01_{tag}.json`.  Clocks {d['clocks']['sm_mhz']:.0f}/{d['clocks']['sm_max_mhz']:.0f} MHz,
throttle reasons {d['clocks']['reasons'] or 'none'}.

**Config 5** (`profiles/bench_cfg5_r01_{tag}.json`, `--workload cfg5`: N = 32768,
L = 12, B = 256, 64→64 @ 8×8): {e5['ms_per_step']:.3f} ms/step = {e5['value']:.4g} evals/s; NTT
{s5['ntt_fwd']:.3f}, MAC {s5['mac_fold']:.3f} ({e5['config']['mac']}), INTT+scatter
{s5['intt_scatter']:.3f} ms.

## Launch list (`profiles/launches_r01_{tag}.csv`; ncu gpu__time_duration, `bench.py --profile --steps 1 --warmup 1`; cold-cache, serialised; step kernels only)

| kernel | launches | total µs | share of step kernels |
|---|---|---|---|
{tab}

MAC {share('mac'):.3f}, INTT+scatter {share('intt'):.3f}, NTT {share('ntt_fwd'):.3f} — live sequential shares
(bench): MAC {ra['mac_fold']['share_of_step']:.3f}, INTT+scatter {ra['intt_scatter']['share_of_step']:.3f}, NTT {ra['ntt_fwd']['share_of_step']:.3f}.

## Roofline (bench `roofline_all`; DRAM traffic `profiles/traffic_r01.json` from `gpurun_out/traffic_r01{ttag}.csv`)

| kernel | bound | achieved | peak | frac |
|---|---|---|---|---|
| ntt_fwd | alu | {ra['ntt_fwd']['achieved']:.1f} Gbutterfly/s | {ra['ntt_fwd']['peak']:.1f} | {ra['ntt_fwd']['frac']:.3f} |
| mac_fold | hbm | {ra['mac_fold']['achieved']:.1f} GB/s | {ra['mac_fold']['peak']:.1f} | {ra['mac_fold']['frac']:.3f} ({ra['mac_fold']['alu_frac']:.3f} of the int8 MMA roof) |
| intt_scatter | alu | {ra['intt_scatter']['achieved']:.1f} Gbutterfly/s | {ra['intt_scatter']['peak']:.1f} | {ra['intt_scatter']['frac']:.3f} |

Full `--set full` captures of the step kernels (stall analysis):
`profiles/r01_v68_ncu.md`.  Phase ablations: `profiles/r01_v60_summary.md`.
"""
open(P + f"r01_{tag}_summary.md", "w").write(txt)
print(txt[:300])
