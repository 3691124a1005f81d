"""Summarise a bench JSON line (scratch tool): step, stages, per-layer, roofline."""
import json, sys
d = json.load(open(sys.argv[1]))
print("ms/step", round(d["ms_per_step"], 4), "seq", round(d["sequential_ms_per_step"], 4),
      "po", round(d["payload_only"]["ms_per_step"], 4) if d.get("payload_only") else None)
print({k: round(v, 4) for k, v in d["stages_ms_per_step"].items()})
for r in d["per_layer"]:
    print(r["layer"], r["s"], r["c_o"], [round(r[k] * 1000, 1) for k in ("ntt_ms", "mac_ms", "intt_ms")])
for k, v in d["roofline_all"].items():
    print(k, v["bound"], round(v["frac"], 3), "hbm_frac", round(v.get("hbm_frac", v["frac"]), 3))
