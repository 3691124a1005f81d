import json, sys
sys.path.insert(0, '.')
import bench
r = bench.u1_peaks(0)
for k, v in r.items():
    print(k, f"{v['per_s']:.4g}/s", f"{v['per_s']/(148*1.965e9):.2f}/clk/SM@1965")
json.dump(r, open('gpurun_out/u1.json', 'w'), indent=1)
