# A/B of bench.py options on the current library: bash scripts/ab_bench.sh "NAME:ARGS" ...
# (two interleaved rounds; ms per step, payload-only ms, stage sums)
for rep in 1 2; do
for spec in "$@"; do
  v=${spec%%:*}; a=${spec#*:}
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-client --no-cpu-baseline --no-extras $a > gpurun_out/b_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/b_$v.json'));print('$v',round(d['ms_per_step'],4),round(d['payload_only']['ms_per_step'],4),d['config'].get('job_streams'))"
done; done
