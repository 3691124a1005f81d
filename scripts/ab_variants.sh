# A/B of prebuilt library variants (paper_2409_05205_b200/var/lib_NAME.so, git-ignored):
# bash scripts/ab_variants.sh "NAME:ENV=VAL" ...  (CFG5=1 also runs config 5); two rounds each.
cp paper_2409_05205_b200/libhe_rotfree.so /tmp/orig.so
for rep in 1 2; do
for spec in "$@"; do
  v=${spec%%:*}; e=${spec#*:}
  cp paper_2409_05205_b200/var/lib_$v.so paper_2409_05205_b200/libhe_rotfree.so
  env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-client --no-cpu-baseline --no-extras > gpurun_out/v_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/v_$v.json'));print('$spec',round(d['ms_per_step'],4),round(d['payload_only']['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms_per_step'].items()}, [(round(r['ntt_ms']*1000,1),round(r['mac_ms']*1000,1),round(r['intt_ms']*1000,1)) for r in d['per_layer'][:19:3]])"
  if [ -n "$CFG5" ]; then env $e timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-e2e --no-client --no-cpu-baseline --no-extras > gpurun_out/v5_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/v5_$v.json'));print('  cfg5',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms_per_step'].items() if v})"; fi
done; done
cp /tmp/orig.so paper_2409_05205_b200/libhe_rotfree.so
