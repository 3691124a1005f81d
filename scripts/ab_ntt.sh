# A/B of prebuilt library variants on the NTT limbs/s figures (bench ntt.sizes):
# bash scripts/ab_ntt.sh NAME ...   (two rounds each)
cp paper_2409_05205_b200/libhe_rotfree.so /tmp/orig_ntt.so
for rep in 1 2; do
for v in "$@"; do
  cp paper_2409_05205_b200/var/lib_$v.so paper_2409_05205_b200/libhe_rotfree.so
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-client --no-cpu-baseline --no-extras > gpurun_out/n_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/n_$v.json'));n=d['ntt']
print('$v', round(d['ms_per_step'],4), [(s['N'], round(s['forward']['frac_u1_fp64_roof'],3), round(s['inverse']['frac_u1_fp64_roof'],3), round(s['inverse']['limbs_per_s']/1e6,2)) for s in n['sizes']])"
done; done
cp /tmp/orig_ntt.so paper_2409_05205_b200/libhe_rotfree.so
