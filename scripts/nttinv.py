import json,sys
for v in sys.argv[1:]:
    d=json.load(open(f'gpurun_out/v_{v}.json'))
    print(v, round(d['ms_per_step'],4), [(r['N'], round(r['inverse']['limbs_per_s']/1e6,2), round(r['inverse']['frac_u1_fp64_roof'],3)) for r in d['ntt']['sizes']], d.get('client',{}) and None)
