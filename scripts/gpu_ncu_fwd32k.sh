# usage: bash scripts/gpu_ncu_fwd32k.sh TAG -- ncu --set full of the full forward NTT at
# N = 32768 and N = 16384 (k_ntt_fwd_dp16_s2 / _s1, scripts/ntt_one.py): the stall
# breakdown DESIGN.md §12 asks for (0.52 vs 0.66 of the U1 roof)
TAG=$1
mkdir -p gpurun_out
for spec in "fwd32k:32768:256:k_ntt_fwd_dp16_s2" "fwd16k:16384:512:k_ntt_fwd_dp16_s1"; do
  IFS=: read n N nl re <<< "$spec"
  timeout 300 python scripts/ntt_one.py $N $nl > gpurun_out/plain_${n}_$TAG.log 2>&1 || { echo "plain $n failed"; continue; }
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$re" -s 1 -c 1 -o gpurun_out/prof_${n}_$TAG python scripts/ntt_one.py $N $nl \
    > gpurun_out/ncu_${n}_$TAG.log 2>&1; echo "ncu $n rc=$?"
  f=gpurun_out/prof_${n}_$TAG.ncu-rep
  { python scripts/ncu_brief.py $f; python scripts/ncu_opcodes.py $f 14; python scripts/ncu_lines2.py $f 16; } > gpurun_out/brief_prof_${n}_$TAG.txt 2>&1
  ncu -i $f --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[-1]
for k,x in zip(h,v):
    if 'barrier' in k or 'membar' in k or 'cluster' in k.lower() or 'dsmem' in k.lower() or 'l1tex__m_xbar' in k or 'smsp__warp_issue_stalled' in k and 'pct' not in k:
        print(k,x)
" >> gpurun_out/brief_prof_${n}_$TAG.txt 2>&1
  rm -f $f
done
