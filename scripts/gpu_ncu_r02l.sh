# usage: bash scripts/gpu_ncu_r02l.sh TAG -- every step kernel class (gpu_ncu_all.sh) plus
# the full inverse NTT at N = 16384 (k_ntt_inv_dp_cl<1>, scripts/ntt_one.py)
TAG=$1
bash scripts/gpu_ncu_all.sh $TAG
timeout 300 python scripts/ntt_one.py 16384 512 > gpurun_out/plain_inv_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_ntt_inv_dp_cl" -s 1 -c 1 -o gpurun_out/prof_inv16k_$TAG python scripts/ntt_one.py 16384 512 \
  > gpurun_out/ncu_inv16k_$TAG.log 2>&1; echo "ncu inv rc=$?"
f=gpurun_out/prof_inv16k_$TAG.ncu-rep
{ python scripts/ncu_brief.py $f; python scripts/ncu_opcodes.py $f 14; python scripts/ncu_lines2.py $f 14; } > gpurun_out/brief_prof_inv16k_$TAG.txt 2>&1
rm -f $f
