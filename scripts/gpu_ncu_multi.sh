# usage: bash scripts/gpu_ncu_multi.sh TAG   -- several targeted ncu captures (one ncu "use")
TAG=$1
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
for spec in "k_mac_imma:1" "k_mac_imma:14" "k_intt_scatter:1" "k_intt_scatter:14" "k_ntt_fwd_s1:20"; do
  re=${spec%%:*}; sk=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $sk -c 1 -o gpurun_out/prof_${TAG}_${re}_${sk} python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}_${re}_${sk}.log 2>&1; echo "ncu $re $sk rc=$?"
done
