# usage: bash scripts/gpu_ncu_cfg5.sh TAG -- ncu --set full of config 5's K4 row writer and tcgen05 MAC
TAG=$1
mkdir -p gpurun_out
timeout 300 python bench.py --workload cfg5 --profile --steps 1 --warmup 1 > gpurun_out/plain5_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
for spec in "k4c5:k_intt_rows<.int.2, .int.15" "tc5:k_mac_tc<.int.1, .bool.1>"; do
  n=${spec%%:*}; re=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$re" -s 1 -c 1 -o gpurun_out/prof_${n}_$TAG python bench.py --workload cfg5 --profile --steps 1 --warmup 1 \
    > gpurun_out/ncu_${n}_$TAG.log 2>&1; echo "ncu $n rc=$?"
done
