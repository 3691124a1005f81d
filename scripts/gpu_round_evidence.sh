# usage: bash scripts/gpu_round_evidence.sh TAG  -- bench line, launch list, 3 full ncu captures
TAG=$1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu_$TAG.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
for spec in "k_ntt_fwd_dp_s1:21" "k_mac_imma:1" "k_intt_scatter:1" "k_mac_imma:14" "k_intt_scatter:14"; do
  re=${spec%%:*}; sk=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $sk -c 1 -o gpurun_out/prof_${TAG}_${re}_${sk} python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}_${re}_${sk}.log 2>&1; echo "ncu $re $sk rc=$?"
done
