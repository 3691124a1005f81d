# usage: bash scripts/gpu_round_evidence.sh TAG  -- bench line, launch list, one ncu launch-list pass
TAG=$1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu_$TAG.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
# full captures: one ncu per gpurun call -- scripts/gpu_ncu_one.sh TAG REGEX SKIP
