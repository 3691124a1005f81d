# usage: bash scripts/gpu_round2_evidence.sh TAG -- the round's evidence in one GPU call:
# GPU tests, bench lines (config 4 default, config 5, reference arm), the ncu launch
# list of the bench command, and the per-workload DRAM traffic passes.
TAG=$1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --workload cfg5 --steps 20 --warmup 5 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err; echo "bench cfg5 rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
bash scripts/gpu_ncu_traffic.sh tr4_$TAG plain20
bash scripts/gpu_ncu_traffic.sh tr5_$TAG cfg5
