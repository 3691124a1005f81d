set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01.json 2> gpurun_out/bench_ref_r01.err; echo "ref rc=$?"
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu.txt
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_mac_fold|k_ntt_fwd_body|k_intt_scatter" -s 20 -c 6 -o gpurun_out/prof_r01 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
