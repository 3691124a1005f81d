# usage: bash scripts/gpu_ncu_traffic.sh TAG -- DRAM bytes + duration of every
# kernel launch of one --profile run (one ncu pass; the plain run first)
TAG=$1
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_traffic_$TAG.log 2>&1; echo "ncu rc=$?"
