# usage: bash scripts/gpu_ncu_traffic.sh TAG [WORKLOAD] -- DRAM bytes + duration
# of every kernel launch of one --profile run of that workload (one ncu pass;
# the plain run first); then summarise into profiles/traffic_WORKLOAD.json
TAG=$1; WL=${2:-plain20}
mkdir -p gpurun_out
timeout 300 python bench.py --workload $WL --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_$TAG.csv python bench.py --workload $WL --profile --steps 1 --warmup 1 > gpurun_out/ncu_traffic_$TAG.log 2>&1; echo "ncu rc=$?"
python scripts/traffic_summary.py gpurun_out/traffic_$TAG.csv gpurun_out/traffic_$WL.json $WL "$TAG" > /dev/null && echo "traffic -> gpurun_out/traffic_$WL.json"
