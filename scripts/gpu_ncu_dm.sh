# usage: bash scripts/gpu_ncu_dm.sh TAG "DEMANGLED-REGEX" SKIP -- one ncu --set full capture,
# kernel matched on its demangled name (template arguments included)
TAG=$1; RE=$2; SK=${3:-0}
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RE" -s $SK -c 1 -o gpurun_out/prof_$TAG python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
