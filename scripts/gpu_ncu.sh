# usage: bash scripts/gpu_ncu.sh TAG REGEX SKIP COUNT  (one ncu --set full capture)
TAG=$1; RE=$2; SKIP=${3:-0}; CNT=${4:-3}
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT -o gpurun_out/prof_$TAG python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
