# usage: bash scripts/gpu_ncu3.sh TAG [SPEC...] -- one ncu --set full capture per
# SPEC (name:regex over demangled names; default: the three s = 8 step kernels,
# config-4 layer 2 instances) after the plain run exits 0
TAG=$1; shift
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
if [ $# -eq 0 ]; then
  set -- "ntt:k_ntt_fwd_dp_s1<.int.2, .int.14, .int.3, .int.2," \
         "mac:k_mac_imma<.int.2, .int.5, .int.16, .int.16, .int.16, .int.4, .int.1, .int.3>" \
         "k4:k_intt_scatter<.bool.1, .int.14, .int.3, .int.2, .int.2184, .int.4, .int.8, .int.34, .int.32"
fi
for spec in "$@"; do
  n=${spec%%:*}; re=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"$re" -s 1 -c 1 -o gpurun_out/prof_${n}_$TAG python bench.py --profile --steps 1 --warmup 1 \
    > gpurun_out/ncu_${n}_$TAG.log 2>&1; echo "ncu $n rc=$?"
done
