# usage: bash scripts/gpu_sanitize.sh TAG -- compute-sanitizer (memcheck, racecheck, synccheck,
# initcheck) over a small subset of the GPU parity tests; logs under gpurun_out/.
TAG=$1
mkdir -p gpurun_out
SEL="test_conv_small or test_conv_configs_full or test_ntt_roundtrip or test_ntt_inverse_matches_definition or test_pack_input or test_errors"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout 1200 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/san_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_${tool}_$TAG.log
done
