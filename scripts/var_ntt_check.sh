# usage: bash scripts/var_ntt_check.sh NAME ... -- the transform GPU tests against each
# prebuilt variant (paper_2409_05205_b200/var/lib_NAME.so), then the NTT A/B
cp paper_2409_05205_b200/libhe_rotfree.so /tmp/orig_chk.so
for v in "$@"; do
  cp paper_2409_05205_b200/var/lib_$v.so paper_2409_05205_b200/libhe_rotfree.so
  timeout 300 python -m pytest tests -m gpu -q -x -k "ntt or fc or client" > gpurun_out/chk_$v.log 2>&1; echo "$v tests rc=$? $(tail -1 gpurun_out/chk_$v.log)"
done
cp /tmp/orig_chk.so paper_2409_05205_b200/libhe_rotfree.so
bash scripts/ab_ntt.sh "$@"
