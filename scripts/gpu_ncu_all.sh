# usage: bash scripts/gpu_ncu_all.sh TAG -- ncu --set full of every step kernel class
# (config 4: s = 8 NTT / MAC / K4, s = 32 MAC / K4, s = 128 MAC / K4, FC inverse;
#  config 5: K4 row writer, tcgen05 MAC, column NTT), one kernel per ncu run
TAG=$1
bash scripts/gpu_ncu3.sh $TAG \
  "ntt8:k_ntt_fwd_dp_s1<.int.2, .int.14, .int.3, .int.2," \
  "mac16:k_mac_imma<.int.2, .int.5, .int.16, .int.16, .int.16, .int.4, .int.1, .int.3>" \
  "k4s8:k_intt_scatter<.bool.1, .int.14, .int.3, .int.2, .int.2184, .int.4, .int.8, .int.34, .int.32" \
  "ntt32:k_ntt_fwd_dp_s1<.int.2, .int.14, .int.5" \
  "mac32:k_mac_imma<.int.2, .int.1, .int.32, .int.32, .int.32, .int.2, .int.1, .int.1>" \
  "rows32:k_intt_rows<.int.2, .int.14, .int.5" \
  "cols128:k_ntt_fwd_cols<.int.2, .int.7" \
  "mac64:k_mac_imma<.int.1, .int.1, .int.64, .int.64, .int.64" \
  "rows128:k_intt_rows<.int.2, .int.14, .int.7" \
  "fcinv:k_fc_inv<.bool.1>"
bash scripts/gpu_ncu_cfg5.sh $TAG
# summaries on the box (the reports together exceed gpurun's 64 MiB return limit)
for f in gpurun_out/prof_*_$TAG.ncu-rep; do
  n=$(basename $f .ncu-rep)
  { python scripts/ncu_brief.py $f; python scripts/ncu_opcodes.py $f 14; python scripts/ncu_lines2.py $f 14; } > gpurun_out/brief_$n.txt 2>&1
  rm -f $f
done
