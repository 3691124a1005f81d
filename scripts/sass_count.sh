# usage: bash scripts/sass_count.sh [LIB] -- static SASS instruction count of the step kernels
LIB=${1:-paper_2409_05205_b200/libhe_rotfree.so}
cuobjdump -sass $LIB | awk '/Function :/{name=$3} /^[ \t]+\/\*[0-9a-f]{4}\*\//{n[name]++} END{for(k in n) print n[k], k}' | \
  grep -E "k_mac_imma.*Li1ELi[13]EE|k_mac_tcILi1|k_intt_scatterILb1ELi14ELi3ELi2ELi2184ELi4ELi8ELi34ELi32|k_intt_rowsILi2ELi14|k_ntt_fwd_dp_s1ILi2ELi14|k_ntt_fwd_colsILi2" | sort -k2
