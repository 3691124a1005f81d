# usage: bash scripts/build_var.sh NAME "-DFLAG=V ..."  -> paper_2409_05205_b200/var/lib_NAME.so
set -e
mkdir -p paper_2409_05205_b200/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Iinclude $2 -o paper_2409_05205_b200/var/lib_$1.so \
  paper_2409_05205_b200/csrc/he_host.cu paper_2409_05205_b200/csrc/he_kernels.cu
