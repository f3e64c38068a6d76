# A/B builds of libfz.so: bash tools/ab_build.sh NAME [nvcc -D flags...] -> ab/libfz_NAME.so (tools select it with
# FZ_LIB_PATH=ab/libfz_NAME.so; the product build is __graft_entry__.build())
N=$1; shift
mkdir -p ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --split-compile=0 -diag-suppress 128,186 "$@" -o ab/libfz_$N.so paper_2407_20474_b200/csrc/fz.cu
