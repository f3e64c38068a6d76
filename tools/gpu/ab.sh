# A/B of libfz builds on one box: bash tools/gpu/ab.sh TAG "CONFIGS" lib1 lib2 ... (interleaved twice)
O=gpurun_out
T=$1; C=$2; shift 2
for pass in 1 2; do
  for lib in "$@"; do
    FZ_LIB_PATH=$lib timeout 600 python tools/ab_time.py $(basename $lib .so) $C >> $O/${T}_ab.log 2>&1
  done
done
