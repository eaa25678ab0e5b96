#!/bin/bash
# Build a tuning variant of libstb200.so with extra nvcc defines, e.g.
#   bash tools/build_variant.sh emu3 -DSTB_EXP_EMU=3
# -> paper_2512_15834_b200/lib/variants/emu3/libstb200.so; select it with STB200_LIB=<path>.
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=${SRC:-$ROOT/paper_2512_15834_b200/csrc}
OUT=$ROOT/paper_2512_15834_b200/lib/variants/$NAME
mkdir -p $OUT/obj
for f in kv attention attn_prefill_tc gemm ops moe; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $C/$f.cu -o $OUT/obj/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libstb200.so $OUT/obj/*.o -lcudart
echo $OUT/libstb200.so
