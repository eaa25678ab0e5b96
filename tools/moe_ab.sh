#!/bin/bash
# A/B of MoE grouped-GEMM tuning variants (tools/build_variant.sh) at gpt-oss-120b expert shapes
IMPL=${IMPL:-mx}
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
  echo "== $v"; env $L timeout 120 python tools/bench_moe.py --T ${TS:-8,32,128} --impl $IMPL 2>&1 | grep "T="
done
