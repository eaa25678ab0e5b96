#!/bin/bash
# A/B of the decode GEMM's pre-wait weight prefetch depth: cold (event-bracketed) launches and
# the PDL-chained decode step.
for v in default pre4 pre2; do
  if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
  echo "== $v"
  env $L timeout 200 python tools/gemm_cold.py --body 2>&1 | grep "copies=8"
  env $L timeout 200 python tools/profile_step.py --ctx 2048 --steps 40 2>&1 | tail -1
done
