#!/bin/bash
# In-step A/B of tuning variants (tools/build_variant.sh): decode steps of 32 rows at ctx 2k with
# one prefill run of each size packed in (tools/profile_step.py --mix), variants alternated.
MIXES=${MIXES:-"1x150 1x300 1x576 1x1000"}
for m in $MIXES; do
  for r in 1 2; do
    for v in default "$@"; do
      if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
      echo "$v mix $m run $r: $(env $L timeout 200 python tools/profile_step.py --ctx 2048 --steps 24 --mix $m 2>&1 | tail -1 | sed 's/.*median step //')"
    done
  done
done
