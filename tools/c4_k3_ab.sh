#!/bin/bash
# In-step A/B of K3 ring depth on the C4 shape (d_head 64): decode steps of 32 rows at ctx 2k
for r in 1 2; do
  for v in default "$@"; do
    if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
    echo "$v run $r: $(env $L timeout 300 python tools/profile_step.py --shape gpt-oss-120b --batch 32 --ctx ${CTX:-2048} --steps 16 2>&1 | tail -1 | sed 's/.*median step //')"
  done
done
