#!/bin/bash
# In-step A/B of tuning variants on decode-only steps (B = 32) at several contexts, alternated.
CTXS=${CTXS:-"2048 4096"}
for c in $CTXS; do
  for r in 1 2; do
    for v in default "$@"; do
      if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
      echo "$v ctx $c run $r: $(env $L timeout 200 python tools/profile_step.py --ctx $c --steps 30 2>&1 | tail -1 | sed 's/.*median step //')"
    done
  done
done
