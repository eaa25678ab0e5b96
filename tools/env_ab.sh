#!/bin/bash
# In-step A/B of an environment switch on decode-only steps (B = 32): VAR=0 vs VAR=1, alternated.
#   tools/env_ab.sh STB200_K3_PLAN     (CTXS / MIX override the contexts / packed prefill,
#                                       VALS the values: default "0 1")
VAR=$1
VALS=${VALS:-"0 1"}
CTXS=${CTXS:-"2048 4096 8192"}
for c in $CTXS; do
  for r in 1 2 3; do
    for v in $VALS; do
      echo "$VAR=$v ctx $c run $r: $(env $VAR=$v timeout 200 python tools/profile_step.py --ctx $c --steps 30 ${MIX:+--mix $MIX} 2>&1 | tail -1 | sed 's/.*median step //')"
    done
  done
done
