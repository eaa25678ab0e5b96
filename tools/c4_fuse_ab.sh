#!/bin/bash
# In-step A/B of the fused down-input split (STB200_MOE_FUSED_SPLIT) on the C4 shape
for m in "" "--mix 1x400"; do
  for r in 1 2 3; do
    for v in 1 0; do
      echo "fused=$v [$m] run $r: $(STB200_MOE_FUSED_SPLIT=$v timeout 300 python tools/profile_step.py --shape gpt-oss-120b --batch 32 --ctx 2048 --steps 16 $m 2>&1 | tail -1 | sed 's/.*median step //')"
    done
  done
done
