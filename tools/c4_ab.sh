for m in "" "--mix 1x400"; do
  for r in 1 2; do
    for v in default nocnt oldstager; do
      if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
      echo "$v [$m] run $r: $(env $L timeout 300 python tools/profile_step.py --shape gpt-oss-120b --batch 32 --ctx 2048 --steps 16 $m 2>&1 | tail -1 | sed 's/.*median step //')"
    done
  done
done
