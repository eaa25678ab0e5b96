for r in 1 2; do
  for v in default ring200; do
    if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
    echo "$v c3 run $r: $(env $L timeout 300 python tools/profile_step.py --shape qwen3-32b --batch 64 --ctx 2048 --steps 20 --headroom 512 2>&1 | tail -1 | sed 's/.*median step //')"
  done
done
