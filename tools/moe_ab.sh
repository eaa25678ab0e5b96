for v in default ring224 xs16 cpar1 ntp1; do
  if [ $v = default ]; then L=""; else L="STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so"; fi
  echo "== $v"; env $L timeout 120 python tools/bench_moe.py --T 32,128 2>&1 | grep "^T="
done
