python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -2
bash tools/build_variant.sh n1c2 -DSTB_MOE_NTP=1 > /dev/null &
bash tools/build_variant.sh n1c3 -DSTB_MOE_NTP=1 -DSTB_MOE_CONV_PAR=3 > /dev/null &
bash tools/build_variant.sh n2c1 -DSTB_MOE_CONV_PAR=1 > /dev/null &
wait
for v in base n1c2 n1c3 n2c1; do
  echo "== $v"
  if [ $v = base ]; then python tools/bench_moe.py --T 8,32,512; else STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so python tools/bench_moe.py --T 8,32,512; fi
done
timeout 900 python -m pytest tests/test_gpu_batch_parity.py -q -x -k "preemption" 2>&1 | tail -15
