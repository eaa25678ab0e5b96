python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh n1 -DSTB_MOE_NTP=1 > /dev/null &
bash tools/build_variant.sh stream2 -DSTB_MOE_SKIP_CONVERT=1 -DSTB_MOE_MMA_PER_STAGE=0 > /dev/null &
bash tools/build_variant.sh stream1 -DSTB_MOE_SKIP_CONVERT=1 -DSTB_MOE_MMA_PER_STAGE=0 -DSTB_MOE_NTP=1 > /dev/null &
bash tools/build_variant.sh noconv2 -DSTB_MOE_SKIP_CONVERT=1 > /dev/null &
wait
for v in base n1 stream2 stream1 noconv2; do
  echo "== $v"
  if [ $v = base ]; then python tools/bench_moe.py --T 32,512; else STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so python tools/bench_moe.py --T 32,512; fi
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -c 1 -o gpurun_out/r2p_moe_t32 python tools/bench_moe.py --T 32 --iters 1 > /dev/null 2>&1; echo ncu=$?
