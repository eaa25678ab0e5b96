python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh mma1 -DSTB_MOE_MMA_PER_STAGE=1 > /dev/null
bash tools/build_variant.sh nost -DSTB_MOE_SKIP_TMEM_STORE=1 > /dev/null
bash tools/build_variant.sh both -DSTB_MOE_SKIP_TMEM_STORE=1 -DSTB_MOE_MMA_PER_STAGE=1 > /dev/null
for v in base mma1 nost both; do
  echo "== $v"
  if [ $v = base ]; then python tools/bench_moe.py --T 32,512; else STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so python tools/bench_moe.py --T 32,512; fi
done
