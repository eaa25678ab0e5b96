python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh noconv -DSTB_MOE_SKIP_CONVERT=1 > /dev/null
bash tools/build_variant.sh ring120 -DSTB_MOE_RING_KB=120 > /dev/null
bash tools/build_variant.sh noconv_mma1 -DSTB_MOE_SKIP_CONVERT=1 -DSTB_MOE_MMA_PER_STAGE=1 > /dev/null
for v in noconv noconv_mma1 ring120; do
  echo "== $v"
  STB200_LIB=paper_2512_15834_b200/lib/variants/$v/libstb200.so python tools/bench_moe.py --T 32,512
done
