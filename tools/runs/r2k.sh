python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -c 1 -o gpurun_out/r2k_moe_t32 python tools/bench_moe.py --T 32 --iters 1 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:moe_gemm -c 1 -o gpurun_out/r2k_moe_t2048 python tools/bench_moe.py --T 2048 --iters 1 > /dev/null 2>&1; echo ncu2=$?
ls -la gpurun_out
