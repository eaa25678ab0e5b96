set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2r_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2r_gputest.log 2>&1; echo pytest=$?
tail -8 gpurun_out/r2r_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2r_bench.log 2> gpurun_out/r2r_bench.err; echo bench=$?
tail -c 1500 gpurun_out/r2r_bench.log
timeout 1200 python bench.py --config c4 --steps 20 --warmup 5 > gpurun_out/r2r_bench_c4.log 2> gpurun_out/r2r_bench_c4.err; echo benchc4=$?
tail -c 1500 gpurun_out/r2r_bench_c4.log
tail -3 gpurun_out/r2r_bench_c4.err
