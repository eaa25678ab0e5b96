set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_canary.py -x -q > gpurun_out/r2e_canary.log 2>&1; echo canary=$?
tail -5 gpurun_out/r2e_canary.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2e_bench.log 2> gpurun_out/r2e_bench.err; echo bench=$?
tail -c 4000 gpurun_out/r2e_bench.log
tail -5 gpurun_out/r2e_bench.err
