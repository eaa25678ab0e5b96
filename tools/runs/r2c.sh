set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m oracle.gen_canary llama3-8b qwen3-32b > gpurun_out/r2c_canary.log 2>&1; echo canary=$?
mkdir -p gpurun_out/golden && cp tests/golden/canary_*.npz gpurun_out/golden/
timeout 1200 python -m pytest tests/test_gpu_batch_parity.py tests/test_gpu_canary.py -x -q > gpurun_out/r2c_newtests.log 2>&1; echo newtests=$?
tail -5 gpurun_out/r2c_newtests.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2c_gputest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r2c_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c_bench.log 2> gpurun_out/r2c_bench.err; echo bench=$?
tail -c 3000 gpurun_out/r2c_bench.log
