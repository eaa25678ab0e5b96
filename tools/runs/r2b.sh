set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m oracle.gen_canary llama3-8b qwen3-32b > gpurun_out/r2b_canary.log 2>&1; echo canary=$?
mkdir -p gpurun_out/golden && cp tests/golden/canary_*.npz gpurun_out/golden/
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2b_gputest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r2b_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_bench.log 2> gpurun_out/r2b_bench.err; echo bench=$?
tail -c 1500 gpurun_out/r2b_bench.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_ref.log 2> gpurun_out/r2b_ref.err; echo ref=$?
tail -c 1500 gpurun_out/r2b_ref.log
