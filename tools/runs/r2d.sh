set -x
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/r2d_smoke.log
timeout 900 python -m oracle.gen_canary llama3-8b qwen3-32b > gpurun_out/r2d_canary.log 2>&1; echo canary=$?
cat gpurun_out/r2d_canary.log | tail -3
mkdir -p gpurun_out/golden && cp tests/golden/canary_*.npz gpurun_out/golden/
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2d_gputest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r2d_gputest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2d_bench.log 2> gpurun_out/r2d_bench.err; echo bench=$?
tail -c 3000 gpurun_out/r2d_bench.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2d_ref.log 2> gpurun_out/r2d_ref.err; echo ref=$?
tail -c 1500 gpurun_out/r2d_ref.log
