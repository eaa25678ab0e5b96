set -x
free -g | head -2; nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_gputest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r2a_gputest.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2a_bench.log 2> gpurun_out/r2a_bench.err; echo bench=$?
tail -c 3000 gpurun_out/r2a_bench.log
