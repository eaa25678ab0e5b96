set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_service_live.py -q -x > gpurun_out/r2i_live.log 2>&1; echo live=$?
tail -5 gpurun_out/r2i_live.log
free -g | head -2
timeout 1800 python -m oracle.gen_canary gpt-oss-120b > gpurun_out/r2i_canary.log 2>&1; echo canary=$?
tail -3 gpurun_out/r2i_canary.log
mkdir -p gpurun_out/golden && cp tests/golden/canary_gpt-oss-120b.npz gpurun_out/golden/
timeout 1500 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/r2i_bench_c4.log 2> gpurun_out/r2i_bench_c4.err; echo bench=$?
tail -c 4000 gpurun_out/r2i_bench_c4.log
tail -20 gpurun_out/r2i_bench_c4.err
