python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k gemm 2>&1 | tail -2
python tools/bench_moe.py
