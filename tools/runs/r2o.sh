python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -2
python tools/bench_moe.py
timeout 900 python -m pytest tests/test_gpu_batch_parity.py -q -x -k "preemption" 2>&1 | tail -15
