python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_canary.py -q -x -k oss > gpurun_out/r2s_canary.log 2>&1; echo canary=$?
tail -3 gpurun_out/r2s_canary.log
timeout 300 python tools/profile_step.py --steps 12 --ctx 2048 --timers 2>&1 | tail -12
timeout 300 python tools/profile_step.py --steps 12 --ctx 2048 --mix 1x470 --timers 2>&1 | tail -12
timeout 300 python tools/profile_step.py --steps 12 --ctx 2048 --mix 8x60 --timers 2>&1 | tail -12
