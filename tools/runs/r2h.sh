python tools/diag_moe.py
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k gpt_oss > gpurun_out/r2h_par.log 2>&1; echo par=$?
tail -5 gpurun_out/r2h_par.log
timeout 900 python -m pytest tests/test_gpu_batch_parity.py -q -x -k gpt > gpurun_out/r2h_bpar.log 2>&1; echo bpar=$?
tail -5 gpurun_out/r2h_bpar.log
