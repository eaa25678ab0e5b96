set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_moe.py -q -x > gpurun_out/r2f_moe.log 2>&1; echo moe=$?
tail -30 gpurun_out/r2f_moe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k gpt_oss > gpurun_out/r2f_par.log 2>&1; echo par=$?
tail -30 gpurun_out/r2f_par.log
timeout 900 python -m pytest tests/test_gpu_batch_parity.py -q -x -k gpt > gpurun_out/r2f_bpar.log 2>&1; echo bpar=$?
tail -30 gpurun_out/r2f_bpar.log
