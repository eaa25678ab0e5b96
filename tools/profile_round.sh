#!/bin/bash
# One GPU call's worth of evidence for profiles/: launch list of steady-state decode
# steps, full ncu captures of the hot kernels, and a kernel microbenchmark table.
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_decode.csv python tools/profile_step.py --profile --steps 8 --profile-steps 2 --ctx 4096 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_decode.csv 2 > $OUT/launches_decode.txt
timeout 400 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"attn_decode|gemm_bf16" -c 6 -o $OUT/full_decode python tools/profile_step.py --profile --steps 6 --profile-steps 1 --ctx 4096 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_tc -c 2 \
  -o $OUT/full_prefill python tools/bench_kernels.py --what prefill > /dev/null 2>&1
timeout 300 python tools/bench_kernels.py > $OUT/kernels.txt 2>&1
ls -la $OUT
