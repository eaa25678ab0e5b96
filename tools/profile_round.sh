#!/bin/bash
# One GPU call's worth of evidence for profiles/: launch lists of steady-state decode and
# mixed (prefill + decode) steps at the bench's context, full ncu captures of the hot
# kernels, and a kernel microbenchmark table. Usage: bash tools/profile_round.sh [outdir]
set -x
OUT=${1:-gpurun_out}
CTX=${CTX:-2048}
mkdir -p $OUT
# microbenchmarks first: after the ncu replay sessions the GPU runs tensor-heavy kernels
# ~25% slower for a while (power / thermal state), which skewed earlier tables
timeout 300 python tools/bench_kernels.py --what gemm,attn,prefill,small \
  --prefill-cases 4x2048x2048,1x2048x34816,8x512x4096,32x33x4096,1x33x2150,1x600x2700 > $OUT/kernels.txt 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_decode.csv python tools/profile_step.py --profile --steps 8 --profile-steps 2 --ctx $CTX > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_decode.csv 2 > $OUT/launches_decode.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_mixed.csv python tools/profile_step.py --profile --steps 8 --profile-steps 2 --ctx $CTX --mix 1x576 > /dev/null 2>&1
python tools/launch_table.py $OUT/launches_mixed.csv 2 > $OUT/launches_mixed.txt
timeout 400 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"attn_decode|gemm_bf16" -c 6 -o $OUT/full_decode python tools/profile_step.py --profile --steps 6 --profile-steps 1 --ctx $CTX > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm -c 1 -s 2 \
  -o $OUT/full_gemm_prefill python tools/gemm_once.py --M 608 --N 28672 --K 4096 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_tc -c 2 \
  -o $OUT/full_prefill python tools/bench_kernels.py --what prefill > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_tc -c 1 \
  -o $OUT/full_prefill_c5 python tools/bench_kernels.py --what prefill --prefill-cases 1x2048x34816 > /dev/null 2>&1
ls -la $OUT
