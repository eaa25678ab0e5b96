#!/bin/bash
# compute-sanitizer over small kernel-test cases of K1-K5 and the MoE kernels (one GPU):
# memcheck (out-of-bounds / misaligned global + shared accesses), racecheck (shared-memory
# hazards) and synccheck (barrier misuse). Usage: bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out}
mkdir -p $OUT
SEL='attn_decode and tiny and ctxs1 or attn_decode and tiny and 16 or attn_prefill and tiny and unit or gemm_bf16 and 7-384 or gemm_w_tiled and 1-256 or spec_validate or kv_commit_roundtrip or moe_gemm_mxfp4 and 1-16 or moe_route and 37 or moe_gather or attn_decode_window_sinks and ctxs1-16 or attn_prefill_window_sinks and runs3-32'
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 700 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -x -k "$SEL" > $OUT/sanitize_$tool.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_$tool.log | tail -3
done
