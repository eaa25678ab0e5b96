#!/bin/bash
# compute-sanitizer memcheck + racecheck on K3's planned-partition and multi-query paths (tiny shape)
mkdir -p gpurun_out/r2_sanitize
SEL='attn_decode_planned and tiny or attn_decode_multi_query and tiny'
for tool in memcheck racecheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_kernels.py -q -k "$SEL" > gpurun_out/r2_sanitize/sanitize_${tool}_k3_planned.log 2>&1
  tail -2 gpurun_out/r2_sanitize/sanitize_${tool}_k3_planned.log
done
