SEL='attn_decode and tiny and ctxs1 or attn_decode and tiny and 16 or gemm_bf16 and 7-384 or gemm_w_tiled and 1-256 or spec_validate or kv_commit_roundtrip or moe_gemm_mxfp4 and 1-16 or moe_route and 37 or moe_gather or attn_decode_window_sinks and ctxs1-16'
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --target-processes all --print-limit 50 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_moe.py -q -k "$SEL" > gpurun_out/r2_sanitize/sanitize_synccheck_nonK2.log 2>&1
tail -3 gpurun_out/r2_sanitize/sanitize_synccheck_nonK2.log
