# In-step attribution under PDL: decode-step time with kernel classes left out
# (STB200_SKIP_KERNELS, debug only). Usage: bash tools/skip_probe.sh [ctx] [batch]
CTX=${1:-2048}; BATCH=${2:-32}
for sk in "" stb_attn_decode stb_gemm_bf16 gemm:wqkv gemm:wo gemm:w_gate_up gemm:w_down gemm:lm_head stb_add_rmsnorm stb_qkv_rope_commit stb_silu_mul; do
  echo -n "skip=[$sk] "; STB200_SKIP_KERNELS=$sk timeout 200 python tools/profile_step.py --steps 40 --ctx $CTX --batch $BATCH 2>&1 | tail -1
done
