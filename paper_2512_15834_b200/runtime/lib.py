"""ctypes binding of libstb200.so (the C ABI in include/stb200.h).

No fallback: if the library is missing or CUDA is unavailable, `load()`
raises `KernelError`. Every wrapper checks the returned status and raises
`KernelError` / `KVCapacityError` with `stb_last_error()`.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ..errors import KernelError, KVCapacityError

# STB200_LIB selects a tuning variant built by tools/build_variant.sh (same ABI)
LIB_PATH = Path(os.environ.get("STB200_LIB") or Path(__file__).resolve().parent.parent / "lib" / "libstb200.so")

P = C.c_void_p
I32 = C.c_int
I64 = C.c_int64
F32 = C.c_float

# name -> (restype, argtypes); mirrors include/stb200.h one to one
SIGNATURES: dict[str, tuple] = {
    "stb_last_error": (C.c_char_p, []),
    "stb_version": (I32, []),
    "stb_launch_count": (I64, []),
    "stb_kv_pool_create": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, C.POINTER(P)]),
    "stb_kv_pool_destroy": (I32, [P]),
    "stb_kv_reserve": (I32, [P, I32, I32]),
    "stb_kv_truncate": (I32, [P, I32, I32]),
    "stb_kv_release": (I32, [P, I32]),
    "stb_kv_free_blocks": (I32, [P]),
    "stb_kv_slot_len": (I32, [P, I32]),
    "stb_kv_slot_blocks": (I32, [P, I32, P, I32]),
    "stb_kv_sync": (I32, [P, P]),
    "stb_kv_layer_ptrs": (I32, [P, I32, C.POINTER(P), C.POINTER(P)]),
    "stb_kv_block_table": (I32, [P, C.POINTER(P), C.POINTER(I32)]),
    "stb_kv_commit": (I32, [P, I32, P, P, I64, P, P, I32, P]),
    "stb_kv_copy_blocks": (I32, [P, P, P, I32, P]),
    "stb_qkv_rope_commit": (I32, [P, I32, P, P, P, P, I32, I32, F32, I32, P]),
    "stb_qkv_norm_rope_commit": (I32, [P, I32, P, P, P, P, I32, I32, F32, P, P, F32, I32, P]),
    "stb_attn_decode_workspace": (I64, [I32, I32, I32, I32]),
    "stb_attn_decode": (I32, [P, I32, P, P, P, P, I32, I32, F32, I32, P, P]),
    "stb_attn_decode_mq": (I32, [P, I32, P, P, P, P, P, P, I32, I32, F32, I32, P, P]),
    "stb_attn_decode_planned": (I32, [P, I32, P, P, P, P, P, P, I32, I32, F32, I32, I32, P, P]),
    "stb_attn_prefill": (I32, [P, I32, P, P, P, P, P, I32, I32, I32, F32, I32, P]),
    "stb_attn_prefill_split": (I32, [P, I32, P, P, P, P, P, I32, I32, I32, F32, I32, I32, P]),
    "stb_spec_validate": (I32, [P, P, P, P, P, P, P, P, I32, P, P, P, P]),
    "stb_key_match": (I32, [P, P, I32, P, P, I32, P, P]),
    "stb_gemm_bf16": (I32, [P, I64, P, I64, P, I64, I32, I32, I32, I32, I32, P]),
    "stb_gemm_is_stream": (I32, [I32, I32, I32]),
    "stb_gemm_bf16_fused": (I32, [P, I64, P, I64, P, I64, I32, I32, I32, I32, P, P]),
    "stb_gemm_block": (I32, [P, I32, I32, P]),
    "stb_embed_prep": (I32, [P, P, P, P, P, I32, I32, I32, P]),
    "stb_weight_tiled_elems": (I64, [I32, I32]),
    "stb_weight_tile": (I32, [P, I64, I32, I32, P, P]),
    "stb_embed": (I32, [P, P, P, I32, I32, P]),
    "stb_add_rmsnorm": (I32, [P, P, P, P, I32, I32, F32, I32, P]),
    "stb_silu_mul": (I32, [P, P, I32, I32, I32, P]),
    "stb_gather_rmsnorm": (I32, [P, P, P, P, I32, I32, F32, P]),
    "stb_sample_forced": (I32, [P, I64, P, I32, I32, F32, P, P, P, I32, P]),
    # gpt-oss family (config C4)
    "stb_qkv_rope_commit_ex": (I32, [P, I32, P, P, P, P, I32, I32, F32, P, F32, P, I32, P]),
    "stb_attn_decode_ex": (I32, [P, I32, P, P, P, P, I32, I32, F32, I32, I32, P, P, P]),
    "stb_attn_prefill_ex": (I32, [P, I32, P, P, P, P, P, I32, I32, I32, F32, I32, I32, I32, P, P]),
    "stb_add_bias_rmsnorm": (I32, [P, P, P, P, P, I32, I32, F32, I32, P]),
    "stb_moe_route": (I32, [P, I64, P, I32, I32, I32, P, P, P, P, P]),
    "stb_moe_gather": (I32, [P, I64, I32, I32, I32, I32, P, P, P, P, P, P, P]),
    "stb_moe_gemm_mxfp4": (I32, [P, I32, P, P, P, I32, I32, I32, I32, F32, P, I64, I32, P]),
    "stb_moe_quant_bytes": (I64, [I32, I32]),
    "stb_moe_quant_scale_words": (I64, [I32, I32]),
    "stb_moe_quant": (I32, [P, I64, I32, I32, I32, P, P, P]),
    "stb_moe_gather_mx": (I32, [P, I64, I32, I32, I32, I32, P, P, P, P, P, I32, P, P, P]),
    "stb_moe_gemm_mx_q": (I32, [P, P, I32, P, P, P, I32, I32, I32, I32, F32, P, I64, I32, P, P, I32, P]),
    "stb_moe_gemm_mx": (I32, [P, P, I32, P, P, P, I32, I32, I32, I32, F32, P, I64, I32, P]),
    "stb_moe_combine": (I32, [P, P, I32, I32, I32, P, P, P, P, F32, P, I32, P]),
}

STATUS_CAPACITY = -4

_lib = None


def load_raw(path: Path | str = LIB_PATH) -> C.CDLL:
    """dlopen the library and bind every signature (no CUDA needed)."""
    if not Path(path).exists():
        raise KernelError(f"{path} not built: run __graft_entry__.build()")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def load() -> C.CDLL:
    """The library for the product path; fails loudly without a GPU."""
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise KernelError("B200 runtime needs CUDA; no device visible (there is no CPU fallback)")
        _lib = load_raw(LIB_PATH)
    return _lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = _lib.stb_last_error().decode() if _lib is not None else ""
        if rc == STATUS_CAPACITY:
            raise KVCapacityError(f"{what}: {msg}")
        raise KernelError(f"{what} failed ({rc}): {msg}")
    return rc


_DEBUG_SYNC = bool(os.environ.get("STB200_DEBUG_SYNC"))


def call(name: str, *args) -> int:
    rc = check(getattr(load(), name)(*args), name)
    if _DEBUG_SYNC:  # debugging aid: attribute asynchronous faults to the launching call
        import torch

        try:
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001
            raise KernelError(f"{name}: asynchronous fault: {exc}") from exc
    return rc
