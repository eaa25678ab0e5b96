"""One fused-epilogue GEMM launch (for ncu): --kind silu|resid|qkv, llama3-8b shapes."""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2512_15834_b200.modelcfg import SHAPES  # noqa: E402
from paper_2512_15834_b200.runtime import lib  # noqa: E402
from paper_2512_15834_b200.runtime.decoder import GemmEpi, KVPool, TiledWeight  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="silu")
    ap.add_argument("--M", type=int, default=608)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    s = SHAPES["llama3-8b"]
    M, d, F = a.M, s.d_model, s.d_ff
    parts = d // 128
    ss = torch.rand(M, parts, device="cuda") * 128
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if a.kind == "silu":
        N, K = 2 * F, d
        out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
        e = GemmEpi(kind=1, ss_in=ss.data_ptr(), ss_parts=parts, inv_dim=1.0 / d, eps=1e-5, out=out.data_ptr(), ldo=F)
    elif a.kind == "resid":
        N, K = d, s.q_dim
        x = torch.randn(M, d, device="cuda")
        xb = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
        e = GemmEpi(kind=3, out=xb.data_ptr(), ldo=d, x=x.data_ptr(), ldx=d, ss_out=ss.data_ptr(), ss_parts=parts)
    else:
        N, K = s.q_dim + 2 * s.kv_dim, d
        pool = KVPool(s.with_layers(1), M // 16 + 64, 4, M // 16 + 8)
        pool.reserve(0, M + 16)
        pool.sync(st.value)
        slot_of = torch.zeros(M, dtype=torch.int32, device="cuda")
        pos = torch.arange(M, dtype=torch.int32, device="cuda")
        q = torch.empty(M, s.q_dim, device="cuda", dtype=torch.bfloat16)
        e = GemmEpi(kind=2, ss_in=ss.data_ptr(), ss_parts=parts, inv_dim=1.0 / d, eps=1e-5, out=q.data_ptr(),
                    ldo=s.q_dim, pool=pool.h.value, layer=0, n_q=s.n_q, slot_of=slot_of.data_ptr(),
                    pos_of=pos.data_ptr(), rope_theta=s.rope_theta)
    tw = TiledWeight(torch.randn(N, K, device="cuda", dtype=torch.bfloat16))
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    work = torch.zeros(M, N, device="cuda")
    for _ in range(a.reps):
        rc = lib.load().stb_gemm_bf16_fused(C.c_void_p(A.data_ptr()), K, C.c_void_p(tw.data_ptr()), 0,
                                            C.c_void_p(work.data_ptr()), N, M, N, K, 4, C.byref(e), st)
        assert rc == 0, lib.load().stb_last_error()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
