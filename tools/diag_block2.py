"""Localise a block-vs-per-op difference: single-phase and two-phase chains vs the per-op kernels."""
import ctypes as C, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2512_15834_b200.runtime import lib
from paper_2512_15834_b200.runtime.decoder import BlockOp, OP_GEMM, OP_NORM, OP_SILU, TiledWeight
P = lambda t: C.c_void_p(t.data_ptr())
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
rel = lambda a, b: float((a.float() - b.float()).norm() / max(b.float().norm(), 1e-30))
torch.manual_seed(0)
for M in (1, 5, 32):
    for N, K in ((4096, 4096), (6144, 4096), (28672, 4096), (4096, 14336)):
        x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
        tw = TiledWeight(w)
        c1 = torch.zeros(M, N, device="cuda"); c2 = torch.zeros(M, N, device="cuda")
        lib.call("stb_gemm_bf16", P(x), K, P(tw), 0, P(c1), N, M, N, K, 0, 1 | 4, st())
        ops = (BlockOp * 1)(BlockOp(kind=OP_GEMM, x=x.data_ptr(), ldx=K, w=tw.data_ptr(), c=c2.data_ptr(), ldc=N, n=N, k=K))
        lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 1, M, st())
        ref = x.float() @ w.float().t()
        torch.cuda.synchronize()
        print(f"M={M} N={N} K={K}: gemm per-op vs fp32 {rel(c1, ref):.2e}  block vs fp32 {rel(c2, ref):.2e}  block vs per-op {rel(c2, c1):.2e}")
# two-phase: GEMM -> NORM -> GEMM
M, d, F = 3, 4096, 14336
xa = torch.randn(M, d, device="cuda", dtype=torch.bfloat16)
w1 = torch.randn(d, d, device="cuda", dtype=torch.bfloat16) * 0.02
w2 = torch.randn(2 * F, d, device="cuda", dtype=torch.bfloat16) * 0.02
w3 = torch.randn(d, F, device="cuda", dtype=torch.bfloat16) * 0.02
nw = (torch.rand(d, device="cuda") + 0.5).to(torch.bfloat16)
t1, t2, t3 = TiledWeight(w1), TiledWeight(w2), TiledWeight(w3)
def state():
    return dict(x=torch.randn(M, d, device="cuda", generator=torch.Generator("cuda").manual_seed(7)),
                proj=torch.zeros(M, d, device="cuda"), h=torch.zeros(M, d, device="cuda", dtype=torch.bfloat16),
                gu=torch.zeros(M, 2 * F, device="cuda"), act=torch.zeros(M, F, device="cuda", dtype=torch.bfloat16),
                out=torch.zeros(M, d, device="cuda"))
a = state()
lib.call("stb_gemm_bf16", P(xa), d, P(t1), 0, P(a["proj"]), d, M, d, d, 0, 5, st())
lib.call("stb_add_rmsnorm", P(a["x"]), P(a["proj"]), P(nw), P(a["h"]), M, d, 1e-5, M, st())
lib.call("stb_gemm_bf16", P(a["h"]), d, P(t2), 0, P(a["gu"]), 2 * F, M, 2 * F, d, 0, 5, st())
lib.call("stb_silu_mul", P(a["gu"]), P(a["act"]), M, F, M, st())
lib.call("stb_gemm_bf16", P(a["act"]), F, P(t3), 0, P(a["out"]), d, M, d, F, 0, 5, st())
b = state()
ops = (BlockOp * 5)(
    BlockOp(kind=OP_GEMM, x=xa.data_ptr(), ldx=d, w=t1.data_ptr(), c=b["proj"].data_ptr(), ldc=d, n=d, k=d),
    BlockOp(kind=OP_NORM, c=b["proj"].data_ptr(), w=nw.data_ptr(), n=d, x_res=b["x"].data_ptr(), y=b["h"].data_ptr(), eps=1e-5),
    BlockOp(kind=OP_GEMM, x=b["h"].data_ptr(), ldx=d, w=t2.data_ptr(), c=b["gu"].data_ptr(), ldc=2 * F, n=2 * F, k=d),
    BlockOp(kind=OP_SILU, c=b["gu"].data_ptr(), y=b["act"].data_ptr(), n=F),
    BlockOp(kind=OP_GEMM, x=b["act"].data_ptr(), ldx=F, w=t3.data_ptr(), c=b["out"].data_ptr(), ldc=d, n=d, k=F))
lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 5, M, st())
torch.cuda.synchronize()
for k in ("x", "h", "act", "out"):
    print(k, f"{rel(b[k], a[k]):.3e}", "max abs", float((b[k].float() - a[k].float()).abs().max()))
print("proj/gu zero:", float(b["proj"].abs().max()), float(b["gu"].abs().max()))
# ROPE phase vs stb_qkv_rope_commit: [NORM, GEMM QKV, ROPE] on a pool
from paper_2512_15834_b200.modelcfg import SHAPES
from paper_2512_15834_b200.runtime.decoder import KVPool, OP_ROPE
import dataclasses
for base in ("llama3-8b", "qwen3-32b"):
    shape = dataclasses.replace(SHAPES[base], layers=1, vocab=1024)
    for M in (1, 7):
        pools = []
        outs = []
        for mode in ("op", "blk"):
            pool = KVPool(shape, num_blocks=64, max_slots=M + 1, max_blocks_per_slot=8)
            for b in range(M): pool.reserve(b, 71)
            pool.sync(torch.cuda.current_stream().cuda_stream)
            g = torch.Generator("cuda").manual_seed(11)
            x = torch.randn(M, shape.d_model, device="cuda", generator=g)
            wq = torch.randn(shape.q_dim + 2 * shape.kv_dim, shape.d_model, device="cuda", generator=g).to(torch.bfloat16) * 0.02
            nw = (torch.rand(shape.d_model, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
            qn = (torch.rand(shape.d_head, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
            kn = (torch.rand(shape.d_head, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
            tw = TiledWeight(wq)
            h = torch.zeros(M, shape.d_model, device="cuda", dtype=torch.bfloat16)
            qkv = torch.zeros(M, shape.q_dim + 2 * shape.kv_dim, device="cuda")
            q = torch.zeros(M, shape.q_dim, device="cuda", dtype=torch.bfloat16)
            slot = torch.arange(M, device="cuda", dtype=torch.int32)
            pos = torch.full((M,), 70, device="cuda", dtype=torch.int32)
            N, K = wq.shape
            qk = shape.qk_norm
            if mode == "op":
                lib.call("stb_add_rmsnorm", P(x), None, P(nw), P(h), M, shape.d_model, 1e-5, 0, st())
                lib.call("stb_gemm_bf16", P(h), K, P(tw), 0, P(qkv), N, M, N, K, 0, 5, st())
                if qk:
                    lib.call("stb_qkv_norm_rope_commit", pool.h, 0, P(qkv), P(q), P(slot), P(pos), M, shape.n_q, shape.rope_theta, P(qn), P(kn), 1e-6, M, st())
                else:
                    lib.call("stb_qkv_rope_commit", pool.h, 0, P(qkv), P(q), P(slot), P(pos), M, shape.n_q, shape.rope_theta, M, st())
            else:
                ops = (BlockOp * 3)(
                    BlockOp(kind=OP_NORM, w=nw.data_ptr(), n=shape.d_model, x_res=x.data_ptr(), y=h.data_ptr(), eps=1e-5),
                    BlockOp(kind=OP_GEMM, x=h.data_ptr(), ldx=K, w=tw.data_ptr(), c=qkv.data_ptr(), ldc=N, n=N, k=K),
                    BlockOp(kind=OP_ROPE, c=qkv.data_ptr(), y=q.data_ptr(), pool=pool.h, layer=0, n_q=shape.n_q,
                            slot_of=slot.data_ptr(), pos_of=pos.data_ptr(), rope_theta=shape.rope_theta,
                            q_norm=qn.data_ptr() if qk else None, k_norm=kn.data_ptr() if qk else None, eps=1e-6))
                lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 3, M, st())
            torch.cuda.synchronize()
            kp, vp = pool.layer_ptrs(0)
            nbytes = 64 * shape.n_kv * 16 * shape.d_head
            kt = torch.empty(nbytes, dtype=torch.bfloat16, device="cuda"); vt = torch.empty_like(kt)
            import ctypes
            cudart = torch.cuda.cudart()
            torch.cuda.synchronize()
            kt.copy_(torch.frombuffer(bytearray(0), dtype=torch.uint8).new_empty(0) if False else kt)
            outs.append((h.clone(), q.clone(), qkv.clone(), pool))
        (h1, q1, c1, p1), (h2, q2, c2, p2) = outs
        print(base, M, "h", rel(h2, h1), "q", rel(q2, q1), "qkv cleared", float(c1.abs().max()), float(c2.abs().max()))
