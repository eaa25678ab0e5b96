"""The decode block (stb_gemm_block): a decode step's chain [O, add+norm, gate-up, SiLU, down,
add+norm, QKV(next layer), RoPE+commit] as ONE launch per layer, against the per-op launches it
replaces (stb_gemm_bf16 / stb_add_rmsnorm / stb_silu_mul / stb_qkv_norm_rope_commit, each checked
against torch fp32 in test_gpu_kernels.py).

* kernel level, same inputs: every phase's output equals the per-op kernel's to fp32
  reduction-order noise (the stream-K partial sums land in another order), the committed K/V
  rows and q to that noise, and every accumulator is left zeroed; shapes include tiny ones
  where most CTAs own no stream-K segment of a phase (the grid barrier must still count every
  CTA exactly once per phase);
* decoder level: a decode step through the block path against the per-op path (same weights,
  same KV) — logits / residual within 1e-2 (both paths carry run-to-run fp32 reduction noise of
  ~1e-3 through the random-init layers), with 2 launches per layer instead of 9.
The block path is opt-in (STB200_GEMM_BLOCK=1: measured slower than the per-op launches,
DESIGN.md §4); with it on, test_gpu_parity.py / test_gpu_batch_parity.py run decode steps through
it against the oracle. (Reference: the per-token decode charges
`engine.py:270,276,302,317`.)"""

import ctypes as C
import dataclasses

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def P(t):
    return C.c_void_p(t.data_ptr())


def st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def rel(a, b):
    return float((a.float() - b.float()).norm() / max(float(b.float().norm()), 1e-30))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_15834_b200.runtime import lib as L

    L.load()
    return L


@pytest.mark.parametrize("M", [1, 5, 32, 64])
@pytest.mark.parametrize("N,K", [(4096, 4096), (6144, 4096), (28672, 4096), (4096, 14336), (512, 256)])
def test_block_single_gemm(lib, M, N, K):
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, BlockOp, TiledWeight

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    tw = TiledWeight(w)
    c_op, c_blk = torch.zeros(M, N, device="cuda"), torch.zeros(M, N, device="cuda")
    lib.call("stb_gemm_bf16", P(x), K, P(tw), 0, P(c_op), N, M, N, K, 0, 1 | 4, st())
    ops = (BlockOp * 1)(BlockOp(kind=OP_GEMM, x=x.data_ptr(), ldx=K, w=tw.data_ptr(), c=c_blk.data_ptr(), ldc=N, n=N,
                                k=K))
    lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 1, M, st())
    ref = x.float() @ w.float().t()
    torch.cuda.synchronize()
    assert rel(c_blk, ref) < 1e-5
    assert rel(c_blk, c_op) < 1e-6


@pytest.mark.parametrize("M", [1, 3, 32, 64])
@pytest.mark.parametrize("d,F", [(4096, 14336), (256, 1024)])
def test_block_mlp_chain(lib, M, d, F):
    """[O, add+norm, gate-up, SiLU, down] vs the five per-op launches."""
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, OP_NORM, OP_SILU, BlockOp, TiledWeight

    g = torch.Generator(device="cuda").manual_seed(M + d)
    xa = torch.randn(M, d, device="cuda", generator=g).to(torch.bfloat16)
    w1, w2, w3 = ((torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
                  for n, k in ((d, d), (2 * F, d), (d, F)))
    nw = (torch.rand(d, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    x0 = torch.randn(M, d, device="cuda", generator=g)
    t1, t2, t3 = TiledWeight(w1), TiledWeight(w2), TiledWeight(w3)

    def state():
        return dict(x=x0.clone(), proj=torch.zeros(M, d, device="cuda"),
                    h=torch.zeros(M, d, device="cuda", dtype=torch.bfloat16), gu=torch.zeros(M, 2 * F, device="cuda"),
                    act=torch.zeros(M, F, device="cuda", dtype=torch.bfloat16), out=torch.zeros(M, d, device="cuda"))

    a = state()
    lib.call("stb_gemm_bf16", P(xa), d, P(t1), 0, P(a["proj"]), d, M, d, d, 0, 5, st())
    lib.call("stb_add_rmsnorm", P(a["x"]), P(a["proj"]), P(nw), P(a["h"]), M, d, 1e-5, M, st())
    lib.call("stb_gemm_bf16", P(a["h"]), d, P(t2), 0, P(a["gu"]), 2 * F, M, 2 * F, d, 0, 5, st())
    lib.call("stb_silu_mul", P(a["gu"]), P(a["act"]), M, F, M, st())
    lib.call("stb_gemm_bf16", P(a["act"]), F, P(t3), 0, P(a["out"]), d, M, d, F, 0, 5, st())
    b = state()
    ops = (BlockOp * 5)(
        BlockOp(kind=OP_GEMM, x=xa.data_ptr(), ldx=d, w=t1.data_ptr(), c=b["proj"].data_ptr(), ldc=d, n=d, k=d),
        BlockOp(kind=OP_NORM, c=b["proj"].data_ptr(), w=nw.data_ptr(), n=d, x_res=b["x"].data_ptr(),
                y=b["h"].data_ptr(), eps=1e-5),
        BlockOp(kind=OP_GEMM, x=b["h"].data_ptr(), ldx=d, w=t2.data_ptr(), c=b["gu"].data_ptr(), ldc=2 * F, n=2 * F,
                k=d),
        BlockOp(kind=OP_SILU, c=b["gu"].data_ptr(), y=b["act"].data_ptr(), n=F),
        BlockOp(kind=OP_GEMM, x=b["act"].data_ptr(), ldx=F, w=t3.data_ptr(), c=b["out"].data_ptr(), ldc=d, n=d, k=F))
    lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 5, M, st())
    torch.cuda.synchronize()
    assert rel(b["x"], a["x"]) < 1e-6
    # bf16 row-op outputs: identical unless an fp32 reduction-order difference crosses a rounding
    # boundary (one bf16 ulp on a few elements)
    for k in ("h", "act"):
        assert float((b[k].float() != a[k].float()).float().mean()) < 2e-2 and rel(b[k], a[k]) < 5e-3, k
    assert rel(b["out"], a["out"]) < 1e-3
    assert not b["proj"].any() and not b["gu"].any()  # accumulators left zeroed


@pytest.mark.parametrize("base", ["llama3-8b", "qwen3-32b", "tiny"])
@pytest.mark.parametrize("M", [1, 7, 64])
def test_block_qkv_chain(lib, base, M):
    """[add+norm, QKV, RoPE(+qk-norm)+commit] vs the per-op launches: h, q, the committed K/V rows."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from test_gpu_kernels import _dense_kv

    from paper_2512_15834_b200.modelcfg import SHAPES, TINY
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, OP_NORM, OP_ROPE, BlockOp, KVPool, TiledWeight

    shape = dataclasses.replace(TINY if base == "tiny" else SHAPES[base], layers=1)
    qk = shape.qk_norm
    N, d = shape.q_dim + 2 * shape.kv_dim, shape.d_model
    pos_v = 70
    res = []
    for mode in ("op", "blk"):
        pool = KVPool(shape, 8 * M + 16, M + 1, 16)
        for b in range(M):
            pool.reserve(b, pos_v + 1)
        pool.sync(torch.cuda.current_stream().cuda_stream)
        g = torch.Generator(device="cuda").manual_seed(11 + M)
        x = torch.randn(M, d, device="cuda", generator=g)
        delta = torch.randn(M, d, device="cuda", generator=g)
        wq = (torch.randn(N, d, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
        nw = (torch.rand(d, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
        qn = (torch.rand(shape.d_head, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
        kn = (torch.rand(shape.d_head, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
        tw = TiledWeight(wq)
        h = torch.zeros(M, d, device="cuda", dtype=torch.bfloat16)
        qkv = torch.zeros(M, N, device="cuda")
        q = torch.zeros(M, shape.q_dim, device="cuda", dtype=torch.bfloat16)
        slot = torch.arange(M, device="cuda", dtype=torch.int32)
        pos = torch.full((M,), pos_v, device="cuda", dtype=torch.int32)
        if mode == "op":
            lib.call("stb_add_rmsnorm", P(x), P(delta), P(nw), P(h), M, d, 1e-5, M, st())
            lib.call("stb_gemm_bf16", P(h), d, P(tw), 0, P(qkv), N, M, N, d, 0, 5, st())
            if qk:
                lib.call("stb_qkv_norm_rope_commit", pool.h, 0, P(qkv), P(q), P(slot), P(pos), M, shape.n_q,
                         shape.rope_theta, P(qn), P(kn), 1e-6, M, st())
            else:
                lib.call("stb_qkv_rope_commit", pool.h, 0, P(qkv), P(q), P(slot), P(pos), M, shape.n_q,
                         shape.rope_theta, M, st())
        else:
            ops = (BlockOp * 3)(
                BlockOp(kind=OP_NORM, c=delta.data_ptr(), w=nw.data_ptr(), n=d, x_res=x.data_ptr(), y=h.data_ptr(),
                        eps=1e-5),
                BlockOp(kind=OP_GEMM, x=h.data_ptr(), ldx=d, w=tw.data_ptr(), c=qkv.data_ptr(), ldc=N, n=N, k=d),
                BlockOp(kind=OP_ROPE, c=qkv.data_ptr(), y=q.data_ptr(), pool=pool.h, layer=0, n_q=shape.n_q,
                        slot_of=slot.data_ptr(), pos_of=pos.data_ptr(), rope_theta=shape.rope_theta,
                        q_norm=qn.data_ptr() if qk else None, k_norm=kn.data_ptr() if qk else None, eps=1e-6))
            lib.call("stb_gemm_block", C.cast(ops, C.c_void_p), 3, M, st())
        torch.cuda.synchronize()
        kv = [_dense_kv(pool, 0, b, pos_v + 1, shape) for b in range(M)]
        k_new = torch.stack([k[pos_v] for k, _ in kv])
        v_new = torch.stack([v[pos_v] for _, v in kv])
        res.append((x.clone(), h.clone(), q.clone(), k_new, v_new, qkv.clone(), delta.clone()))
        del pool
    (x1, h1, q1, k1, v1, _, _), (x2, h2, q2, k2, v2, c2, d2) = res
    assert rel(x2, x1) < 1e-6 and rel(h2, h1) < 1e-3
    for name, a, b in (("q", q2, q1), ("k", k2, k1), ("v", v2, v1)):
        assert rel(a, b) < 1e-3, (name, rel(a, b))
    assert not c2.any() and not d2.any()


def _steps(shape, B, prompt, seed):
    from paper_2512_15834_b200.runtime.decoder import StepBatch

    rng = np.random.default_rng(seed)
    i32 = np.int32
    n = B * prompt
    pre = StepBatch(ids=rng.integers(3, shape.vocab, n).astype(i32),
                    pos=np.tile(np.arange(prompt), B).astype(i32), slot_of=np.repeat(np.arange(B), prompt).astype(i32),
                    dec_slots=np.zeros(0, i32), dec_ctx=np.zeros(0, i32), pre_slots=np.arange(B).astype(i32),
                    pre_qstart=(np.arange(B + 1) * prompt).astype(i32), pre_ctx=np.full(B, prompt, i32),
                    sample_rows=(np.arange(B) * prompt + prompt - 1).astype(i32), targets=np.full(B, -1, i32))
    dec = StepBatch(ids=rng.integers(3, shape.vocab, B).astype(i32), pos=np.full(B, prompt, i32),
                    slot_of=np.arange(B).astype(i32), dec_slots=np.arange(B).astype(i32),
                    dec_ctx=np.full(B, prompt + 1, i32), pre_slots=np.zeros(0, i32), pre_qstart=np.zeros(1, i32),
                    pre_ctx=np.zeros(0, i32), sample_rows=np.arange(B).astype(i32), targets=np.full(B, -1, i32))
    return pre, dec


@pytest.mark.parametrize("base", ["llama3-8b", "qwen3-32b"])
@pytest.mark.parametrize("B", [1, 13, 64])
def test_decode_block_step_matches_per_op(lib, base, B):
    from paper_2512_15834_b200.modelcfg import SHAPES
    from paper_2512_15834_b200.runtime import decoder as D
    from paper_2512_15834_b200.runtime import weights as W

    shape = dataclasses.replace(SHAPES[base], name=f"{base}[L=2,V=32k]", layers=2, vocab=32768)
    prompt = 70
    pool = D.KVPool(shape, num_blocks=B * (prompt // 16 + 2) + 16, max_slots=B + 1, max_blocks_per_slot=16)
    for b in range(B):
        pool.reserve(b, prompt + 1)
    w = W.build(shape, seed=5, init_device="cuda")
    dec = D.Decoder(shape, w, pool, use_graphs=False)
    dec.keep_logits = True
    pre, step = _steps(shape, B, prompt, seed=B)
    dec.forward(pre)
    torch.cuda.synchronize()

    def run(block_max):
        saved = D.BLOCK_MAX_T
        D.BLOCK_MAX_T = block_max
        try:
            n0 = lib.load().stb_launch_count()
            dec.forward(step)
            torch.cuda.synchronize()
            return dec.last_logits.clone(), dec.x[:B].clone(), lib.load().stb_launch_count() - n0
        finally:
            D.BLOCK_MAX_T = saved

    lg_b, x_b, n_block = run(64)
    lg_p, x_p, n_op = run(0)
    # embed + first block + (attention + block) per layer + final norm, LM head, sampler
    assert n_block == 2 * shape.layers + 5 and n_op > 4 * shape.layers, (n_block, n_op)
    assert rel(lg_b, lg_p) < 1e-2 and rel(x_b, x_p) < 1e-2, (rel(lg_b, lg_p), rel(x_b, x_p))
    for t in (dec.qkv[:B], dec.proj[:B], dec.gu[:B]):
        assert not t.any()


def test_gemm_block_rejects_bad_chains(lib):
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, OP_SILU, BlockOp

    raw = lib.load()
    s = C.c_void_p(0)
    ops = (BlockOp * 1)(BlockOp(kind=OP_SILU))
    assert raw.stb_gemm_block(C.cast(ops, C.c_void_p), 1, 32, s) < 0  # bad SILU operands / no GEMM
    ops = (BlockOp * 1)(BlockOp(kind=OP_GEMM))
    assert raw.stb_gemm_block(C.cast(ops, C.c_void_p), 1, 65, s) < 0  # M > 64
    assert raw.stb_gemm_block(C.cast(ops, C.c_void_p), 0, 32, s) < 0
    assert raw.stb_gemm_block(C.cast(ops, C.c_void_p), 1, 32, s) < 0  # null operands
    assert b"gemm_block" in raw.stb_last_error()
