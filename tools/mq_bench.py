"""K3 with a verify run folded in (stb_attn_decode_mq) vs K3 alone + a separate K2 verify launch,
C2 shapes: B decode rows at ctx c plus one run of n queries at ctx c (CUDA-graph timed)."""
import math, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/tools")
import test_gpu_kernels as K
from bench_kernels import time_it
from paper_2512_15834_b200.runtime import lib
from paper_2512_15834_b200.modelcfg import ModelShape
lib.load()
shape = ModelShape("llama-ish", 1, 4096, 32, 8, 128, 64, 64)
for B, c, n in ((31, 3000, 33), (31, 3000, 16), (31, 2000, 33), (0, 3000, 33)):
    ctxs = [c] * (B + 1)
    pool = K._pool(lib, shape, nb=sum(-(-x // 16) for x in ctxs) + 8, slots=len(ctxs), bps=400)
    K._fill_pool(lib, pool, shape, ctxs, seed=3)
    G = 4; qe = 4
    T = B + n
    q = torch.randn(T, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    e = [(b, c, b, 1) for b in range(B)] + [(B, c - n + j + min(qe, n - j), B + j, min(qe, n - j)) for j in range(0, n, qe)]
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    meta = [t([x[i] for x in e]) for i in range(4)]
    E = len(e)
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(E + 64, 32, 8, 128) // 4), device="cuda")
    sc = 1 / math.sqrt(128)
    st = K.stream
    mq = lambda i: lib.call("stb_attn_decode_mq", pool.h, 0, K.P(q), K.P(out), *[K.P(a) for a in meta], E, 32, sc, c, K.P(ws), st())
    dslots, dctx = t(list(range(B))), t([c] * B)
    dec = lambda i: lib.call("stb_attn_decode", pool.h, 0, K.P(q), K.P(out), K.P(dslots), K.P(dctx), B, 32, sc, c, K.P(ws), st()) if B else None
    pslot, pq, pctx = t([B]), t([0, n]), t([c])
    q2, o2 = q[B:], out[B:]
    ver = lambda i: lib.call("stb_attn_prefill_split", pool.h, 0, K.P(q2), K.P(o2), K.P(pslot), K.P(pq), K.P(pctx), 1, n, 32, sc, n, 8, st())
    t_mq = time_it(mq)
    t_dec = time_it(dec) if B else 0.0
    t_ver = time_it(ver)
    t_both = time_it(lambda i: (dec(i), ver(i)))
    print(f"B={B} ctx={c} run n={n}: mq {t_mq:.1f} us | K3 alone {t_dec:.1f} + K2 verify {t_ver:.1f} (chained {t_both:.1f}) us")
