import sys, math, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import test_gpu_kernels as K
from paper_2512_15834_b200.runtime import lib
lib.load()
shape = K.SHAPES[0]
for dec, runs in (([700] * 3, []), ([700]*3, [(1, 800)]), ([], [(4, 800)]), ([700]*3, [(33, 2984)])):
    ctxs = dec + [c for _, c in runs]
    pool = K._pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(ctxs), bps=600)
    dense = K._fill_pool(lib, pool, shape, ctxs, seed=11)
    G = shape.n_q // shape.n_kv; qe = 16 // G
    B = len(dec); T = B + sum(n for n, _ in runs)
    q = torch.randn(T, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    e = [(b, dec[b], b, 1) for b in range(B)]
    row = B
    for r, (n, c) in enumerate(runs):
        for j in range(0, n, qe):
            nq = min(qe, n - j); e.append((B + r, c - n + j + nq, row + j, nq))
        row += n
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    E = len(e)
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(E, shape.n_q, shape.n_kv, shape.d_head) // 4), device="cuda")
    meta = [t([x[i] for x in e]) for i in range(4)]
    rc = lib.call("stb_attn_decode_mq", pool.h, 0, K.P(q), K.P(out), *[K.P(a) for a in meta], E, shape.n_q, 1 / math.sqrt(shape.d_head), max(ctxs), K.P(ws), K.stream())
    torch.cuda.synchronize()
    nanrows = torch.isnan(out.float()).any(-1).any(-1).nonzero().flatten().tolist()
    print(dec, runs, "E", E, "rc", rc, "nan rows", nanrows[:20], "of", T)
    bad = torch.isnan(out.float()).any(-1)  # [T, n_q]
    for r in nanrows[:3]:
        print("   row", r, "nan heads", bad[r].nonzero().flatten().tolist())
