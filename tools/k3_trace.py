"""Per-warp timeline of one K3 launch (variant built with -DSTB_K3_TRACE): entry, partition
done, first page landed, last chunk done, exit — us from the first warp's entry."""
import ctypes as C, math, sys, torch
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import test_gpu_kernels as K
from paper_2512_15834_b200.runtime import lib
from paper_2512_15834_b200.modelcfg import ModelShape
lib.load()
shape = ModelShape("llama-ish", 1, 4096, 32, 8, 128, 64, 64)
fn = lib.load().stb_debug_k3_trace
fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
for B, c in ((32, 128), (32, 2048), (32, 4096)):
    ctxs = [c] * B
    pool = K._pool(lib, shape, nb=sum(-(-x // 16) for x in ctxs) + 8, slots=B, bps=300)
    K._fill_pool(lib, pool, shape, ctxs, seed=3)
    q = torch.randn(B, 32, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ctx = torch.full((B,), c, dtype=torch.int32, device="cuda")
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B, 32, 8, 128) // 4), device="cuda")
    call = lambda: lib.call("stb_attn_decode", pool.h, 0, K.P(q), K.P(out), K.P(slots), K.P(ctx), B, 32, 1 / math.sqrt(128), c, K.P(ws), K.stream())
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    buf = torch.zeros(8192 * 8, dtype=torch.int64, device="cuda")
    fn(C.c_void_p(buf.data_ptr()), 8192)
    call()
    torch.cuda.synchronize()
    n = fn(None, 0)
    r = buf[:n * 8].view(n, 8).cpu().numpy().astype(np.int64)
    e0 = r[:, 0].min()
    def st(col, name):
        v = r[:, col]
        v = (v[v > 0] - e0) / 1e3
        return f"{name} p10 {np.percentile(v, 10):5.1f} p50 {np.median(v):5.1f} p90 {np.percentile(v, 90):5.1f} max {v.max():5.1f}"
    if len(sys.argv) > 1:
        np.save(f"{sys.argv[1]}_B{B}_c{c}.npy", r)
    print(f"B={B} ctx={c}: {n} warps | " + " | ".join(st(i, nm) for i, nm in ((0, "entry"), (6, "metadata"), (1, "partition"), (2, "first page"), (3, "last chunk"), (5, "exit"))))
