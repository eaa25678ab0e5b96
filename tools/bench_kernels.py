"""Kernel microbenchmarks (CUDA events, cold operands cycled past L2).

GEMM: the decode- and prefill-shaped projections of a model shape.
Decode attention: B sequences at a context length, K3 alone.
Prints achieved GB/s (HBM-bound) or TFLOP/s against MEASURED_PEAKS.json.
"""

import argparse
import ctypes as C
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2512_15834_b200.modelcfg import SHAPES  # noqa: E402
from paper_2512_15834_b200.runtime import lib  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {
    "hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def P(t):
    return C.c_void_p(t.data_ptr())


def st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def time_it(fn, iters=40, warm=3):
    """Device time per call: the loop is captured in a CUDA graph (no host launch cost)."""
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def bench_gemm(shape, M, split=0, layout="tiled"):
    s = shape
    gemms = {"qkv": (s.q_dim + 2 * s.kv_dim, s.d_model), "o": (s.d_model, s.q_dim),
             "gate_up": (2 * s.d_ff, s.d_model), "down": (s.d_model, s.d_ff), "lm_head": (s.vocab, s.d_model)}
    out = {}
    for name, (N, K) in gemms.items():
        copies = max(2, int(math.ceil(400e6 / (N * K * 2))))
        ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        c = torch.empty(M, N, device="cuda")
        flags = 1 if lib.load().stb_gemm_is_stream(M, N, K) else 0  # as the decoder runs it
        byts = N * K * 2 + M * K * 2 + M * N * 4
        fl = 2 * M * N * K
        if layout in ("rowmajor", "both"):
            us = time_it(lambda i: lib.call("stb_gemm_bf16", P(a), K, P(ws[i % copies]), K, P(c), N, M, N, K, split,
                                            flags, st()))
            out[name] = (us, byts / us / 1e3, fl / us / 1e6)
            print(f"  M={M:5d} {name:8s} N={N:6d} K={K:5d}: {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s "
                  f"({byts / us / 1e3 / PEAK['hbm_gbs']:.2f})  {fl / us / 1e6:7.1f} TF/s "
                  f"({fl / us / 1e6 / PEAK['bf16_tflops']:.2f})  row-major W")
        if layout in ("tiled", "both"):
            from paper_2512_15834_b200.runtime.decoder import TiledWeight

            tw = [TiledWeight(w) for w in ws]
            us = time_it(lambda i: lib.call("stb_gemm_bf16", P(a), K, P(tw[i % copies]), 0, P(c), N, M, N, K, split,
                                            flags | 4, st()))
            out[name] = (us, byts / us / 1e3, fl / us / 1e6)
            print(f"  M={M:5d} {name:8s} N={N:6d} K={K:5d}: {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s "
                  f"({byts / us / 1e3 / PEAK['hbm_gbs']:.2f})  {fl / us / 1e6:7.1f} TF/s "
                  f"({fl / us / 1e6 / PEAK['bf16_tflops']:.2f})  tiled W")
            del tw
        del ws
    tot = sum(v[0] for v in out.values())
    print(f"  M={M}: sum {tot:.1f} us")
    return out


def bench_fused(shape, M):
    """Decode/prefill projections with their fused epilogues (stb_gemm_bf16_fused) vs the plain
    GEMM on the same tiled weights."""
    from paper_2512_15834_b200.runtime.decoder import GemmEpi, KVPool, TiledWeight

    s = shape
    d, F = s.d_model, s.d_ff
    pool = KVPool(s.with_layers(1), M // 16 + 64, 4, M // 16 + 8)
    pool.reserve(0, M + 16)
    pool.sync(torch.cuda.current_stream().cuda_stream)
    slot_of = torch.zeros(M, dtype=torch.int32, device="cuda")
    pos = torch.arange(M, dtype=torch.int32, device="cuda")
    parts = d // 128
    ss = torch.rand(M, parts, device="cuda") * 128
    sso = torch.empty(M, parts, device="cuda")
    x = torch.randn(M, d, device="cuda")
    xb = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    q = torch.empty(M, s.q_dim, device="cuda", dtype=torch.bfloat16)
    act = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    cases = {
        "qkv": (s.q_dim + 2 * s.kv_dim, d, GemmEpi(kind=2, ss_in=ss.data_ptr(), ss_parts=parts, inv_dim=1.0 / d,
                                                   eps=1e-5,
                                                   out=q.data_ptr(), ldo=s.q_dim, pool=pool.h.value, layer=0,
                                                   n_q=s.n_q, slot_of=slot_of.data_ptr(), pos_of=pos.data_ptr(),
                                                   rope_theta=s.rope_theta)),
        "o": (d, s.q_dim, GemmEpi(kind=3, out=xb.data_ptr(), ldo=d, x=x.data_ptr(), ldx=d, ss_out=sso.data_ptr(),
                                  ss_parts=parts)),
        "gate_up": (2 * F, d, GemmEpi(kind=1, ss_in=ss.data_ptr(), ss_parts=parts, inv_dim=1.0 / d, eps=1e-5,
                                      out=act.data_ptr(), ldo=F)),
        "down": (d, F, GemmEpi(kind=3, out=xb.data_ptr(), ldo=d, x=x.data_ptr(), ldx=d, ss_out=sso.data_ptr(),
                               ss_parts=parts)),
    }
    fn = lib.load().stb_gemm_bf16_fused
    tot = [0.0, 0.0]
    for name, (N, K, e) in cases.items():
        copies = max(2, int(math.ceil(400e6 / (N * K * 2))))
        # the model's value ranges (weights N(0, 0.02)): silu/rsqrt stay on their fast paths
        tw = [TiledWeight((0.02 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)) for _ in range(copies)]
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        work = torch.zeros(M, N, device="cuda")
        us_f = time_it(lambda i: fn(P(a), K, P(tw[i % copies]), 0, P(work), N, M, N, K, 4, C.byref(e), st()))
        flags = 1 if lib.load().stb_gemm_is_stream(M, N, K) else 0
        us_p = time_it(lambda i: lib.call("stb_gemm_bf16", P(a), K, P(tw[i % copies]), 0, P(work), N, M, N, K, 0,
                                          flags | 4, st()))
        work.zero_()
        tot[0] += us_f
        tot[1] += us_p
        print(f"  M={M:5d} {name:8s} N={N:6d} K={K:5d}: fused {us_f:8.1f} us   plain {us_p:8.1f} us")
        del tw
    print(f"  M={M}: fused sum {tot[0]:.1f} us, plain sum {tot[1]:.1f} us")


def bench_attn(shape, B, ctx, reps=4):
    from paper_2512_15834_b200.runtime.decoder import KVPool

    s = shape
    pages = B * (ctx // 16 + 1)
    pools = []
    for r in range(reps):  # several pools cycled so K/V are cold in L2
        pool = KVPool(s.with_layers(1), pages + 16, B, ctx // 16 + 2)
        for b in range(B):
            pool.reserve(b, ctx)
        pool.sync(torch.cuda.current_stream().cuda_stream)
        pools.append(pool)
    q = torch.randn(B, s.n_q, s.d_head, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(q)
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ctxs = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B, s.n_q, s.n_kv, s.d_head) // 4), device="cuda")
    sc = 1 / math.sqrt(s.d_head)
    us = time_it(lambda i: lib.call("stb_attn_decode", pools[i % reps].h, 0, P(q), P(o), P(slots), P(ctxs), B, s.n_q,
                                    sc, 0, P(ws), st()))
    byts = B * ctx * 2 * s.kv_dim * 2 + 2 * B * s.q_dim * 2
    print(f"  attn_decode B={B:3d} ctx={ctx:6d}: {us:8.1f} us  {byts / us / 1e3:7.0f} GB/s "
          f"({byts / us / 1e3 / PEAK['hbm_gbs']:.2f})")
    return us


def bench_prefill(shape, S, n, ctx, reps=2):
    """K2 append-prefill: S runs of n new queries at context ctx (incl. the new rows)."""
    from paper_2512_15834_b200.runtime.decoder import KVPool

    s = shape
    pools = []
    for r in range(reps):
        pool = KVPool(s.with_layers(1), S * (ctx // 16 + 1) + 16, S, ctx // 16 + 2)
        for b in range(S):
            pool.reserve(b, ctx)
        pool.sync(torch.cuda.current_stream().cuda_stream)
        pools.append(pool)
    T = S * n
    q = torch.randn(T, s.n_q, s.d_head, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(q)
    slots = torch.arange(S, dtype=torch.int32, device="cuda")
    qs = torch.arange(0, T + 1, n, dtype=torch.int32, device="cuda")
    ctxs = torch.full((S,), ctx, dtype=torch.int32, device="cuda")
    sc = 1 / math.sqrt(s.d_head)
    us = time_it(lambda i: lib.call("stb_attn_prefill", pools[i % reps].h, 0, P(q), P(o), P(slots), P(qs), P(ctxs), S,
                                    T, s.n_q, sc, n, st()), iters=10)
    prev = ctx - n
    fl = S * 4 * s.n_q * s.d_head * (n * prev + n * (n + 1) / 2)
    print(f"  attn_prefill S={S:3d} n={n:5d} ctx={ctx:6d}: {us:9.1f} us  {fl / us / 1e6:7.1f} TF/s "
          f"({fl / us / 1e6 / PEAK['bf16_tflops']:.2f})")


def bench_pdl(shape, M=32):
    """rmsnorm -> QKV GEMM pairs in one graph: is the GEMM's weight prefetch overlapping?"""
    s = shape
    N, K = s.q_dim + 2 * s.kv_dim, s.d_model
    copies = 8
    ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
    x = torch.randn(M, K, device="cuda")
    h = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    nw = torch.ones(K, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda")

    def norm(i):
        lib.call("stb_add_rmsnorm", P(x), None, P(nw), P(h), M, K, 1e-5, 0, st())

    def gemm(i):
        lib.call("stb_gemm_bf16", P(h), K, P(ws[i % copies]), K, P(c), N, M, N, K, 0, 0, st())

    t_norm = time_it(norm)
    t_gemm = time_it(gemm)
    t_pair = time_it(lambda i: (norm(i), gemm(i)))
    print(f"  pdl probe M={M}: rmsnorm {t_norm:.1f} us, qkv gemm {t_gemm:.1f} us, pair {t_pair:.1f} us "
          f"(overlap {t_norm + t_gemm - t_pair:.1f} us)")


def bench_gemm_sweep(M=32, N=148 * 128):
    """Fixed cost of a decode-shaped GEMM: time vs weight bytes at one tile per SM."""
    for K in (64, 256, 1024, 4096, 8192):
        copies = max(2, int(math.ceil(400e6 / (N * K * 2))))
        ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(copies)]
        a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        c = torch.empty(M, N, device="cuda")
        for split, flags in ((0, 0), (0, 1), (1, 0)):  # flags=1: caller-zeroed C (no memset/barrier)
            us = time_it(lambda i: lib.call("stb_gemm_bf16", P(a), K, P(ws[i % copies]), K, P(c), N, M, N, K, split,
                                            flags, st()))
            print(f"  sweep M={M} N={N} K={K:5d} split={split} flags={flags}: {us:7.2f} us  "
                  f"{N * K * 2 / us / 1e3:7.0f} GB/s")
        del ws


def bench_small(shape):
    """Row ops of a decode step at B=32: add+RMSNorm, SiLU-gate, forced sampler (HBM-bound)."""
    B, d, f, V = 32, shape.d_model, shape.d_ff, shape.vocab
    x = torch.randn(B, d, device="cuda")
    delta = torch.randn(B, d, device="cuda")
    nw = torch.ones(d, device="cuda", dtype=torch.bfloat16)
    h = torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
    us = time_it(lambda i: lib.call("stb_add_rmsnorm", P(x), P(delta), P(nw), P(h), B, d, 1e-5, 0, st()))
    print(f"  add_rmsnorm B={B} d={d}: {us:6.2f} us  {B * d * 14 / us / 1e3:6.0f} GB/s")
    gu = torch.randn(B, 2 * f, device="cuda")
    a = torch.empty(B, f, device="cuda", dtype=torch.bfloat16)
    us = time_it(lambda i: lib.call("stb_silu_mul", P(gu), P(a), B, f, 0, st()))
    print(f"  silu_mul B={B} f={f}: {us:6.2f} us  {B * f * 10 / us / 1e3:6.0f} GB/s")
    logits = torch.randn(B, V, device="cuda")
    tgt = torch.randint(0, V, (B,), device="cuda", dtype=torch.int32)
    o = torch.empty(B, device="cuda", dtype=torch.int32)
    ra = torch.empty(B, device="cuda", dtype=torch.int32)
    rm = torch.empty(B, device="cuda")
    for clear in (0, 1):
        us = time_it(lambda i: lib.call("stb_sample_forced", P(logits), V, P(tgt), B, V, 1e4, P(o), P(ra), P(rm),
                                        clear, st()))
        print(f"  sample_forced R={B} V={V} clear={clear}: {us:6.2f} us  "
              f"{B * V * 4 * (1 + clear) / us / 1e3:6.0f} GB/s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama3-8b")
    ap.add_argument("--what", default="gemm,attn,prefill")
    ap.add_argument("--M", default="32,2080")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--layout", default="tiled", choices=["tiled", "rowmajor", "both"])
    ap.add_argument("--attn-cases", default="32x2048,32x4096,16x32768,1x4096,64x4096", help="BxCTX list")
    ap.add_argument("--prefill-cases", default="4x2048x2048,1x2048x34816,8x512x4096,32x33x4096",
                    help="SxNxCTX list for --what prefill")
    args = ap.parse_args()
    lib.load()
    shape = SHAPES[args.shape]
    if "gemm" in args.what:
        for M in [int(x) for x in args.M.split(",")]:
            bench_gemm(shape, M, args.split, args.layout)
    if "fused" in args.what:
        for M in [int(x) for x in args.M.split(",")]:
            bench_fused(shape, M)
    if "sweep" in args.what:
        bench_gemm_sweep()
    if "pdl" in args.what:
        bench_pdl(shape)
    if "prefill" in args.what:
        for case in args.prefill_cases.split(","):
            S, n, ctx = (int(x) for x in case.split("x"))
            bench_prefill(shape, S, n, ctx)
    if "small" in args.what:
        bench_small(shape)
    if "attn" in args.what:
        for case in args.attn_cases.split(","):
            B, ctx = (int(x) for x in case.split("x"))
            bench_attn(shape, B, ctx)


if __name__ == "__main__":
    main()
