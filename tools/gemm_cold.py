"""Cold-launch cost of decode-shaped GEMMs, timed the way bench.py's roofline timer sees them:
each launch bracketed by its own CUDA event pair inside a captured graph (the event nodes
break the programmatic-dependent-launch overlap with the previous kernel), against the same
launches back to back under PDL, and against an empty event pair.

    python tools/gemm_cold.py [--shape llama3-8b] [--M 32]

Per shape prints: PDL-chained us/launch, event-bracketed us/launch (minus the empty pair),
and the bracketed time of a K = 64 launch of the same N (the fixed per-launch cost)."""
import argparse
import ctypes as C
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2512_15834_b200.modelcfg import SHAPES  # noqa: E402
from paper_2512_15834_b200.runtime import lib  # noqa: E402
from paper_2512_15834_b200.runtime.decoder import TiledWeight  # noqa: E402


def P(t):
    return C.c_void_p(t.data_ptr())


def run(fns, iters, bracket):
    """Capture iters rounds of fns (optionally each call inside an event pair); returns
    (us per call from the bracket pairs, us per call from the whole replay)."""
    s = torch.cuda.current_stream()
    for f in fns:
        f()
    torch.cuda.synchronize()
    pairs = []
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            for f in fns:
                if bracket:
                    a = torch.cuda.Event(enable_timing=True, external=True)
                    b = torch.cuda.Event(enable_timing=True, external=True)
                    a.record()
                    f()
                    b.record()
                    pairs.append((a, b))
                else:
                    f()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    n = iters * len(fns)
    whole = e0.elapsed_time(e1) * 1e3 / n
    br = sum(a.elapsed_time(b) for a, b in pairs) * 1e3 / n if bracket else float("nan")
    return br, whole


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama3-8b")
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--extra", action="store_true")
    ap.add_argument("--blockcmp", action="store_true")
    ap.add_argument("--body", action="store_true")
    ap.add_argument("--chains", action="store_true")
    a = ap.parse_args()
    s = SHAPES[a.shape]
    M = a.M
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    x_norm = torch.randn(M, s.d_model, device="cuda")
    nw = torch.ones(s.d_model, device="cuda", dtype=torch.bfloat16)
    h = torch.empty(M, s.d_model, device="cuda", dtype=torch.bfloat16)
    norm = lambda: lib.call("stb_add_rmsnorm", P(x_norm), None, P(nw), P(h), M, s.d_model, 1e-5, 0, st())  # noqa

    empty_br, _ = run([lambda: None], a.iters, True)
    norm_br, norm_whole = run([norm], a.iters, True)
    print(f"empty event pair {empty_br:.2f} us; add_rmsnorm bracketed {norm_br - empty_br:.2f} us "
          f"(chained {norm_whole:.2f})")
    gemms = {"qkv": (s.q_dim + 2 * s.kv_dim, s.d_model), "o": (s.d_model, s.q_dim),
             "gate_up": (2 * s.d_ff, s.d_model), "down": (s.d_model, s.d_ff)}
    for name, (N, K) in gemms.items():
        copies = max(2, int(math.ceil(400e6 / (N * K * 2))))
        ws = [TiledWeight(torch.randn(N, K, device="cuda", dtype=torch.bfloat16)) for _ in range(copies)]
        xa = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        c = torch.zeros(M, N, device="cuda")
        flags = 4 | (1 if lib.load().stb_gemm_is_stream(M, N, K) else 0)
        cnt = [0]

        def gemm(kk=K, fl=flags):
            w = ws[cnt[0] % copies]
            cnt[0] += 1
            lib.call("stb_gemm_bf16", P(xa), K, P(w), 0, P(c), N, M, N, kk, 0, fl, st())

        wbytes = N * K * 2
        # norm -> gemm pairs as in the decoder (norm rows are the GEMM's predecessor)
        _, chained = run([norm, gemm], a.iters, False)
        br, _ = run([norm, gemm], a.iters, True)
        gem_br = 2 * br - (norm_br)  # bracket average covers norm + gemm alternately
        gem_br -= empty_br
        gem_chain = 2 * chained - norm_whole
        br_k64, _ = run([lambda: gemm(64)], a.iters, True)
        br_k64 -= empty_br
        br_nz, _ = run([lambda: gemm(K, flags & ~1)], a.iters, True)
        br_nz -= empty_br
        print(f"{name:8s} N={N:6d} K={K:6d}: chained {gem_chain:6.2f} us ({wbytes / gem_chain / 1e3:6.0f} GB/s) | "
              f"bracketed {gem_br:6.2f} us ({wbytes / gem_br / 1e3:6.0f} GB/s) | in-kernel zero+barrier "
              f"{br_nz:6.2f} us | K=64 bracketed {br_k64:6.2f} us")
        del ws


if __name__ == "__main__" and not {"--extra", "--body", "--blockcmp", "--chains"} & set(sys.argv):
    main()


def trace_phases(label, launch):
    """One eager launch with the in-kernel globaltimer trace on: CTA entry spread and phase
    medians from the first CTA entry (us; %globaltimer granularity applies)."""
    import numpy as np

    fn = lib.load().stb_debug_gemm_trace
    fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
    buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    fn(C.c_void_p(buf.data_ptr()), 4096)
    launch()
    torch.cuda.synchronize()
    n = fn(None, 0)
    r = buf[:n * 8].view(n, 8).cpu().numpy().astype(np.int64)
    e0 = r[:, 3].min()
    cols = (("entry", 3), ("prefilled", 2), ("dep-wait", 4), ("first-stage", 5), ("last-mma", 6), ("last-epi", 1), ("exit", 7))
    parts = []
    for name, col in cols:
        v = (r[:, col] - e0) / 1e3
        v = v[r[:, col] > 0]
        if len(v):
            parts.append(f"{name} {np.median(v):5.1f}/{v.max():5.1f}")
    print(f"  trace {label} ({n} CTAs, p50/max us): " + "  ".join(parts))


def extra():
    torch.cuda.init()
    tiny = torch.zeros(1, device="cuda")
    e, _ = run([lambda: None], 20, True)
    k, _ = run([lambda: tiny.add_(1.0)], 20, True)
    print(f"empty pair {e:.2f} us; 1-thread torch kernel bracketed {k - e:.2f} us above it")
    s = SHAPES["llama3-8b"]
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    for N, K in ((s.d_model, s.q_dim), (2 * s.d_ff, s.d_model)):
        w = TiledWeight(torch.randn(N, K, device="cuda", dtype=torch.bfloat16))
        xa = torch.randn(32, K, device="cuda", dtype=torch.bfloat16)
        c = torch.zeros(32, N, device="cuda")
        for kk in (64, K):
            trace_phases(f"N={N} K={kk}", lambda: lib.call("stb_gemm_bf16", P(xa), K, P(w), 0, P(c), N, 32, N, kk, 0,
                                                           5, st()))


if __name__ == "__main__" and "--extra" in sys.argv:
    extra()


def bracket_vs_body():
    """Event-bracketed launches in a graph with the in-kernel trace on: per launch, the bracket
    (minus the empty pair) against the kernel body (first CTA entry -> last CTA exit)."""
    import numpy as np

    s = SHAPES["llama3-8b"]
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    e, _ = run([lambda: None], 20, True)
    fn = lib.load().stb_debug_gemm_trace
    fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
    for N, K in ((s.d_model, s.q_dim), (2 * s.d_ff, s.d_model)):
        for copies in (1, 8):
            ws = [TiledWeight(torch.randn(N, K, device="cuda", dtype=torch.bfloat16)) for _ in range(copies)]
            xa = torch.randn(32, K, device="cuda", dtype=torch.bfloat16)
            c = torch.zeros(32, N, device="cuda")
            it = [0]

            def g():
                w = ws[it[0] % copies]
                it[0] += 1
                lib.call("stb_gemm_bf16", P(xa), K, P(w), 0, P(c), N, 32, N, K, 0, 5, st())

            buf = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            fn(C.c_void_p(buf.data_ptr()), (1 << 20) // 8)
            br, _ = run([g], 8, True)  # warm call + 2 replays are traced
            torch.cuda.synchronize()
            n = fn(None, 0)
            r = buf[:n * 8].view(n, 8).cpu().numpy().astype(np.int64)
            bodies = []
            for tag in np.unique(r[:, 0]):
                q = r[r[:, 0] == tag]
                # several replays share a tag: split by entry-time clusters (> 50 us apart)
                q = q[np.argsort(q[:, 3])]
                cuts = np.where(np.diff(q[:, 3]) > 50_000)[0] + 1
                for part in np.split(q, cuts):
                    bodies.append((part[:, 7].max() - part[:, 3].min()) / 1e3)
            print(f"  N={N} K={K} copies={copies}: bracketed {br - e:6.2f} us, body median {np.median(bodies):6.2f} us "
                  f"(n={len(bodies)}), outside {br - e - np.median(bodies):5.2f} us")
            fn(None, 0)
            del ws


if __name__ == "__main__" and "--body" in sys.argv:
    bracket_vs_body()


def block_vs_standalone():
    """Same decode-shaped GEMM as stb_gemm_bf16 and as a one-phase stb_gemm_block, both chained
    in a graph (PDL between launches), weights cycled past L2: us per launch."""
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, BlockOp

    s = SHAPES["llama3-8b"]
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    for N, K in ((s.q_dim + 2 * s.kv_dim, s.d_model), (s.d_model, s.q_dim), (2 * s.d_ff, s.d_model), (s.d_model, s.d_ff)):
        copies = max(2, int(math.ceil(400e6 / (N * K * 2))))
        ws = [TiledWeight(torch.randn(N, K, device="cuda", dtype=torch.bfloat16)) for _ in range(copies)]
        xa = torch.randn(32, K, device="cuda", dtype=torch.bfloat16)
        c = torch.zeros(32, N, device="cuda")
        ops = [(BlockOp * 1)(BlockOp(kind=OP_GEMM, x=xa.data_ptr(), ldx=K, w=w.data_ptr(), c=c.data_ptr(), ldc=N, n=N,
                                     k=K)) for w in ws]
        it = [0, 0]

        def g1():
            lib.call("stb_gemm_bf16", P(xa), K, P(ws[it[0] % copies]), 0, P(c), N, 32, N, K, 0, 5, st())
            it[0] += 1

        def g2():
            lib.call("stb_gemm_block", C.cast(ops[it[1] % copies], C.c_void_p), 1, 32, st())
            it[1] += 1

        _, t1 = run([g1], 40, False)
        _, t2 = run([g2], 40, False)
        print(f"  N={N:6d} K={K:6d}: standalone {t1:6.2f} us  block(1 GEMM) {t2:6.2f} us  ({N * K * 2 / t2 / 1e3:.0f} GB/s)")
        del ws


if __name__ == "__main__" and "--blockcmp" in sys.argv:
    block_vs_standalone()


def block_chains():
    """Chain-composition costs of stb_gemm_block at M = 32 (llama3-8b widths): us per launch
    of [O], [GU], [O, GU] (independent inputs), [O, NORM, GU], [GU, SILU, DOWN], chained in a
    graph with weights cycled past L2."""
    from paper_2512_15834_b200.runtime.decoder import OP_GEMM, OP_NORM, OP_SILU, BlockOp

    s = SHAPES["llama3-8b"]
    d, F, M = s.d_model, s.d_ff, 32
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    copies = 3
    wo = [TiledWeight(torch.randn(d, d, device="cuda", dtype=torch.bfloat16) * 0.02) for _ in range(copies)]
    wgu = [TiledWeight(torch.randn(2 * F, d, device="cuda", dtype=torch.bfloat16) * 0.02) for _ in range(copies)]
    wd = [TiledWeight(torch.randn(d, F, device="cuda", dtype=torch.bfloat16) * 0.02) for _ in range(copies)]
    xa = torch.randn(M, d, device="cuda", dtype=torch.bfloat16)
    h = torch.randn(M, d, device="cuda", dtype=torch.bfloat16)
    act = torch.randn(M, F, device="cuda", dtype=torch.bfloat16)
    x = torch.randn(M, d, device="cuda")
    proj, gu, out = torch.zeros(M, d, device="cuda"), torch.zeros(M, 2 * F, device="cuda"), torch.zeros(M, d, device="cuda")
    nw = torch.ones(d, device="cuda", dtype=torch.bfloat16)
    G = lambda a, w, c, n, k: BlockOp(kind=OP_GEMM, x=a.data_ptr(), ldx=k, w=w.data_ptr(), c=c.data_ptr(), ldc=n, n=n, k=k)  # noqa
    chains = {
        "O": lambda i: [G(xa, wo[i], proj, d, d)],
        "GU": lambda i: [G(h, wgu[i], gu, 2 * F, d)],
        "O+GU (indep)": lambda i: [G(xa, wo[i], proj, d, d), G(h, wgu[i], gu, 2 * F, d)],
        "O,NORM,GU": lambda i: [G(xa, wo[i], proj, d, d),
                                BlockOp(kind=OP_NORM, c=proj.data_ptr(), w=nw.data_ptr(), n=d, x_res=x.data_ptr(),
                                        y=h.data_ptr(), eps=1e-5), G(h, wgu[i], gu, 2 * F, d)],
        "GU,SILU,DOWN": lambda i: [G(h, wgu[i], gu, 2 * F, d), BlockOp(kind=OP_SILU, c=gu.data_ptr(), y=act.data_ptr(), n=F),
                                   G(act, wd[i], out, d, F)],
    }
    for name, mk in chains.items():
        arrs = [(BlockOp * len(mk(i)))(*mk(i)) for i in range(copies)]
        it = [0]

        def f():
            a = arrs[it[0] % copies]
            lib.call("stb_gemm_block", C.cast(a, C.c_void_p), len(a), M, st())
            it[0] += 1

        _, t = run([f], 30, False)
        print(f"  chain {name:14s}: {t:7.2f} us per launch")


if __name__ == "__main__" and "--chains" in sys.argv:
    block_chains()
