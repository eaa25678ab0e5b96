"""Microbenchmark of the MXFP4 grouped GEMM (moe.cu) at gpt-oss-120b expert shapes: routes T
tokens over 128 experts (top-4), then times gate-up and down launches with CUDA events on the
launching stream; reports algorithmic HBM bytes (touched experts' tiles + token rows in/out) per
second vs the measured HBM peak. Usage: python tools/bench_moe.py [--T 32,128,512,2048]"""

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2512_15834_b200.runtime import lib as L  # noqa: E402
from paper_2512_15834_b200.runtime import weights as W  # noqa: E402


def P(t):
    return C.c_void_p(t.data_ptr())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="1,8,32,128,512,2048")
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--d", type=int, default=2880)
    ap.add_argument("--ff", type=int, default=2880)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--impl", default="mx,mxfp4", help="mx = block-scaled tcgen05 path (stb_moe_gemm_mx, the "
                    "default), mxfp4 = the dequantising kernel (stb_moe_gemm_mxfp4)")
    a = ap.parse_args()
    L.load()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    E, d, ff, k = a.E, a.d, a.ff, a.k
    # random codes (any byte is a valid pair of e2m1 codes); scale bytes in range
    def tiles(N, K):
        t = torch.randint(0, 256, (E, -(-N // 128), K // 64, W.TILE_BYTES), dtype=torch.uint8, device="cuda")
        t[..., 4096:] = 120
        return t
    def stages(N, K):  # MX stage format (stb_moe_gemm_mx)
        t = torch.randint(0, 256, (E, -(-N // 128), -(-K // 128), W.MX_STAGE_BYTES), dtype=torch.uint8, device="cuda")
        t[..., 8192:] = 120
        return t
    impls = a.impl.split(",")
    gu, dn = (tiles(2 * ff, d), tiles(d, ff)) if "mxfp4" in impls else (None, None)
    gum, dnm = (stages(2 * ff, d), stages(d, ff)) if "mx" in impls else (None, None)
    bgu, bdn = torch.zeros(E, 2 * ff, device="cuda"), torch.zeros(E, d, device="cuda")
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    for T in [int(x) for x in a.T.split(",")]:
        logits = torch.randn(T, E, device="cuda")
        counts = torch.zeros(E, dtype=torch.int32, device="cuda")
        ex = torch.empty(T * k, dtype=torch.int32, device="cuda")
        rk, wt = torch.empty_like(ex), torch.empty(T * k, device="cuda")
        L.call("stb_moe_route", P(logits), E, None, T, E, k, P(counts), P(ex), P(rk), P(wt), st)
        h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
        cap = T * k + 64
        offs = torch.empty(E + 1, dtype=torch.int32, device="cuda")
        perm = torch.empty(T * k, dtype=torch.int32, device="cuda")
        xp = torch.zeros(cap, d, dtype=torch.float16, device="cuda")
        act = torch.zeros(cap, ff, dtype=torch.float16, device="cuda")
        y = torch.zeros(cap, d, device="cuda")
        L.call("stb_moe_gather", P(h), d, T, d, k, E, P(counts), P(ex), P(rk), P(offs), P(perm), P(xp), st)
        touched = int((counts > 0).sum())
        rows = T * k
        kq = max(d, ff)
        xq = [torch.zeros(L.load().stb_moe_quant_bytes(cap, kq), dtype=torch.uint8, device="cuda") for _ in range(2)]
        xsf = [torch.zeros(L.load().stb_moe_quant_scale_words(cap, kq), dtype=torch.int32, device="cuda")
               for _ in range(2)]
        L.call("stb_moe_quant", P(xp), d, rows, d, cap, P(xq[0]), P(xsf[0]), st)
        L.call("stb_moe_quant", P(act), ff, rows, ff, cap, P(xq[1]), P(xsf[1]), st)
        impl = "mxfp4"

        def run(kind):
            if impl == "quant":
                L.call("stb_moe_quant", P(xp), d, rows, d, cap, P(xq[0]), P(xsf[0]), st)
            elif impl == "mx" and kind == 1:
                L.call("stb_moe_gemm_mx", P(xq[0]), P(xsf[0]), cap, P(gum), P(bgu), P(counts), E, 2 * ff, d, 1, 7.0,
                       P(act), ff, rows, st)
            elif impl == "mx":
                L.call("stb_moe_gemm_mx", P(xq[1]), P(xsf[1]), cap, P(dnm), P(bdn), P(counts), E, d, ff, 2, 0.0, P(y),
                       d, rows, st)
            elif kind == 1:
                L.call("stb_moe_gemm_mxfp4", P(xp), cap, P(gu), P(bgu), P(counts), E, 2 * ff, d, 1, 7.0, P(act), ff,
                       rows, st)
            else:
                L.call("stb_moe_gemm_mxfp4", P(act), cap, P(dn), P(bdn), P(counts), E, d, ff, 2, 0.0, P(y), d, rows, st)

        for impl in a.impl.split(",") + (["quant"] if "mx" in a.impl.split(",") else []):
          res = {}
          for kind, N, K, ob in ((1, 2 * ff, d, ff * 2), (2, d, ff, d * 4)) if impl != "quant" else ((1, 0, d, 0),):
              for _ in range(3):
                  run(kind)
              torch.cuda.synchronize()
              e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
              e0.record()
              for _ in range(a.iters):
                  run(kind)
              e1.record()
              torch.cuda.synchronize()
              us = e0.elapsed_time(e1) / a.iters * 1e3
              byts = touched * (-(-N // 128)) * (K // 64) * W.TILE_BYTES + rows * K * 2 + rows * ob
              res["gate_up" if kind == 1 else "down"] = (round(us, 1), round(byts / us / 1e3, 1), round(byts / us / 1e3 / peak, 3))
              prof = getattr(L.load(), "stb_debug_moe_prof", None)  # -DSTB_MOE_PROF variants only
              if prof is not None:
                  buf = (C.c_ulonglong * 16)()
                  prof(buf)
                  run(kind)
                  torch.cuda.synchronize()
                  prof(buf)
                  v = list(buf)
                  pct = lambda w, t: f"{100 * w / max(t, 1):4.1f}%"  # noqa: E731
                  print(f"   T={T} {'gate_up' if kind == 1 else 'down'} waits: producer w_empty {pct(v[0], v[3])} | "
                        f"MMA acc_empty {pct(v[4], v[7])} x_full {pct(v[5], v[7])} a_full {pct(v[6], v[7])} | "
                        f"converters w_full {pct(v[8], v[11])} a_empty {pct(v[9], v[11])}", flush=True)
          print(f"[{impl:5s}] T={T:5d} experts touched {touched:3d}: " + "  ".join(f"{n} {u} us {g} GB/s ({f})" for n, (u, g, f) in res.items()),
              flush=True)


if __name__ == "__main__":
    main()
