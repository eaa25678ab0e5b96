"""Launch one GEMM shape a few times (no graph) — a clean target for `ncu --set full`.

    ncu --set full -k regex:gemm -c 1 -s 2 python tools/gemm_once.py --M 608 --N 28672 --K 4096
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2512_15834_b200.runtime import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=608)
ap.add_argument("--N", type=int, default=28672)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--trace", action="store_true", help="per-CTA phase medians of the last launch (us)")
a = ap.parse_args()
x = torch.randn(a.M, a.K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(a.N, a.K, device="cuda", dtype=torch.bfloat16)
c = torch.zeros(a.M, a.N, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(a.reps):
    lib.call("stb_gemm_bf16", C.c_void_p(x.data_ptr()), a.K, C.c_void_p(w.data_ptr()), a.K, C.c_void_p(c.data_ptr()),
             a.N, a.M, a.N, a.K, a.split, 0, st)
torch.cuda.synchronize()
print("ok", a.M, a.N, a.K)
if a.trace:
    import numpy as np

    fn = lib.load().stb_debug_gemm_trace
    fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
    buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
    fn(C.c_void_p(buf.data_ptr()), 4096)
    lib.call("stb_gemm_bf16", C.c_void_p(x.data_ptr()), a.K, C.c_void_p(w.data_ptr()), a.K,
             C.c_void_p(c.data_ptr()), a.N, a.M, a.N, a.K, a.split, 0, st)
    torch.cuda.synchronize()
    n = fn(None, 0)
    r = buf[:n * 8].view(n, 8).cpu().numpy().astype(np.int64)
    e0 = r[:, 3].min()
    for name, col in (("dep-wait", 4), ("first-stage", 5), ("last-mma-issue", 6), ("last-epi-start", 1),
                      ("exit", 7)):
        v = (r[:, col] - e0) / 1e3
        print(f"  {name:15s} p10 {np.percentile(v, 10):6.1f}  p50 {np.median(v):6.1f}  max {v.max():6.1f} us")
