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
