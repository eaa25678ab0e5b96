"""Per-phase timeline of decode-block launches (stb_debug_block_trace) in one decode step:
for each op, the CTA-median times (us from the launch's first CTA entry) at which the op may
start (previous barrier observed), finishes its work, and has arrived on the next barrier."""
import ctypes as C, dataclasses, sys, torch, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_block import _steps
from paper_2512_15834_b200.modelcfg import SHAPES
from paper_2512_15834_b200.runtime import decoder as D, weights as W, lib
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shape = dataclasses.replace(SHAPES["llama3-8b"], name="x", layers=4, vocab=32768)
prompt = 1000
pool = D.KVPool(shape, num_blocks=B * (prompt // 16 + 2) + 16, max_slots=B + 1, max_blocks_per_slot=80)
for b in range(B): pool.reserve(b, prompt + 1)
w = W.build(shape, seed=5, init_device="cuda")
dec = D.Decoder(shape, w, pool, use_graphs=False)
pre, step = _steps(shape, B, prompt, seed=B)
dec.forward(pre); torch.cuda.synchronize()
for _ in range(3):
    dec.forward(step)
torch.cuda.synchronize()
fn = lib.load().stb_debug_block_trace
fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
buf = torch.zeros(4096 * 32, dtype=torch.int64, device="cuda")
fn(C.c_void_p(buf.data_ptr()), 4096)
dec.forward(step); torch.cuda.synchronize()
n = fn(None, 0)
r = buf[:n * 32].view(n, 32).cpu().numpy().astype(np.int64)
# group by launch: records sorted by entry time, split on gaps > 30 us
tags = r[:, 0] >> 8
t_first = {t: r[tags == t, 2].min() for t in np.unique(tags)}
for L, t in enumerate(sorted(t_first, key=t_first.get)):
    q = r[tags == t]
    e0 = q[:, 2].min()
    nops = int(q[0, 0] & 255)
    ent = (q[:, 2] - e0) / 1e3
    print(f"  CTA entry spread: p50 {np.median(ent):.1f} p90 {np.percentile(ent, 90):.1f} max {ent.max():.1f} us")
    s = f"launch {L} ({len(q)} CTAs, {nops} ops): dep {np.median(q[:, 3] - e0) / 1e3:5.1f} |"
    for op in range(nops):
        st_, dn, ar = q[:, 4 + 3 * op], q[:, 5 + 3 * op], q[:, 6 + 3 * op]
        s += f" op{op} {np.median(st_ - e0) / 1e3:5.1f}/{np.median(dn - e0) / 1e3:5.1f}/{np.max(dn - e0) / 1e3:5.1f}"
        if op + 1 < nops:
            s += f"/{np.max(ar - e0) / 1e3:5.1f}"
        s += " |"
    s += f" exit {np.max(q[:, 31] - e0) / 1e3:5.1f}"
    print(s)
