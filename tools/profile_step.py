"""Steady-state decode steps of the B200 engine, for ncu and kernel timing.

Builds the engine on a shape, admits `--batch` requests whose script is one
long reasoning turn, prefills them to `--ctx`, then runs decode steps. With
`--profile`, cudaProfilerStart/Stop bracket the last `--profile-steps` steps so
`ncu --profile-from-start off` captures only those launches.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/profile_step.py --profile
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2512_15834_b200.domain import EOS, Token, TokenKind  # noqa: E402
from paper_2512_15834_b200.engine import B200Engine, EngineConfig  # noqa: E402
from harness.mocks import GenerationScript  # noqa: E402
from paper_2512_15834_b200.modelcfg import SHAPES  # noqa: E402
from paper_2512_15834_b200.runtime.executor import BatchRuntime  # noqa: E402
from paper_2512_15834_b200.runtime.realtime import RealtimeLoop  # noqa: E402


class Quiet:
    def on_turn_start(self, *a): pass
    def on_emit(self, *a): pass
    def on_ingest(self, *a): pass
    def on_final(self, *a): pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="llama3-8b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--headroom", type=int, default=4096, help="KV tokens per sequence beyond --ctx in the pool")
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--timers", action="store_true", help="per-kernel CUDA-event times inside the step")
    ap.add_argument("--mix", default="", help="NxL: N new L-token prefills packed into every step")
    ap.add_argument("--gemm-trace", action="store_true",
                    help="per-CTA %%globaltimer timeline of every GEMM launch in the last step")
    args = ap.parse_args()
    shape = SHAPES[args.shape]
    if args.layers:
        shape = shape.with_layers(args.layers)
    nb = args.batch * (args.ctx + args.headroom) // 16 + 64 + args.headroom
    rt = BatchRuntime(shape, init_device="cuda", num_blocks=nb, max_slots=max(64, args.batch) + 1024,
                      max_ctx=args.ctx + 8192, max_step_tokens=16384)
    loop = RealtimeLoop()
    eng = B200Engine(loop, EngineConfig(prefill_rate=0, decode_rate=0, batch_size=max(64, args.batch)), runtime=rt)
    script = GenerationScript([[Token(TokenKind.TEXT, "mull ")] * 8000 + [EOS]])
    for b in range(args.batch):
        eng.submit_request(f"r{b}", script, args.ctx, Quiet())
    while rt.runs:  # prefill
        rt.step()
    torch.cuda.synchronize()
    mix_n, mix_l = (int(x) for x in args.mix.split("x")) if args.mix else (0, 0)
    short = GenerationScript([[Token(TokenKind.TEXT, "mull ")] * 2 + [EOS]])
    extra = [0]

    def inject():
        for _ in range(mix_n):
            eng.submit_request(f"x{extra[0]}", short, mix_l, Quiet())
            extra[0] += 1

    times = []
    if args.timers:
        rt.dec.timers = {}
    for i in range(args.steps):
        last = i >= args.steps - args.profile_steps
        if args.profile and i == args.steps - args.profile_steps:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        inject()
        t0 = time.perf_counter()
        rt.step()
        rt.drain()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        if args.profile and last and i == args.steps - 1:
            torch.cuda.profiler.stop()
    rt.drain()
    if args.gemm_trace:
        gemm_trace(rt)
    if args.timers:
        ov_t, _, ov_n = rt.dec.timers.pop("event_overhead", (0.0, 0, 0))
        ov = ov_t / ov_n if ov_n else 0.0
        rt.dec.timers.pop("attn_prefill:launches", None)
        print(f"  (event-pair overhead {ov * 1e3:.2f} us per launch subtracted)")
        for name, (t, work, n) in rt.dec.timers.items():
            t = max(t - n * ov, 1e-3 * t)
            if name in ("gemm_prefill", "attn_prefill"):
                print(f"  {name:12s} {t / n * 1e3:8.2f} us avg x{n}  {work / (t / 1e3) / 1e12:8.1f} TFLOP/s")
            else:
                print(f"  {name:12s} {t / n * 1e3:8.2f} us avg x{n}  {work / (t / 1e3) / 1e9:8.1f} GB/s algorithmic")
    ms = sorted(times[len(times) // 3:])
    print(f"{shape.name} B={args.batch} ctx~{args.ctx} mix={args.mix or '-'}: median step {ms[len(ms) // 2] * 1e3:.3f} ms "
          f"({args.batch / ms[len(ms) // 2]:.0f} tok/s)")


def gemm_trace(rt):
    """One more decode step with GEMM tracing on: per launch, the CTA-median entry,
    dependency-wait, first-stage and last-MMA times and the last CTA exit (us, from
    the first GEMM entry), plus the idle gap since the previous GEMM's last exit."""
    import ctypes as C

    import numpy as np

    from paper_2512_15834_b200.runtime import lib

    cap = 1 << 16
    buf = torch.zeros(cap * 8, dtype=torch.int64, device="cuda")
    fn = lib.load().stb_debug_gemm_trace
    fn.argtypes, fn.restype = [C.c_void_p, C.c_int], C.c_int
    torch.cuda.synchronize()
    fn(C.c_void_p(buf.data_ptr()), cap)
    rt.step()
    rt.drain()
    torch.cuda.synchronize()
    n = fn(None, 0)
    rec = buf[:n * 8].view(n, 8).cpu().numpy().astype(np.int64)
    t_base = rec[:, 3].min()
    prev_end = None
    print(f"  GEMM trace: {n} CTA records")
    print("   (us from entry of the launch; p50/max over CTAs)")
    print("   tag  gap  | wait p50 | first p50 | mma-issued p50/max | epi-start p50/max | exit p50/max | dur")
    for tag in np.unique(rec[:, 0]):
        r = rec[rec[:, 0] == tag]
        e0 = r[:, 3].min()
        q = lambda col, f: (f(r[:, col]) - e0) / 1e3  # noqa: E731
        end = r[:, 7].max()
        gap = (e0 - prev_end) / 1e3 if prev_end is not None else 0.0
        print(f"  {tag:4d} {gap:5.1f} | {q(4, np.median):6.1f} | {q(5, np.median):6.1f} | "
              f"{q(6, np.median):6.1f} {q(6, np.max):6.1f} | {q(1, np.median):6.1f} {q(1, np.max):6.1f} | "
              f"{q(7, np.median):6.1f} {q(7, np.max):6.1f} | {(end - e0) / 1e3:6.1f}")
        prev_end = end


if __name__ == "__main__":
    main()
