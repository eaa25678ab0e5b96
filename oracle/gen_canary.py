"""ORACLE (test infrastructure). Full-size canary goldens: the fp32 CPU oracle decoder
(`oracle/cpu_decoder.py`) at the BASELINE model's full depth and width, run over a fixed
32-token canary sequence, logits of its last row saved to tests/golden/canary_<shape>.npz —
twice: pure fp32, and fp32 arithmetic with bf16 rounding at the points where the engine stores
bf16 (`CpuDecoder.bf16_points`). Their difference is the intrinsic error of bf16 storage at
full depth (~4% at 32 layers of Llama-3-8B width); the engine is checked against the second
within 2e-2 and reported against the first.

The engine's weights for the large configs are drawn on the GPU (runtime/weights.py), so
this script needs a CUDA device only to *draw the same inputs*: every tensor is drawn with
the product's seeded generator on cuda, copied to the host, upcast to fp32, and the whole
forward runs on the CPU, one layer at a time (`stream=True`: no layer stays resident, so
Qwen3-32B fits host memory). Run on the GPU box; the .npz it writes is committed:

    python -m oracle.gen_canary llama3-8b qwen3-32b gpt-oss-120b
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

from .cpu_decoder import CpuDecoder
from .ids import SALT_PROMPT, fill

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
CANARY_LEN = 32


def canary_ids(vocab: int) -> list[int]:
    return fill(0, "canary", SALT_PROMPT, 0, CANARY_LEN, vocab)


def gpu_drawn_source(seed: int = 0):
    from paper_2512_15834_b200.runtime.weights import draw

    def src(name, shp, norm):
        return draw(shp, seed, name, device="cuda", norm=norm).float().cpu()

    return src


def gpu_expert_source(shape, seed: int = 0):
    """MoE experts drawn like the engine's (product generator on cuda, bf16), put through the
    oracle's own MXFP4 restatement (cpu_decoder.mxfp4_roundtrip, on the device for speed), fp32
    on the host."""
    from paper_2512_15834_b200.runtime.weights import draw

    from .cpu_decoder import mxfp4_roundtrip

    d, f = shape.d_model, shape.d_ff

    def src(layer, e):
        p = f"l{layer}.e{e}."
        wg = mxfp4_roundtrip(draw((2 * f, d), seed, p + "w_gate_up", device="cuda").float()).cpu()
        wd = mxfp4_roundtrip(draw((d, f), seed, p + "w_down", device="cuda").float()).cpu()
        bg = draw((2 * f,), seed, p + "b_gate_up", device="cuda").float().cpu()
        bd = draw((d,), seed, p + "b_down", device="cuda").float().cpu()
        return wg, bg, wd, bd

    return src


def main(names: list[str]) -> None:
    from paper_2512_15834_b200.modelcfg import SHAPES

    torch.set_num_threads(max(1, torch.get_num_threads()))
    for name in names:
        shape = SHAPES[name]
        t0 = time.time()
        dec = CpuDecoder(shape, source=gpu_drawn_source(0), stream=True,
                         expert_source=gpu_expert_source(shape) if shape.moe else None)
        ids = canary_ids(shape.vocab)
        logits = dec.forward("canary", ids, 0, [len(ids) - 1])[0]
        dec.bf16_points = True  # same fp32 arithmetic, bf16 rounding where the engine stores bf16
        dec.drop("canary")
        emu = dec.forward("canary", ids, 0, [len(ids) - 1])[0]
        intrinsic = float((emu - logits).norm() / logits.norm())
        path = OUT / f"canary_{name}.npz"
        np.savez_compressed(path, ids=np.asarray(ids, np.int32), logits=logits.numpy().astype(np.float16),
                            logits_bf16_points=emu.numpy().astype(np.float16), intrinsic_bf16_err=np.float64(intrinsic),
                            norm=np.float64(logits.norm()), argmax=np.int64(logits.argmax()))
        print(f"{name}: wrote {path} in {time.time() - t0:.0f} s (argmax {int(logits.argmax())}, "
              f"norm {float(logits.norm()):.3f}, bf16-storage vs fp32 {intrinsic:.4f})", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["llama3-8b"])
