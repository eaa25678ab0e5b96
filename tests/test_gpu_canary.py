"""Full-size numerics parity (the benchmarked models at their full depth and width).

1. End to end: the engine's logits for the fixed 32-token canary sequence vs the fp32 CPU oracle's
   (tests/golden/canary_<shape>.npz, oracle/gen_canary.py, same GPU-drawn weights): no further from
   fp32 than bf16 storage itself is (bench.canary_compare), argmax within the oracle's top 5.
2. Per layer, teacher-forced: every layer's update of the residual stream, computed by the engine,
   vs the fp32 oracle's `layer_forward` fed the ENGINE's own input to that layer: relative L2 error
   <= 2e-2 (BASELINE north star, bf16 vs the fp32 reference), and the final norm + LM head on the
   engine's last residual row likewise."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
SHAPES = sorted(p.stem[len("canary_"):] for p in GOLDEN.glob("canary_*.npz"))
TOL = 2e-2


@pytest.mark.parametrize("name", SHAPES)
def test_full_size_canary(name):
    import torch

    from oracle.cpu_decoder import CpuDecoder
    from oracle.gen_canary import gpu_drawn_source, gpu_expert_source
    from oracle.ids import SALT_PROMPT, fill
    from paper_2512_15834_b200.modelcfg import SHAPES as ALL
    from paper_2512_15834_b200.runtime.executor import EagerRuntime

    shape = ALL[name]
    g = np.load(GOLDEN / f"canary_{name}.npz")
    ids = fill(0, "canary", SALT_PROMPT, 0, int(g["ids"].shape[0]), shape.vocab)
    assert ids == g["ids"].tolist()
    rt = EagerRuntime(shape, init_device="cuda", num_blocks=256, max_slots=8, max_ctx=4096)
    taps: list = []
    routes: list = []
    got = rt.probe_logits(ids, taps=taps, routes=routes).numpy().astype(np.float64)
    del rt
    torch.cuda.empty_cache()
    from bench import canary_compare

    res = canary_compare(got, g)
    assert res["status"] == "pass", res

    assert len(taps) == shape.layers + 1
    dec = CpuDecoder(shape, source=gpu_drawn_source(0), stream=True,
                     expert_source=gpu_expert_source(shape) if shape.moe else None)
    dec.bf16_points = shape.moe  # MoE: bf16 storage rounding as on the engine (router near-ties)
    pos = torch.arange(len(ids))
    G, D = shape.n_kv, shape.d_head
    errs = []
    for i, w in dec.iter_layers():
        x_in = taps[i]
        ref, _ = dec.layer_forward(w, x_in, pos, 0, (torch.zeros(0, G, D), torch.zeros(0, G, D)),
                                   hint=routes[i] if routes else None)
        d_ref, d_got = ref - x_in, taps[i + 1] - x_in
        errs.append(float((d_got - d_ref).norm() / d_ref.norm()))
    head = (dec._norm(taps[-1][-1:], dec.fn) @ dec.head.T)[0].double().numpy()
    e_head = float(np.linalg.norm(got - head) / np.linalg.norm(head))
    assert max(errs) <= TOL, (max(errs), int(np.argmax(errs)), errs)
    assert e_head <= TOL, e_head
