"""Diagnostics: per-layer teacher-forced error of the gpt-oss-mini engine vs the oracle."""
import sys

import torch

sys.path.insert(0, ".")
from oracle.cpu_decoder import CpuDecoder  # noqa: E402
from paper_2512_15834_b200.modelcfg import GPT_OSS_MINI  # noqa: E402
from paper_2512_15834_b200.runtime.executor import EagerRuntime  # noqa: E402

shape = GPT_OSS_MINI
for n in (20, 32, 33, 40, 64, 100, 256):
    rt = EagerRuntime(shape, num_blocks=512, max_slots=8, max_ctx=4096)
    ids = [(7 * i + 3) % shape.vocab for i in range(n)]
    taps = []
    routes = []
    got = rt.probe_logits(ids, taps=taps, routes=routes)
    dec = CpuDecoder(shape)
    dec.bf16_points = True
    pos = torch.arange(n)
    errs = []
    for i, w in dec.iter_layers():
        x_in = taps[i]
        ref, _ = dec.layer_forward(w, x_in, pos, 0, (torch.zeros(0, 2, 64), torch.zeros(0, 2, 64)), hint=routes[i])
        d_ref, d_got = ref - x_in, taps[i + 1] - x_in
        row = ((d_got - d_ref).norm(dim=1) / d_ref.norm(dim=1))
        errs.append((round(float((d_got - d_ref).norm() / d_ref.norm()), 4), [round(float(v), 3) for v in row[::max(1, n // 8)]]))
    print(n, errs, 'arbitrated', dec.arbitrated, 'of', dec.routed, flush=True)
