"""Decode step at B=1 / 32 through the block path and the per-op path, 4 runs each, against the
fp32 oracle: is the block path's difference systematic or run-to-run noise?"""
import dataclasses, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_block import _steps
from oracle.cpu_decoder import CpuDecoder
from paper_2512_15834_b200.modelcfg import SHAPES
from paper_2512_15834_b200.runtime import decoder as D, weights as W
rel = lambda a, b: float((a.float().cpu() - b.float().cpu()).norm() / b.float().cpu().norm())
for base, B in (("llama3-8b", 1), ("llama3-8b", 4)):
    shape = dataclasses.replace(SHAPES[base], name="x", layers=2, vocab=32768)
    prompt = 70
    pool = D.KVPool(shape, num_blocks=B * (prompt // 16 + 2) + 16, max_slots=B + 1, max_blocks_per_slot=16)
    for b in range(B): pool.reserve(b, prompt + 1)
    w = W.build(shape, seed=0, init_device="cuda")
    dec = D.Decoder(shape, w, pool, use_graphs=False); dec.keep_logits = True
    pre, step = _steps(shape, B, prompt, seed=B)
    dec.forward(pre); torch.cuda.synchronize()
    ora = CpuDecoder(shape)
    want = []
    for b in range(B):
        ids = [int(t) for t in pre.ids[b * prompt:(b + 1) * prompt]] + [int(step.ids[b])]
        want.append(ora.forward(f"r{b}", ids, 0, [prompt])[0])
    want = torch.stack(want)
    res = {}
    for mode in (64, 0, 64, 0, 64, 0):
        D.BLOCK_MAX_T = mode
        for name in ("qkv", "proj", "gu"):
            r = dec._dirty[name]
            if r:
                getattr(dec, name)[:r].zero_(); dec._dirty[name] = 0
        dec.forward(step); torch.cuda.synchronize()
        res.setdefault(mode, []).append(dec.last_logits.clone())
    print(base, B, "block vs oracle", [round(rel(l, want), 5) for l in res[64]],
          "per-op vs oracle", [round(rel(l, want), 5) for l in res[0]])
    print("   block-vs-block", round(rel(res[64][1], res[64][0]), 5), "op-vs-op", round(rel(res[0][1], res[0][0]), 5),
          "block-vs-op", round(rel(res[64][0], res[0][0]), 5))
