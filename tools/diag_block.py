import dataclasses, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_block import _steps
from paper_2512_15834_b200.modelcfg import SHAPES
from paper_2512_15834_b200.runtime import decoder as D, weights as W
for base, B in (("llama3-8b", 1), ("llama3-8b", 32)):
    shape = dataclasses.replace(SHAPES[base], name="x", layers=2, vocab=32768)
    prompt = 70
    pool = D.KVPool(shape, num_blocks=B * (prompt // 16 + 2) + 16, max_slots=B + 1, max_blocks_per_slot=16)
    for b in range(B): pool.reserve(b, prompt + 1)
    w = W.build(shape, seed=5, init_device="cuda")
    dec = D.Decoder(shape, w, pool, use_graphs=False); dec.keep_logits = True
    dec.taps = []
    pre, step = _steps(shape, B, prompt, seed=B)
    dec.forward(pre); torch.cuda.synchronize()
    def run(bm):
        D.BLOCK_MAX_T = bm; dec.taps = []
        dec.forward(step); torch.cuda.synchronize()
        return dec.last_logits.clone(), [t[:B].clone() for t in dec.taps], dec.q[:B].clone()
    rel = lambda a, b: float((a.float() - b.float()).norm() / b.float().norm())
    a = run(64); b = run(0); c = run(0); d = run(64)
    print(base, B, "logits blk-op", rel(a[0], b[0]), "op-op", rel(c[0], b[0]), "blk-blk", rel(d[0], a[0]))
    for i, (ta, tb) in enumerate(zip(a[1], b[1])):
        print("  tap", i, rel(ta, tb))
    print("  q", rel(a[2], b[2]))
