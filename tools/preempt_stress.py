"""KV-preemption stress (GPU): the batch-parity fleet on pools far smaller than its working set,
several seeds; every run must complete and replay against the oracle (tests/test_gpu_batch_parity.py
helpers). Usage: python tools/preempt_stress.py [--blocks 36,40,48] [--seeds 1,2,3]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from test_gpu_batch_parity import LOGIT_RTOL, _replay, _run_fleet  # noqa: E402

from paper_2512_15834_b200.modelcfg import TINY  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", default="36,40,48")
    ap.add_argument("--seeds", default="1,2,3")
    a = ap.parse_args()
    bad = 0
    for nb in [int(x) for x in a.blocks.split(",")]:
        for seed in [int(x) for x in a.seeds.split(",")]:
            try:
                rt, _ = _run_fleet(TINY, agents=12, steps=400, seed=seed, num_blocks=nb)
                err = _replay(rt, TINY, num_blocks=nb)
                ok = err <= LOGIT_RTOL
                print(f"blocks={nb} seed={seed}: spills={rt.spills} deferred={rt.deferred} max rel err={err:.2e} "
                      f"{'ok' if ok else 'PARITY FAIL'}", flush=True)
                bad += not ok
            except Exception as e:  # noqa: BLE001
                print(f"blocks={nb} seed={seed}: {type(e).__name__}: {e}", flush=True)
                bad += 1
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
