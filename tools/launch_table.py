"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import re
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"<unnamed>::|_GLOBAL__N__\w+::|void ", "", name)[:56]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"total {tot / 1e6 / steps:.3f} ms per step ({steps} steps, {sum(n for n, _ in agg.values())} launches)")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / tot * 100:6.2f}%  {v / n / 1e3:8.2f} us x{n // steps:4d}/step  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
