"""Print the launch sequence (name, duration) of an ncu gpu__time_duration CSV: rows [a, b)."""
import csv
import re
import sys


def main(path, a=0, b=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for j, r in enumerate(rows[hi + 1:][a:b]):
        v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"<unnamed>::|_GLOBAL__N__\w+::|void ", "", name)[:48]
        print(f"{a + j:5d} {v / 1e3:9.2f} us  {name}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:4]))
