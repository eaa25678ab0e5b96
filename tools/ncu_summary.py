"""Summarise `ncu --set full` reports for profiles/: one block per captured kernel with
duration, DRAM traffic (read + write), HBM / L2 / tensor-pipe utilisation and the
top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/r1b/full_decode.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs/thread")]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(f"{path}: no kernels")
        return
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        print(f"### {name[:110]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:20s} {d[k]} {units[hdr.index(k)]}")
        st = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]))
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"## {p}\n")
        summarise(p)
