"""Summarise .ncu-rep captures into a markdown table (run here, no GPU):
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/...md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def stalls(path, top=8):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h = rows[1]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    data = [(int(r[si]) if r[si].isdigit() else 0, r[src].strip()) for r in rows[2:] if len(r) > si]
    tot = sum(d[0] for d in data) or 1
    return [(100.0 * n / tot, s) for n, s in sorted(data, reverse=True)[:top]]


for path in sys.argv[1:]:
    h, u, rows = raw(path)
    for r in rows:
        name = r[h.index("Kernel Name")]
        print(f"### `{name[:120]}`\n\nsource: `{path.split('/')[-1]}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {label} (`{k}`) | {r[i]} {u[i]} |")
        print("\nTop warp-stall sampling locations (SASS):\n")
        print("| % samples | instruction |\n|---|---|")
        for pct, s in stalls(path):
            print(f"| {pct:.1f} | `{s[:70]}` |")
        print()
