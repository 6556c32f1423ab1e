"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.

    python tools/launch_summary.py launches.csv [--skip N] [--count N]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    for r in rd:
        if r[im] != "gpu__time_duration.sum":
            continue
        rows.append((r[ik], float(r[iv].replace(",", ""))))
    unit = "ns"
    by = {}
    for k, v in rows:
        d = by.setdefault(k.split("(")[0], [0.0, 0])
        d[0] += v
        d[1] += 1
    tot = sum(v for _, v in rows)
    print(f"# {len(rows)} launches, {tot / 1e6:.3f} ms total (gpu__time_duration.sum, {unit})")
    for k, (v, n) in sorted(by.items(), key=lambda kv: -kv[1][0]):
        print(f"{k[:70]:70s} n={n:5d} total_ms={v / 1e6:8.3f} share={v / tot:.4f} avg_us={v / n / 1e3:8.2f}")


if __name__ == "__main__":
    main()
