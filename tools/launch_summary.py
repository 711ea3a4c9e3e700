"""Summarise an ncu --csv launch list: per-kernel total / count / share."""
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Grid Size")
    out = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[ui]]
        out.append((r[ki].split("(")[0], r[gi], v * scale))
    return out


def main(path):
    rows = load(path)
    tot = sum(r[2] for r in rows)
    agg = {}
    for name, grid, ms in rows:
        a = agg.setdefault(name, [0.0, 0])
        a[0] += ms
        a[1] += 1
    print(f"{'ms':>9} {'share':>6} {'n':>4}  kernel")
    for k, (ms, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{ms:9.3f} {100 * ms / tot:5.1f}% {c:4d}  {k}")
    print(f"{tot:9.3f} total ms over {len(rows)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
