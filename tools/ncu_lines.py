"""Per-CUDA-source-line instruction / stall share from an ncu report.

usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import subprocess
import sys


def main(rep, kern, top=30):
    out = subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", f"regex:{kern}",
         "--launch-count", "1"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.split("\n")))
    hi = [i for i, x in enumerate(r) if x and "Instructions Executed" in x][0]
    hdr = r[hi]
    ei = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    rows = []
    for x in r[hi + 1:]:
        if len(x) < len(hdr) or not x[0]:
            continue  # SASS rows carry no line number; CUDA rows aggregate them
        try:
            rows.append((int(x[ei] or 0), int(x[si] or 0), x[0], x[1].strip()[:100]))
        except ValueError:
            pass
    T = sum(x[0] for x in rows) or 1
    S = sum(x[1] for x in rows) or 1
    rows.sort(key=lambda x: -x[1])
    print(f"total warp-instructions {T}")
    for x in rows[:top]:
        print(f"{100 * x[0] / T:5.1f}% inst {100 * x[1] / S:5.1f}% stall  L{x[2]:>4} {x[3]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
