"""Aggregate an ncu source page (cuda,sass) by CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > page.csv
    python tools/ncu_lines.py page.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = next(r for r in rows if r and r[0] == "Line No")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    iN = hdr.index("Instructions Executed")
    lines = []
    for r in rows:
        if r and r[0] not in ("", "Line No") and len(r) > iN and r[0].isdigit():
            try:
                lines.append((float(r[iW] or 0), float(r[iN] or 0), int(r[0]), r[1]))
            except ValueError:
                pass
    tw = sum(x[0] for x in lines) or 1
    tn = sum(x[1] for x in lines) or 1
    print(f"samples {tw:.0f} instructions {tn:.0f}")
    for w, n, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{w / tw * 100:5.1f}% smp {n / tn * 100:5.1f}% ins  L{ln:<5d} {src.strip()[:90]}")


if __name__ == "__main__":
    main()
