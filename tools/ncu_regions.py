"""Summarise an ncu --set full report by barrier-delimited SASS region:
share of stall samples / executed instructions, top opcodes, top stalls.

    python tools/ncu_regions.py gpurun_out/x.ncu-rep
"""
import csv
import subprocess
import sys
from collections import Counter


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    data = rows[2:]
    iS = h.index("Warp Stall Sampling (All Samples)")
    iE = h.index("Instructions Executed")
    iSrc = h.index("Source")
    iA = h.index("Address")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot_s = sum(int(r[iS] or 0) for r in data)
    tot_e = sum(int(r[iE] or 0) for r in data)
    print("total samples", tot_s, "instr", tot_e)
    region, R = 0, {}
    for r in data:
        toks = r[iSrc].split()
        d = R.setdefault(region, {"s": 0, "e": 0, "first": r[iA][-5:], "ops": Counter(), "st": Counter()})
        d["s"] += int(r[iS] or 0)
        d["e"] += int(r[iE] or 0)
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "")).split(".")[0]
        d["ops"][op] += int(r[iE] or 0)
        for i in stall_cols:
            d["st"][h[i][6:]] += int(r[i] or 0)
        if toks and "BAR" in (toks[1] if toks[0].startswith("@") else toks[0]):
            region += 1
    for k, d in R.items():
        if d["s"] / tot_s > 0.015:
            print(k, d["first"], f"samples {d['s'] / tot_s * 100:5.1f}%  instr {d['e'] / tot_e * 100:5.1f}%",
                  d["ops"].most_common(5))
            print("     stalls:", [(a, f"{b / max(d['s'], 1) * 100:.0f}%") for a, b in d["st"].most_common(5)])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(det.splitlines())
    next(r)
    keep = ("Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM",
            "Eligible Warps Per Scheduler", "No Eligible", "Registers Per Thread")
    for row in r:
        if len(row) > 14 and row[12] in keep:
            print(f"  {row[12]}: {row[14]} {row[13]}")


if __name__ == "__main__":
    main(sys.argv[1])
