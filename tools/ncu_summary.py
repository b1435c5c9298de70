"""One-file summary of an `ncu --set full` capture for profiles/: the headline
metrics (duration, DRAM bytes, pipe and issue utilisation, FP64 instruction
counts) and the per-region stall table of tools/ncu_regions.py.

    python tools/ncu_summary.py gpurun_out/p2/fused2_c2.ncu-rep "K1g C2 ..." > profiles/r2/k1g_c2_full.txt
    python tools/ncu_summary.py REP LABEL --json profiles/fp64_c2.json --traffic profiles/traffic_c2.json --kernel fused2_kernel
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts % of peak"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "CTAs/SM limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM limit (shared memory)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instr"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-instr"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-instr"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(s):
    return float(s.replace(",", ""))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("label")
    ap.add_argument("--json", help="write FP64 flops per launch to this file (key --kernel)")
    ap.add_argument("--traffic", help="write DRAM bytes per launch to this file")
    ap.add_argument("--kernel", default="fused2_kernel")
    a = ap.parse_args()
    m = raw(a.rep)
    print(f"# {a.label}")
    print(f"# source: {a.rep} (ncu --set full --clock-control none, one launch; cold cache, replayed)")
    for k, name in KEYS:
        if k in m:
            print(f"{name:34s} {m[k][0]:>16s} {m[k][1]}")
    flops = None
    try:
        fma = num(m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"][0])
        add = num(m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"][0])
        mul = num(m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"][0])
        flops = 2 * fma + add + mul
        print(f"{'FP64 flops (2 fma + add + mul)':34s} {flops:16.4e}")
    except KeyError:
        pass
    rd = num(m["dram__bytes_read.sum"][0]) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else
                                             1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1)
    wr = num(m["dram__bytes_write.sum"][0]) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else
                                              1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1)
    print(f"{'DRAM bytes per launch':34s} {rd + wr:16.4e}")
    print()
    sys.stdout.flush()
    here = os.path.dirname(os.path.abspath(__file__))
    subprocess.run([sys.executable, os.path.join(here, "ncu_regions.py"), a.rep])
    if a.json and flops is not None:
        d = json.load(open(a.json)) if os.path.exists(a.json) else {}
        d[a.kernel] = flops
        d["source"] = a.label
        json.dump(d, open(a.json, "w"), indent=1)
    if a.traffic:
        json.dump({"dram_bytes_per_launch": rd + wr, "kernel": a.kernel, "source": a.label},
                  open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
