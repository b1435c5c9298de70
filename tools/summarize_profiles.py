"""Summarise gpurun_out/<tag>_* ncu outputs into profiles/ (committed).

    python tools/summarize_profiles.py r01
    python tools/summarize_profiles.py s2_c4 --launches gpurun_out/s2/c4_launches.csv \
        --rep gpurun_out/s2/c4_stream.ncu-rep --kernel stream_kernel --config c4 \
        --label "C4 (1,048,576 elements, 537M GLL points)"
"""
import argparse
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(tag, path=None):
    path = path or os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iN, iV, iM = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    per = defaultdict(list)
    for r in rows[1:]:
        if r[iM] == "gpu__time_duration.sum":
            per[r[iN].split("(")[0]].append(float(r[iV].replace(",", "")))
    tot = sum(sum(v) for v in per.values())
    lines = [f"# ncu launch list ({tag}): bench.py --steps 3 --warmup 3, gpu__time_duration.sum",
             "# cold-cache, serialised per-launch times; compare SHARES, not absolutes",
             f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / tot * 100:6.1f}%")
    ours = {k: v for k, v in per.items() if "nkb::" in k}
    t2 = sum(sum(v) for v in ours.values()) or 1.0
    lines += ["", "# libnekb200 kernels only (the rest is the synthetic-data generator and torch glue)",
              f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.2f} {sum(v) / t2 * 100:6.1f}%")
    return "\n".join(lines) + "\n"


def full(tag, rep=None):
    rep = rep or os.path.join(ROOT, "gpurun_out", f"{tag}_fused.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "launch__grid_size", "launch__block_size"]
    out = {}
    for w in want:
        if w in h:
            i = h.index(w)
            out[w] = (vals[i], units[i])
    return out


def main(tag, launches_csv=None, rep=None, kernel="fused_kernel", config="c2",
         label="C2 (32768 elements, 16.8M GLL points)"):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    txt = launches(tag, launches_csv)
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write(txt)
    print(txt)
    rep = rep or os.path.join(ROOT, "gpurun_out", f"{tag}_fused.ncu-rep")
    m = full(tag, rep)
    short = kernel.replace("_kernel", "")
    lines = [f"# ncu --set full, {kernel}, {label}, tag {tag}"]
    for k, (v, u) in m.items():
        lines.append(f"{k:70s} {v} {u}")
    open(os.path.join(ROOT, "profiles", f"{tag}_{short}_full.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

    def num(k):
        v, u = m[k]
        f = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return f * scale
    # per-source-line stall samples of the same capture (where the warps wait)
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                          capture_output=True, text=True).stdout
    tmp = os.path.join(ROOT, "gpurun_out", f"{tag}_source.csv")
    open(tmp, "w").write(page)
    top = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "40"],
                         capture_output=True, text=True).stdout
    open(os.path.join(ROOT, "profiles", f"{tag}_{short}_lines.txt"), "w").write(
        f"# {kernel} stall samples / instructions by CUDA source line (ncu source page), tag {tag}\n" + top)
    bj = os.path.join(ROOT, "gpurun_out", f"{tag}_bench.json")
    if os.path.exists(bj):
        js = [ln for ln in open(bj).read().splitlines() if ln.startswith("{")]
        if js:
            open(os.path.join(ROOT, "profiles", f"{tag}_bench.json"), "w").write(js[-1] + "\n")
    if "dram__bytes_read.sum" in m:
        traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        json.dump({"dram_bytes_per_launch": traffic, "source": f"profiles/{tag}_{short}_full.txt"},
                  open(os.path.join(ROOT, "profiles", f"traffic_{config}.json"), "w"), indent=1)
        print("traffic", traffic)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag", nargs="?", default="r01")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--rep", default=None)
    ap.add_argument("--kernel", default="fused_kernel")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--label", default="C2 (32768 elements, 16.8M GLL points)")
    a = ap.parse_args()
    main(a.tag, a.launches, a.rep, a.kernel, a.config, a.label)
