"""Markdown tables for DESIGN.md from bench JSON lines under a directory.

    python tools/tables.py profiles/r2            # every *.json bench line, one row each
"""
from __future__ import annotations

import glob
import json
import os
import sys


def load(path):
    with open(path) as f:
        lines = [l for l in f.read().splitlines() if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main(d):
    rows = []
    for p in sorted(glob.glob(os.path.join(d, "**", "*.json"), recursive=True)):
        j = load(p)
        if not j or "metric" not in j or j.get("impl") == "reference":
            continue
        r = j.get("roofline", {})
        c = j.get("config", {})
        e2e = (j.get("e2e") or {}).get("value")
        rows.append((os.path.relpath(p, d), c.get("workload", "")[:60], j["n_gpus"], j["value"] / 1e9, j["ms_per_step"],
                     r.get("kernel_ms"), r.get("frac"), j.get("scaling"),
                     None if e2e is None else e2e / 1e9, (j.get("parity") or {}).get("ok"),
                     j.get("fused_ms_per_rank"), (j.get("stages_ms") or {}).get("composite")))
    print("| file | workload | GPUs | G GLL pts/s | ms/step | kernel ms | frac | scaling | e2e G/s | parity | per-rank kernel ms | composite ms |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        f = lambda v, n=3: "—" if v is None else (f"{v:.{n}f}" if isinstance(v, float) else str(v))
        print(f"| {r[0]} | {r[1]} | {r[2]} | {f(r[3], 2)} | {f(r[4], 4)} | {f(r[5], 4)} | {f(r[6])} | {r[7]} | "
              f"{f(r[8], 2)} | {f(r[9])} | {r[10]} | {f(r[11], 4)} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r2")
