#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> <kernels_per_step> <steps> > profiles/rNN_launches.md
  python tools/ncu_summary.py full <report.ncu-rep | raw.csv> [key] >> profiles/rNN_ncu_full.md

`launches` aggregates the per-launch gpu__time_duration of the LAST <steps> steps (cold-cache,
serialised: compare shares, not absolutes).  `full` prints the counters the roofline uses
(duration, DRAM bytes -> traffic, tensor-pipe and throughput percentages) and, with `key`, merges
traffic per launch into profiles/traffic.json under that key.
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "launch__registers_per_thread", "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path, per_step, steps):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    data = []
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
            data.append((r[ki], ns))
    last = data[-per_step * steps:]
    tot = sum(d[1] for d in last)
    agg, cnt = defaultdict(float), defaultdict(int)
    for k, v in last:
        agg[k] += v
        cnt[k] += 1
    print("| share | launches | ms (sum of %d steps) | kernel |" % steps)
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print("| %.2f%% | %d | %.3f | `%s` |" % (100 * v / tot, cnt[k], v / 1e6, k[:110]))
    print("\nserialised total: %.3f ms per step (%d launches per step)" % (tot / 1e6 / steps, per_step))


def full(path, key=None):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` exported on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print("\n#### `%s`\n" % d.get("Kernel Name", "?")[:120])
        print("| counter | value |\n|---|---|")
        for k in FULL_KEYS:
            if k in d:
                print("| %s | %s %s |" % (k, d[k], u.get(k, "")))
        if key:
            def to_bytes(k):
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u.get(k, "byte"), 1)
                return float(d[k].replace(",", "")) * mult
            tr = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            p = os.path.join(ROOT, "profiles", "traffic.json")
            j = json.load(open(p)) if os.path.exists(p) else {}
            j[key] = tr
            json.dump(j, open(p, "w"), indent=1, sort_keys=True)
            print("\ntraffic (dram read+write per launch) = %.4g bytes -> profiles/traffic.json[%s]" % (tr, key))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
