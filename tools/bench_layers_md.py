#!/usr/bin/env python
"""Render profiles/rNN_bench_layers.md from bench.py outputs brought back in gpurun_out/ (no GPU needed).

  python tools/bench_layers_md.py <bench_3x.json> <layers_3x.json> <layers_tf32.json> [<bench line> ...] > profiles/r01_bench_layers.md

bench_*.json: a file whose last line is bench.py's JSON line; layers_*.json: bench.py --layers-out.
"""
import json
import sys


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    b3, l3, lt = sys.argv[1:4]
    extra = sys.argv[4:]
    line = last_json(b3)
    def rows(path):
        d = json.load(open(path))
        return d["layers"] if isinstance(d, dict) else d
    L3 = rows(l3)
    LT = {(r["layer"], r["op"]): r for r in rows(lt)}
    print("# r01 bench — per-call times inside the timed region (CUDA events on the launching stream)\n")
    print("Default workload: %s, 1 B200.  Bench line (%s):\n" % (line["config"]["workload"], line["config"]["math"]))
    print("```json\n%s\n```\n" % json.dumps(line))
    for e in extra:
        d = last_json(e)
        c = d.get("config", {})
        print("* `%s` %s: **%.0f %s**, %.3f ms/step, dominant call %s-bound at %.3f of its peak (%s; %s), SM clock %s MHz\n" % (
            c.get("workload", d.get("impl", "")), c.get("math", ""), d["value"], d["unit"], d["ms_per_step"],
            (d.get("roofline") or {}).get("bound"), (d.get("roofline") or {}).get("frac") or 0.0,
            (d.get("roofline") or {}).get("unit"), ((d.get("roofline") or {}).get("kernel") or "")[:60],
            (d.get("clocks") or {}).get("sm_mhz")))
    print("| layer | op | 3xTF32 ms | 3xTF32 TFLOP/s | TF32 ms | TF32 TFLOP/s | GB/s (3x, compulsory) | plan (3xTF32) |")
    print("|---|---|---|---|---|---|---|---|")
    tot3 = tott = 0.0
    for r in sorted(L3, key=lambda r: (r["i"], r["op"])):
        t = LT.get((r["layer"], r["op"]))
        tot3 += r["ms"]
        tott += t["ms"] if t else 0.0
        print("| %s | %s | %.3f | %.1f | %s | %s | %.0f | %s |" % (
            r["layer"], r["op"], r["ms"], r["tflops"], "%.3f" % t["ms"] if t else "-",
            "%.1f" % t["tflops"] if t else "-", r["gbs"], r["plan"]))
    print("\nsum of per-call times: 3xTF32 %.2f ms, TF32 %.2f ms per step" % (tot3, tott))


if __name__ == "__main__":
    main()
