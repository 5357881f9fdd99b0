#!/usr/bin/env python
"""Render the parity-margin table from the -m gpu tests' parity log (no GPU needed).

  python tools/parity_margins.py <parity_errors.json> "<title line>" > profiles/rNN_parity_margins.md

One row per (config, op, math): the worst random-input error of the group against its tolerance
(normwise max|g-r|/max|r|, reading L8; the fused-epilogue statistics rows carry their own
conditioned error), and the count of integer-input rows that were not bit-exact.
"""
import json
import sys
from collections import defaultdict


def main():
    rows = json.load(open(sys.argv[1]))["rows"]
    title = sys.argv[2] if len(sys.argv) > 2 else "parity margins"
    worst = {}
    ints = defaultdict(lambda: [0, 0])
    for r in rows:
        key = (r["config"], r["op"], r["math"])
        if r.get("check") == "integer":
            ints[key][0] += 1
            ints[key][1] += 0 if r.get("exact", r.get("normwise", 0) == 0) else 1
            continue
        e = r.get("normwise")
        if e is None:
            continue
        if key not in worst or e > worst[key]["normwise"]:
            worst[key] = r
    n_rand = sum(1 for r in rows if r.get("check") != "integer")
    n_int = sum(v[0] for v in ints.values())
    bad_int = sum(v[1] for v in ints.values())
    print("# %s" % title)
    print()
    print("Normwise error per (config, op, math), worst layer of each group, from the `-m gpu` parity tests'")
    print("log (%d random-input rows; %d integer-input rows, %d not bit-exact)." % (n_rand, n_int, bad_int))
    print()
    print("| config | op | math | worst layer | error | tol | margin (tol/err) | coverage |")
    print("|---|---|---|---|---|---|---|---|")
    for key in sorted(worst):
        r = worst[key]
        tol = r.get("tol", 1e-5 if r["math"] == "3xtf32" else 5e-3)
        e = r["normwise"]
        m = "%.1fx" % (tol / e) if e > 0 else "exact"
        print("| %s | %s | %s | %s | %.2e | %.0e | %s | %s |" % (key[0], key[1], key[2], r.get("layer", ""), e, tol, m,
                                                              r.get("coverage", "whole tensor")))


if __name__ == "__main__":
    main()
