#!/usr/bin/env python
"""Compare per-layer in-step times of two bench runs (A/B on one box): ab_compare.py DIR"""
import json
import sys

d = sys.argv[1]


def agg(fn):
    a = {}
    for l in json.load(open(fn))["layers"]:
        k = l["layer"].split(".")[0] + " " + l["op"]
        a[k] = a.get(k, 0) + l["ms"]
    return a


h = [agg("%s/layers_head_%d.json" % (d, r)) for r in (1, 2)]
n = [agg("%s/layers_new_%d.json" % (d, r)) for r in (1, 2)]
for k in h[0]:
    hh = (h[0][k] + h[1][k]) / 2
    nn = (n[0][k] + n[1][k]) / 2
    print("%-10s head %7.3f  new %7.3f  %+6.1f%%" % (k, hh, nn, 100 * (nn / hh - 1)))
