#!/usr/bin/env python
"""Per-call GPU time of back-to-back conv calls (no flush / with an L2 flush between calls) for tiny and
small-map shapes: separates fixed per-kernel cost from bandwidth (round-2 VGG b128 investigation)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_08819_b200 import smconv as sm
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    shapes = [("tiny", (32, 2, 2, 32, 32, 3, 3, 1, 1, 1, 1)), ("vgg11", (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1)),
              ("vgg6", (128, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1)), ("vgg3", (128, 16, 16, 64, 128, 3, 3, 1, 1, 1, 1))]
    reps = 100
    quick = "--quick" in sys.argv  # under ncu: a few calls per shape, no graphs
    if quick:
        reps = 2
    only = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--shape=")]
    for name, d in shapes:
        if only and name not in only[0].split(","):
            continue
        N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = d
        x = torch.randn(N, IH, IW, IC, device=dev)
        w = torch.randn(OC, FH, FW, IC, device=dev)
        for math in ("tf32", "3xtf32"):
            for op in (0, 2):
                y = torch.empty(N, IH, IW, OC, device=dev)
                dw = torch.empty(OC, FH, FW, IC, device=dev)
                f = (lambda: sm.conv2d_fwd(x, w, (1, 1), (1, 1), math=math, out=y)) if op == 0 else \
                    (lambda: sm.conv2d_bwd_filter(x, y, (3, 3), (1, 1), (1, 1), math=math, out=dw))
                for _ in range(5):
                    f()
                torch.cuda.synchronize()
                res = {}
                for mode in ("b2b", "flush"):
                    evs = []
                    for i in range(reps):
                        if mode == "flush":
                            flush.zero_()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        f()
                        e1.record()
                        evs.append((e0, e1))
                    torch.cuda.synchronize()
                    t = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
                    res[mode] = {"median_us": t[len(t) // 2], "min_us": t[0]}
                # whole loop, no per-call events
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for i in range(reps):
                    f()
                e1.record()
                torch.cuda.synchronize()
                res["loop_avg_us"] = e0.elapsed_time(e1) * 1e3 / reps
                if quick:
                    print(json.dumps({"shape": name, "op": op, "math": math}), flush=True)
                    continue
                # graph of the loop
                g = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    f()
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
                with torch.cuda.graph(g):
                    for i in range(reps):
                        f()
                g.replay()
                torch.cuda.synchronize()
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                res["graph_avg_us"] = e0.elapsed_time(e1) * 1e3 / reps
                res.update(shape=name, op=op, math=math,
                           plan=sm.plan_describe(op, d, sm.MATH[math]))
                print(json.dumps(res), flush=True)
    # torch reference kernels
    a = torch.empty(1 << 18, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        a.add_(1.0)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"shape": "torch add_ 1MB", "loop_avg_us": e0.elapsed_time(e1) * 1e3 / reps}))


if __name__ == "__main__":
    main()
