#!/usr/bin/env python
"""Per-CTA phase timestamps of one TMA-variant call (smconv_set_trace): where a small-map kernel's time goes.
Slots: 0 entry, 1 setup, 2 first TMA, 4 first MMA, 5 last MMA commit, 6 acc ready, 7 epilogue done,
8 CTA barrier, 9/10 csk reduce, 11 exit (SM clock64 cycles); 15 globaltimer at entry (ns)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_08819_b200 import smconv as sm
    dev = torch.device("cuda")
    shapes = {"tiny": (32, 2, 2, 32, 32, 3, 3, 1, 1, 1, 1), "vgg11": (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),
              "vgg6": (128, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1), "vgg9": (128, 4, 4, 512, 512, 3, 3, 1, 1, 1, 1)}
    buf = torch.zeros(148 * 16 * 4, dtype=torch.int64, device=dev)
    for name in sys.argv[1].split(","):
        d = shapes[name]
        N, IH, IW, IC, OC = d[:5]
        x = torch.randn(N, IH, IW, IC, device=dev)
        w = torch.randn(OC, 3, 3, IC, device=dev)
        y = torch.empty(N, IH, IW, OC, device=dev)
        for math in ("tf32", "3xtf32"):
            for _ in range(3):
                sm.conv2d_fwd(x, w, math=math, out=y)
            torch.cuda.synchronize()
            buf.zero_()
            sm.lib().smconv_set_trace(buf.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sm.conv2d_fwd(x, w, math=math, out=y)
            e1.record()
            torch.cuda.synchronize()
            sm.lib().smconv_set_trace(None)
            t = buf.view(-1, 16).cpu().numpy()
            t = t[t[:, 0] != 0]
            rel = (t[:, :15] - t[:, :1])
            rel[t[:, :15] == 0] = -1
            gt = t[:, 15] - t[:, 15].min()
            out = {"shape": name, "math": math, "event_us": e0.elapsed_time(e1) * 1e3, "ctas": int(len(t)),
                   "plan": sm.plan_describe(0, d, sm.MATH[math]),
                   "start_spread_ns": [int(gt.min()), int(gt.max())],
                   "median_cycles": [int(sorted(c)[len(c) // 2]) for c in rel.T],
                   "max_cycles": [int(c.max()) for c in rel.T]}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
