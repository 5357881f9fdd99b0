#!/usr/bin/env python
"""One small call per (kernel family, op, math) through the C ABI, for compute-sanitizer
(racecheck / synccheck / memcheck): tools/gpu_sanitize.sh runs it under each tool."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # (variant, op, dims)
    ("tma", 0, (128, 4, 4, 64, 128, 3, 3, 1, 1, 1, 1)),
    ("tma", 1, (128, 4, 4, 64, 128, 3, 3, 1, 1, 1, 1)),
    ("tma", 2, (128, 4, 4, 64, 128, 3, 3, 1, 1, 1, 1)),
    ("tma-csk", 0, (128, 2, 2, 256, 256, 3, 3, 1, 1, 1, 1)),
    ("tma-pair", 0, (256, 4, 4, 128, 128, 3, 3, 1, 1, 1, 1)),
    ("tma-pair", 2, (64, 4, 4, 128, 256, 3, 3, 1, 1, 1, 1)),
    ("tma-ragged", 2, (32, 6, 6, 48, 112, 3, 3, 1, 1, 1, 1)),
    ("tma-pair", 1, (256, 4, 4, 128, 128, 3, 3, 1, 1, 1, 1)),          # TMA-store epilogue, K-major dX filter
    ("tma-zfill", 1, (64, 8, 8, 64, 128, 1, 1, 2, 2, 0, 0)),            # 1x1 s2 dX: zero phases from the epilogue
    ("tma-s2dx", 1, (32, 32, 32, 64, 64, 3, 3, 2, 2, 1, 1)),            # super-pixel dX (automatic plan)
    ("strip", 0, (64, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1)),
    ("strip", 1, (64, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1)),
    ("dws", 2, (32, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1)),
    ("direct", 0, (32, 8, 8, 4, 64, 3, 3, 1, 1, 1, 1)),
    ("generic", 1, (8, 8, 8, 4, 64, 3, 3, 1, 1, 1, 1)),
]
VARIANT = {"tma": 2, "tma-csk": 0, "tma-pair": 0, "tma-ragged": 0, "tma-zfill": 2, "tma-s2dx": 0, "strip": 3, "dws": 5,
           "direct": 4, "generic": 1}


def main():
    import torch
    from paper_2305_08819_b200 import smconv as sm
    only = sys.argv[1:]
    for name, op, d in CASES:
        for math in ("tf32", "3xtf32"):
            if only and name not in only:
                continue
            N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = d
            OH, OW = sm.out_hw(IH, IW, FH, FW, (sh, sw), (ph, pw))
            x = torch.randn(N, IH, IW, IC, device="cuda")
            w = torch.randn(OC, FH, FW, IC, device="cuda")
            dy = torch.randn(N, OH, OW, OC, device="cuda")
            sm.force_variant(op, VARIANT[name])
            if op == 0:
                sm.conv2d_fwd(x, w, (sh, sw), (ph, pw), math=math)
            elif op == 1:
                sm.conv2d_bwd_data(dy, w, (IH, IW), (sh, sw), (ph, pw), math=math)
            else:
                sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw), math=math)
            torch.cuda.synchronize()
            print(name, op, math, sm.plan_describe(op, d, sm.MATH[math]), flush=True)
            sm.force_variant(op, 0)


if __name__ == "__main__":
    main()
