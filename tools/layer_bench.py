#!/usr/bin/env python
"""Time single conv calls (one layer, one op) through the C ABI with CUDA events — for tuning.

  python tools/layer_bench.py --net resnet18 --layer l1.0a --op fwd --batch 4096 --math tf32 [--reps 20]

Prints one JSON line per (layer, op): median ms, TFLOP/s (valid-tap), GB/s (compulsory), plan.
Inputs larger than L2 are used as-is; for small layers the L2 is flushed between reps.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet18")
    ap.add_argument("--layer", default=None, help="layer name (default: all)")
    ap.add_argument("--op", default="fwd,dx,dw")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--math", default="3xtf32")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--variant", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_2305_08819_b200 import nets, synth
    from paper_2305_08819_b200 import smconv as sm
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    m = sm.MATH[a.math]
    for op in (0, 1, 2):
        sm.force_variant(op, a.variant)
    for i, l in enumerate(nets.NETS[a.net]()):
        if a.layer and l.name not in a.layer.split(","):
            continue
        X, W, dY = synth.torch_layer_inputs(l, a.batch, dev, seed=i)
        for opn in a.op.split(","):
            op = {"fwd": 0, "dx": 1, "dw": 2}[opn]
            if op == 1 and i == 0:
                continue
            dims = l.dims(a.batch)
            nb = sm.workspace_bytes(op, dims, m)
            ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
            if op == 0:
                args = (X, W, torch.empty((a.batch, l.OH, l.OW, l.OC), device=dev))
            elif op == 1:
                args = (dY, W, torch.empty_like(X))
            else:
                args = (X, dY, torch.empty_like(W))
            st = torch.cuda.current_stream().cuda_stream
            small = nets.bytes_compulsory(l, a.batch, opn) < (256 << 20)

            def call():
                sm.raw_call(op, args[0].data_ptr(), args[1].data_ptr(), args[2].data_ptr(), dims, m,
                            ws.data_ptr(), nb, st)
            for _ in range(3):
                call()
            ts = []
            for _ in range(a.reps):
                if small:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            fl = nets.flops(l, a.batch, True)
            by = nets.bytes_compulsory(l, a.batch, opn)
            print(json.dumps({"layer": l.name, "op": opn, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                              "gbs": round(by / ms / 1e6, 1), "plan": sm.plan_describe(op, dims, m),
                              "env": {k: v for k, v in os.environ.items() if k.startswith("SMCONV")}}), flush=True)


if __name__ == "__main__":
    main()
