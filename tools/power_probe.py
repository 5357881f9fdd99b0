#!/usr/bin/env python
"""Energy per call of single conv calls: each (layer, op) runs back to back for ~2 s while NVML samples the
board power and SM clock.  The 3xTF32 ResNet step runs at the power cap, where the
energy per call, not its isolated time, decides the step time.

  python tools/power_probe.py --net resnet18 --layer l1.0a,l2.1a --op fwd,dx,dw --batch 4096 --math 3xtf32

Prints one JSON line per (layer, op): ms per call, mean W, median SM MHz, mJ per call, pJ per useful flop.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="resnet18")
    ap.add_argument("--layer", default=None)
    ap.add_argument("--op", default="fwd,dx,dw")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--math", default="3xtf32")
    ap.add_argument("--seconds", type=float, default=2.0)
    a = ap.parse_args()
    import pynvml
    import torch

    from paper_2305_08819_b200 import nets, synth
    from paper_2305_08819_b200 import smconv as sm
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    dev = torch.device("cuda")
    m = sm.MATH[a.math]
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

            def call():
                sm.raw_call(op, args[0].data_ptr(), args[1].data_ptr(), args[2].data_ptr(), dims, m,
                            ws.data_ptr(), nb, st)
            for _ in range(5):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                call()
            e1.record()
            torch.cuda.synchronize()
            t1 = e0.elapsed_time(e1) / 5
            reps = max(10, int(a.seconds * 1000 / max(t1, 1e-3)))
            samples, stop = [], threading.Event()

            def sampler():
                while not stop.is_set():
                    samples.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    time.sleep(0.02)
            for _ in range(reps // 4):  # reach the steady power state before sampling
                call()
            th = threading.Thread(target=sampler)
            th.start()
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            stop.set()
            th.join()
            ms = e0.elapsed_time(e1) / reps
            pw = statistics.mean(s[0] for s in samples[len(samples) // 4:]) if samples else float("nan")
            mhz = statistics.median(s[1] for s in samples[len(samples) // 4:]) if samples else 0
            fl = nets.flops(l, a.batch, True)
            print(json.dumps({"layer": l.name, "op": opn, "math": a.math, "ms": round(ms, 4), "watts": round(pw, 1),
                              "sm_mhz": mhz, "mj_per_call": round(pw * ms, 2),
                              "pj_per_flop": round(pw * ms * 1e9 / fl, 3), "tflops": round(fl / ms / 1e9, 1),
                              "plan": sm.plan_describe(op, dims, m)}), flush=True)


if __name__ == "__main__":
    main()
