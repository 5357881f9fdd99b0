#!/usr/bin/env python
"""DWS promotion-chunk experiment: time + error of the l1 dW (3x3 64->64 at 32x32) for the chunk
length set by SMCONV_TMA_CHUNK at load time.  Error: normwise over 64 full-batch dW entries at batch
4096 against the oracle (conv2d_bwd_filter_at), and over the whole dW at batch 64."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this is an experiment checker)
from paper_2305_08819_b200 import nets, synth  # noqa: E402
from paper_2305_08819_b200 import smconv as sm  # noqa: E402

dev = torch.device("cuda")
l = [x for x in nets.resnet18() if x.name == "l1.0a"][0]
out = {"chunk": os.environ.get("SMCONV_TMA_CHUNK", "default")}
for B in (64, 4096):
    X, W, dY = synth.torch_layer_inputs(l, B, dev, seed=123)
    st, pd = (l.sh, l.sw), (l.ph, l.pw)
    dw = sm.conv2d_bwd_filter(X, dY, (l.FH, l.FW), st, pd, math="3xtf32")
    torch.cuda.synchronize()
    if B == 64:
        ref = oracle.conv2d_bwd_filter(X.cpu().numpy(), dY.cpu().numpy(), (l.FH, l.FW), st, pd)
        got = dw.cpu().numpy().astype(np.float64)
        out["err_b64"] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    else:
        g = np.random.default_rng(7)
        idx = g.choice(dw.numel(), 64, replace=False)
        ref = oracle.conv2d_bwd_filter_at(X.cpu().numpy(), dY.cpu().numpy(), (l.FH, l.FW), idx, st, pd)
        got = dw.reshape(-1)[torch.from_numpy(idx).to(dev)].double().cpu().numpy()
        out["err_b4096"] = float(np.max(np.abs(got - ref)) / float(dw.abs().max()))
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sm.conv2d_bwd_filter(X, dY, (l.FH, l.FW), st, pd, math="3xtf32", out=dw) if False else \
                sm.conv2d_bwd_filter(X, dY, (l.FH, l.FW), st, pd, math="3xtf32")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out["ms_b4096"] = statistics.median(ts)
print(json.dumps(out))
