"""The network step captured as a CUDA graph with programmatic dependent launch on every kernel -- the
configuration bench.py times below 1024 images per GPU -- computes exactly what the eager step without
PDL computes.

With PDL a kernel may start while its predecessor is still running and must not touch global memory
before `griddepcontrol.wait` (csrc/launch.cuh); a kernel that read its input early, or wrote before its
predecessor's last read, would change the result only under PDL.  Each mode runs in its own process
(the library reads SMCONV_PDL once), on the same seeded inputs; the step is deterministic (fixed plans,
fixed-order reductions, SURVEY.md §8(b) contract 6), so the full flat dW buffer -- which every fwd, dX
and dW call of the chain feeds -- must agree bit for bit.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2305_08819_b200 import build, dp
build.build()
net, batch, math, mode, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
dev = torch.device("cuda", 0)
step = dp.ConvNetStep(net, batch, dev, math=math, seed=1, dw_stream=True)
step.step(None)
torch.cuda.synchronize()
if mode == "graph":
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        step.step(None)
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step.step(None)
    step.dw_flat.fill_(float("nan"))
    g.replay()
    g.replay()
else:
    step.step(None)
torch.cuda.synchronize()
np.save(out, step.dw_flat.cpu().numpy())
""" % ROOT


@pytest.mark.parametrize("net,batch,math", [("vgg16", 128, "3xtf32"), ("vgg16", 128, "tf32"),
                                            ("resnet18", 256, "3xtf32")])
def test_graph_pdl_step_equals_eager(tmp_path, net, batch, math):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = {}
    for mode, pdl in (("eager", "0"), ("graph", "2")):
        out = str(tmp_path / ("%s.npy" % mode))
        env = dict(os.environ, SMCONV_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", SCRIPT, net, str(batch), math, mode, out], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = np.load(out)
    assert np.isfinite(res["graph"]).all()
    assert np.array_equal(res["eager"], res["graph"]), float(np.max(np.abs(res["eager"] - res["graph"])))
