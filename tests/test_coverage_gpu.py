"""Every output element is written, by every plan the networks use.

The conv ops overwrite their outputs (reading L6, include/smconv.h contract 2): dX positions
no tap reaches are written as 0 (reading L5; O2).  Several plans write an output
element from somewhere other than a plain per-row store -- the row-coalesced epilogue (a lane stores
other lanes' rows), the in-epilogue zero phases of the 1x1 stride-2 dX (`zfill`), the
super-pixel dX scatter, the in-cluster split-K reduction, the split-K reduce kernel.  A missed element
would keep whatever the caller's buffer held, which a freshly allocated (often zero) buffer can hide.
Here the output buffer is poisoned with NaN before the call: the result must be finite and bitwise
equal to the result written over a zero-filled buffer (every element written, nothing read from it).
No oracle: the values themselves are checked against the oracle in test_parity_gpu / test_configs_gpu.
"""
import pytest

pytestmark = pytest.mark.gpu

# (net, batch): the bench batches where they fit the test budget; batch 256 keeps the 3xTF32 CTA-pair
# plans (N % 256) and the 1x1 stride-2 zfill plans of ResNet-18
CASES = [("resnet18", 256), ("vgg16", 128), ("googlenet", 64), ("alexnet", 64), ("resnet18", 40)]


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_08819_b200 import build
    build.build()
    from paper_2305_08819_b200 import smconv as sm
    return torch, sm


def _cases():
    from paper_2305_08819_b200 import nets
    out = []
    for net, N in CASES:
        for i, l in enumerate(nets.NETS[net]()):
            out.append((net, N, i, l))
    return out


@pytest.mark.parametrize("nil", _cases(), ids=lambda c: "%s-b%d-%s" % (c[0], c[1], c[3].name))
def test_every_output_element_written(env, nil):
    torch, sm = env
    from paper_2305_08819_b200 import synth
    net, N, i, l = nil
    st, pd = (l.sh, l.sw), (l.ph, l.pw)
    g = synth.rng(77, i)
    x = torch.from_numpy(synth.activations(g, N, l.IH, l.IW, l.IC, l.ic_logical, stem=l.ic_logical < 4)).cuda()
    w = torch.from_numpy(synth.filters(g, l.OC, l.FH, l.FW, l.IC, l.ic_logical)).cuda()
    dy = torch.from_numpy(synth.activations(g, N, l.OH, l.OW, l.OC)).cuda()
    for math in ("3xtf32", "tf32"):
        calls = [("fwd", lambda o: sm.conv2d_fwd(x, w, st, pd, math=math, out=o), (N, l.OH, l.OW, l.OC)),
                 ("dw", lambda o: sm.conv2d_bwd_filter(x, dy, (l.FH, l.FW), st, pd, math=math, out=o),
                  (l.OC, l.FH, l.FW, l.IC))]
        if i > 0:
            calls.append(("dx", lambda o: sm.conv2d_bwd_data(dy, w, (l.IH, l.IW), st, pd, math=math, out=o),
                          (N, l.IH, l.IW, l.IC)))
        for op, f, shape in calls:
            poisoned = torch.full(shape, float("nan"), device="cuda")
            zeroed = torch.zeros(shape, device="cuda")
            f(poisoned)
            f(zeroed)
            torch.cuda.synchronize()
            opi = {"fwd": 0, "dx": 1, "dw": 2}[op]
            plan = sm.plan_describe(opi, l.dims(N), sm.MATH[math])
            assert bool(torch.isfinite(poisoned).all()), (op, math, plan, int((~torch.isfinite(poisoned)).sum()))
            assert torch.equal(poisoned, zeroed), (op, math, plan)
