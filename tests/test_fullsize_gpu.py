"""Full-size GPU parity: every ResNet-18 conv at the benchmark's batch (BASELINE config 5, 4096 images
on one GPU), through the same C-ABI calls and the same plans ``bench.py`` times, checked against the
oracle on outputs it can afford:

  * fwd / dX are per-image independent: whole images sampled from the batch (first, middle, last) are
    recomputed by the oracle on that image alone -- exact, not an approximation;
  * dW sums over all 4096 images: sampled entries are recomputed by ``oracle.conv2d_bwd_filter_at``
    over the FULL batch (dW parity always uses the full batch);
  * a property that holds at any size: the trilinear adjoint identity
    <fwd(X, W), dY> = <X, dX(dY, W)> = <W, dW(X, dY)> from the GPU outputs (fp64 dot products).

The same checks run on the large-map regime ("input-feature-size
>= 128 x 128"): the CIFAR ResNet-18 on 128 x 128 inputs at batch 64 and 224 x 224 at batch 16
(nets.NETS["resnet18@128"], ["resnet18@224"]; bench.py --net resnet18@128).

Tolerances: north_star / DESIGN.md reading L8 -- normwise max|g - r| / max|r|: 3xTF32 1e-5, TF32 5e-3
(per sampled image; for dW samples relative to max|dW| of the GPU tensor).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B = 4096
TOL = {"3xtf32": 1e-5, "tf32": 5e-3}
ADJ_TOL = {"3xtf32": 1e-6, "tf32": 1e-3}


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2305_08819_b200 import build
    build.build()
    from paper_2305_08819_b200 import nets
    from paper_2305_08819_b200 import smconv as sm
    return torch, oracle, sm, nets


CONFIGS = [("resnet18", B), ("resnet18@128", 64), ("resnet18@224", 16)]


def _layers():
    from paper_2305_08819_b200 import nets
    return [(net, nb, i, l) for net, nb in CONFIGS for i, l in enumerate(nets.NETS[net]())]


def _nw(got, ref):
    den = float(np.max(np.abs(ref)))
    return float(np.max(np.abs(got.astype(np.float64) - ref))) / den if den > 0 else 0.0


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("il", _layers(), ids=lambda il: "%s-%s" % (il[0], il[3].name))
def test_resnet18_layer_full_batch(env, il, math, parity_log):
    torch, oracle, sm, nets = env
    net, B, i, l = il
    from paper_2305_08819_b200 import synth
    dev = torch.device("cuda")
    X, W, dY = synth.torch_layer_inputs(l, B, dev, seed=5000 + i)
    st, pd = (l.sh, l.sw), (l.ph, l.pw)
    y = sm.conv2d_fwd(X, W, st, pd, math=math)
    dx = sm.conv2d_bwd_data(dY, W, (l.IH, l.IW), st, pd, math=math) if i > 0 else None  # bench skips stem dX
    dw = sm.conv2d_bwd_filter(X, dY, (l.FH, l.FW), st, pd, math=math)
    torch.cuda.synchronize()
    Wh = W.cpu().numpy()

    m = sm.MATH[math]

    def log(op, e, cov):
        parity_log.append({"config": "%s-b%d" % (net, B), "layer": l.name, "op": op, "math": math,
                           "check": "random", "coverage": cov, "normwise": e, "tol": TOL[math],
                           "plan": sm.plan_describe({"fwd": 0, "dx": 1, "dw": 2}[op], l.dims(B), m)})

    # fwd / dX on whole sampled images
    ef, ed = 0.0, 0.0
    for n in (0, B // 2 + 7, B - 1):
        ref = oracle.conv2d_fwd(X[n:n + 1].cpu().numpy(), Wh, st, pd)
        e = _nw(y[n:n + 1].cpu().numpy(), ref)
        ef = max(ef, e)
        assert e <= TOL[math], ("fwd", n, e)
        if dx is not None:
            ref = oracle.conv2d_bwd_data(dY[n:n + 1].cpu().numpy(), Wh, (l.IH, l.IW), st, pd)
            e = _nw(dx[n:n + 1].cpu().numpy(), ref)
            ed = max(ed, e)
            assert e <= TOL[math], ("dx", n, e)
    log("fwd", ef, "3 whole images")
    if dx is not None:
        log("dx", ed, "3 whole images")

    # dW entries over the full batch
    g = np.random.default_rng(77 + i)
    idx = np.concatenate([[0, dw.numel() - 1], g.choice(dw.numel(), 14, replace=False)])
    ref = oracle.conv2d_bwd_filter_at(X.cpu().numpy(), dY.cpu().numpy(), (l.FH, l.FW), idx, st, pd)
    got = dw.reshape(-1)[torch.from_numpy(idx).to(dev)].double().cpu().numpy()
    scale = float(dw.abs().max())
    e = float(np.max(np.abs(got - ref))) / scale
    log("dw", e, "%d dW entries over the full batch" % len(idx))
    assert e <= TOL[math], ("dw", e)

    # adjoint identity over the whole tensors (fp64 reductions on the device); the scale is the
    # absolute-value sum, which bounds the effect of a relative error in either operand
    a = float((y.double() * dY.double()).sum())
    sa = float((y.double().abs() * dY.double().abs()).sum())
    c = float((W.double() * dw.double()).sum())
    assert abs(a - c) <= ADJ_TOL[math] * sa, (a, c, sa)
    if dx is not None:
        b = float((X.double() * dx.double()).sum())
        assert abs(a - b) <= ADJ_TOL[math] * sa, (a, b, sa)
