"""Parity at each BASELINE config's OWN bench batch, through the same C-ABI calls and hence the same
plans ``bench.py --net <net>`` times (the plan is a pure function of the conv tuple and math; the
library caches it):

  * config 2, VGG-16 b128: WHOLE tensors of fwd, dX and dW against the oracle, random inputs in both
    math modes and integer inputs bit-exact (pin P7) -- the oracle finishes the whole net in seconds;
  * config 4, AlexNet b256: whole tensors likewise;
  * config 4, GoogLeNet b256 and config 3, ResNet-18 b512: fwd / dX on whole sampled images (per-image
    independent ops, so a one-image oracle run is exact), dW on sampled entries summed over the FULL
    batch (``oracle.conv2d_bwd_filter_at``; dW parity always uses the full batch);
    integer inputs bit-exact on the same samples.

Every comparison appends its normwise error (reading L8) to the session's parity log
(``gpurun_out/parity_errors.json``) with the plan that produced it.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 5e-3}
CONFIGS = {"vgg16": 128, "alexnet": 256, "googlenet": 256, "resnet18": 512}
WHOLE = {"vgg16", "alexnet"}


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2305_08819_b200 import build
    build.build()
    from paper_2305_08819_b200 import smconv as sm
    return torch, oracle, sm


def _layers():
    from paper_2305_08819_b200 import nets
    return [(net, i, l) for net in CONFIGS for i, l in enumerate(nets.NETS[net]())]


def _nw(got, ref):
    den = float(np.max(np.abs(ref)))
    return float(np.max(np.abs(got.astype(np.float64) - ref))) / den if den > 0 else float(np.max(np.abs(got)))


def _int_lim(l, N):
    kmax = max(l.FH * l.FW * l.IC, l.FH * l.FW * l.OC, N * l.OH * l.OW)
    return 2 if kmax * 4 < 2 ** 23 else 1


@pytest.mark.parametrize("nil", _layers(), ids=lambda t: "%s-%s" % (t[0], t[2].name))
def test_config_layer_at_bench_batch(env, nil, parity_log):
    torch, oracle, sm = env
    from paper_2305_08819_b200 import synth
    net, i, l = nil
    N = CONFIGS[net]
    dims = l.dims(N)
    st, pd = (l.sh, l.sw), (l.ph, l.pw)
    stem = l.ic_logical < 4
    for integer in (0, _int_lim(l, N)):
        g = synth.rng(20 + list(CONFIGS).index(net), i, salt=integer)
        X = synth.activations(g, N, l.IH, l.IW, l.IC, l.ic_logical, stem=stem, integer=integer)
        W = synth.filters(g, l.OC, l.FH, l.FW, l.IC, l.ic_logical, integer=integer)
        dY = synth.activations(g, N, l.OH, l.OW, l.OC, integer=integer)
        x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
        whole = net in WHOLE
        samples = list(range(N)) if whole else [0, N // 2 + 3, N - 1]
        if whole:
            ref = {"fwd": oracle.conv2d_fwd(X, W, st, pd),
                   "dx": oracle.conv2d_bwd_data(dY, W, (l.IH, l.IW), st, pd) if i > 0 else None,
                   "dw": oracle.conv2d_bwd_filter(X, dY, (l.FH, l.FW), st, pd)}
        else:
            ref = {"fwd": np.concatenate([oracle.conv2d_fwd(X[n:n + 1], W, st, pd) for n in samples]),
                   "dx": np.concatenate([oracle.conv2d_bwd_data(dY[n:n + 1], W, (l.IH, l.IW), st, pd)
                                         for n in samples]) if i > 0 else None}
            rng = np.random.default_rng(1000 + i)
            nwt = l.OC * l.FH * l.FW * l.IC
            idx = np.unique(np.concatenate([[0, nwt - 1], rng.choice(nwt, min(nwt, 254), replace=False)]))
            ref["dw"] = oracle.conv2d_bwd_filter_at(X, dY, (l.FH, l.FW), idx, st, pd)
        for math in ("3xtf32", "tf32"):
            m = sm.MATH[math]
            got = {"fwd": sm.conv2d_fwd(x, w, st, pd, math=math),
                   "dx": sm.conv2d_bwd_data(dy, w, (l.IH, l.IW), st, pd, math=math) if i > 0 else None,
                   "dw": sm.conv2d_bwd_filter(x, dy, (l.FH, l.FW), st, pd, math=math)}
            torch.cuda.synchronize()
            for op, opi in (("fwd", 0), ("dx", 1), ("dw", 2)):
                if got[op] is None:
                    continue
                if op == "dw" and not whole:
                    gv = got[op].reshape(-1)[torch.from_numpy(idx).cuda()].double().cpu().numpy()
                    scale = float(got[op].abs().max())
                    e = float(np.max(np.abs(gv - ref[op]))) / scale if scale > 0 else 0.0
                    exact = np.array_equal(gv, ref[op])
                else:
                    gv = got[op].cpu().numpy()
                    if not whole:
                        gv = gv[samples]
                    e = _nw(gv, ref[op])
                    exact = np.array_equal(gv.astype(np.float64), ref[op])
                parity_log.append({"config": "%s-b%d" % (net, N), "layer": l.name, "op": op, "math": math,
                                   "check": "integer" if integer else "random",
                                   "coverage": "whole tensor" if whole else (
                                       "%d whole images" % len(samples) if op != "dw"
                                       else "%d dW entries over the full batch" % len(idx)),
                                   "normwise": e, "tol": 0.0 if integer else TOL[math],
                                   "plan": sm.plan_describe(opi, dims, m)})
                if integer:
                    assert exact, (net, l.name, op, math, e)
                else:
                    assert e <= TOL[math], (net, l.name, op, math, e)
