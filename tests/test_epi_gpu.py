"""GPU parity of the fused conv epilogues (include/smconv_epi.h) against the oracle:
oracle conv (O1 / O2) followed by the oracle's BatchNorm statistics, LeakyReLU and LeakyReLU-backward
statistics (oracle/net_oracle.c, pinned in tests/test_oracle_pins_net.py).

Shapes cover every plan form: fused in the STRIP and TMA epilogues (incl. CTA pairs, the stride-2 dX
with tap-less phases, the super-pixel stride-2 dX whose 4 IC-wide column groups fold onto IC), and the
pass form after in-cluster split-K, GENERIC and DIRECT.  Checks:
  * Y / G: normwise error (reading L8) within the math mode's bar, as the plain ops;
  * S1, S2 against the oracle's statistics of the ORACLE outputs, per channel relative to the sum of
    the absolute terms (the condition of a sum: |dS_c| <= tol * sum_r |term_rc|);
  * S1, S2 against the oracle's statistics of the GPU's OWN outputs at 1e-6 (the reduction alone);
  * integer inputs ({-1,0,1}, k = 1/4): Y, G, S1, S2 bit-exact (every partial sum is an exact integer
    or quarter in fp32);
  * in place (G written over A) equals out of place; repeated calls are bitwise identical.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 5e-3}

# (name, N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw)
SHAPES = [
    ("strip-64", 64, 16, 16, 64, 64, 3, 3, 1, 1, 1, 1),
    ("tma-8x8", 128, 8, 8, 128, 256, 3, 3, 1, 1, 1, 1),
    ("tma-pair", 256, 8, 8, 128, 128, 3, 3, 1, 1, 1, 1),
    ("csk-2x2", 128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),
    ("s2-3x3", 64, 16, 16, 64, 128, 3, 3, 2, 2, 1, 1),
    ("s2dx-32", 64, 32, 32, 64, 128, 3, 3, 2, 2, 1, 1),
    ("sc-1x1s2", 128, 16, 16, 64, 128, 1, 1, 2, 2, 0, 0),
    ("stem", 32, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1),
    ("generic", 8, 8, 8, 48, 112, 3, 3, 1, 1, 1, 1),
    ("ragged", 40, 7, 7, 32, 96, 3, 3, 1, 1, 1, 1),
]


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2305_08819_b200 import build
    build.build()
    oracle.build()
    from paper_2305_08819_b200 import smconv as sm
    return torch, oracle, sm


def _nw(got, ref):
    den = float(np.max(np.abs(ref)))
    return float(np.max(np.abs(got.astype(np.float64) - ref))) / (den if den > 0 else 1.0)


def _cond_err(got, ref, absum):
    return float(np.max(np.abs(got - ref) / np.maximum(absum, 1e-300)))


def _inputs(s, integer, seed):
    from paper_2305_08819_b200 import synth
    _, N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    g = synth.rng(40, seed)
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    X = synth.activations(g, N, IH, IW, IC, integer=integer)
    W = synth.filters(g, OC, FH, FW, IC, integer=integer)
    dY = synth.activations(g, N, OH, OW, OC, integer=integer)
    # the activation A = leakyRelu(Z) the dX output is the gradient of (signs mixed, zeros in integer mode)
    A = synth.activations(g, N, IH, IW, IC, integer=integer)
    return X, W, dY, A


def _log(parity_log, s, op, math, check, err, tol, plan):
    parity_log.append({"config": "epi", "layer": s[0], "op": op, "math": math, "check": check, "normwise": err,
                       "tol": tol, "coverage": "whole tensor", "plan": plan})


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("s", SHAPES, ids=lambda s: s[0])
def test_fwd_bn_stats_and_leaky(env, s, math, parity_log):
    torch, oracle, sm = env
    X, W, dY, A = _inputs(s, 0, 1)
    st, pd = (s[8], s[9]), (s[10], s[11])
    dims = tuple(s[1:])
    x, w = (torch.from_numpy(a).cuda() for a in (X, W))
    y, stats = sm.conv2d_fwd_epi(x, w, st, pd, math=math, epi="bn_stats")
    y2, stats2 = sm.conv2d_fwd_epi(x, w, st, pd, math=math, epi="bn_stats")
    yl, _ = sm.conv2d_fwd_epi(x, w, st, pd, math=math, epi="leaky", k=0.1)
    torch.cuda.synchronize()
    Y = y.cpu().numpy()
    S = stats.cpu().numpy()
    assert np.array_equal(S, stats2.cpu().numpy()) and np.array_equal(Y, y2.cpu().numpy()), "not deterministic"
    ref = oracle.conv2d_fwd(X, W, st, pd)
    plan = sm.epi_plan_describe(0, dims, math, "bn_stats")
    e = _nw(Y, ref)
    _log(parity_log, s, "fwd+bn_stats:y", math, "random", e, TOL[math], plan)
    assert e <= TOL[math], (e, plan)
    r1, r2 = oracle.channel_stats(ref)
    a1, _ = oracle.channel_stats(np.abs(ref))
    e1, e2 = _cond_err(S[0], r1, a1), _cond_err(S[1], r2, r2)
    _log(parity_log, s, "fwd+bn_stats:s1", math, "random", e1, TOL[math], plan)
    _log(parity_log, s, "fwd+bn_stats:s2", math, "random", e2, TOL[math], plan)
    assert e1 <= TOL[math] and e2 <= TOL[math], (e1, e2, plan)
    o1, o2 = oracle.channel_stats(Y.astype(np.float64))  # the reduction alone, on the GPU's own Y
    oa, _ = oracle.channel_stats(np.abs(Y.astype(np.float64)))
    assert _cond_err(S[0], o1, oa) <= 1e-6 and _cond_err(S[1], o2, o2) <= 1e-6, plan
    el = _nw(yl.cpu().numpy(), oracle.leaky_relu(ref, 0.1))
    _log(parity_log, s, "fwd+leaky", math, "random", el, TOL[math], sm.epi_plan_describe(0, dims, math, "leaky"))
    assert el <= TOL[math]


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("s", SHAPES, ids=lambda s: s[0])
def test_dx_leaky_bwd_stats(env, s, math, parity_log):
    torch, oracle, sm = env
    X, W, dY, A = _inputs(s, 0, 2)
    st, pd = (s[8], s[9]), (s[10], s[11])
    dims = tuple(s[1:])
    IH, IW = s[2], s[3]
    k = 0.05
    dy, w, a = (torch.from_numpy(v).cuda() for v in (dY, W, A))
    g, stats = sm.conv2d_bwd_data_epi(dy, w, a, (IH, IW), st, pd, math=math, epi="leaky_bwd_stats", k=k)
    g2, _ = sm.conv2d_bwd_data_epi(dy, w, a, (IH, IW), st, pd, math=math, epi="leaky_bwd", k=k)
    a_inplace = a.clone()
    g3, stats3 = sm.conv2d_bwd_data_epi(dy, w, a_inplace, (IH, IW), st, pd, math=math, epi="leaky_bwd_stats", k=k,
                                        out=a_inplace)
    torch.cuda.synchronize()
    G = g.cpu().numpy()
    S = stats.cpu().numpy()
    assert np.array_equal(G, g2.cpu().numpy()), "leaky_bwd and leaky_bwd_stats give different G"
    assert np.array_equal(G, g3.cpu().numpy()) and np.array_equal(S, stats3.cpu().numpy()), "in-place differs"
    dref = oracle.conv2d_bwd_data(dY, W, (IH, IW), st, pd)
    Gr, r1, r2 = oracle.leaky_bwd_stats(dref, A, k)
    plan = sm.epi_plan_describe(1, dims, math, "leaky_bwd_stats")
    e = _nw(G, Gr)
    _log(parity_log, s, "dx+leaky_bwd:g", math, "random", e, TOL[math], plan)
    assert e <= TOL[math], (e, plan)
    z = np.where(A > 0, A.astype(np.float64), A.astype(np.float64) / k)
    a1, _ = oracle.channel_stats(np.abs(Gr))
    a2, _ = oracle.channel_stats(np.abs(Gr * z))
    e1, e2 = _cond_err(S[0], r1, a1), _cond_err(S[1], r2, a2)
    _log(parity_log, s, "dx+leaky_bwd:s1", math, "random", e1, TOL[math], plan)
    _log(parity_log, s, "dx+leaky_bwd:s2", math, "random", e2, TOL[math], plan)
    assert e1 <= TOL[math] and e2 <= TOL[math], (e1, e2, plan)
    Gd = G.astype(np.float64).reshape(-1, s[4])  # the reduction alone, on the GPU's own G
    zd = z.reshape(-1, s[4])
    o1, o2 = Gd.sum(axis=0), (Gd * zd).sum(axis=0)
    oa, ob = np.abs(Gd).sum(axis=0), np.abs(Gd * zd).sum(axis=0)
    assert _cond_err(S[0], o1, oa) <= 1e-6 and _cond_err(S[1], o2, ob) <= 1e-6, plan


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("s", [x for x in SHAPES if x[4] * x[6] * x[7] <= 576 and x[5] * x[6] * x[7] <= 1152],
                         ids=lambda s: s[0])
def test_epi_integer_bit_exact(env, s, math, parity_log):
    """{-1,0,1} inputs with K <= 576 (fwd) / 1152 (dX): y^2 sums of 32 rows stay below 2^24, and with
    k = 1/4 every G and G*z is an exact multiple of 1/4: GPU == oracle bitwise (pin P7 extended)."""
    torch, oracle, sm = env
    X, W, dY, A = _inputs(s, 1, 3)
    st, pd = (s[8], s[9]), (s[10], s[11])
    IH, IW = s[2], s[3]
    k = 0.25
    x, w, dy, a = (torch.from_numpy(v).cuda() for v in (X, W, dY, A))
    y, sy = sm.conv2d_fwd_epi(x, w, st, pd, math=math, epi="bn_stats")
    g, sg = sm.conv2d_bwd_data_epi(dy, w, a, (IH, IW), st, pd, math=math, epi="leaky_bwd_stats", k=k)
    torch.cuda.synchronize()
    ref = oracle.conv2d_fwd(X, W, st, pd)
    r1, r2 = oracle.channel_stats(ref)
    assert np.array_equal(y.cpu().numpy().astype(np.float64), ref)
    assert np.array_equal(sy.cpu().numpy()[0], r1) and np.array_equal(sy.cpu().numpy()[1], r2)
    Gr, q1, q2 = oracle.leaky_bwd_stats(oracle.conv2d_bwd_data(dY, W, (IH, IW), st, pd), A, k)
    assert np.array_equal(g.cpu().numpy().astype(np.float64), Gr)
    assert np.array_equal(sg.cpu().numpy()[0], q1) and np.array_equal(sg.cpu().numpy()[1], q2)
    _log(parity_log, s, "epi", math, "integer", 0.0, 0.0, sm.epi_plan_describe(0, tuple(s[1:]), math, "bn_stats"))


def test_epi_errors(env):
    torch, oracle, sm = env
    x = torch.zeros((32, 8, 8, 32), device="cuda")
    w = torch.zeros((32, 3, 3, 32), device="cuda")
    with pytest.raises(sm.ConvError) as ei:
        sm.conv2d_fwd_epi(x, w, epi="leaky_bwd")
    assert ei.value.code == sm.CONV_EARG
    with pytest.raises(sm.ConvError) as ei:
        sm.conv2d_fwd_epi(x, w, epi="leaky", k=0.0)
    assert ei.value.code == sm.CONV_EARG
    a = torch.zeros((32, 8, 8, 32), device="cuda")
    with pytest.raises(sm.ConvError) as ei:  # A overlapping dY
        sm.conv2d_bwd_data_epi(a, w, a, (8, 8), epi="leaky_bwd")
    assert ei.value.code == sm.CONV_EALIAS
