"""Pins for the CPU oracle — checks against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle (a dropped term, a
wrong sign, a wrong index, a transposed operand, a wrong padding/stride rule)
fails at least one of them:

  * golden worked values from SPEC.md (tests/golden/spec_worked_examples.txt);
  * closed forms for all-ones inputs (counting formulas, written independently);
  * 1x1 conv == BLAS matmul (numpy float64);
  * delta kernels == shifts / subsampling;
  * exact finite differences of the bilinear form <conv(X,W),G> (h = 1);
  * the trilinear adjoint identity <O1(X,W),G> = <X,O2(G,W)> = <W,O3(X,G)>;
  * dense-operator transpose on tiny shapes;
  * torch's CPU float64 conv2d / autograd (an independent library routine);
  * integer inputs: exact integer results;
  * padding transparency (IC 3 vs zero-padded 4), floor output size.
"""
import os

import numpy as np
import pytest

from paper_2305_08819_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.txt")

SHAPES = [  # N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw
    (2, 5, 5, 3, 4, 3, 3, 1, 1, 1, 1),      # SPEC.md:112 naive-loop case
    (2, 8, 8, 4, 8, 3, 3, 1, 1, 1, 1),      # BASELINE config 1
    (1, 7, 6, 4, 4, 3, 3, 2, 2, 1, 1),      # stride 2, odd extent
    (2, 8, 8, 4, 8, 1, 1, 2, 2, 0, 0),      # 1x1 s2 shortcut
    (1, 6, 7, 4, 4, 5, 5, 1, 1, 2, 2),      # 5x5 p2 (GoogLeNet)
    (1, 9, 9, 4, 4, 3, 2, 2, 3, 2, 0),      # asymmetric kernel / stride / pad
    (1, 13, 13, 4, 4, 11, 11, 4, 4, 5, 5),  # AlexNet 11x11 s4 p5
    (1, 2, 2, 8, 4, 3, 3, 1, 1, 1, 1),      # 2x2 map (small-map regime)
    (1, 3, 3, 4, 4, 3, 3, 1, 1, 4, 4),      # pad >= FH: outputs from padding only
]


def _rand(shape, g):
    return g.uniform(-1, 1, size=shape).astype(np.float32)


def _inputs(s, seed=0):
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    g = synth.rng(0, seed, salt=1)
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    return (_rand((N, IH, IW, IC), g), _rand((OC, FH, FW, IC), g),
            _rand((N, OH, OW, OC), g), OH, OW)


def _read_golden():
    cases = {}
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, vals = line.split(":")
        op, name, *dims = head.split()
        arr = np.array([float(v) for v in vals.split()], np.float32).reshape([int(d) for d in dims])
        cases.setdefault(op, {})[name] = arr
    return cases


# ---------------------------------------------------------------- golden (SPEC)
def test_golden_spec_worked_examples(oracle_mod):
    c = _read_golden()
    f = c["fwd"]
    np.testing.assert_array_equal(oracle_mod.conv2d_fwd(f["X"], f["W"], (1, 1), (0, 0)), f["Y"])
    d = c["dx"]
    np.testing.assert_array_equal(oracle_mod.conv2d_bwd_data(d["dY"], d["W"], (1, 1), (1, 1), (0, 0)),
                                  d["dX"])
    w = c["dw"]
    np.testing.assert_array_equal(oracle_mod.conv2d_bwd_filter(w["X"], w["dY"], (1, 1), (1, 1), (0, 0)),
                                  w["dW"])


# ---------------------------------------------------------------- shapes (L1)
def test_output_size_floor(oracle_mod):
    assert oracle_mod.out_hw(32, 32, 3, 3, 1, 1, 1, 1) == (32, 32)
    assert oracle_mod.out_hw(32, 32, 3, 3, 2, 2, 1, 1) == (16, 16)   # SPEC.md:584 -> floor
    assert oracle_mod.out_hw(32, 32, 1, 1, 2, 2, 0, 0) == (16, 16)
    assert oracle_mod.out_hw(32, 32, 11, 11, 4, 4, 5, 5) == (8, 8)
    with pytest.raises(ValueError):
        oracle_mod.out_hw(2, 2, 5, 5, 1, 1, 0, 0)                    # OH < 1
    with pytest.raises(ValueError):
        oracle_mod.out_hw(8, 8, 3, 3, 0, 1, 1, 1)                    # stride 0


# ---------------------------------------------------------------- closed forms (P6)
def _cover(I, O, F, s, p):
    """v[o] = #{f : 0 <= o*s-p+f < I}; c[f] = #{o : 0 <= o*s-p+f < I}."""
    v = np.array([sum(1 for f in range(F) if 0 <= o * s - p + f < I) for o in range(O)], np.float64)
    c = np.array([sum(1 for o in range(O) if 0 <= o * s - p + f < I) for f in range(F)], np.float64)
    return v, c


@pytest.mark.parametrize("s", SHAPES)
def test_all_ones_closed_forms(oracle_mod, s):
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    vh, ch = _cover(IH, OH, FH, sh, ph)
    vw, cw = _cover(IW, OW, FW, sw, pw)
    X = np.ones((N, IH, IW, IC), np.float32)
    W = np.ones((OC, FH, FW, IC), np.float32)
    G = np.ones((N, OH, OW, OC), np.float32)
    Y = oracle_mod.conv2d_fwd(X, W, (sh, sw), (ph, pw))
    np.testing.assert_array_equal(Y, np.broadcast_to((IC * vh[:, None] * vw[None, :])[None, :, :, None], Y.shape))
    dW = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw))
    np.testing.assert_array_equal(dW, np.broadcast_to((N * ch[:, None] * cw[None, :])[None, :, :, None], dW.shape))
    dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
    hits_h = np.zeros(IH)
    hits_w = np.zeros(IW)
    for o in range(OH):
        for f in range(FH):
            if 0 <= o * sh - ph + f < IH:
                hits_h[o * sh - ph + f] += 1
    for o in range(OW):
        for f in range(FW):
            if 0 <= o * sw - pw + f < IW:
                hits_w[o * sw - pw + f] += 1
    np.testing.assert_array_equal(dX, np.broadcast_to((OC * hits_h[:, None] * hits_w[None, :])[None, :, :, None], dX.shape))


def test_closed_form_examples(oracle_mod):
    # 3x3 p1 on 8x8 with all ones: corners 4*IC, edges 6*IC, interior 9*IC
    Y = oracle_mod.conv2d_fwd(np.ones((1, 8, 8, 4), np.float32), np.ones((1, 3, 3, 4), np.float32))
    assert Y[0, 0, 0, 0] == 16 and Y[0, 0, 3, 0] == 24 and Y[0, 4, 4, 0] == 36
    # 1x1 s2 dX: OC at even positions, 0 at odd (every other row/col uncovered, reading L5)
    dX = oracle_mod.conv2d_bwd_data(np.ones((1, 4, 4, 8), np.float32), np.ones((8, 1, 1, 4), np.float32),
                                    (8, 8), (2, 2), (0, 0))
    assert dX[0, 0, 0, 0] == 8 and dX[0, 1, 0, 0] == 0 and dX[0, 0, 1, 0] == 0 and dX[0, 6, 6, 3] == 8
    # zero inputs -> zero outputs
    assert not oracle_mod.conv2d_bwd_data(np.zeros((1, 8, 8, 8), np.float32),
                                          np.ones((8, 3, 3, 4), np.float32), (8, 8)).any()
    assert not oracle_mod.conv2d_bwd_filter(np.ones((1, 8, 8, 4), np.float32),
                                            np.zeros((1, 8, 8, 8), np.float32), (3, 3)).any()


# ---------------------------------------------------------------- 1x1 = matmul (P3)
def test_1x1_is_matmul(oracle_mod):
    g = synth.rng(0, 0, salt=2)
    X = _rand((3, 5, 4, 12), g)
    W = _rand((8, 1, 1, 12), g)
    Y = oracle_mod.conv2d_fwd(X, W, (1, 1), (0, 0))
    ref = X.astype(np.float64).reshape(-1, 12) @ W.astype(np.float64).reshape(8, 12).T
    np.testing.assert_allclose(Y.reshape(-1, 8), ref, rtol=1e-13, atol=1e-13)
    G = _rand((3, 5, 4, 8), g)
    dX = oracle_mod.conv2d_bwd_data(G, W, (5, 4), (1, 1), (0, 0))
    np.testing.assert_allclose(dX.reshape(-1, 12), G.astype(np.float64).reshape(-1, 8) @ W.astype(np.float64).reshape(8, 12),
                               rtol=1e-13, atol=1e-13)
    dW = oracle_mod.conv2d_bwd_filter(X, G, (1, 1), (1, 1), (0, 0))
    np.testing.assert_allclose(dW.reshape(8, 12), G.astype(np.float64).reshape(-1, 8).T @ X.astype(np.float64).reshape(-1, 12),
                               rtol=1e-12, atol=1e-12)
    # FH=IH, FW=IW, p0: a fully-connected layer
    Xf = _rand((6, 3, 3, 8), g)
    Wf = _rand((4, 3, 3, 8), g)
    Yf = oracle_mod.conv2d_fwd(Xf, Wf, (1, 1), (0, 0))
    np.testing.assert_allclose(Yf.reshape(6, 4), Xf.astype(np.float64).reshape(6, -1) @ Wf.astype(np.float64).reshape(4, -1).T,
                               rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- delta kernels (P4)
@pytest.mark.parametrize("s", [(1, 1, 1, 1), (2, 2, 1, 1), (1, 1, 0, 0), (2, 2, 0, 0), (1, 2, 2, 0)])
def test_delta_kernel_is_shift(oracle_mod, s):
    sh, sw, ph, pw = s
    g = synth.rng(0, 0, salt=3)
    N, IH, IW, C, FH, FW = 2, 7, 6, 4, 3, 3
    X = _rand((N, IH, IW, C), g)
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    for a in range(FH):
        for b in range(FW):
            W = np.zeros((C, FH, FW, C), np.float32)
            for c in range(C):
                W[c, a, b, c] = 1.0
            Y = oracle_mod.conv2d_fwd(X, W, (sh, sw), (ph, pw))
            exp = np.zeros((N, OH, OW, C))
            for oh in range(OH):
                for ow in range(OW):
                    ih, iw = oh * sh - ph + a, ow * sw - pw + b
                    if 0 <= ih < IH and 0 <= iw < IW:
                        exp[:, oh, ow, :] = X[:, ih, iw, :]
            np.testing.assert_array_equal(Y, exp)
            # dX of a delta kernel is the adjoint scatter of dY
            G = _rand((N, OH, OW, C), g)
            dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
            expx = np.zeros((N, IH, IW, C))
            for oh in range(OH):
                for ow in range(OW):
                    ih, iw = oh * sh - ph + a, ow * sw - pw + b
                    if 0 <= ih < IH and 0 <= iw < IW:
                        expx[:, ih, iw, :] += G[:, oh, ow, :]
            np.testing.assert_array_equal(dX, expx)


# ---------------------------------------------------------------- adjoint identity (P2)
@pytest.mark.parametrize("s", SHAPES)
def test_trilinear_adjoint_identity(oracle_mod, s):
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    X, W, G, OH, OW = _inputs(s, 5)
    Y = oracle_mod.conv2d_fwd(X, W, (sh, sw), (ph, pw))
    dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
    dW = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw))
    a = float(np.sum(Y * G.astype(np.float64)))
    b = float(np.sum(X.astype(np.float64) * dX))
    c = float(np.sum(W.astype(np.float64) * dW))
    scale = float(np.sum(np.abs(Y) * np.abs(G))) + 1e-300
    assert abs(a - b) <= 1e-12 * scale and abs(a - c) <= 1e-12 * scale


# ---------------------------------------------------------------- dense operator transpose (P1)
@pytest.mark.parametrize("s", [(1, 4, 4, 4, 4, 3, 3, 1, 1, 1, 1), (1, 5, 4, 4, 4, 3, 3, 2, 2, 1, 1),
                               (1, 4, 4, 4, 4, 1, 1, 2, 2, 0, 0), (1, 3, 3, 4, 4, 3, 3, 1, 1, 2, 2)])
def test_dense_operator_transpose(oracle_mod, s):
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    X, W, G, OH, OW = _inputs(s, 6)
    nx = N * IH * IW * IC
    A = np.zeros((N * OH * OW * OC, nx))
    for j in range(nx):
        e = np.zeros(nx, np.float32)
        e[j] = 1
        A[:, j] = oracle_mod.conv2d_fwd(e.reshape(X.shape), W, (sh, sw), (ph, pw)).ravel()
    dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
    np.testing.assert_allclose(dX.ravel(), A.T @ G.astype(np.float64).ravel(), rtol=1e-12, atol=1e-12)
    nw = W.size
    B = np.zeros((N * OH * OW * OC, nw))
    for j in range(nw):
        e = np.zeros(nw, np.float32)
        e[j] = 1
        B[:, j] = oracle_mod.conv2d_fwd(X, e.reshape(W.shape), (sh, sw), (ph, pw)).ravel()
    dW = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw))
    np.testing.assert_allclose(dW.ravel(), B.T @ G.astype(np.float64).ravel(), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- finite differences (P5)
def test_finite_differences_exact_for_bilinear(oracle_mod):
    s = (1, 5, 5, 4, 4, 3, 3, 2, 2, 1, 1)
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    X, W, G, OH, OW = _inputs(s, 7)
    Gd = G.astype(np.float64)

    def L(Xa, Wa):
        return float(np.sum(oracle_mod.conv2d_fwd(Xa, Wa, (sh, sw), (ph, pw)) * Gd))
    dW = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw))
    dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
    g = synth.rng(0, 0, salt=4)
    for j in g.choice(W.size, 12, replace=False):
        E = np.zeros(W.size, np.float32)
        E[j] = 1.0
        E = E.reshape(W.shape)
        fd = (L(X, W + E) - L(X, W - E)) / 2.0
        assert abs(fd - dW.ravel()[j]) <= 1e-6 * (1 + abs(fd))
    for j in g.choice(X.size, 12, replace=False):
        E = np.zeros(X.size, np.float32)
        E[j] = 1.0
        E = E.reshape(X.shape)
        fd = (L(X + E, W) - L(X - E, W)) / 2.0
        assert abs(fd - dX.ravel()[j]) <= 1e-6 * (1 + abs(fd))


# ---------------------------------------------------------------- torch float64 (library routine)
@pytest.mark.parametrize("s", SHAPES)
def test_against_torch_float64(oracle_mod, s):
    import torch
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    X, W, G, OH, OW = _inputs(s, 8)
    xt = torch.from_numpy(X).double().permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    wt = torch.from_numpy(W).double().permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    yt = torch.nn.functional.conv2d(xt, wt, stride=(sh, sw), padding=(ph, pw))
    gt = torch.from_numpy(G).double().permute(0, 3, 1, 2)
    yt.backward(gt)
    Y = oracle_mod.conv2d_fwd(X, W, (sh, sw), (ph, pw))
    np.testing.assert_allclose(Y, yt.detach().permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)
    dX = oracle_mod.conv2d_bwd_data(G, W, (IH, IW), (sh, sw), (ph, pw))
    np.testing.assert_allclose(dX, xt.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)
    dW = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw))
    np.testing.assert_allclose(dW, wt.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- integer mode (P7)
def test_integer_inputs_exact(oracle_mod):
    s = (2, 6, 6, 8, 4, 3, 3, 1, 1, 1, 1)
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    g = synth.rng(0, 0, salt=5)
    X = synth.activations(g, N, IH, IW, IC, integer=2)
    W = synth.filters(g, OC, FH, FW, IC, integer=2)
    Y = oracle_mod.conv2d_fwd(X, W)
    assert np.all(Y == np.round(Y))
    # int64 im2col brute force (tiny)
    Xp = np.pad(X.astype(np.int64), ((0, 0), (1, 1), (1, 1), (0, 0)))
    exp = np.zeros((N, IH, IW, OC), np.int64)
    for fh in range(3):
        for fw in range(3):
            exp += np.einsum("nhwc,oc->nhwo", Xp[:, fh:fh + IH, fw:fw + IW, :], W[:, fh, fw, :].astype(np.int64))
    np.testing.assert_array_equal(Y, exp)


# ---------------------------------------------------------------- padding transparency (P8, L7)
def test_padding_transparency(oracle_mod):
    g = synth.rng(0, 0, salt=6)
    X3 = _rand((2, 6, 6, 3), g)
    W3 = _rand((8, 3, 3, 3), g)
    G = _rand((2, 6, 6, 8), g)
    X4 = np.concatenate([X3, np.zeros((2, 6, 6, 1), np.float32)], -1)
    W4 = np.concatenate([W3, np.zeros((8, 3, 3, 1), np.float32)], -1)
    np.testing.assert_array_equal(oracle_mod.conv2d_fwd(X3, W3), oracle_mod.conv2d_fwd(X4, W4))
    dX4 = oracle_mod.conv2d_bwd_data(G, W4, (6, 6))
    np.testing.assert_array_equal(dX4[..., :3], oracle_mod.conv2d_bwd_data(G, W3, (6, 6)))
    assert not dX4[..., 3].any()
    dW4 = oracle_mod.conv2d_bwd_filter(X4, G, (3, 3))
    np.testing.assert_array_equal(dW4[..., :3], oracle_mod.conv2d_bwd_filter(X3, G, (3, 3)))
    assert not dW4[..., 3].any()


def test_thread_count_independent(oracle_mod):
    s = (2, 8, 8, 8, 8, 3, 3, 1, 1, 1, 1)
    X, W, G, OH, OW = _inputs(s, 9)
    n0 = oracle_mod.num_threads()
    a = oracle_mod.conv2d_bwd_filter(X, G, (3, 3))
    oracle_mod.set_num_threads(1)
    b = oracle_mod.conv2d_bwd_filter(X, G, (3, 3))
    oracle_mod.set_num_threads(n0)
    np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- sampled O3 (full-size GPU parity helper)
@pytest.mark.parametrize("s", SHAPES)
def test_bwd_filter_at_matches_full_and_torch(oracle_mod, s):
    """conv2d_bwd_filter_at (O3 at chosen entries, used for full-batch sampled parity) equals the
    pinned full O3 bit for bit, and torch's float64 weight gradient (independent routine)."""
    import torch
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    X, W, G, OH, OW = _inputs(s, 10)
    full = oracle_mod.conv2d_bwd_filter(X, G, (FH, FW), (sh, sw), (ph, pw)).ravel()
    g = np.random.default_rng(11)
    idx = np.concatenate([[0, full.size - 1], g.choice(full.size, min(20, full.size), replace=False)])
    got = oracle_mod.conv2d_bwd_filter_at(X, G, (FH, FW), idx, (sh, sw), (ph, pw))
    np.testing.assert_array_equal(got, full[idx])
    xt = torch.from_numpy(X).double().permute(0, 3, 1, 2)
    wt = torch.from_numpy(W).double().permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    yt = torch.nn.functional.conv2d(xt, wt, stride=(sh, sw), padding=(ph, pw))
    yt.backward(torch.from_numpy(G).double().permute(0, 3, 1, 2))
    ref = wt.grad.permute(0, 2, 3, 1).numpy().ravel()[idx]
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    with pytest.raises(ValueError):
        oracle_mod.conv2d_bwd_filter_at(X, G, (FH, FW), [full.size], (sh, sw), (ph, pw))
