"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (north_star; reading L8 = normwise max relative error
max|g - r| / max|r| per output tensor):  3xTF32 <= 1e-5,  TF32 <= 5e-3.
Integer-valued inputs are exact in TF32 and every partial sum is an integer < 2^24, so
there the GPU must equal the oracle BIT FOR BIT in both modes (pin P7).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 5e-3}


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


def normwise(got, ref):
    den = float(np.max(np.abs(ref)))
    num = float(np.max(np.abs(got.astype(np.float64) - ref)))
    return num / den if den > 0 else num


def dims_of(s):
    return s  # (N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw)


def gen(s, seed, integer=0, stem=False):
    from paper_2305_08819_b200 import synth
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    g = synth.rng(9, seed)
    X = synth.activations(g, N, IH, IW, IC, stem=stem, integer=integer)
    W = synth.filters(g, OC, FH, FW, IC, integer=integer)
    dY = synth.activations(g, N, OH, OW, OC, integer=integer)
    return X, W, dY


def gpu_all(env, s, X, W, dY, math):
    torch, _, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
    y = sm.conv2d_fwd(x, w, (sh, sw), (ph, pw), math=math)
    dx = sm.conv2d_bwd_data(dy, w, (IH, IW), (sh, sw), (ph, pw), math=math)
    dw = sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw), math=math)
    torch.cuda.synchronize()
    return y.cpu().numpy(), dx.cpu().numpy(), dw.cpu().numpy()


def oracle_all(env, s, X, W, dY):
    _, oracle, _ = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    return (oracle.conv2d_fwd(X, W, (sh, sw), (ph, pw)),
            oracle.conv2d_bwd_data(dY, W, (IH, IW), (sh, sw), (ph, pw)),
            oracle.conv2d_bwd_filter(X, dY, (FH, FW), (sh, sw), (ph, pw)))


CONFIG1 = (2, 8, 8, 4, 8, 3, 3, 1, 1, 1, 1)

# small-but-multi-tile versions of every distinct VGG-16 / ResNet-18 shape class + edge cases
SWEEP = [
    CONFIG1,
    (4, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1),      # stem (IC 3->4)
    (2, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),     # vgg2 / r.l1
    (4, 16, 16, 64, 128, 3, 3, 1, 1, 1, 1),    # vgg3
    (4, 16, 16, 128, 128, 3, 3, 1, 1, 1, 1),   # vgg4 / r.l2
    (8, 8, 8, 128, 256, 3, 3, 1, 1, 1, 1),     # vgg5
    (8, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1),     # vgg6/7 / r.l3
    (16, 4, 4, 256, 512, 3, 3, 1, 1, 1, 1),    # vgg8
    (16, 4, 4, 512, 512, 3, 3, 1, 1, 1, 1),    # vgg9/10 / r.l4
    (32, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),    # vgg11-13
    (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),   # vgg11-13 at a batch-folded tile (N % 128 == 0)
    (4, 32, 32, 64, 128, 3, 3, 2, 2, 1, 1),    # r.l2a 3x3 s2
    (4, 32, 32, 64, 128, 1, 1, 2, 2, 0, 0),    # r.l2 shortcut 1x1 s2
    (8, 16, 16, 128, 256, 3, 3, 2, 2, 1, 1),   # r.l3a
    (8, 16, 16, 128, 256, 1, 1, 2, 2, 0, 0),   # r.l3 sc
    (16, 8, 8, 256, 512, 3, 3, 2, 2, 1, 1),    # r.l4a
    (16, 8, 8, 256, 512, 1, 1, 2, 2, 0, 0),    # r.l4 sc
    (3, 7, 9, 20, 36, 3, 3, 1, 1, 1, 1),       # ragged everything, non-32 channels
    (5, 6, 6, 48, 112, 5, 5, 1, 1, 2, 2),      # GoogLeNet-style 5x5 / non-32 channels
    (2, 13, 13, 4, 64, 11, 11, 4, 4, 5, 5),    # AlexNet conv1 11x11 s4
    (1, 3, 3, 8, 8, 3, 3, 1, 1, 4, 4),         # pad >= FH: many outputs only see padding
    (130, 2, 2, 32, 36, 3, 3, 1, 1, 1, 1),     # N = 130: tiles straddle positions
    # channels that are not multiples of 32 on the TMA variant (TMA out-of-bounds fill pads the reduction
    # channels; ragged GEMM-column channels: per-32-block boxes, padded dW columns)
    (32, 7, 9, 20, 36, 3, 3, 1, 1, 1, 1),      # ragged everything, N % 32 == 0
    (64, 6, 6, 48, 112, 5, 5, 1, 1, 2, 2),     # GoogLeNet-style 5x5
    (32, 8, 8, 24, 16, 1, 1, 1, 1, 0, 0),      # 1x1 with 16 / 24 channels (GoogLeNet 5x5 reduce)
    (256, 4, 4, 112, 208, 3, 3, 1, 1, 1, 1),   # CTA pairs with ragged channels
    (32, 8, 8, 144, 48, 3, 3, 2, 2, 1, 1),     # stride-2 phases, ragged channels
    # the 64-channel dW kernel (DWS) on wide maps: 32-column blocks, rows innermost (large-map regime)
    (8, 16, 96, 64, 64, 3, 3, 1, 1, 1, 1),
    (4, 64, 64, 64, 64, 3, 3, 1, 1, 1, 1),
]


def _id(s):
    return "x".join(map(str, s))


def test_probe_tf32_rounding(env):
    """N8: record how tcgen05 converts fp32 operands and rounds its accumulator."""
    _, _, sm = env
    r = sm.probe_tf32()
    u = 2.0 ** -23
    conv = r[0:5]
    print("operand conversion:", [float(v) for v in conv])
    print("accumulate across MMAs (1 + d):", [(float(v) - 1) / u for v in r[16:21]], "ulps")
    print("sum inside one MMA (1 + d):", [(float(v) - 1) / u for v in r[32:37]], "ulps")
    assert np.all(r[49:64] == 0)  # D[0][1..15] must be zero: descriptor / layout sanity
    trunc = [1.0, 1.0, 1 + 2 ** -10, 1.0, -1.0]
    rne = [1.0, 1 + 2 ** -10, 1 + 2 ** -9, 1.0, -(1 + 2 ** -10)]
    rna = [1 + 2 ** -10, 1 + 2 ** -10, 1 + 2 ** -9, 1.0, -(1 + 2 ** -10)]
    assert any(np.array_equal(conv, np.array(m, np.float32)) for m in (trunc, rne, rna)), conv


def test_config1_both_modes(env):
    s = CONFIG1
    X, W, dY = gen(s, 1)
    ref = oracle_all(env, s, X, W, dY)
    for math in ("3xtf32", "tf32"):
        got = gpu_all(env, s, X, W, dY, math)
        for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
            e = normwise(g, r)
            print("config1 %s %s err %.3e" % (math, name, e))
            assert e <= TOL[math], (math, name, e)


@pytest.mark.parametrize("s", SWEEP, ids=_id)
def test_integer_mode_bit_exact(env, s):
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    OH = (IH + 2 * ph - FH) // sh + 1
    OW = (IW + 2 * pw - FW) // sw + 1
    # keep every partial sum an integer < 2^24: |x*w| <= lim^2, K terms
    kmax = max(FH * FW * IC, FH * FW * OC, N * OH * OW)
    lim = 2 if kmax * 4 < 2 ** 23 else 1
    X, W, dY = gen(s, 2, integer=lim)
    ref = oracle_all(env, s, X, W, dY)
    for math in ("3xtf32", "tf32"):
        got = gpu_all(env, s, X, W, dY, math)
        for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
            assert np.array_equal(g.astype(np.float64), r), (math, name, float(np.max(np.abs(g - r))))


@pytest.mark.parametrize("s", SWEEP, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_random_within_tolerance(env, s, math):
    stem = s[3] == 4
    X, W, dY = gen(s, 3, stem=stem)
    if stem:  # logical IC = 3, pad lane zero
        X[..., 3] = 0
        W[..., 3] = 0
    ref = oracle_all(env, s, X, W, dY)
    got = gpu_all(env, s, X, W, dY, math)
    for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
        e = normwise(g, r)
        assert e <= TOL[math], (name, e)
    if stem:  # pad lanes of dX / dW come out exactly zero
        assert not got[1][..., 3].any() and not got[2][..., 3].any()


def test_deterministic(env):
    s = (8, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1)
    X, W, dY = gen(s, 4)
    a = gpu_all(env, s, X, W, dY, "3xtf32")
    b = gpu_all(env, s, X, W, dY, "3xtf32")
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_adjoint_identity_on_gpu_outputs(env):
    """<conv(X,W),G> = <X,deconv(G,W)> = <W,dW(X,G)> from GPU outputs alone (pin P2)."""
    s = (16, 8, 8, 128, 256, 3, 3, 2, 2, 1, 1)
    X, W, dY = gen(s, 5)
    y, dx, dw = gpu_all(env, s, X, W, dY, "3xtf32")
    a = float(np.sum(y.astype(np.float64) * dY))
    b = float(np.sum(X.astype(np.float64) * dx))
    c = float(np.sum(W.astype(np.float64) * dw))
    scale = float(np.sum(np.abs(y.astype(np.float64)) * np.abs(dY)))
    assert abs(a - b) <= 2e-6 * scale and abs(a - c) <= 2e-6 * scale


def test_variants_equivalent(env):
    """SPEC.md:247,843 path equivalence: the generic and TMA variants agree with the oracle on the
    same inputs (when TMA serves the shape)."""
    torch, oracle, sm = env
    for s in [(128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1), (16, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1),
              (16, 8, 8, 256, 512, 3, 3, 2, 2, 1, 1)]:
        X, W, dY = gen(s, 6)
        ref = oracle_all(env, s, X, W, dY)
        for v in (sm.CONV_VARIANT_GENERIC, sm.CONV_VARIANT_TMA):
            for op in (0, 1, 2):
                sm.force_variant(op, v)
            try:
                got = gpu_all(env, s, X, W, dY, "3xtf32")
            except sm.ConvError as e:
                assert e.code == sm.CONV_EUNSUPPORTED
                continue
            finally:
                for op in (0, 1, 2):
                    sm.force_variant(op, sm.CONV_VARIANT_AUTO)
            for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
                assert normwise(g, r) <= 1e-5, (v, name)


def test_dp_shard_sum_equals_full_batch(env):
    """Batch sharding (north_star (e)): sum over shards of dW == full-batch dW, bit-exact on
    integer inputs (what the NCCL all-reduce SUM computes, reading L10)."""
    torch, oracle, sm = env
    s = (64, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1)
    X, W, dY = gen(s, 7, integer=1)
    x, dy = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
    full = sm.conv2d_bwd_filter(x, dy, (3, 3), math="3xtf32")
    for g in (2, 4, 8):
        parts = [sm.conv2d_bwd_filter(x[r * 64 // g:(r + 1) * 64 // g].contiguous(),
                                      dy[r * 64 // g:(r + 1) * 64 // g].contiguous(), (3, 3), math="3xtf32")
                 for r in range(g)]
        tot = parts[0].clone()
        for p in parts[1:]:
            tot += p
        assert torch.equal(tot, full)
    assert np.array_equal(full.cpu().numpy().astype(np.float64), oracle.conv2d_bwd_filter(X, dY, (3, 3)))


def test_errors_on_gpu_call(env):
    torch, _, sm = env
    buf = torch.zeros(4096, device="cuda")
    x = buf[:512].view(2, 8, 8, 4)
    w = torch.zeros((8, 3, 3, 4), device="cuda")
    with pytest.raises(sm.ConvError) as e:
        sm.conv2d_fwd(x, w, (1, 1), (1, 1), out=buf[256:1280].view(2, 8, 8, 8))
    assert e.value.code == sm.CONV_EALIAS


# ---------------------------------------------------------------- TMA variant (N % 32 == 0, channels % 32 == 0)
SWEEP_TMA = [
    (32, 8, 8, 32, 32, 3, 3, 1, 1, 1, 1),      # smallest: one 32-image group per tile position
    (64, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),    # r.l1 / vgg2 class, tiles straddle positions (N % 128 != 0)
    (128, 16, 16, 64, 128, 3, 3, 1, 1, 1, 1),  # vgg3, batch-folded tiles
    (32, 16, 16, 128, 128, 3, 3, 1, 1, 1, 1),
    (32, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1),
    (32, 4, 4, 512, 512, 3, 3, 1, 1, 1, 1),
    (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),   # vgg11-13 at b128
    (96, 2, 2, 256, 96, 3, 3, 1, 1, 1, 1),     # ragged N tiles (96 images), OC 96
    (32, 32, 32, 64, 128, 3, 3, 2, 2, 1, 1),   # r.l2a 3x3 s2
    (32, 32, 32, 64, 128, 1, 1, 2, 2, 0, 0),   # r.l2 sc
    (64, 8, 8, 256, 512, 3, 3, 2, 2, 1, 1),    # r.l4a
    (64, 8, 8, 256, 512, 1, 1, 2, 2, 0, 0),    # r.l4 sc
    (32, 6, 6, 96, 160, 5, 5, 1, 1, 2, 2),     # 5x5 p2, non-power-of-2 channels (multiples of 32)
    (32, 7, 5, 32, 64, 3, 3, 2, 2, 1, 1),      # odd extents, stride 2
    # dW single-tap tiles skip the k-blocks whose source pixel is padding (IC % BN == 0):
    (32, 7, 5, 128, 64, 3, 3, 2, 2, 2, 1),     # stride 2, asymmetric pad: partial row / column ranges
    (64, 3, 3, 128, 32, 3, 3, 1, 1, 2, 2),     # pad 2: some taps in range at few positions only
    # CTA pairs (cta_group::2, M = 256) for fwd / dX in 3xTF32 need N % 256 == 0:
    (256, 6, 6, 128, 128, 3, 3, 1, 1, 1, 1),   # BN 128 pairs
    (256, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1),     # BN 64 pairs (32-column B halves)
    (256, 8, 8, 64, 128, 3, 3, 2, 2, 1, 1),    # stride-2 dX: 4 phases of pair tiles
    (512, 3, 3, 96, 160, 3, 3, 1, 1, 1, 1),    # 2 pair image blocks, ragged N tile (160 = 128 + 32)
    # dW pairs (3xTF32, OC % 256 == 0, BN 128: two 128-channel blocks of OC per M = 256 tile)
    (64, 4, 4, 128, 256, 3, 3, 1, 1, 1, 1),    # l3/l4 class, single-tap tiles (IC % BN == 0)
    (32, 5, 5, 96, 512, 3, 3, 2, 2, 1, 1),     # stride 2, 2 pair m-tiles, n-tiles straddling taps
]


@pytest.fixture(params=["single", "pair", "single-3mma", "pair-3mma"])
def force_tma(env, request):
    """TMA variant forced; run with 1-CTA tiles and with CTA-pair (cta_group::2) tiles (pairs apply to
    fwd / dX in 3xTF32 when N % 256 == 0, other cases are unchanged), and 3xTF32 fwd / dX once in the
    hybrid form (W' plane + bf16 cross-term MMA) and once as three TF32 MMAs ("3mma", the small-call
    default, smconv_set_hybrid_min_gflop)."""
    _, _, sm = env
    for op in (0, 1, 2):
        sm.force_variant(op, sm.CONV_VARIANT_TMA)
    old = sm.set_pair(request.param.startswith("pair"))
    old_h = sm.set_hybrid_min_gflop(1e9 if request.param.endswith("3mma") else 0.0)
    yield
    sm.set_hybrid_min_gflop(old_h)
    sm.set_pair(old)
    for op in (0, 1, 2):
        sm.force_variant(op, sm.CONV_VARIANT_AUTO)


@pytest.mark.parametrize("s", SWEEP_TMA, ids=_id)
def test_tma_integer_bit_exact(env, force_tma, s):
    X, W, dY = gen(s, 12, integer=1)
    ref = oracle_all(env, s, X, W, dY)
    for math in ("3xtf32", "tf32"):
        got = gpu_all(env, s, X, W, dY, math)
        for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
            assert np.array_equal(g.astype(np.float64), r), (math, name, float(np.max(np.abs(g - r))))


@pytest.mark.parametrize("s", SWEEP_TMA, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_tma_random_within_tolerance(env, force_tma, s, math):
    X, W, dY = gen(s, 13)
    ref = oracle_all(env, s, X, W, dY)
    got = gpu_all(env, s, X, W, dY, math)
    for name, g, r in zip(("fwd", "dx", "dw"), got, ref):
        e = normwise(g, r)
        print("tma %s %s %s err %.3e" % (_id(s), math, name, e))
        assert e <= TOL[math], (name, e)


# ---------------------------------------------------------------- STRIP variant (stride 1, 3-wide filters)
SWEEP_STRIP = [
    (32, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),     # ResNet l1 / VGG conv2 class (BN 64)
    (64, 16, 16, 128, 128, 3, 3, 1, 1, 1, 1),   # l2 class (BN 128, TF32 only; 3xTF32 falls back)
    (32, 8, 8, 64, 32, 3, 3, 1, 1, 1, 1),       # BN 32
    (32, 7, 10, 32, 64, 3, 3, 1, 1, 1, 1),      # ragged strip (OW 10 not a multiple of 4R)
    (32, 6, 6, 64, 64, 3, 3, 1, 1, 0, 0),       # no padding
    (32, 5, 9, 32, 64, 5, 3, 1, 1, 2, 1),       # FH 5 rows, pad 2 / 1
    (96, 4, 4, 64, 64, 3, 3, 1, 1, 1, 1),       # 3 image groups, 4x4 map
    # CTA-pair strips (3xTF32, BN 64, N % 64 == 0: two 32-image groups per M = 256 tile)
    (64, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),     # l1 class, one pair image block
    (192, 7, 10, 64, 64, 3, 3, 1, 1, 1, 1),     # 3 pair blocks, ragged strip
    (64, 5, 9, 64, 64, 5, 3, 1, 1, 2, 1),       # FH 5 rows, pad 2 / 1 (skipped filter rows)
    (128, 6, 6, 96, 64, 3, 3, 1, 1, 0, 0),      # no padding, 3 channel blocks of fwd K (dX BN 96: not 3xTF32)
]


@pytest.fixture(params=["single", "pair"])
def force_strip(env, request):
    """STRIP variant forced; once with 1-CTA strips and once with CTA-pair strips (pairs apply in
    3xTF32 at BN 64 when N % 64 == 0; other cases are unchanged)."""
    _, _, sm = env
    for op in (0, 1):
        sm.force_variant(op, sm.CONV_VARIANT_STRIP)
    old = sm.set_pair(request.param == "pair")
    yield
    sm.set_pair(old)
    for op in (0, 1):
        sm.force_variant(op, sm.CONV_VARIANT_AUTO)


def _strip_ok(sm, s, math, op):
    try:
        return "strip" in sm.plan_describe(op, s, sm.MATH[math])
    except sm.ConvError as e:
        assert e.code == sm.CONV_EUNSUPPORTED
        return False


@pytest.mark.parametrize("s", SWEEP_STRIP, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_strip_parity(env, force_strip, s, math):
    torch, oracle, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    for integer in (1, 0):
        X, W, dY = gen(s, 20 + integer, integer=integer)
        x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
        ran = 0
        if _strip_ok(sm, s, math, 0):
            y = sm.conv2d_fwd(x, w, (sh, sw), (ph, pw), math=math).cpu().numpy()
            ref = oracle.conv2d_fwd(X, W, (sh, sw), (ph, pw))
            ran += 1
            if integer:
                assert np.array_equal(y.astype(np.float64), ref)
            else:
                assert normwise(y, ref) <= TOL[math]
        if _strip_ok(sm, s, math, 1):
            dx = sm.conv2d_bwd_data(dy, w, (IH, IW), (sh, sw), (ph, pw), math=math).cpu().numpy()
            ref = oracle.conv2d_bwd_data(dY, W, (IH, IW), (sh, sw), (ph, pw))
            ran += 1
            if integer:
                assert np.array_equal(dx.astype(np.float64), ref)
            else:
                assert normwise(dx, ref) <= TOL[math]
        if math == "tf32" or (s[3] <= 64 and s[4] <= 64):  # 3xTF32 strips: BN (fwd OC, dX IC) <= 64
            assert ran == 2, "strip variant should serve this shape"


# ---------------------------------------------------------------- super-pixel stride-2 dX (smconv.cu s2dx)
SWEEP_S2DX = [  # eligible when dY has >= 16x16 positions
    (32, 32, 32, 64, 64, 3, 3, 2, 2, 1, 1),     # l2.0a geometry, G = 32 image boxes
    (256, 32, 32, 64, 128, 3, 3, 2, 2, 1, 1),   # N % 256: CTA-pair fwd tiles; l2.0a channels
    (128, 32, 40, 128, 96, 3, 3, 2, 2, 1, 1),   # non-square, 2 x 128 virtual columns per phase row
    (32, 48, 32, 64, 32, 3, 3, 2, 2, 1, 1),     # OC 32, 24x16 dY
]


@pytest.mark.parametrize("s", SWEEP_S2DX, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_s2dx_parity(env, s, math):
    """dX of 3x3 stride-2 pad-1 convs as one super-pixel 2x2 fwd conv (all four phases at once)."""
    torch, oracle, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    desc = sm.plan_describe(1, s, sm.MATH[math])
    # (TF32 plans with BN 256 may split K on the smaller shapes: then the phase path runs)
    assert "s2dx" in desc or math == "tf32", desc
    for integer in (1, 0):
        X, W, dY = gen(s, 60 + integer, integer=integer)
        w, dy = torch.from_numpy(W).cuda(), torch.from_numpy(dY).cuda()
        dx = sm.conv2d_bwd_data(dy, w, (IH, IW), (sh, sw), (ph, pw), math=math).cpu().numpy()
        ref = oracle.conv2d_bwd_data(dY, W, (IH, IW), (sh, sw), (ph, pw))
        if integer:
            assert np.array_equal(dx.astype(np.float64), ref)
        else:
            assert normwise(dx, ref) <= TOL[math], normwise(dx, ref)


# ---------------------------------------------------------------- DIRECT variant (few-channel stems)
SWEEP_DIRECT = [
    (4, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1),     # the CIFAR stem (IC 3 -> 4)
    (3, 9, 13, 4, 20, 3, 3, 2, 2, 1, 1),      # stride 2, ragged
    (2, 12, 12, 4, 96, 5, 5, 1, 1, 2, 2),     # 5x5, OC not a multiple of 64
    (2, 10, 10, 8, 64, 3, 3, 1, 1, 1, 1),     # IC 8
    (5, 7, 7, 4, 192, 3, 3, 1, 1, 0, 0),      # GoogLeNet-stem OC, no padding
]


@pytest.fixture
def force_direct(env):
    """DIRECT forced: the heuristic sends small-batch stem dW to GENERIC (r01z)."""
    _, _, sm = env
    for op in (0, 2):
        sm.force_variant(op, sm.CONV_VARIANT_DIRECT)
    yield
    for op in (0, 2):
        sm.force_variant(op, sm.CONV_VARIANT_AUTO)


@pytest.mark.parametrize("s", SWEEP_DIRECT, ids=_id)
def test_direct_parity(env, force_direct, s):
    torch, oracle, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    assert "direct" in sm.plan_describe(0, s) and "direct" in sm.plan_describe(2, s)
    for integer in (2, 0):
        X, W, dY = gen(s, 30 + integer, integer=integer, stem=not integer)
        x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
        for math in ("3xtf32", "tf32"):  # DIRECT is exact fp32 FMA in both modes
            y = sm.conv2d_fwd(x, w, (sh, sw), (ph, pw), math=math).cpu().numpy()
            dw = sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw), math=math).cpu().numpy()
            ry = oracle.conv2d_fwd(X, W, (sh, sw), (ph, pw))
            rw = oracle.conv2d_bwd_filter(X, dY, (FH, FW), (sh, sw), (ph, pw))
            if integer:
                assert np.array_equal(y.astype(np.float64), ry) and np.array_equal(dw.astype(np.float64), rw)
            else:
                assert normwise(y, ry) <= 1e-6 and normwise(dw, rw) <= 1e-6, (normwise(y, ry), normwise(dw, rw))


# ---------------------------------------------------------------- STEM variant (IC = 4 stems, tensor cores)
SWEEP_STEM = [
    (4, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1),     # the CIFAR stem (IC 3 -> 4)
    (77, 30, 30, 4, 64, 3, 3, 1, 1, 1, 1),    # 541 tiles of 128 pixels, ragged last tile; 2166 dW k-blocks
    (3, 9, 13, 4, 64, 3, 3, 2, 2, 1, 1),      # stride 2, ragged map
    (30, 32, 32, 4, 128, 3, 3, 1, 1, 1, 1),   # OC 128, 240 tiles (148 persistent CTAs)
    (5, 7, 7, 4, 192, 3, 3, 1, 1, 0, 0),      # GoogLeNet-stem OC (two dW m-tiles), no padding
    (40, 32, 32, 4, 192, 3, 3, 1, 1, 1, 1),   # OC 192 (one accumulator, 4 A slots), 320 tiles: 2-3 per CTA
    (3, 11, 6, 4, 20, 3, 3, 1, 1, 2, 2),      # dW only (fwd OC must be 64 / 128 / 192), pad 2
]


@pytest.fixture
def force_stem(env):
    _, _, sm = env
    for op in (0, 2):
        sm.force_variant(op, sm.CONV_VARIANT_STEM)
    yield
    for op in (0, 2):
        sm.force_variant(op, sm.CONV_VARIANT_AUTO)


@pytest.mark.parametrize("s", SWEEP_STEM, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_stem_parity(env, force_stem, s, math, parity_log):
    torch, oracle, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    fwd_ok = OC in (64, 128, 192)
    if fwd_ok:
        assert "stem" in sm.plan_describe(0, s, sm.MATH[math])
    assert "stem" in sm.plan_describe(2, s, sm.MATH[math])
    for integer in (2, 0):
        X, W, dY = gen(s, 50 + integer, integer=integer, stem=not integer)
        x, w, dy = (torch.from_numpy(a).cuda() for a in (X, W, dY))
        rw = oracle.conv2d_bwd_filter(X, dY, (FH, FW), (sh, sw), (ph, pw))
        dw = sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw), math=math).cpu().numpy()
        outs = [("dw", dw, rw)]
        if fwd_ok:
            ry = oracle.conv2d_fwd(X, W, (sh, sw), (ph, pw))
            y = sm.conv2d_fwd(x, w, (sh, sw), (ph, pw), math=math).cpu().numpy()
            outs.append(("fwd", y, ry))
        for name, got, ref in outs:
            if integer:
                assert np.array_equal(got.astype(np.float64), ref), name
            else:
                e = normwise(got, ref)
                parity_log.append({"config": "stem-sweep", "layer": "x".join(map(str, s)), "op": name, "math": math,
                                   "normwise": e, "tol": TOL[math],
                                   "plan": sm.plan_describe({"fwd": 0, "dw": 2}[name], s, sm.MATH[math])})
                assert e <= TOL[math], (name, e)


def test_stem_deterministic(env):
    """dW partials are summed in a fixed order: two calls are bitwise identical."""
    torch, oracle, sm = env
    s = (64, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1)
    X, W, dY = gen(s, 7)
    x, dy = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
    a = sm.conv2d_bwd_filter(x, dy, (3, 3), (1, 1), (1, 1))
    b = sm.conv2d_bwd_filter(x, dy, (3, 3), (1, 1), (1, 1))
    assert "stem" in sm.plan_describe(2, s) and torch.equal(a, b)


# ---------------------------------------------------------------- DWS variant (dW, 3x3 s1 64->64)
SWEEP_DWS = [
    (2, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),    # r.l1 / vgg2 geometry: one output row per k-block
    (3, 16, 16, 64, 64, 3, 3, 1, 1, 1, 1),    # two rows per k-block
    (5, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1),      # four rows per k-block
    (2, 34, 34, 64, 64, 3, 3, 1, 1, 0, 0),    # no padding (slab never out of bounds at the left)
    (1, 30, 14, 64, 64, 3, 3, 1, 1, 2, 2),    # pad 2: OH 32 x OW 16, whole out-of-range slab rows
    (40, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1),   # chains of 13 k-blocks: 2 promotion chunks per item
]


@pytest.mark.parametrize("s", SWEEP_DWS, ids=_id)
@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
def test_dws_parity(env, s, math):
    torch, oracle, sm = env
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    assert "dws" in sm.plan_describe(2, s, sm.MATH[math])
    for integer in (2, 0):
        X, W, dY = gen(s, 40 + integer, integer=integer)
        x, dy = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
        dw = sm.conv2d_bwd_filter(x, dy, (FH, FW), (sh, sw), (ph, pw), math=math).cpu().numpy()
        ref = oracle.conv2d_bwd_filter(X, dY, (FH, FW), (sh, sw), (ph, pw))
        if integer:
            assert np.array_equal(dw.astype(np.float64), ref)
        else:
            assert normwise(dw, ref) <= TOL[math], normwise(dw, ref)
