"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol the
headers declare, its index arithmetic self-test passes, and validation rejects bad calls
with the documented codes before any CUDA call (SURVEY.md §8(b) contract items 1-5)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sm():
    from paper_2305_08819_b200 import build
    build.build()
    from paper_2305_08819_b200 import smconv
    smconv.lib()
    return smconv


def _declared():
    names = []
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not h.endswith(".h"):
            continue
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(\w+)\s*\(", src, flags=re.M)
    return names


def test_exports_every_declared_symbol(sm):
    names = _declared()
    assert {"conv2d_fwd", "conv2d_bwd_data", "conv2d_bwd_filter", "conv2d_out_hw",
            "conv2d_workspace_bytes", "conv2d_strerror", "conv2d_last_error_detail"} <= set(names)
    L = ctypes.CDLL(sm.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(sm.EXPORTS + sm.EXT_EXPORTS + sm.GEMM_EXPORTS + sm.EPI_EXPORTS + sm.MCAST_EXPORTS) <= set(names)


def test_library_is_sm100a(sm):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", sm.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "LDTM" in sass  # tcgen05.mma / tcgen05.ld


def test_selftest_fastdiv(sm):
    assert sm.lib().smconv_selftest_host() == 0


def test_out_hw(sm):
    assert sm.out_hw(32, 32, 3, 3, (1, 1), (1, 1)) == (32, 32)
    assert sm.out_hw(32, 32, 3, 3, (2, 2), (1, 1)) == (16, 16)   # SPEC.md:584, floor (L1)
    assert sm.out_hw(32, 32, 1, 1, (2, 2), (0, 0)) == (16, 16)
    assert sm.out_hw(32, 32, 11, 11, (4, 4), (5, 5)) == (8, 8)
    with pytest.raises(sm.ConvError) as e:
        sm.out_hw(2, 2, 5, 5, (1, 1), (0, 0))
    assert e.value.code == sm.CONV_EARG


def _call(sm, op, a, b, o, dims, math=0, ws=0, nws=0):
    f = (sm.lib().conv2d_fwd, sm.lib().conv2d_bwd_data, sm.lib().conv2d_bwd_filter)[op]
    return f(ctypes.c_void_p(a), ctypes.c_void_p(b), ctypes.c_void_p(o), *dims, math,
             ctypes.c_void_p(ws), nws, None)


GOOD = (2, 8, 8, 4, 8, 3, 3, 1, 1, 1, 1)
A, B, O = 0x100000, 0x200000, 0x300000   # fake, 16-B aligned, disjoint; never dereferenced on the error path


@pytest.mark.parametrize("op", [0, 1, 2])
def test_validation_codes(sm, op):
    bad = list(GOOD)
    bad[7] = 0  # stride 0 -> positivity error
    assert _call(sm, op, A, B, O, bad) == sm.CONV_EARG
    assert "sh" in sm.lib().conv2d_last_error_detail().decode()
    bad = list(GOOD)
    bad[9] = -1
    assert _call(sm, op, A, B, O, bad) == sm.CONV_EARG
    bad = list(GOOD)
    bad[3] = 3  # IC not padded to 4x
    assert _call(sm, op, A, B, O, bad) == sm.CONV_EALIGN
    bad = list(GOOD)
    bad[1], bad[2], bad[9], bad[10] = 2, 2, 0, 0  # 3x3 on 2x2 without padding -> OH < 1
    assert _call(sm, op, A, B, O, bad) == sm.CONV_EARG
    assert _call(sm, op, A + 4, B, O, GOOD) == sm.CONV_EALIGN
    assert _call(sm, op, A, B, A, GOOD) == sm.CONV_EALIAS
    assert _call(sm, op, A, B, O, GOOD, math=7) == sm.CONV_EARG
    assert _call(sm, op, 0, B, O, GOOD) == sm.CONV_EARG
    big = (1 << 16, 64, 64, 64, 64, 3, 3, 1, 1, 1, 1)  # 2^34 elements
    assert _call(sm, op, A, B, O, big) == sm.CONV_EUNSUPPORTED


def test_workspace_contract(sm):
    # a dW with a long reduction always splits K -> needs workspace; NULL workspace is refused
    dims = (512, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1)
    n = sm.workspace_bytes(2, dims)
    assert n > 0
    a, b, o = 1 << 40, 2 << 40, 3 << 40
    assert _call(sm, 2, a, b, o, dims, ws=0, nws=0) == sm.CONV_EWORKSPACE
    assert _call(sm, 2, a, b, o, dims, ws=4 << 40, nws=n - 16) == sm.CONV_EWORKSPACE
    assert sm.lib().conv2d_workspace_bytes(0, 0, 8, 8, 4, 8, 3, 3, 1, 1, 1, 1, 0) == ctypes.c_size_t(-1).value


def test_strerror(sm):
    for c, n in enumerate(["CONV_OK", "CONV_EARG", "CONV_EALIGN", "CONV_EALIAS", "CONV_EWORKSPACE",
                           "CONV_EUNSUPPORTED", "CONV_ECUDA"]):
        assert sm.lib().conv2d_strerror(c).decode() == n
    assert sm.lib().conv2d_strerror(99).decode() == "CONV_UNKNOWN"


def test_plans_cover_network_shapes(sm):
    from paper_2305_08819_b200 import nets
    for name, f in nets.NETS.items():
        for l in f():
            for op in (0, 1, 2):
                for math in (0, 1):
                    d = sm.plan_describe(op, l.dims(128), math)
                    assert "variant=" in d
                    # main kernel [+ split-K reduce, unless the split is reduced in-cluster (csk)]
                    # [+ zero fill of tap-less dX stride phases, unless the epilogue writes them (zfill)]
                    # [+ the bf16 W' prep of 3xTF32 fwd / dX on the TMA and STRIP variants]
                    k = sm.plan_kernels(op, l.dims(128), math)
                    wx = math == 0 and op != 2 and ("variant=tma" in d or "variant=strip" in d) and " 3mma" not in d
                    hbm_split = "splits=1 " not in d and " csk" not in d
                    assert k == 1 + hbm_split + (op == 1 and l.sh * l.sw > 1 and
                                                               "variant=tma" in d and l.FH == 1 and
                                                               " zfill" not in d) + wx + \
                        ("s2dx" in d), (l.name, op, d)


def test_stem_plans(sm):
    """The IC = 4 3x3 stems (every network's first conv) go to the tensor-core STEM variant: fwd for
    OC 64 / 128 / 192, dW for any OC % 4 == 0 (per-CTA pixel ranges + the fixed-order partial sum);
    other few-channel shapes keep DIRECT / GENERIC."""
    for N in (128, 512, 4096):
        s = (N, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1)
        for math in (0, 1):
            assert sm.plan_describe(0, s, math).startswith("variant=stem"), sm.plan_describe(0, s, math)
            d = sm.plan_describe(2, s, math)
            assert d.startswith("variant=stem") and sm.plan_kernels(2, s, math) == 2, d
            assert sm.plan_kernels(0, s, math) == 1
    assert sm.plan_describe(0, (256, 32, 32, 4, 192, 3, 3, 1, 1, 1, 1), 0).startswith("variant=stem")
    assert not sm.plan_describe(0, (8, 32, 32, 4, 96, 3, 3, 1, 1, 1, 1), 0).startswith("variant=stem")
    assert sm.plan_describe(2, (8, 32, 32, 4, 96, 3, 3, 1, 1, 1, 1), 0).startswith("variant=stem")
    assert not sm.plan_describe(0, (8, 32, 32, 8, 64, 3, 3, 1, 1, 1, 1), 0).startswith("variant=stem")
    assert not sm.plan_describe(0, (8, 32, 32, 4, 64, 5, 5, 1, 1, 2, 2), 0).startswith("variant=stem")


def test_force_variant(sm):
    sm.force_variant(0, sm.CONV_VARIANT_GENERIC)
    assert "generic" in sm.plan_describe(0, GOOD)
    sm.force_variant(0, sm.CONV_VARIANT_AUTO)
    with pytest.raises(sm.ConvError):
        sm.force_variant(5, 0)


VARIANT_NAMES = {1: "generic", 2: "tma", 3: "strip", 4: "direct", 5: "dws", 6: "stem"}


@pytest.mark.parametrize("op", [0, 1, 2])
@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6])
def test_forced_variant_is_served_or_refused(sm, op, variant):
    """Forcing a variant either yields a plan of THAT variant or CONV_EUNSUPPORTED -- never a plan whose
    launch would write the wrong buffer extent (e.g. STRIP forced for dW)."""
    shapes = [(32, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1), (4, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1),
              (32, 8, 8, 128, 256, 3, 3, 2, 2, 1, 1), (3, 7, 9, 20, 36, 3, 3, 1, 1, 1, 1)]
    sm.force_variant(op, variant)
    try:
        for s in shapes:
            try:
                d = sm.plan_describe(op, s, 0)
            except sm.ConvError as e:
                assert e.code == sm.CONV_EUNSUPPORTED, (s, e)
                continue
            assert d.startswith("variant=" + VARIANT_NAMES[variant]), (s, d)
            assert not (variant == 3 and op == 2)
    finally:
        sm.force_variant(op, 0)


def test_direct_only_when_launch_fits(sm):
    """AUTO must not pick DIRECT for shapes whose launch would exceed its shared memory (the launch would
    then return CONV_EUNSUPPORTED for a valid call)."""
    assert "direct" not in sm.plan_describe(0, (8, 8, 8, 8, 1024, 3, 3, 1, 1, 1, 1), 0)
    assert "direct" not in sm.plan_describe(2, (2048, 32, 32, 8, 256, 3, 3, 1, 1, 1, 1), 0)
    sm.force_variant(0, sm.CONV_VARIANT_DIRECT)
    try:  # the stem still fits DIRECT when forced (AUTO now sends it to STEM)
        assert "direct" in sm.plan_describe(0, (4096, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1), 0)
    finally:
        sm.force_variant(0, 0)


def test_plan_cache_tracks_forced_variant(sm):
    s = (32, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1)
    a = sm.plan_describe(0, s, 0)
    sm.force_variant(0, 1)
    try:
        assert sm.plan_describe(0, s, 0).startswith("variant=generic")
    finally:
        sm.force_variant(0, 0)
    assert sm.plan_describe(0, s, 0) == a


def test_binding_cross_checks_shapes(sm):
    """The torch wrappers check every tensor against the others before calling the C ABI (shape /
    channel mismatch -> error, SPEC conv2d_*); CPU tensors are refused (no CPU fallback)."""
    import torch
    x = torch.zeros((2, 8, 8, 4))
    w = torch.zeros((8, 3, 3, 4))
    with pytest.raises(ValueError):
        sm.conv2d_fwd(x, w)


def test_gemm_host_validation(sm):
    """GEMM entry points: plans map onto the 1x1 conv variants; row lengths must be multiples of 4
     and dims positive -- rejected on the host with the gemm name in the detail."""
    assert "variant=" in sm.gemm_plan_describe(0, 4096, 256, 512)
    assert "variant=" in sm.gemm_plan_describe(1, 256, 512, 4096)
    assert "variant=" in sm.gemm_plan_describe(2, 4096, 256, 512)
    with pytest.raises(sm.ConvError) as e:
        sm.gemm_plan_describe(0, 8, 6, 8)  # N % 4 != 0
    assert e.value.code == sm.CONV_EALIGN and "matMul" in e.value.detail
    with pytest.raises(sm.ConvError) as e:
        sm.gemm_workspace_bytes(2, 8, 8, 0)
    assert e.value.code == sm.CONV_EARG
    L = sm.lib()
    rc = L.gemm_matmul_t1(None, None, None, 8, 8, 8, 0, None, 0, None)
    assert rc == sm.CONV_EARG and b"matMulT1" in L.conv2d_last_error_detail()


def test_epi_argument_errors_on_host(sm):
    """Fused-epilogue argument checks (include/smconv_epi.h) return before anything is enqueued."""
    import ctypes as C
    L = sm.lib()
    P = C.c_void_p
    d = (32, 8, 8, 32, 32, 3, 3, 1, 1, 1, 1)
    x, w, y, st = P(0x100000), P(0x200000), P(0x300000), P(0x400000)
    call = lambda epi, k, stats: L.conv2d_fwd_epi(x, w, y, stats, *d, 0, epi, k, P(0), 0, P(0))
    assert call(3, 0.1, st) == sm.CONV_EARG          # a dX epilogue on fwd
    assert call(9, 0.1, st) == sm.CONV_EARG          # unknown
    assert call(2, 0.0, st) == sm.CONV_EARG          # leaky slope must be > 0
    assert call(2, float("nan"), st) == sm.CONV_EARG
    assert call(1, 0.1, P(0)) == sm.CONV_EARG        # stats required
    assert call(1, 0.1, P(0x400004)) == sm.CONV_EALIGN
    assert call(1, 0.1, P(0x300000 + 64)) == sm.CONV_EALIAS  # stats inside Y
    dx = lambda epi, a: L.conv2d_bwd_data_epi(y, w, a, x, st, *d, 0, epi, C.c_float(0.1), P(0), 0, P(0))
    assert dx(1, P(0x500000)) == sm.CONV_EARG       # a fwd epilogue on dX
    assert dx(3, P(0)) == sm.CONV_EARG               # A required
    assert dx(3, P(0x500008)) == sm.CONV_EALIGN
    assert dx(3, P(0x300000)) == sm.CONV_EALIAS      # A overlapping dY
    assert dx(3, P(0x100000 + 4096)) == sm.CONV_EALIAS  # A partially overlapping dX
    assert sm.lib().conv2d_epi_workspace_bytes(2, *d, 0, 1) == C.c_size_t(-1).value  # no dW epilogue
    assert sm.epi_workspace_bytes(0, d, 0, "bn_stats") >= sm.workspace_bytes(0, d, 0)


def test_epi_plans(sm):
    """Fused where the conv kernel writes final values (TMA / STRIP without split-K), else a pass;
    statistics add two fixed-order reduction kernels."""
    d_strip = (128, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1)
    d_csk = (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1)
    d_stem = (512, 32, 32, 4, 64, 3, 3, 1, 1, 1, 1)
    assert "epi=fused" in sm.epi_plan_describe(0, d_strip, 1, "bn_stats")
    assert "epi=pass" in sm.epi_plan_describe(0, d_csk, 1, "bn_stats")
    assert "epi=pass" in sm.epi_plan_describe(0, d_stem, 0, "leaky")
    assert sm.epi_plan_kernels(0, d_strip, 1, "bn_stats") == sm.plan_kernels(0, d_strip, 1) + 2
    assert sm.epi_plan_kernels(0, d_csk, 1, "bn_stats") == sm.plan_kernels(0, d_csk, 1) + 3
    assert sm.epi_plan_kernels(1, d_strip, 1, "leaky_bwd") == sm.plan_kernels(1, d_strip, 1)


def test_mcast_plans(sm):
    """Fused dW + all-reduce (include/smconv_mcast.h): the TMA dW epilogue adds into the multicast buffer
    when the plan has one split; otherwise the split-K reduce kernel does (a single-split non-TMA plan
    stages its tile in the workspace)."""
    one = (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1)     # VGG conv11 3xTF32: TMA pairs, one split
    many = (128, 32, 32, 64, 64, 3, 3, 1, 1, 1, 1)    # DWS split-K
    assert "mcast=epilogue" in sm.mcast_plan_describe(one, 0)
    d = sm.mcast_plan_describe(many, 0)
    assert "mcast=reduce" in d
    assert sm.mcast_workspace_bytes(many, 0) == sm.workspace_bytes(2, many, 0)
    stem = (8, 8, 8, 4, 64, 3, 3, 1, 1, 1, 1)
    if "splits=1 " in sm.plan_describe(2, stem, 0):
        assert sm.mcast_workspace_bytes(stem, 0) >= 64 * 9 * 4 * 4


def test_hybrid_threshold(sm):
    """3xTF32 TMA fwd / dX: small calls run three TF32 MMAs (no W' plane, one kernel fewer), large ones
    the hybrid form; the threshold is settable and the plan cache follows it."""
    small = (128, 4, 4, 512, 512, 3, 3, 1, 1, 1, 1)   # VGG vgg9 at b128: 6.7 GFLOP
    big = (4096, 8, 8, 256, 256, 3, 3, 1, 1, 1, 1)    # ResNet l3 at b4096: 309 GFLOP
    assert " 3mma" in sm.plan_describe(0, small, 0) and " 3mma" in sm.plan_describe(1, small, 0)
    assert " 3mma" not in sm.plan_describe(0, big, 0)
    assert " 3mma" not in sm.plan_describe(0, small, 1)  # TF32 mode has no split at all
    k_small = sm.plan_kernels(0, small, 0)
    old = sm.set_hybrid_min_gflop(0.0)
    try:
        assert " 3mma" not in sm.plan_describe(0, small, 0)
        assert sm.plan_kernels(0, small, 0) == k_small + 1  # + wx_prep
    finally:
        sm.set_hybrid_min_gflop(old)
    assert " 3mma" in sm.plan_describe(0, small, 0)
