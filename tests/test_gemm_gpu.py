"""GPU parity of the paper's matrix-multiply operators (include/smgemm.h; Fig. 3
matMulT1, :64 nn.fullconnect) against the oracle's plain triple loop
(oracle.matmul, pinned to BLAS / int64 / SPEC's worked values in test_oracle_pins_net.py).
Integer inputs bit-exact in both math modes (pin P7); random inputs normwise <= 1e-5 (3xTF32) /
5e-3 (TF32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"3xtf32": 1e-5, "tf32": 5e-3}

# (M, N, K): the Fig. 2 FC layer (256 -> 10, padded to 12) at batch 512, wider FC layers, ragged and
# tiny shapes, a 4096-row batch (position-major tiles of 128 rows), K long enough for split-K
SHAPES = [(512, 12, 256), (512, 256, 512), (4096, 512, 512), (37, 20, 44), (4, 4, 4), (130, 36, 1024),
          (256, 1024, 4096), (1, 8, 8)]


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


def _nw(g, r):
    den = float(np.max(np.abs(r)))
    return float(np.max(np.abs(g.astype(np.float64) - r))) / den if den else float(np.max(np.abs(g)))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("op", ["matmul", "matmul_t1", "matmul_t2"])
def test_gemm_parity(env, shape, op, parity_log):
    torch, oracle, sm = env
    M, N, K = shape
    if op == "matmul_t1" and M % 4:
        M += 4 - M % 4  # matMulT1 needs its A rows (length M) padded to 4x
    rng = np.random.default_rng(M * 1000003 + N * 1009 + K + 7 * ["matmul", "matmul_t1", "matmul_t2"].index(op))
    ashape = (K, M) if op == "matmul_t1" else (M, K)
    bshape = (N, K) if op == "matmul_t2" else (K, N)
    for integer in (1, 0):
        if integer:
            A = rng.integers(-2, 3, ashape).astype(np.float32)
            B = rng.integers(-2, 3, bshape).astype(np.float32)
        else:
            A = rng.uniform(-1, 1, ashape).astype(np.float32)
            B = rng.uniform(-1, 1, bshape).astype(np.float32)
        ref = oracle.matmul(A, B, ta=op == "matmul_t1", tb=op == "matmul_t2")
        a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        for math in ("3xtf32", "tf32"):
            c = getattr(sm, op)(a, b, math=math)
            torch.cuda.synchronize()
            got = c.cpu().numpy()
            assert got.shape == (M, N)
            e = _nw(got, ref)
            g = {"matmul": 0, "matmul_t1": 1, "matmul_t2": 2}[op]
            parity_log.append({"config": "gemm", "layer": "%dx%dx%d" % (M, N, K), "op": op, "math": math,
                               "check": "integer" if integer else "random", "coverage": "whole tensor",
                               "normwise": e, "tol": 0.0 if integer else TOL[math],
                               "plan": sm.gemm_plan_describe(g, M, N, K, sm.MATH[math])})
            if integer:
                assert np.array_equal(got.astype(np.float64), ref), (math, e)
            else:
                assert e <= TOL[math], (math, e)


def test_gemm_spec_worked_values(env):
    """SPEC.md:100-101 worked values, zero-padded to the 4x row rule."""
    torch, _, sm = env
    a = torch.zeros((4, 4), device="cuda")
    a[:2, :2] = torch.tensor([[1.0, 2.0], [3.0, 4.0]])
    b = torch.zeros((4, 4), device="cuda")
    b[:2, 0] = torch.tensor([5.0, 6.0])
    c = sm.matmul(a, b)
    assert c[:2, 0].tolist() == [17.0, 39.0] and float(c[:, 1:].abs().sum()) == 0.0
    b2 = torch.zeros((4, 4), device="cuda")
    b2[:2, 0] = torch.tensor([1.0, 0.0])
    c = sm.matmul_t1(a, b2)
    assert c[:2, 0].tolist() == [1.0, 2.0]
