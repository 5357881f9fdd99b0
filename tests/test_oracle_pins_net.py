"""Pins of oracle/net_oracle.c (GEMM, BatchNorm statistics, LeakyReLU and its BN-backward statistics)
against things other than itself: SPEC's worked values (tests/golden/spec_gemm_leaky.txt), numpy's
float64 BLAS matmul and exact int64 matmul, numpy sums, torch's float64 batch_norm (training mode)
and torch float64 autograd through leakyRelu(BN(x))."""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_gemm_leaky.txt")


def _golden():
    cases = {}
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, vals = line.split(":")
        name, tensor, *shape = head.split()
        cases.setdefault(name, {})[tensor] = np.array([float(v) for v in vals.split()]).reshape([int(s) for s in shape])
    return cases


def test_gemm_spec_worked_values():
    g = _golden()
    for name, ta in (("gemm_identity", False), ("gemm_plain", False), ("gemm_t1", True)):
        c = g[name]
        assert np.array_equal(oracle.matmul(c["A"], c["B"], ta=ta), c["C"]), name


def test_leaky_spec_worked_values():
    c = _golden()["leaky"]
    assert np.allclose(oracle.leaky_relu(c["X"], 0.01), c["Y"], rtol=0, atol=1e-15)
    x = np.linspace(-3, 3, 13)
    assert np.array_equal(oracle.leaky_relu(x, 1.0), x)  # slope 1: identity


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_blas_and_int64(ta, tb):
    rng = np.random.default_rng(5)
    M, N, K = 37, 23, 61  # all different: a transposed operand cannot pass by symmetry
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    got = oracle.matmul(A, B, ta=ta, tb=tb)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    Ai = rng.integers(-50, 51, A.shape)
    Bi = rng.integers(-50, 51, B.shape)
    refi = (Ai.T if ta else Ai) @ (Bi.T if tb else Bi)
    assert np.array_equal(oracle.matmul(Ai, Bi, ta=ta, tb=tb), refi.astype(np.float64))


def test_channel_stats_vs_numpy_and_torch_batchnorm():
    import torch
    rng = np.random.default_rng(6)
    Y = rng.normal(0.3, 2.0, (5, 7, 6, 12))
    s1, s2 = oracle.channel_stats(Y)
    assert np.allclose(s1, Y.sum(axis=(0, 1, 2)), rtol=1e-13, atol=1e-12)
    assert np.allclose(s2, (Y * Y).sum(axis=(0, 1, 2)), rtol=1e-13)
    # the BN training-mode statistics follow: mean = S1/M, biased var = S2/M - mean^2
    M = Y.size // 12
    t = torch.from_numpy(Y).permute(0, 3, 1, 2).contiguous()  # NCHW for torch
    rm, rv = torch.zeros(12, dtype=torch.float64), torch.ones(12, dtype=torch.float64)
    out = torch.nn.functional.batch_norm(t, rm, rv, training=True, momentum=1.0, eps=1e-8)
    mean = s1 / M
    var = s2 / M - mean ** 2
    xhat = (Y - mean) / np.sqrt(var + 1e-8)
    assert np.allclose(xhat, out.permute(0, 2, 3, 1).numpy(), rtol=1e-9, atol=1e-9)
    ones = np.ones((2, 3, 4, 5))
    a, b = oracle.channel_stats(ones)
    assert np.array_equal(a, np.full(5, 24.0)) and np.array_equal(b, np.full(5, 24.0))


@pytest.mark.parametrize("k", [0.01, 0.2])
def test_leaky_bwd_stats_give_bn_gradients(k):
    """Autograd (torch float64) through A = leakyRelu(gamma * xhat + beta), L = <A, R>: the oracle's
    G must be dL/dZ, S1 = dL/dbeta and (S2 - beta * S1) / gamma = dL/dgamma."""
    import torch
    rng = np.random.default_rng(7)
    C = 9
    x = torch.from_numpy(rng.normal(0, 1.5, (4, 5, 3, C))).requires_grad_(False)
    gamma = torch.from_numpy(rng.uniform(0.5, 2.0, C)).requires_grad_(True)
    beta = torch.from_numpy(rng.uniform(-0.5, 0.5, C)).requires_grad_(True)
    mean = x.mean(dim=(0, 1, 2))
    var = x.var(dim=(0, 1, 2), unbiased=False)
    xhat = (x - mean) / torch.sqrt(var + 1e-8)
    Z = (gamma * xhat + beta).detach().requires_grad_(True)
    A = torch.where(Z > 0, Z, k * Z)
    R = torch.from_numpy(rng.uniform(-1, 1, A.shape))
    (A * R).sum().backward()
    dZ = Z.grad.numpy()
    Z2 = gamma * xhat + beta
    A2 = torch.where(Z2 > 0, Z2, k * Z2)
    (A2 * R).sum().backward()
    A32 = A.detach().numpy().astype(np.float32)
    # z recomputed from the fp32-rounded output must match Z closely; G uses only its sign
    G, S1, S2 = oracle.leaky_bwd_stats(R.numpy(), A32, k)
    assert np.allclose(G, dZ, rtol=0, atol=1e-15)
    assert np.allclose(S1, beta.grad.numpy(), rtol=1e-12, atol=1e-12)
    dgamma = (S2 - beta.detach().numpy() * S1) / gamma.detach().numpy()
    assert np.allclose(dgamma, gamma.grad.numpy(), rtol=1e-5, atol=1e-6)  # fp32 rounding of A in z
