"""Seeded synthetic inputs — the ONLY module shared by the oracle side and the CUDA side.

It draws random numbers; it holds none of the method's arithmetic.

Recipe:
  * X: stem layers (logical IC=3) U[0,1)  (pixels / 255);
       inner layers U[-1,1) (zero-mean: the hard case for relative error).
  * W: Kaiming-uniform U(-b, b), b = sqrt(6 / fan_in), fan_in = FH*FW*IC_logical
       ("Use Kaiming-uniform").
  * dY: U[-1,1).
  * pad lanes (IC 3 -> 4) are exactly 0.
  * integer mode (DESIGN.md pin P7): uniform integers in [-lim, lim].
  * seed = 230508819 + 1000*config + layer_index, numpy PCG64, float32 draws.
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 230508819


def rng(config: int = 0, layer_index: int = 0, salt: int = 0) -> np.random.Generator:
    return np.random.default_rng(BASE_SEED + 1000 * config + layer_index + 7919 * salt)


def _uniform(g, shape, lo, hi):
    return g.uniform(lo, hi, size=shape).astype(np.float32)


def activations(g, N, H, W, C, c_logical=None, stem=False, integer=0):
    """NHWC activation [N,H,W,C]; channels >= c_logical are zero pad lanes."""
    c_logical = C if c_logical is None else c_logical
    if integer:
        a = g.integers(-integer, integer + 1, size=(N, H, W, C)).astype(np.float32)
    elif stem:
        a = _uniform(g, (N, H, W, C), 0.0, 1.0)
    else:
        a = _uniform(g, (N, H, W, C), -1.0, 1.0)
    if c_logical < C:
        a[..., c_logical:] = 0.0
    return a


def filters(g, OC, FH, FW, IC, ic_logical=None, integer=0):
    """Filter [OC,FH,FW,IC], Kaiming-uniform with fan_in = FH*FW*ic_logical."""
    ic_logical = IC if ic_logical is None else ic_logical
    if integer:
        w = g.integers(-integer, integer + 1, size=(OC, FH, FW, IC)).astype(np.float32)
    else:
        b = math.sqrt(6.0 / (FH * FW * ic_logical))
        w = _uniform(g, (OC, FH, FW, IC), -b, b)
    if ic_logical < IC:
        w[..., ic_logical:] = 0.0
    return w


def layer_inputs(layer, N, config=0, layer_index=0, integer=0):
    """(X, W, dY) host float32 arrays for one layer of nets.py."""
    g = rng(config, layer_index)
    stem = layer.ic_logical < 4 or layer.ic_logical == 3
    X = activations(g, N, layer.IH, layer.IW, layer.IC, layer.ic_logical, stem=stem, integer=integer)
    W = filters(g, layer.OC, layer.FH, layer.FW, layer.IC, layer.ic_logical, integer=integer)
    dY = activations(g, N, layer.OH, layer.OW, layer.OC, integer=integer)
    return X, W, dY


def torch_layer_inputs(layer, N, device, seed, dtype=None, act_seed=None):
    """Device-side seeded draws with the same distributions (bench workloads too large for
    host generation).  Uses a torch.Generator on ``device``; the oracle sees these inputs only as
    host copies in tests/test_fullsize_gpu.py (sampled outputs at the full bench size).

    ``act_seed``: if given, X and dY come from their own generator seeded with it (data-parallel
    ranks: the filters W are replicated -- same ``seed`` on every rank -- while each rank's batch
    shard gets different activations)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    agen = gen
    if act_seed is not None:
        agen = torch.Generator(device=device)
        agen.manual_seed(int(act_seed))
    f32 = torch.float32
    stem = layer.ic_logical < 4
    X = torch.empty((N, layer.IH, layer.IW, layer.IC), dtype=f32, device=device)
    if stem:
        X.uniform_(0.0, 1.0, generator=agen)
    else:
        X.uniform_(-1.0, 1.0, generator=agen)
    if layer.ic_logical < layer.IC:
        X[..., layer.ic_logical:] = 0
    b = math.sqrt(6.0 / (layer.FH * layer.FW * layer.ic_logical))
    Wt = torch.empty((layer.OC, layer.FH, layer.FW, layer.IC), dtype=f32, device=device)
    Wt.uniform_(-b, b, generator=gen)
    if layer.ic_logical < layer.IC:
        Wt[..., layer.ic_logical:] = 0
    dY = torch.empty((N, layer.OH, layer.OW, layer.OC), dtype=f32, device=device)
    dY.uniform_(-1.0, 1.0, generator=agen)
    return X, Wt, dY
