"""The data-parallel step with a REAL NCCL process group on the B200 (world_size 1: gpurun and the
driver's GPU tier give one GPU; the world-2 exchange logic is covered with gloo in test_dp_gloo.py).

``ConvNetStep.step(pg)`` runs every conv of ResNet-18 (fwd, dX, dW) on the GPU and issues the
bucketed async NCCL all-reduce (SUM, reading L10) of the flat backward-ordered dW buffer
(north_star (e)).  Checks:
  * the NCCL all-reduce at world 1 leaves dW bit-for-bit equal to the same step without a group
    (SUM over one rank is the identity; any bucket offset / size / ordering slip shows up here);
  * every layer's all-reduced dW equals the oracle's O3 on the step's own X and dY buffers (copied
    back after the step), normwise <= 1e-5 (3xTF32), i.e. the buffers NCCL touched hold the right
    values for the right layers.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_convnet_step_nccl_world1(parity_log):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import oracle
    from paper_2305_08819_b200 import build, dp
    build.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % _free_port(), rank=0, world_size=1,
                            device_id=dev)
    try:
        B = 64
        step = dp.ConvNetStep("resnet18", B, dev, math="3xtf32", seed=3, bucket_mb=1.0)
        assert len(step.buckets) > 3  # several buckets, so the per-layer issue order is exercised
        step.step(None)
        torch.cuda.synchronize()
        ref_flat = step.dw_flat.clone()
        step.dw_flat.fill_(float("nan"))
        step.step(dist.group.WORLD)
        torch.cuda.synchronize()
        assert torch.equal(step.dw_flat, ref_flat)
        for i, b in enumerate(step.bufs):
            l = b.layer
            X, dY = b.X.cpu().numpy(), b.dY.cpu().numpy()
            ref = oracle.conv2d_bwd_filter(X, dY, (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw))
            got = b.dW.cpu().numpy().astype(np.float64)
            e = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
            parity_log.append({"config": "resnet18-b%d-nccl1" % B, "layer": l.name, "op": "dw", "math": "3xtf32",
                               "check": "random", "coverage": "whole tensor after NCCL all-reduce",
                               "normwise": e, "tol": 1e-5, "plan": ""})
            assert e <= 1e-5, (l.name, e)
    finally:
        dist.destroy_process_group()
