"""Data-parallel host logic on CPU with the gloo backend, world_size 2 (north_star (e)).

Each rank takes its shard of a seeded batch, computes its partial dW of every layer of a small
conv stack with the CPU oracle (test infrastructure), writes them into the backward-ordered flat
buffer of paper_2305_08819_b200.dp, and all-reduces the buckets (SUM, async handles) exactly
as the GPU step does with NCCL.  The result must equal the oracle's full-batch dW: bit-exact on
integer inputs (reading L10: SUM, not mean)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_08819_b200 import dp, nets, synth

LAYERS = [nets.L("a", 6, 8, 8), nets.L("b", 6, 8, 16, s=2), nets.L("c", 3, 16, 16, k=1), nets.L("d", 3, 16, 8)]
BATCH = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(integer):
    out = []
    for i, l in enumerate(LAYERS):
        g = synth.rng(77, i)
        X = synth.activations(g, BATCH, l.IH, l.IW, l.IC, integer=integer)
        dY = synth.activations(g, BATCH, l.OH, l.OW, l.OC, integer=integer)
        out.append((X, dY))
    return out


def _worker(rank, world, port, integer, bucket_elems, q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = dp.shard_range(BATCH, world, rank)
    sizes = [l.OC * l.FH * l.FW * l.IC for l in LAYERS]
    offs = dp.flat_offsets_backward(sizes)
    flat = torch.zeros(sum(sizes), dtype=torch.float32)
    buckets = dp.plan_buckets(sizes, bucket_elems)
    handles = []
    data = _inputs(integer)
    for i in reversed(range(len(LAYERS))):       # backward order, like ConvNetStep.step
        l = LAYERS[i]
        X, dY = data[i]
        dW = oracle.conv2d_bwd_filter(X[lo:hi], dY[lo:hi], (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw))
        flat[offs[i]:offs[i] + sizes[i]] = torch.from_numpy(dW.astype(np.float32).ravel())
        handles += dp.allreduce_buckets(flat, buckets, dist.group.WORLD, ready_layer=i)
    for h in handles:
        h.wait()
    if rank == 0:
        q.put(flat.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("integer,bucket_elems", [(1, 1 << 30), (1, 700), (0, 1000)])
def test_gloo_world2_dw_allreduce_equals_full_batch(integer, bucket_elems):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, integer, bucket_elems, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = [l.OC * l.FH * l.FW * l.IC for l in LAYERS]
    offs = dp.flat_offsets_backward(sizes)
    data = _inputs(integer)
    for i, l in enumerate(LAYERS):
        X, dY = data[i]
        ref = oracle.conv2d_bwd_filter(X, dY, (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw))
        g = got[offs[i]:offs[i] + sizes[i]].astype(np.float64)
        if integer:
            assert np.array_equal(g, ref.ravel()), l.name
        else:
            assert np.max(np.abs(g - ref.ravel())) <= 1e-5 * np.max(np.abs(ref))


def test_bucket_plan_covers_flat_buffer():
    sizes = [l.OC * l.FH * l.FW * l.IC for l in nets.resnet18()]
    for lim in (1, 1 << 18, 1 << 22, 1 << 40):
        b = dp.plan_buckets(sizes, lim)
        assert b[0][1] == 0 and b[-1][2] == sum(sizes)
        for (i, s, e), (j, s2, e2) in zip(b, b[1:]):
            assert e == s2 and i > j
    offs = dp.flat_offsets_backward(sizes)
    assert offs[len(sizes) - 1] == 0 and offs[0] == sum(sizes) - sizes[0]
    assert dp.shard_range(4096, 8, 3) == (1536, 2048)
    with pytest.raises(ValueError):
        dp.shard_range(100, 8, 0)
