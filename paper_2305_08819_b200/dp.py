"""Batch-sharded data-parallel conv step (north_star (e)).

One process per GPU.  Rank r of g owns images [r*B/g, (r+1)*B/g) of the batch; the
filters are replicated.  Forward and deconvolution (dX) are per-image independent, so
they need no communication; dW is a sum over images, so the only collective is one
all-reduce(SUM, fp32) of dW (reading L10: SUM, so the result equals the full-batch dW).
All dW of the step live in ONE flat fp32 buffer in backward order, cut into buckets;
each bucket's all-reduce is issued (async, NCCL over NVLink/NVSwitch) as soon as the
last dW kernel writing into it has been enqueued, so it overlaps the rest of the
backward pass.

The network is a CONV-ONLY chain of the paper's CIFAR-10 layer shapes (nets.py):
  forward:  X_{l+1} = Y_l along the main path (a 1x1 stride-2 shortcut reads its block's
            input; its output ends there);
  backward: dY of the last conv is the synthetic loss gradient; dY_l = dX_{l+1} along the
            main path; a shortcut shares its block's output gradient.
BatchNorm / ReLU / residual adds / pooling are outside the hot path
and are not run; VGG's max-pools are replaced by fresh synthetic activations at each
stage start (its chain breaks there).  Every conv of the network runs exactly as in a
training step: fwd for all layers, dX for all but the stem, dW for all.
"""
from __future__ import annotations

import math as _math
from dataclasses import dataclass, field
from typing import List, Optional

from . import nets, synth
from . import smconv as sm


@dataclass
class LayerBuf:
    layer: nets.Layer
    X: object = None
    W: object = None
    Y: object = None
    dY: object = None
    dX: object = None
    dW: object = None          # view into the flat dW buffer
    x_src: int = -1            # index of the layer whose Y is this layer's X (-1: own buffer)
    dy_src: int = -1           # index of the layer whose dX is this layer's dY (-1: own buffer)
    dy_share: int = -1         # shortcut: shares dY with this layer
    ws: object = None
    ws_bytes: List[int] = field(default_factory=lambda: [0, 0, 0])


def shard_range(batch: int, world: int, rank: int):
    """Images [lo, hi) of the global batch owned by `rank` (contiguous equal shards)."""
    if batch % world:
        raise ValueError("global batch %d not divisible by %d ranks" % (batch, world))
    per = batch // world
    return rank * per, (rank + 1) * per


def flat_offsets_backward(sizes):
    """Offset of each layer's dW in the flat buffer laid out in BACKWARD (last layer first) order."""
    offs, o = {}, 0
    for i in reversed(range(len(sizes))):
        offs[i] = o
        o += sizes[i]
    return offs


def plan_buckets(sizes, bucket_elems):
    """Cut the backward-ordered flat dW buffer into buckets of >= bucket_elems elements (the last
    may be smaller).  Returns [(i, start, end)]: bucket [start, end) is complete once layer i's dW
    (the last layer of the bucket in backward order) has been written."""
    buckets, start, acc = [], 0, 0
    order = list(reversed(range(len(sizes))))
    for k, i in enumerate(order):
        acc += sizes[i]
        if acc - start >= bucket_elems or k == len(order) - 1:
            buckets.append((i, start, acc))
            start = acc
    return buckets


def allreduce_buckets(flat, buckets, pg, ready_layer=None):
    """Issue async SUM all-reduces (reading L10) of the buckets whose last layer is `ready_layer`
    (all buckets if None).  Returns the work handles."""
    import torch.distributed as dist
    hs = []
    for (i, s, e) in buckets:
        if ready_layer is None or i == ready_layer:
            hs.append(dist.all_reduce(flat[s:e], op=dist.ReduceOp.SUM, async_op=True, group=pg))
    return hs


def _chain_resnet(layers):
    """(x_src, dy_src, dy_share) per layer for the conv-only ResNet chain."""
    n = len(layers)
    x_src, dy_src, share = [-1] * n, [-1] * n, [-1] * n
    prev = -1            # layer whose Y is the current activation
    block_in = -1
    i = 0
    while i < n:
        name = layers[i].name
        if name.endswith("a"):
            block_in = prev
        if name.endswith("sc"):
            x_src[i] = block_in
            i += 1
            continue
        x_src[i] = prev
        prev = i
        i += 1
    # backward: dY_l = dX of the next main-path layer that consumes Y_l
    for j in range(n):
        for k in range(n):
            if x_src[k] == j and not layers[k].name.endswith("sc"):
                dy_src[j] = k
    for j in range(n):
        if layers[j].name.endswith("sc"):
            # shortcut output feeds the block output = conv b of the same block
            b = j + 1
            share[j] = b
    return x_src, dy_src, share


def _chain_vgg(layers):
    n = len(layers)
    x_src, dy_src, share = [-1] * n, [-1] * n, [-1] * n
    for i in range(1, n):
        if layers[i].IH == layers[i - 1].OH and layers[i].IC == layers[i - 1].OC:
            x_src[i] = i - 1
            dy_src[i - 1] = i
    return x_src, dy_src, share


class ConvNetStep:
    """Buffers + one fwd/bwd pass of a conv-only network on this rank's batch shard."""

    def __init__(self, net: str, batch: int, device, math: str = "3xtf32", seed: int = 0,
                 bucket_mb: float = 16.0, chain: bool = True, rank: int = 0, epi: bool = False,
                 leaky_k: float = 0.01, mcast_group=None, dw_stream: bool = False):
        import torch
        self.torch = torch
        self.net = net
        self.layers = nets.NETS[net]()
        self.batch = batch
        self.device = device
        self.math = sm.MATH[math]
        # fused epilogues (include/smconv_epi.h): every fwd also emits its BatchNorm statistics, every dX
        # applies the LeakyReLU backward (slope read from the layer's forward input A = X) and emits the
        # BN-backward statistics — the paper's leakyRelu(bn(conv(X))) block
        self.epi = epi
        self.leaky_k = leaky_k
        L = self.layers
        if chain and net.startswith("resnet18"):
            xs, ds, sh = _chain_resnet(L)
        elif chain and net == "vgg16":
            xs, ds, sh = _chain_vgg(L)
        else:
            xs, ds, sh = [-1] * len(L), [-1] * len(L), [-1] * len(L)
        self.bufs: List[LayerBuf] = []
        f32 = torch.float32
        # flat dW buffer in BACKWARD order (bucket = contiguous run of finished layers)
        sizes = [l.OC * l.FH * l.FW * l.IC for l in L]
        # fused dW all-reduce (include/smconv_mcast.h): dW lives in symmetric memory with an NVLink
        # multicast mapping; the dW kernels add each rank's shard into every rank's copy (no NCCL pass)
        self.mc_handle, self.mc_ptr = None, 0
        if mcast_group is not None:
            from torch.distributed import _symmetric_memory as symm
            if hasattr(symm, "enable_symm_mem_for_group"):
                symm.enable_symm_mem_for_group(mcast_group.group_name)
            self.dw_flat = symm.empty(sum(sizes), dtype=f32, device=device)
            self.mc_handle = symm.rendezvous(self.dw_flat, mcast_group.group_name)
            self.mc_ptr = int(getattr(self.mc_handle, "multicast_ptr", 0) or 0)
            if not self.mc_ptr:
                raise RuntimeError("fused dW all-reduce: no NVLink multicast object (multicast_ptr == 0)")
            self.dw_flat.zero_()
        else:
            self.dw_flat = torch.zeros(sum(sizes), dtype=f32, device=device)
        self.dw_offs = flat_offsets_backward(sizes)
        offs = flat_offsets_backward(sizes)
        for i, l in enumerate(L):
            b = LayerBuf(l, x_src=xs[i], dy_src=ds[i], dy_share=sh[i])
            # W replicated (rank-independent seed); X / dY differ per rank's batch shard
            X, Wt, dY = synth.torch_layer_inputs(l, batch, device, seed=seed * 1000 + i,
                                                 act_seed=(seed * 1000 + i) * 65537 + 7 * rank + 1)
            b.W = Wt
            if b.x_src < 0:
                b.X = X
            b.Y = torch.empty((batch, l.OH, l.OW, l.OC), dtype=f32, device=device)
            if i > 0:
                b.dX = torch.empty((batch, l.IH, l.IW, l.IC), dtype=f32, device=device)
            if b.dy_src < 0 and b.dy_share < 0:
                b.dY = dY
            b.dW = self.dw_flat[offs[i]:offs[i] + sizes[i]].view(l.OC, l.FH, l.FW, l.IC)
            self.bufs.append(b)
        for i, b in enumerate(self.bufs):
            if b.x_src >= 0:
                b.X = self.bufs[b.x_src].Y
        for i in reversed(range(len(L))):
            b = self.bufs[i]
            if b.dy_share >= 0:
                b.dY = self.bufs[b.dy_share].dY
            elif b.dy_src >= 0:
                b.dY = self.bufs[b.dy_src].dX
        # external inputs of the step (what a user would upload): chain heads and loss gradients
        self.inputs = [b.X for b in self.bufs if b.x_src < 0] + \
                      [b.dY for b in self.bufs if b.dy_src < 0 and b.dy_share < 0]
        # one split-K workspace shared by every call (they are stream-ordered), sized by the library
        for b in self.bufs:
            b.ws_bytes = [sm.workspace_bytes(op, b.layer.dims(batch), self.math) for op in range(3)]
            if self.mc_ptr:
                b.ws_bytes[2] = sm.mcast_workspace_bytes(b.layer.dims(batch), self.math)
            if epi:
                b.ws_bytes[0] = sm.epi_workspace_bytes(0, b.layer.dims(batch), self.math, "bn_stats")
                b.ws_bytes[1] = sm.epi_workspace_bytes(1, b.layer.dims(batch), self.math, "leaky_bwd_stats")
                b.stats_fwd = torch.zeros((2, b.layer.OC), dtype=torch.float64, device=device)
                b.stats_dx = torch.zeros((2, b.layer.IC), dtype=torch.float64, device=device)
        mx = max(max(b.ws_bytes) for b in self.bufs)
        ws = torch.empty(max(mx, 16), dtype=torch.uint8, device=device) if mx else None
        for b in self.bufs:
            b.ws = ws
        # dW on a second stream (dw_stream): dW_l needs only X_l and dY_l, nothing on the critical dX
        # chain needs it, so it runs beside the next dX calls (small-map layers leave SMs idle: 64-CTA
        # cluster grids, prologues, split-K tails).  Its calls get their own workspace.
        self.side = None
        self.ws_dw = None
        if dw_stream:
            self.side = torch.cuda.Stream(device=device)
            mdw = max(b.ws_bytes[2] for b in self.bufs)
            self.ws_dw = torch.empty(max(mdw, 16), dtype=torch.uint8, device=device) if mdw else None
        # buckets over the backward-ordered flat buffer
        self.buckets = plan_buckets(sizes, int(bucket_mb * (1 << 20) / 4))
        if self.mc_ptr:
            self.kernels_per_step = sum(
                sm.plan_kernels(0, b.layer.dims(batch), self.math)
                + int(sm.mcast_plan_describe(b.layer.dims(batch), self.math).rsplit("kernels=", 1)[1])
                + (sm.plan_kernels(1, b.layer.dims(batch), self.math) if k > 0 else 0)
                for k, b in enumerate(self.bufs))
        elif epi:
            self.kernels_per_step = sum(
                sm.epi_plan_kernels(0, b.layer.dims(batch), self.math, "bn_stats")
                + sm.plan_kernels(2, b.layer.dims(batch), self.math)
                + (sm.epi_plan_kernels(1, b.layer.dims(batch), self.math, "leaky_bwd_stats") if k > 0 else 0)
                for k, b in enumerate(self.bufs))
        else:
            self.kernels_per_step = sum(
                sm.plan_kernels(0, b.layer.dims(batch), self.math) + sm.plan_kernels(2, b.layer.dims(batch), self.math)
                + (sm.plan_kernels(1, b.layer.dims(batch), self.math) if k > 0 else 0)
                for k, b in enumerate(self.bufs))

    # ---------------------------------------------------------------- one step
    def _call(self, op, b: LayerBuf, a, bb, out, stream):
        ws = self.ws_dw if (op == 2 and self.side is not None) else b.ws
        if op == 2 and self.mc_ptr:  # dW + all-reduce in the dW kernels, into the multicast address
            i = self.bufs.index(b)
            sm.raw_call_mcast(a.data_ptr(), bb.data_ptr(), self.mc_ptr + 4 * self.dw_offs[i], b.layer.dims(self.batch),
                              self.math, ws.data_ptr() if (ws is not None and b.ws_bytes[2]) else 0,
                              b.ws_bytes[2] if ws is not None else 0, stream)
            return
        if self.epi and op != 2:
            ep = sm.EPI["bn_stats"] if op == 0 else sm.EPI["leaky_bwd_stats"]
            st = b.stats_fwd if op == 0 else b.stats_dx
            sm.raw_call_epi(op, a.data_ptr(), bb.data_ptr(), b.X.data_ptr(), out.data_ptr(), st.data_ptr(),
                            b.layer.dims(self.batch), self.math, ep, self.leaky_k,
                            ws.data_ptr() if (ws is not None and b.ws_bytes[op]) else 0,
                            b.ws_bytes[op] if ws is not None else 0, stream)
            return
        sm.raw_call(op, a.data_ptr(), bb.data_ptr(), out.data_ptr(), b.layer.dims(self.batch), self.math,
                    ws.data_ptr() if (ws is not None and b.ws_bytes[op]) else 0,
                    b.ws_bytes[op] if ws is not None else 0, stream)

    def step(self, pg=None, events: Optional[list] = None, external_events: bool = False, only=None,
             serial: bool = False):
        """Enqueue fwd for all layers, then dX/dW in reverse with bucketed async all-reduce.
        external_events: timing events that stay valid inside CUDA-graph capture.  serial: every call on
        the current stream even with dw_stream (per-call profiling: no kernel overlaps another)."""
        torch = self.torch
        stream = torch.cuda.current_stream(self.device).cuda_stream
        rec = events is not None

        def mark(key):
            # only: record just these (op, layer) calls (a CUDA event between two kernels also stops the
            # second one from being scheduled early: programmatic dependent launch, csrc/launch.cuh)
            if rec and (only is None or key[:2] in only):
                e = torch.cuda.Event(enable_timing=True, external=True) if external_events else \
                    torch.cuda.Event(enable_timing=True)
                e.record()
                events.append((key, e))

        for i, b in enumerate(self.bufs):
            mark(("fwd", i, 0))
            self._call(0, b, b.X, b.W, b.Y, stream)
            mark(("fwd", i, 1))
        handles = []
        if self.mc_ptr:
            # every rank's dW copy is zero before any rank adds into it (smconv_mcast.h contract)
            self.dw_flat.zero_()
            self.mc_handle.barrier()
        side = None if serial else self.side
        if side is not None:
            side.wait_stream(torch.cuda.current_stream(self.device))  # X of every layer, the loss gradients
        for i in reversed(range(len(self.bufs))):
            b = self.bufs[i]
            # dW first: its bucket's all-reduce (NCCL waits on this stream's work so far) then
            # overlaps this layer's dX and the rest of the backward pass
            if side is not None:
                side.wait_stream(torch.cuda.current_stream(self.device))  # dY_l (the previous dX)
                with torch.cuda.stream(side):
                    mark(("dw", i, 0))
                    self._call(2, b, b.X, b.dY, b.dW, side.cuda_stream)
                    mark(("dw", i, 1))
            else:
                mark(("dw", i, 0))
                self._call(2, b, b.X, b.dY, b.dW, stream)
                mark(("dw", i, 1))
            if pg is not None and not self.mc_ptr:
                if side is not None and any(r == i for (r, _, _) in self.buckets):
                    torch.cuda.current_stream(self.device).wait_stream(side)  # the bucket's dW are written
                handles += allreduce_buckets(self.dw_flat, self.buckets, pg, ready_layer=i)
            if i > 0:
                mark(("dx", i, 0))
                self._call(1, b, b.dY, b.W, b.dX, stream)
                mark(("dx", i, 1))
        if side is not None:
            torch.cuda.current_stream(self.device).wait_stream(side)
        for h in handles:
            h.wait()
        if self.mc_ptr:
            self.mc_handle.barrier()  # every rank's additions have landed before dW is read

    def flops(self, valid=True):
        tot = 0
        for k, b in enumerate(self.bufs):
            f = nets.flops(b.layer, self.batch, valid)
            tot += f * (3 if k > 0 else 2)
        return tot


def input_bytes(step: ConvNetStep) -> int:
    return sum(t.numel() * 4 for t in step.inputs)
