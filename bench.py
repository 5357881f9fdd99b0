#!/usr/bin/env python
"""bench.py — images/s of the conv fwd+bwd step of the paper's CIFAR-10 networks on B200.

Default workload (BASELINE.json configs[4], the metric's "images/s at 1/2/4/8 B200"):
ResNet-18 CIFAR-10 conv layers, fwd + deconv (dX) + dW, GLOBAL batch 4096 sharded over
the N ranks (strong scaling), dW all-reduced (SUM) over NCCL.  At N=1 this is the whole
4096-image step on one GPU.  One "step" = every conv of the network forward, then dX
(all but the stem) and dW in reverse (all §8(a) rows: A0-A8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                  [--net resnet18|vgg16|googlenet|alexnet] [--global-batch B] [--math 3xtf32|tf32]

Under torchrun (N>1) every rank runs its shard; rank 0 prints ONE JSON line.
`--impl reference` times the CPU oracle (the reference arm for this tier) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv TFLOP/s (fwd/dX/dW) on Cifar-10 layer shapes; images/s at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="smconv", choices=["smconv", "reference"])
    ap.add_argument("--net", default="resnet18")
    ap.add_argument("--global-batch", type=int, default=None)
    ap.add_argument("--math", default="3xtf32", choices=["3xtf32", "tf32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bucket-mb", type=float, default=16.0)
    ap.add_argument("--fused-allreduce", action="store_true",
                    help="dW all-reduce inside the dW kernels through an NVLink multicast object "
                         "(include/smconv_mcast.h; torch symmetric memory) instead of bucketed NCCL all-reduces")
    ap.add_argument("--epi", action="store_true",
                    help="fused epilogues (include/smconv_epi.h): fwd emits BatchNorm statistics, dX applies the "
                         "LeakyReLU backward and emits the BN-backward statistics (PAPER.md:52 block)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the timed steps as one CUDA graph, with programmatic dependent launch for every "
                         "kernel.  auto: on at 1 GPU below 1024 images per GPU (measured r02bt: VGG-16 b128 TF32 "
                         "0.79 -> 0.72 ms, 3xTF32 1.27 -> 1.24 ms, AlexNet b256 0.34 -> 0.28 ms: launch-bound small "
                         "calls; ResNet-18 b4096 unchanged, so it stays eager there)")
    ap.add_argument("--dw-stream", default="auto", choices=["auto", "on", "off"],
                    help="run every dW on a second stream beside the dX chain (dp.ConvNetStep dw_stream); "
                         "measured r02aa/r02z: VGG-16 b128 -4..5 %%, ResNet-18 b512 -4.3 %%, b4096 -0.4 %% step "
                         "time.  auto = on below 1024 images per GPU (at b4096 the gain is noise and the dominant "
                         "call's live duration would include its overlap with the dX kernels)")
    ap.add_argument("--layers-out", default=os.path.join(ROOT, "gpurun_out", "bench_layers.json"))
    a = ap.parse_args()
    if a.global_batch is None:
        a.global_batch = {"resnet18": 4096, "vgg16": 128, "googlenet": 256, "alexnet": 256, "resnet18@64": 1024,
                          "resnet18@128": 256, "resnet18@224": 64}.get(a.net, 512)
    return a


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        src = "measured"
    except Exception:
        src = "fallback"
    hbm = float(p.get("hbm_gbs", 6650.0))
    bf16 = float(p.get("bf16_tflops", 1590.0))
    bf16_s = float(p.get("bf16_tflops_sustained", 1400.0))
    # guide's nominal dense ratio tf32 : bf16 = 1.1 : 2.25 (B200_PROFILING.md)
    r = 1.1 / 2.25
    return {"src": src, "hbm_gbs": hbm, "tf32_burst": bf16 * r, "tf32_sustained": bf16_s * r}


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", "clocks_%d.csv" % os.getpid())

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + q, "--format=csv,noheader,nounits",
                                          "-i", ",".join(str(g) for g in self.gpus), "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1]))
                mx = float(c[2])
            except ValueError:
                continue
            for n, v in zip(names, c[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- oracle legs
def oracle_images_per_s(net, n_img, seed=0):
    """Run the CPU oracle over the conv-only chain of `net` for n_img images (fwd all layers,
    dX all but the stem, dW all); returns (seconds, threads)."""
    import numpy as np

    import oracle
    from paper_2305_08819_b200 import nets, synth
    L = nets.NETS[net]()
    X = {}
    t0 = time.perf_counter()
    g = synth.rng(5, 0, salt=seed)
    for i, l in enumerate(L):
        W = synth.filters(g, l.OC, l.FH, l.FW, l.IC, l.ic_logical)
        x = synth.activations(g, n_img, l.IH, l.IW, l.IC, l.ic_logical, stem=(i == 0))
        y = oracle.conv2d_fwd(x, W, (l.sh, l.sw), (l.ph, l.pw))
        X[i] = (x, W, y.astype(np.float32))
    for i in reversed(range(len(L))):
        l = L[i]
        x, W, y = X[i]
        dy = synth.activations(g, n_img, l.OH, l.OW, l.OC)
        if i > 0:
            oracle.conv2d_bwd_data(dy, W, (l.IH, l.IW), (l.sh, l.sw), (l.ph, l.pw))
        oracle.conv2d_bwd_filter(x, dy, (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw))
    return time.perf_counter() - t0, oracle.num_threads()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(net, target_s=15.0):
    """The oracle as it stands on ALL host cores (torchrun's OMP_NUM_THREADS=1 default overridden),
    plus a 1-core sample."""
    oracle_mod = __import__("oracle")
    oracle_mod.build()
    cores = host_cores()
    oracle_mod.set_num_threads(1)
    t1c, _ = oracle_images_per_s(net, 1, seed=3)
    oracle_mod.set_num_threads(cores)
    t1, thr = oracle_images_per_s(net, 1, seed=1)
    n = max(1, min(256, int(target_s / max(t1, 1e-3))))
    t, thr = oracle_images_per_s(net, n, seed=2)
    return {"value": n / t, "unit": "images/s", "cores": thr, "kind": "oracle",
            "value_1core": 1.0 / t1c,
            "sample": "%d image(s) through all %d %s convs (fwd, dX, dW; plain C double-accumulated "
                      "direct loops, OpenMP over outputs), %.1f s on %d threads; value_1core: 1 image on 1 thread "
                      "(%.1f s)" % (n, len(__import__("paper_2305_08819_b200.nets", fromlist=["x"]).NETS[net]()),
                                    net, t, thr, t1c)}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    oracle.set_num_threads(host_cores())  # the driver's torchrun launch sets OMP_NUM_THREADS=1
    per_step = 2
    t_first, thr = oracle_images_per_s(a.net, 1, seed=9)
    per_step = max(1, min(16, int(6.0 / max(t_first, 1e-3))))
    for w in range(a.warmup):
        oracle_images_per_s(a.net, per_step, seed=10 + w)
    times = []
    for k in range(a.steps):
        t, thr = oracle_images_per_s(a.net, per_step, seed=100 + k)
        times.append(t)
    tot = sum(times)
    v = per_step * a.steps / tot
    out = {"metric": METRIC, "value": v, "unit": "images/s", "n_gpus": a.gpus, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": 1000 * tot / a.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": "%s-cifar10 conv stack fwd+dX+dW, oracle sample %d img/step (of global batch %d)"
                                  % (a.net, per_step, a.global_batch), "global_batch": a.global_batch},
           "cpu_baseline": {"value": v, "unit": "images/s", "cores": thr, "kind": "oracle",
                            "sample": "%d image(s) per step through every %s conv" % (per_step, a.net)},
           "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------------- launcher
def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n):
    """`bench.py --gpus N` run without torchrun: start the N ranks ourselves (one process per GPU,
    torch.distributed.run on 127.0.0.1) with the same arguments; rank 0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: launching %d ranks: %s" % (n, " ".join(cmd)), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def _world1_group(dev):
    """A world-size-1 NCCL group for --fused-allreduce on one GPU (the multicast object then spans this GPU)."""
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    return dist.group.WORLD


# ---------------------------------------------------------------------- GPU arm
def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(a.gpus)
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    from paper_2305_08819_b200 import build, nets
    from paper_2305_08819_b200 import dp
    from paper_2305_08819_b200 import smconv as sm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE %d (launch with torchrun --nproc-per-node %d, or "
                         "without torchrun to let bench.py spawn the ranks)" % (a.gpus, world, a.gpus))
    if torch.cuda.device_count() < world:
        raise SystemExit("bench.py: %d ranks but only %d visible GPU(s)" % (world, torch.cuda.device_count()))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    if a.global_batch % world:
        raise SystemExit("global batch %d not divisible by %d ranks" % (a.global_batch, world))
    B = a.global_batch // world
    use_graph = a.graph == "on" or (a.graph == "auto" and world == 1 and B < 1024)
    # Programmatic dependent launch for every kernel when the step is a CUDA graph (launch.cuh: by default
    # only the plain-TF32 plans use it).  Same-box A/B, VGG-16 b128 3xTF32 (r02bt): eager 1.27 ms, eager +
    # PDL 1.34, graph 1.38, graph + PDL 1.24.  Set before the library's first launch reads SMCONV_PDL.
    pdl_note = os.environ.get("SMCONV_PDL")
    if use_graph and pdl_note is None:
        os.environ["SMCONV_PDL"] = "2"
    build.build()
    sm.lib()
    dw_stream = a.dw_stream == "on" or (a.dw_stream == "auto" and B < 1024)
    # filters replicated (rank-independent seed); activations / loss gradients differ per shard
    step = dp.ConvNetStep(a.net, B, dev, math=a.math, seed=1, bucket_mb=a.bucket_mb, rank=rank, epi=a.epi,
                          mcast_group=(pg if pg is not None else _world1_group(dev)) if a.fused_allreduce else None,
                          dw_stream=dw_stream)
    torch.cuda.synchronize()

    def barrier():
        if pg is not None:
            dist.barrier(device_ids=[local])

    for _ in range(a.warmup):
        step.step(pg)
    torch.cuda.synchronize()
    barrier()
    # per-call profile pass (untimed): events around every C-ABI call give the per-layer table and pick
    # the dominant call.  Inside the timed region only the dominant call is bracketed by events: an
    # event between two kernels serialises them (no programmatic dependent launch overlap) and adds its
    # own cost, so per-call events on every call would distort the step being measured.
    prof_events = []
    for _ in range(2):  # serial: per-call times of kernels that do not share the GPU with a dW stream
        step.step(pg, events=prof_events, serial=True)
    torch.cuda.synchronize()
    prof = {}
    pend = {}
    for key, ev in prof_events:
        if key[2] == 0:
            pend[key[:2]] = ev
        else:
            prof.setdefault(key[:2], []).append(pend.pop(key[:2]).elapsed_time(ev))
    top_key = max(prof, key=lambda k: sum(prof[k]) / len(prof[k]))
    barrier()

    clock = ClockSampler(list(range(world)) if rank == 0 else [])
    if rank == 0:
        clock.start()
        time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    events = []
    graph = None
    if use_graph:
        # the K timed steps captured as ONE CUDA graph (per-call timing events are event-record
        # nodes in it), so the host enqueues nothing per call inside the timed region
        try:
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                step.step(None)
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(a.steps):
                    step.step(None, events=events, external_events=True, only={top_key})
            torch.cuda.synchronize()
        except Exception as exc:  # graph capture unavailable: time the eager steps instead
            print("warning: CUDA graph capture failed (%s); timing eager steps" % exc, file=sys.stderr)
            graph, events = None, []
            torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph is not None:
        graph.replay()
    else:
        for _ in range(a.steps):
            step.step(pg, events=events, only={top_key})
    e1.record()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    clocks = clock.stop() if rank == 0 else None

    # the dominant call's duration inside the timed region (events on the launching stream); the other
    # calls' from the profile pass
    live = {}
    pend = {}
    for key, ev in events:
        k = key[:2]
        if key[2] == 0:
            pend[k] = ev
        else:
            live.setdefault(k, []).append(pend.pop(k).elapsed_time(ev))
    per = dict(prof)
    per.update(live)
    layer_rows = []
    P = peaks()

    def tensor_div(op, plan):
        # tensor-pipe cost per product in TF32-MMA units: 3xTF32 dW = 3 TF32 MMAs; 3xTF32 fwd / dX on the
        # TMA / STRIP variants = 1 TF32 MMA + 1 bf16 MMA of twice the K at twice the rate = 2
        hyb = (op != "dw" and ("variant=tma" in plan or "variant=strip" in plan) and " 3mma" not in plan) or \
            " hybw" in plan  # TMA dW with the bf16 cross terms (TmaParams::dw_hyb)
        return (2.0 if hyb else 3.0) if a.math == "3xtf32" else 1.0

    for (op, i), v in per.items():
        l = step.bufs[i].layer
        avg = sum(v) / len(v)
        fl = nets.flops(l, B, valid=True)
        by = nets.bytes_compulsory(l, B, op)
        plan = sm.plan_describe({"fwd": 0, "dx": 1, "dw": 2}[op], l.dims(B), step.math)
        # per-call rows: each call is timed alone in the serial profile pass (<= ~2 ms), so its tensor
        # peak is the burst figure (the sustained one, a cuBLAS bf16 GEMM held for seconds at the power
        # cap, sits below what short TF32 calls reach: 3xTF32 dW rows read up to 1.1 against it, r02bd)
        pk = P["tf32_burst"] / tensor_div(op, plan)
        # the layer's roofline time: max(flops / tensor peak, bytes / HBM peak); frac = that / measured
        t_roof = max(fl / (pk * 1e12), by / (P["hbm_gbs"] * 1e9)) * 1e3
        layer_rows.append({"op": op, "layer": l.name, "i": i, "ms": avg, "flops": fl, "bytes": by,
                           "timed": "live (timed region)" if (op, i) in live else "profile pass",
                           "tflops": fl / avg / 1e9, "gbs": by / avg / 1e6,
                           "bound": "tensor" if fl / (pk * 1e12) >= by / (P["hbm_gbs"] * 1e9) else "hbm",
                           "roofline_ms": t_roof, "frac": t_roof / avg, "plan": plan})
    layer_rows.sort(key=lambda r: -r["ms"])
    top = [r for r in layer_rows if (r["op"], r["i"]) == top_key][0]
    mathdiv = tensor_div(top["op"], top["plan"])
    peak_t = P["tf32_sustained"] / mathdiv
    ridge = peak_t * 1e12 / (P["hbm_gbs"] * 1e9)
    ai = top["flops"] / top["bytes"]
    if ai >= ridge:
        roof = {"bound": "tensor", "achieved": top["tflops"], "peak": peak_t, "unit": "TFLOP/s",
                "frac": top["tflops"] / peak_t}
    else:
        roof = {"bound": "hbm", "achieved": top["gbs"], "peak": P["hbm_gbs"], "unit": "GB/s",
                "frac": top["gbs"] / P["hbm_gbs"]}
    roof["traffic"] = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            key = "%s:%s:%s:b%d" % (a.net, top["layer"], top["op"], B)
            roof["traffic"] = tr.get(key)
        except Exception:
            pass
    roof["kernel"] = "%s %s (%s)" % (top["op"], top["layer"], top["plan"])
    roof["peak_src"] = "%s; TF32 = bf16_tflops_sustained x 1.1/2.25%s" % (
        P["src"], {3.0: " / 3 (3xTF32 dW issues 3 TF32 MMAs per product)",
                   2.0: " / 2 (3xTF32 hybrid: 1 TF32 MMA + 1 K-doubled bf16 MMA per product)"}.get(mathdiv, ""))
    roof["share_of_step"] = top["ms"] * a.steps / ms

    imgs = a.global_batch * a.steps
    value = imgs / (ms_max / 1000.0)
    out = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": "%s-cifar10 conv stack fwd+dX+dW (conv-only chain), global batch %d"
                                  % (a.net, a.global_batch),
                      "global_batch": a.global_batch, "per_gpu_batch": B, "math": a.math,
                      "fwd_dx_cross_terms": "bf16" if a.math == "3xtf32" else None,
                      "cross_terms": ("bf16 (1 TF32 + 1 K-doubled bf16 MMA per product): fwd/dX on TMA and STRIP, "
                                      "dW on TMA; strict 3xTF32 (3 TF32 MMAs): DWS / STEM / GENERIC dW")
                      if a.math == "3xtf32" else None,
                      "epilogue": ("fused: fwd + BN statistics, dX + LeakyReLU backward + BN-backward statistics"
                                   if a.epi else "none (plain conv outputs)"),
                      "cuda_graph": graph is not None, "dw_stream": dw_stream,
                      "pdl": {"0": "off", "1": "plain-TF32 plans", "2": "all kernels"}.get(
                          os.environ.get("SMCONV_PDL", "1"), os.environ.get("SMCONV_PDL")),
                      "parallelism": "dp%d" % world,
                      "dw_allreduce": ("fused in the dW kernels (NVLink multicast multimem.red)" if a.fused_allreduce
                                       else "NCCL all_reduce SUM, bucketed, async" if world > 1 else "none (1 GPU)"), "l2": "inputs larger than L2 (per-step working set "
                      "%.1f GB >> 126 MB)" % (sum(t.numel() for b in step.bufs for t in (b.X, b.Y) if t is not None)
                                              * 4 / 1e9),
                      "conv_tflops_valid": step.flops(True) * world / (ms_max / a.steps / 1000) / 1e12,
                      "conv_tflops_nominal": step.flops(False) * world / (ms_max / a.steps / 1000) / 1e12},
           "roofline": roof, "gpu_launches": step.kernels_per_step * a.steps, "clocks": clocks}

    # ---- e2e: host buffers through the public API, H2D of the step inputs + D2H of dW each step
    if not a.no_e2e:
        host_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in step.inputs]
        for h, t in zip(host_in, step.inputs):
            h.copy_(t)
        host_dw = torch.empty(step.dw_flat.shape, dtype=torch.float32, pin_memory=True)
        h2d = sum(h.numel() * 4 for h in host_in)
        d2h = host_dw.numel() * 4
        barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        g1 = None
        if graph is not None:  # one step per replay here: each step's H2D / D2H sit between replays
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1):
                step.step(None)
            torch.cuda.synchronize()
        f0.record()
        for _ in range(a.steps):
            for h, t in zip(host_in, step.inputs):
                t.copy_(h, non_blocking=True)
            if g1 is not None:
                g1.replay()
            else:
                step.step(pg)
            host_dw.copy_(step.dw_flat, non_blocking=True)
        f1.record()
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if pg is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["e2e"] = {"value": imgs / (float(t.item()) / 1000.0), "unit": "images/s",
                      "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world}

    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(a.net)
    if rank == 0:
        try:
            os.makedirs(os.path.dirname(a.layers_out), exist_ok=True)
            json.dump({"config": out["config"], "layer_peaks": {
                "tensor_tflops": P["tf32_burst"], "hbm_gbs": P["hbm_gbs"],
                "note": "frac = max(flops / tensor peak, bytes / HBM peak) / measured ms; tensor peak = TF32 burst "
                        "(bf16_tflops x 1.1/2.25) / 2 (3xTF32 fwd/dX hybrid) or / 3 (3xTF32 dW, 3mma fwd/dX)"},
                "layers": layer_rows}, open(a.layers_out, "w"), indent=1)
        except Exception:
            pass
        print(json.dumps(out), flush=True)
    if pg is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
