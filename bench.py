#!/usr/bin/env python3
"""bench.py — throughput of the oriented 1D depthwise conv training step on B200.

A "step" = one pass of the whole hot path over one batch:
forward (x -> y), backward_input (dy -> dx), backward_weight (x, dy -> dW), and,
at N > 1 GPUs, the NCCL all-reduce of dW (row a8).  Workload = BASELINE.json
configs[1], the ConvNeXt-T-1D stage-1 layer: N=64, C=96, 56x56, K=31, 8 angles
cycled over channels; synthetic seeded inputs (paper_2309_15812_b200/inputs.py).

metric/value: algorithmic HBM bytes of the step (each pass reads its inputs and
writes its outputs once: 3 x 154.2 MB fp32) divided by the device time, summed
over ranks (weak scaling: every rank runs the full configs[1] batch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype f32|bf16] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU) and fails loudly when fewer than N
GPUs are visible.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "oriented 1D dwconv fwd+bwd HBM GB/s vs peak; ConvNeXt-T-1D train imgs/s 1-8 GPU"
PASSES = ("forward", "backward_input", "backward_weight")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--flags", type=int, default=0, help="o1d_desc.flags (1 = force generic kernels)")
    ap.add_argument("--angle", type=float, default=None,
                    help="give every channel this single angle (per-angle uniformity runs) instead of D=8")
    ap.add_argument("--dirs", type=int, default=None, help="number of directions D (default: the workload's 8)")
    ap.add_argument("--K", type=int, default=None, help="kernel length (experiments; default: the workload's 31)")
    ap.add_argument("--workload", default="s1", choices=["s1", "pp_main", "pp_res", "ks"],
                    help="s1 = BASELINE configs[1] (default); pp_main / pp_res = the 1D++ block's K=15 main and "
                         "C=384 residual oriented convs (SURVEY NEXT-3); ks = configs[2], the kernel-length sweep "
                         "(N=128, C=384, 14x14, K from --K) with a KxK depthwise conv2d comparator")
    ap.add_argument("--disc", default="rotation", choices=["rotation", "shear", "bilinear"],
                    help="tap discretisation: rotation (Def. 1), shear (Appendix, P:386-440) or bilinear (P:309-311)")
    ap.add_argument("--fused", type=int, default=None,
                    help="1: the step's backward is the fused single pass (o1d_backward, NEXT-2); default: the library's")
    ap.add_argument("--model", default=None, choices=["convnext_t_1d", "convnext_b_1d"],
                    help="time the ConvNeXt-1D training step (images/s) instead of the layer step")
    ap.add_argument("--batch", type=int, default=None, help="per-GPU batch for --model (default 128 T / 64 B)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary bf16 measurement")
    return ap.parse_args()


def layer_config(wl, args, world):
    """`config` of the layer-step line, identical for both arms (--impl ours / reference)."""
    return {"workload": wl.name, "N_per_gpu": wl.N, "C": wl.C, "H": wl.H, "W": wl.W, "K": wl.K,
            "angles": (f"D={wl.D} {wl.assign}" if args.angle is None else f"all {args.angle} deg"),
            "discretization": args.disc, "stride": 1, "layout": "NCHW", "dtype": args.dtype,
            "parallelism": f"dp{world} (batch-sharded, all-reduce of dW)",
            "l2": "inputs > L2: 2 rotating buffer sets of 4 x 77 MB"}


def relaunch_distributed(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (one rank per GPU)."""
    import socket

    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible on this host\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def algorithmic_bytes(wl, es):
    """Bytes each pass must move: read inputs once, write outputs once."""
    x = wl.N * wl.C * wl.H * wl.W * es
    y = wl.N * wl.C * wl.H * wl.W * es  # P = H, Q = W at stride 1
    wb = wl.C * wl.K * 4
    return {"forward": x + wb + y, "backward_input": y + wb + x, "backward_weight": x + y + wb}


def algorithmic_fmas(wl):
    return wl.N * wl.C * wl.H * wl.W * wl.K  # dense taps per output (zero padding is free in smem)


def bilinear_fmas(wl, angles):
    """FMAs per pass of the bilinear discretisation (reading R14): every output takes each
    DISTINCT neighbour offset of its channel's weighted taps once (the four corners of each tap with a
    non-zero weight, coincident corners of consecutive taps merged) -- from the library's host tap
    generator (o1d_make_bilinear), the same count the generated kernels hold (31 / 71 / 67 / 71 per
    channel at K=31 for 0 / 22.5 / 45 / 67.5 deg)."""
    import numpy as np

    from paper_2309_15812_b200 import binding as B
    h0, w0, fa, fb = B.make_bilinear(wl.K, angles)
    tot = 0
    for c in range(h0.shape[0]):
        offs = set()
        for k in range(wl.K):
            for dh, wa in ((0, 1 - fa[c, k]), (1, fa[c, k])):
                for dw, wb in ((0, 1 - fb[c, k]), (1, fb[c, k])):
                    if np.float32(wa * wb) != 0:
                        offs.add((int(h0[c, k]) + dh, int(w0[c, k]) + dw))
        tot += len(offs)
    return wl.N * wl.H * wl.W * tot


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [c.strip() for c in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(pass_name):
    """DRAM bytes per launch of `pass_name` from the committed ncu capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            v = json.load(f).get(pass_name)
        return float(v) if v is not None else None
    except Exception:
        return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_steps(wl, dtype_name, n, threads, target_s):
    """Whole 3-pass layer steps of the oracle on n samples until target_s elapsed."""
    import numpy as np

    import oracle
    from oracle import taps as T
    from paper_2309_15812_b200 import inputs

    angles = T.direction_angles(wl.D, wl.C, wl.assign)
    oh, ow = (np.array(a, np.int32) for a in T.taps_table(wl.K, wl.pad, angles))
    x = inputs.activation((n, wl.C, wl.H, wl.W), 0, dtype_name).astype(np.float64)
    dy = inputs.activation((n, wl.C, wl.H, wl.W), 2, dtype_name).astype(np.float64)
    w = inputs.weights(wl.C, wl.K, 1).astype(np.float64)
    steps = 0
    t0 = time.perf_counter()
    while True:
        oracle.forward(x, w, oh, ow, 1, threads)
        oracle.backward_input(dy, w, oh, ow, wl.H, wl.W, 1, threads)
        oracle.backward_weight(x, dy, oh, ow, 1, threads)
        steps += 1
        el = time.perf_counter() - t0
        if el >= target_s or steps >= 100000:
            return steps, el


def cpu_baseline(wl, dtype_name, target_s=12.0, full=True):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload
    (SURVEY 8(d).5): all threads on the workload (the headline `value`), and -- with full --
    one thread, the fp32-accumulator build, and the K-sweep config at K=31."""
    from dataclasses import replace

    import oracle
    from paper_2309_15812_b200 import inputs

    es = 4 if dtype_name == "f32" else 2
    th = max(1, oracle.max_threads())
    n = min(wl.N, 16)
    steps, el = _oracle_steps(wl, dtype_name, n, th, target_s)
    bytes_step = sum(algorithmic_bytes(replace(wl, N=n), es).values())
    out = {"value": bytes_step * steps / el / 1e9, "unit": "GB/s", "cores": th, "kind": "oracle",
           "cpu": cpu_model(),
           "sample": f"{steps} steps of the 3-pass layer step at N={n} (of {wl.N}), C={wl.C}, {wl.H}x{wl.W}, "
                     f"K={wl.K}, f64 accumulation, {th} threads, {el:.1f} s"}
    if full:
        variants = {}
        n1 = 1
        s1, e1 = _oracle_steps(wl, dtype_name, n1, 1, target_s / 4)
        variants["1_thread"] = {"value": sum(algorithmic_bytes(replace(wl, N=n1), es).values()) * s1 / e1 / 1e9,
                                "cores": 1, "sample": f"{s1} steps at N={n1}, {e1:.1f} s"}
        oracle.use_variant("f32acc")
        try:
            s2, e2 = _oracle_steps(wl, dtype_name, n, th, target_s / 4)
        finally:
            oracle.use_variant("f64")
        variants["f32_accumulate"] = {"value": bytes_step * s2 / e2 / 1e9, "cores": th,
                                      "sample": f"{s2} steps at N={n}, fp32 accumulators, {e2:.1f} s"}
        ks = inputs.ksweep(31)
        nk = 8
        s3, e3 = _oracle_steps(ks, dtype_name, nk, th, target_s / 4)
        variants["ksweep_k31"] = {"value": sum(algorithmic_bytes(replace(ks, N=nk), es).values()) * s3 / e3 / 1e9,
                                  "cores": th, "sample": f"{s3} steps of configs[2] K=31 at N={nk}, {e3:.1f} s"}
        out["variants"] = variants
    return out


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from paper_2309_15812_b200 import inputs
    wl = inputs.ksweep(args.K or 31) if args.workload == "ks" else inputs.WORKLOADS[args.workload]
    cb = cpu_baseline(wl, args.dtype, target_s=max(2.0, 60.0 / max(1, args.steps + args.warmup)), full=False)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded SplitMix64 U[-1,1))",
            "config": layer_config(wl, args, args.gpus),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def ffma_peak():
    """Measured FP32 FMA peak (TFLOP/s) of this pool's B200 (profiles/r2/ffma_peak.json,
    tools/ffma2_bench.cu), else the nominal 148 SMs x 128 FMA/clk x 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "ffma_peak.json")) as f:
            d = json.load(f)
        return float(d["ffma_tflops"]), "measured (profiles/r2/ffma_peak.json, tools/ffma2_bench.cu)"
    except Exception:
        return 2 * 148 * 128 * 1.965e9 / 1e12, "nominal (148 SMs x 128 FMA/clk x 1.965 GHz)"


def run_model(args):
    """ConvNeXt-1D synthetic training step (fwd + cross-entropy + bwd + AdamW), bf16
    activations, fp32 oriented-conv weights; DDP (NCCL) over the ranks at N > 1."""
    import torch
    import torch.distributed as dist

    from paper_2309_15812_b200 import convnext1d

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B = args.batch or (128 if args.model == "convnext_t_1d" else 64)
    torch.manual_seed(0)
    model = convnext1d.ConvNeXt1D(args.model).to(dev).to(torch.bfloat16)
    for m in convnext1d.oriented_layers(model):
        m.weight.data = m.weight.data.float()  # the library takes fp32 weights
    if world > 1:
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4)
    g = torch.Generator(device=dev).manual_seed(rank)
    imgs = [torch.randn(B, 3, 224, 224, device=dev, generator=g).to(torch.bfloat16) for _ in range(2)]
    labels = [torch.randint(0, 1000, (B,), device=dev, generator=g) for _ in range(2)]

    def step(i):
        opt.zero_grad(set_to_none=True)
        out = model(imgs[i & 1])
        loss = torch.nn.functional.cross_entropy(out.float(), labels[i & 1])
        loss.backward()
        opt.step()
        return loss

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0.record()
    for i in range(args.steps):
        loss = step(i)
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    t = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    n_or = len(convnext1d.oriented_layers(model))
    line = {"metric": METRIC, "value": B * world / (ms * 1e-3), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (N(0,1) images, random labels, random-init weights)",
            "config": {"workload": f"{args.model}_train_step", "global_batch": B * world, "per_gpu_batch": B,
                       "image": 224, "oriented_layers": n_or, "optimizer": "AdamW",
                       "parallelism": f"ddp{world} (NCCL all-reduce of every gradient incl. dW)"},
            "clocks": ck, "loss": float(loss.item())}
    if rank == 0 and world == 1:
        # share of the step's GPU kernel time in liboriented1d's kernels (torch.profiler, 2 steps
        # after the timed region)
        try:
            with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
                for i in range(2):
                    step(i)
                torch.cuda.synchronize()
            tot = ours = 0.0
            for e in prof.events():
                if e.device_type == torch.autograd.DeviceType.CUDA:
                    dt_ = getattr(e, "device_time_total", 0.0)
                    tot += dt_
                    if "o1d" in e.name:
                        ours += dt_
            line["oriented_share"] = {"kernel_time_frac": ours / tot if tot else None,
                                      "oriented_ms_per_step": ours / 2 / 1e3, "kernel_ms_per_step": tot / 2 / 1e3,
                                      "how": "torch.profiler CUDA kernel time, kernels of liboriented1d vs all"}
        except Exception as ex_:  # pragma: no cover
            line["oriented_share"] = {"error": repr(ex_)}
        # comparator: the same network with torch's 1xK depthwise conv2d (cuDNN) in
        # place of every oriented layer, timed the same way
        try:
            del opt, model
            torch.cuda.empty_cache()
            ref = convnext1d.ConvNeXt1D(args.model, impl="torch1xk").to(dev).to(torch.bfloat16)
            ropt = torch.optim.AdamW(ref.parameters(), lr=1e-4)

            def rstep(i):
                ropt.zero_grad(set_to_none=True)
                torch.nn.functional.cross_entropy(ref(imgs[i & 1]).float(), labels[i & 1]).backward()
                ropt.step()
            for i in range(args.warmup):
                rstep(i)
            torch.cuda.synchronize()
            t0.record()
            for i in range(args.steps):
                rstep(i)
            t1.record()
            torch.cuda.synchronize()
            rms = t0.elapsed_time(t1) / args.steps
            line["comparator"] = {"what": "same network, torch depthwise conv2d 1xK (cuDNN) instead of the oriented layers",
                                  "images_per_s": B / (rms * 1e-3), "ms_per_step": rms,
                                  "oriented_over_1xk": (B / (ms * 1e-3)) / (B / (rms * 1e-3))}
        except Exception as ex_:  # pragma: no cover
            line["comparator"] = {"error": repr(ex_)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2309_15812_b200 import binding as B
    from paper_2309_15812_b200 import dp, inputs

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[args.dtype]
    es = 4 if args.dtype == "f32" else 2
    wl = inputs.ksweep(args.K or 31) if args.workload == "ks" else inputs.WORKLOADS[args.workload]
    from dataclasses import replace
    if args.dirs is not None:
        wl = replace(wl, D=args.dirs)
    if args.K is not None:
        wl = replace(wl, K=args.K)
    angles = B.direction_angles(wl.D, wl.C, wl.assign)
    if args.angle is not None:
        angles = np.full(wl.C, float(args.angle))
    if args.fused is not None:
        os.environ["O1D_FUSED"] = str(args.fused)
    plan = B.Plan(wl.N, wl.C, wl.H, wl.W, wl.K, angles, dtype=tdt, flags=args.flags, device=dev,
                  discretization=args.disc)
    plan_ms, cache_hit = plan.stats()
    fused_step = "step=fused" in plan.describe()
    # two rotating buffer sets so every pass streams from HBM (each set 4 x 77 MB > L2)
    sets = []
    for s in range(2):
        x = torch.from_numpy(inputs.activation(plan.x_shape(), 0 + 10 * s, args.dtype)).to(dev, tdt)
        dy = torch.from_numpy(inputs.activation(plan.y_shape(), 2 + 10 * s, args.dtype)).to(dev, tdt)
        sets.append({"x": x, "dy": dy, "y": torch.empty_like(dy), "dx": torch.empty_like(x)})
    w = torch.from_numpy(inputs.weights(wl.C, wl.K, 1)).to(dev)
    dW = torch.empty_like(w)
    ws = B.workspace(plan)
    stream = torch.cuda.current_stream()
    NPASS = ("forward", "backward_input", "backward_weight", "backward_fused")

    def step(i, ev=None):
        b = sets[i & 1]
        if ev is None:
            B.step(plan, b["x"], w, b["dy"], b["y"], b["dx"], dW, ws)  # o1d_step: passes overlap
            if world > 1:
                dp.allreduce_weight_grad(dW)  # row a8: NCCL sum of the weight gradient over NVLink
            return
        ev[0].record(stream)
        B.forward(plan, b["x"], w, b["y"])
        ev[1].record(stream)
        B.backward_input(plan, b["dy"], w, b["dx"])
        ev[2].record(stream)
        B.backward_weight(plan, b["x"], b["dy"], dW, ws)
        ev[3].record(stream)
        B.backward(plan, b["x"], b["dy"], w, b["dx"], dW, ws)
        ev[4].record(stream)

    for i in range(args.warmup):
        step(i)
    # the fused backward is compiled on its first use: warm it (and every separate pass) up
    # outside the timed regions
    step(0, [torch.cuda.Event(enable_timing=True) for _ in range(5)])
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for i in range(args.steps):
        step(i)  # the step as a user runs it (o1d_step: one call, passes overlap)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-pass times (the roofline of the dominant kernel): the same passes as separate calls
    # with CUDA events between them, timed in a second loop (each kernel in isolation)
    for i in range(args.steps):
        step(i, evs[i])
    torch.cuda.synchronize()
    # ... and each pass as a stream of back-to-back launches of that kernel alone (alternating
    # the two buffer sets, > L2): the mean launch duration, each launch's set-up overlapping its
    # predecessor's tail through programmatic dependent launch, as inside a training step
    stream_ms = {}
    for p in NPASS:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            b = sets[i & 1]
            if p == "forward":
                B.forward(plan, b["x"], w, b["y"])
            elif p == "backward_input":
                B.backward_input(plan, b["dy"], w, b["dx"])
            elif p == "backward_weight":
                B.backward_weight(plan, b["x"], b["dy"], dW, ws)
            else:
                B.backward(plan, b["x"], b["dy"], w, b["dx"], dW, ws)
        e1.record(stream)
        torch.cuda.synchronize()
        stream_ms[p] = e0.elapsed_time(e1) / args.steps
    ck = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    per_pass_iso = {p: 0.0 for p in NPASS}
    for e in evs:
        for j, p in enumerate(NPASS):
            per_pass_iso[p] += e[j].elapsed_time(e[j + 1])
    per_pass = {p: stream_ms[p] * args.steps for p in NPASS}  # totals over the steps, as per_pass_iso
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    ab = algorithmic_bytes(wl, es)
    # fused backward: reads x and dy once, writes dx (+ w read, dW written): 3 planes per (n, c)
    plane_b = wl.N * wl.C * wl.H * wl.W * es
    ab["backward_fused"] = 3 * plane_b + 2 * wl.C * wl.K * 4
    bytes_step = sum(ab[p] for p in PASSES)  # the step's algorithmic bytes (three-pass accounting)
    value = bytes_step * args.steps * world / (max_ms * 1e-3) / 1e9
    ms_step = max_ms / args.steps
    peak, peak_src = measured_peaks()
    timed = ("forward", "backward_fused") if fused_step else PASSES
    dom = max(timed, key=lambda p: per_pass[p])
    dom_ms = per_pass[dom] / args.steps
    achieved = ab[dom] / (dom_ms * 1e-3) / 1e9
    launches = (plan.launches_per_call(0) + (plan.launches_per_call(3) if fused_step else
                                            plan.launches_per_call(1) + plan.launches_per_call(2))) * args.steps
    fpk, fpk_src = ffma_peak()
    # bilinear: four weighted corners per tap, the arithmetic intensity is past the FFMA/HBM ridge
    fmas_pass = bilinear_fmas(wl, angles) if args.disc == "bilinear" else algorithmic_fmas(wl)

    # end to end through the C ABI with pinned HOST buffers (H2D + 3 passes + D2H per step)
    e2e = None
    if not args.no_e2e:
        xh = sets[0]["x"].cpu().pin_memory()
        dyh = sets[0]["dy"].cpu().pin_memory()
        wh = w.cpu().pin_memory()
        yh, dxh, dWh = torch.empty_like(dyh).pin_memory(), torch.empty_like(xh).pin_memory(), torch.empty_like(wh).pin_memory()
        dws = B.step_host_workspace(plan)
        for _ in range(2):
            B.step_host(plan, xh, wh, dyh, yh, dxh, dWh, dws)
        n_e2e = max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(n_e2e):
            B.step_host(plan, xh, wh, dyh, yh, dxh, dWh, dws)
        t1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": bytes_step * n_e2e * world / (float(te.item()) * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(xh.numel() * xh.element_size() + dyh.numel() * dyh.element_size()
                                         + wh.numel() * 4),
               "d2h_bytes_per_step": int(yh.numel() * yh.element_size() + dxh.numel() * dxh.element_size()
                                         + dWh.numel() * 4),
               "steps": n_e2e, "path": "o1d_step_host (pinned host buffers, one C-ABI call per step)"}

    extra = {}
    if rank == 0:
        extra["per_pass_ms"] = {p: per_pass[p] / args.steps for p in NPASS}
        extra["per_pass_timing"] = ("mean launch duration over --steps back-to-back launches of the pass alone "
                                    "(CUDA events around the loop; PDL overlaps each launch's set-up with the "
                                    "previous tail); per_pass_ms_isolated: one launch between two events")
        extra["per_pass_ms_isolated"] = {p: per_pass_iso[p] / args.steps for p in NPASS}
        extra["per_pass_gbs"] = {p: ab[p] / (per_pass[p] / args.steps * 1e-3) / 1e9 for p in NPASS}
        extra["per_pass_frac_of_hbm"] = {p: extra["per_pass_gbs"][p] / peak for p in NPASS}
        extra["per_pass_frac_of_ffma"] = {p: (2 if p == "backward_fused" else 1) * 2 * fmas_pass /
                                          (per_pass[p] / args.steps * 1e-3) / 1e12 / fpk for p in NPASS}
        extra["ffma_peak_tflops"] = {"value": fpk, "source": fpk_src}
        extra["algorithmic_bytes"] = ab
        extra["fp32_tflops_dense"] = 3 * 2 * fmas_pass / (ms_step * 1e-3) / 1e12
        extra["imgs_per_s_layer_step"] = wl.N * world / (ms_step * 1e-3)
        extra["plan"] = plan.describe()
        extra["plan_create_ms"] = plan_ms
        extra["plan_jit_cache_hit"] = cache_hit
        extra["step_backward"] = "fused single pass (o1d_backward)" if fused_step else "backward_input + backward_weight"
        if args.workload == "ks":
            # configs[2] "vs equivalent kxk depthwise (linear-cost check)": torch conv2d (cuDNN),
            # groups=C, K x K, same activations, forward + both gradients -- a library comparator
            xk = sets[0]["x"].detach().clone().requires_grad_(True)
            wk = torch.randn(wl.C, 1, wl.K, wl.K, device=dev, dtype=tdt, requires_grad=True)
            gk = sets[0]["dy"]

            def kxk():
                yk = torch.nn.functional.conv2d(xk, wk, padding=wl.K // 2, groups=wl.C)
                yk.backward(gk)
            for _ in range(3):
                kxk()
            torch.cuda.synchronize()
            t0k, t1k = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nk = 10
            t0k.record(stream)
            for _ in range(nk):
                kxk()
            t1k.record(stream)
            torch.cuda.synchronize()
            extra["comparator"] = {"what": f"torch conv2d depthwise {wl.K}x{wl.K} fwd+bwd (cuDNN), same shape",
                                   "ms_per_step": t0k.elapsed_time(t1k) / nk, "ours_ms_per_step": ms_step,
                                   "ours_speedup": (t0k.elapsed_time(t1k) / nk) / ms_step}
    bound_alu = args.dtype != "f32" or args.disc == "bilinear"
    roof = {"kernel": dom, "unit": "GB/s", "algorithmic_bytes_per_launch": ab[dom], "peak_source": peak_src,
            "timing": "mean launch duration, back-to-back launches of the kernel (see per_pass_timing)",
            "frac_isolated": ab[dom] / (per_pass_iso[dom] / args.steps * 1e-3) / 1e9 / peak}
    if bound_alu:
        # 16-bit activations (15.5 flop/B) and the bilinear taps (~31 flop/B at fp32, 60 distinct
        # offsets per output): past the FFMA/HBM ridge -> FFMA bound
        fl = (2 if dom == "backward_fused" else 1) * 2 * fmas_pass / (dom_ms * 1e-3) / 1e12
        roof.update({"bound": "alu", "achieved": fl, "peak": fpk, "unit": "TFLOP/s", "frac": fl / fpk,
                     "peak_source": fpk_src, "hbm_gbs": achieved, "hbm_frac": achieved / peak, "traffic": None})
    else:
        roof.update({"bound": "hbm", "achieved": achieved, "peak": peak, "frac": achieved / peak,
                     "traffic": ncu_traffic(dom) if args.angle is None and args.disc == "rotation" else None,
                     "traffic_source": "profiles/traffic.json (ncu --set full, fp32 S1)"})
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded SplitMix64 U[-1,1))",
        "config": layer_config(wl, args, world),
        "roofline": roof,
        "gpu_launches": launches, "clocks": ck, "e2e": e2e,
    }
    line.update(extra)
    if rank == 0 and world == 1 and not args.no_cpu:  # the oracle baseline: rank 0 at N=1 only
        try:
            line["cpu_baseline"] = cpu_baseline(wl, args.dtype)
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(ex)}

    def sub(extra_args, timeout):
        out = subprocess.run([sys.executable, os.path.abspath(__file__)] + extra_args, capture_output=True, text=True,
                             timeout=timeout, env={**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": str(local)})
        return json.loads(out.stdout.strip().splitlines()[-1])
    # single-GPU extras (bf16, bilinear, the model step) on the N=1 line only: the scaling runs stay short
    if rank == 0 and world == 1 and not args.no_extra and args.dtype == "f32":
        common = ["--steps", str(args.steps), "--warmup", str(args.warmup), "--no-e2e", "--no-cpu", "--no-extra",
                  "--flags", str(args.flags)]
        for key, ex in (("bf16", ["--dtype", "bf16"]), ("bilinear", ["--disc", "bilinear"])):
            try:
                b = sub(ex + common, 600)
                line[key] = {k: b[k] for k in ("value", "ms_per_step", "roofline", "per_pass_ms", "per_pass_gbs",
                                               "per_pass_frac_of_hbm", "per_pass_frac_of_ffma", "plan_create_ms")}
            except Exception as ex_:  # pragma: no cover
                line[key] = {"error": repr(ex_)}
        try:
            m = sub(["--model", "convnext_t_1d", "--steps", "10", "--warmup", "3"], 900)
            line["convnext_t_1d_train"] = {k: m[k] for k in ("value", "unit", "ms_per_step", "config") if k in m}
            for k in ("oriented_share", "comparator"):
                if k in m:
                    line["convnext_t_1d_train"][k] = m[k]
        except Exception as ex_:  # pragma: no cover
            line["convnext_t_1d_train"] = {"error": repr(ex_)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.model:
        return run_model(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
