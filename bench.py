#!/usr/bin/env python
"""Benchmark of the B200 space-time multiplexing path (BASELINE.json metric).

Metric: packed multi-tenant conv TFLOP/s vs time-/space-only; p99 query latency.
Workload (BASELINE.json configs[1]): 4 tenants x ResNet-50@224 conv layers + fc
per GPU, batch 8 per tenant query, bf16 in / fp32 accumulate, synthetic data.
A step = one space-time round: every tenant submits one query batch, the
scheduler forms super-kernels layer by layer, each runs as one sm_100a launch.

  python bench.py [--gpus N --steps K --warmup W]          # our B200 path
  python bench.py --impl reference [...]                  # reference CPU arm

Multi-GPU (torchrun): tenant-sharded, no collective on the hot path; each rank
serves its own tenants (weak scaling); timing is on-device, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tenants", type=int, default=4, help="tenants per GPU")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--image", type=int, default=224)
    ap.add_argument("--table1", default="2,4,8,10,16,20,32,40,64,80,100,120",
                    help="R values of the conv2_2 microbench sweep ('' to skip)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--csv", default="", help="also write the reference's CSV v1 rows (report.py) to this path")
    ap.add_argument("--extra", default="mix,bert",
                    help="extra BASELINE configs at N=1: mix (configs[2]) and bert (configs[3]); '' to skip")
    ap.add_argument("--total-tenants", type=int, default=64,
                    help="BASELINE configs[4]: this many ResNet-50 tenants placed across the job's GPUs "
                         "(strong scaling), served per GPU; 0 = skip")
    ap.add_argument("--serve-seconds", type=float, default=1.5,
                    help="real-clock serving run per load point (0 = skip the serving section)")
    ap.add_argument("--slo", type=float, default=0.040, help="query SLO (s) of the serving run")
    ap.add_argument("--max-waves", type=int, default=1,
                    help="planner wave cap per super-kernel (1 = reference plan parity; >1 = b200 extension)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def model_layers(name, image):
    from paper_1901_00041_b200 import workload as W
    if name in ("resnet50", "resnet18", "vgg16"):
        return getattr(W, name)(image)
    return W.MODELS[name]()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    """Samples SM clocks and throttle reasons DURING the timed region: NVML
    every 10 ms when available (the timed regions are short), else
    `nvidia-smi -lms 200` (the profiling recipe's clocks line)."""

    NVML_REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(handle, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        self.nvml.append((pynvml.nvmlDeviceGetClockInfo(handle, pynvml.NVML_CLOCK_SM), mx,
                                          pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(handle)))
                    except Exception:
                        pass
                    self.stop.wait(0.01)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if self.nvml:
            sm = sorted(s for s, _, _ in self.nvml)
            reasons = sorted(n for n, bit in self.NVML_REASONS.items() if any(r & bit for _, _, r in self.nvml))
            return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.nvml[0][1], "reasons": reasons,
                    "samples": len(sm), "source": "nvml 10 ms"}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def nearest_rank(values, pct):
    from paper_1901_00041_b200.scheduler import percentile_nearest_rank
    return percentile_nearest_rank(values, pct)


def time_graph(torch, graph, stream, steps, flush=None, isolate=False):
    """Per-step device times (ms) of `steps` replays, plus first-to-last span.
    ``isolate``: synchronize the host before each step, so a step's time never
    includes the host still submitting a wide graph (many parallel branches)."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        t0.record(stream)
        for a, b in ev:
            if flush is not None:
                flush()
            if isolate:
                stream.synchronize()
            a.record(stream)
            graph.launch(stream.cuda_stream)
            b.record(stream)
        t1.record(stream)
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in ev]
    return per, t0.elapsed_time(t1)


def graph_name(args):
    return f"{args.model}_{args.image}"


def load_graph(args):
    """The tenant graph as plain data (oracle/graphs/*.json, exported from the
    product's workload builders and pinned to them by tests/test_workload.py):
    the reference arm and the CPU baseline read it without importing the
    product package."""
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import cpu_conv  # test infra: CPU baseline / reference arm only
    return cpu_conv.load_graph(graph_name(args))


def workload_desc(args, graph):
    """config.workload, identical in both arms (same_config)."""
    convs = sum(L["kind"] == "conv" for L in graph)
    return (f"{args.tenants} tenants/GPU x {args.model}@{args.image} dataflow graph ({len(graph)} ops: {convs} convs, "
            f"pools, residual adds, fc), batch {args.batch} per tenant query (BASELINE configs[1])")


def cpu_graph(args, graph):
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import cpu_conv  # test infra: CPU baseline / reference arm only
    return cpu_conv.CpuGraph(graph, args.batch), cpu_conv.threads()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference's own CPU path on this box's host cores.

    The reference artifact computes no tensors (it is a roofline simulator),
    so its CPU implementation of the path is: the reference planner
    (oracle/_ref/libgpumux_ref.so, the unmodified gpumux_core) forming the
    round's super-kernels over the tenant graph's GEMM shapes (the reference's
    own im2col lowering, gemm.hpp:44-56), plus the fp32 CPU port of the
    members' math (oracle/cpu_conv.py CpuGraph: the same dataflow graph) on all
    host threads.  Each step is a bounded sample: one tenant's full pass at the
    configured batch.  Nothing here imports the product package.
    """
    import ctypes
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    graph = load_graph(args)
    ref_path = os.path.join(HERE, "oracle", "_ref", "libgpumux_ref.so")
    planner_ok = os.path.exists(ref_path)
    if planner_ok:
        ref = ctypes.CDLL(ref_path)
        ref.gm_ref_call.restype = ctypes.c_char_p
        ref.gm_ref_call.argtypes = [ctypes.c_char_p]

        def call(req):
            return json.loads(ref.gm_ref_call(json.dumps(req).encode()))

        shapes = []
        for L in graph:
            if L["kind"] == "gemm":
                shapes.append([L["rows"] * args.batch, L["n"], L["k"]])
                continue
            H, W_, R, S, Cin, Cout, st, pad = L["conv"]
            m, n, k = call({"op": "im2col", "conv": [H, W_, R, S, Cin, Cout, st, pad]})["shape"]
            if L["kind"] != "conv":
                k = R * S  # per-channel ops: the reference's K = R*S model (workload.cpp:66)
            shapes.append([m * args.batch, n, k])  # batch_inputs (gemm.hpp:54-56)
    port, cores = cpu_graph(args, graph)
    steps = []
    total = args.warmup + args.steps
    for i in range(total):
        t0 = time.perf_counter()
        if planner_ok:  # one round of the reference planner over the configured tenants
            call({"op": "run_space_time", "tenants": args.tenants * args.gpus, "layers": shapes,
                  "duration": 1e-3, "microbench": False, "scheduler": {"target_batch": 0}})
        port.run_pass()
        if i >= args.warmup:
            steps.append(time.perf_counter() - t0)
    mean_s = sum(steps) / len(steps)
    value = port.flops_pass / mean_s / 1e12
    kind = "reference" if planner_ok else "port"
    line = {
        "impl": "reference", "metric": "packed multi-tenant conv TFLOP/s vs time-/space-only; p99 query latency",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_desc(args, graph)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"one {args.model}@{args.image} b{args.batch} tenant pass per step "
                                   f"({port.flops_pass / 1e9:.1f} GFLOP, numpy fp32 dataflow graph) + reference "
                                   f"planner round (oracle/_ref run_space_time)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test aid: GM_BENCH_SHARE_GPU=1 runs every rank on cuda:0 with gloo for
    # the timing reductions (exercises the N>1 path on a one-GPU box; the
    # timings are contended and not a scaling measurement)
    share = os.environ.get("GM_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_1901_00041_b200.engine import SpaceTimeEngine
    from paper_1901_00041_b200 import workload as W

    burst, sustained, hbm, peak_src = load_peaks()
    layers = model_layers(args.model, args.image)
    T = args.tenants
    eng = SpaceTimeEngine([layers] * T, [args.batch] * T, device_index=local, tenant_offset=rank * T)
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if share else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_1901_00041_b200.scheduler import BatchPolicy
    # The reference planner exactly (one-wave cap per super-kernel, plan parity).
    rnd = eng.plan_round(BatchPolicy(target_batch=0, max_waves=args.max_waves))
    # headline: the round program (all of the round's super-kernels in one
    # persistent launch, per-tenant layer dependencies on device)
    g_packed = eng.capture_round(rnd)
    tile_info = rnd.tile_info()
    # the reference's literal dispatch unit: one launch per formed super-kernel
    g_parity = eng.capture_packed(rnd)
    g_timed = eng.capture_round(rnd, timed=True)  # event pair around the round kernel
    g_time = eng.capture_serial("time_only")
    g_space = eng.capture_serial("space_only")
    flops_round = eng.flops_per_round()

    for g in (g_packed, g_parity, g_time, g_space, g_timed):
        for _ in range(args.warmup):
            g.launch(stream.cuda_stream)
    torch.cuda.synchronize()

    results = {}
    with ClockSampler(local) as clocks:
        for name, g in (("packed", g_packed), ("packed_per_plan", g_parity), ("time_only", g_time),
                        ("space_only", g_space)):
            barrier()
            per, span = time_graph(torch, g, stream, args.steps)
            barrier()
            span = max_over_ranks(span)
            results[name] = {"ms_per_step": span / args.steps, "per_step_ms": per, "launches": g.kernels}
        # dominant kernel: the round-program super-kernel, timed by an external
        # event pair captured around it on its launch stream, K replays
        round_ms = []
        for _ in range(args.steps):
            g_timed.launch(stream.cuda_stream)
            round_ms += g_timed.kernel_times_ms()
    sk_avg = [sum(round_ms) / len(round_ms)]

    # e2e through the public serving call with pinned host buffers
    h_in = [m.query_input.cpu().pin_memory() for m in eng.models]
    h_out = [torch.empty_like(m.query_output, device="cpu").pin_memory() for m in eng.models]
    for _ in range(args.warmup):
        eng.serve_round(h_in, h_out, stream)
    # the e2e program is captured once the plan is steady; keep warming until
    # then so no capture lands inside the timed region (bounded)
    for _ in range(20):
        if eng.e2e_steady(h_in, h_out):
            break
        eng.serve_round(h_in, h_out, stream)
    eng.serve_round(h_in, h_out, stream)
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        eng.serve_round(h_in, h_out, stream)
        e2e_times.append(time.perf_counter() - t0)
    barrier()
    e2e_sync_s = max_over_ranks(sum(e2e_times) / len(e2e_times))
    # back-to-back rounds through the double-buffered public call: two sets of
    # pinned host batches alternating, every step's H2D and D2H inside the
    # timed region (pipeline fill and drain included)
    h_in2 = [h.clone().pin_memory() for h in h_in]
    h_out2 = [torch.empty_like(h).pin_memory() for h in h_out]
    sets = [(h_in, h_out), (h_in2, h_out2)]
    eng.serve_rounds([sets[i & 1] for i in range(max(args.warmup, 2))], stream)
    barrier()
    t0 = time.perf_counter()
    eng.serve_rounds([sets[i & 1] for i in range(args.steps)], stream)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    barrier()
    h2d = sum(t.numel() * t.element_size() for t in h_in)
    d2h = sum(t.numel() * t.element_size() for t in h_out)

    bytes_round = eng.compulsory_bytes_per_round()
    # Real-clock serving (dynamic batcher + round programs + CUDA-event completions)
    serving = None
    if args.serve_seconds > 0:
        serving = run_serving(args, layers, local, rank, world, dist if world > 1 else None)

    extra = {}
    if (args.extra and rank == 0 and world == 1) or args.total_tenants > 0:
        del eng
        torch.cuda.empty_cache()
    if args.extra and rank == 0 and world == 1:
        for name in args.extra.split(","):
            extra[name] = {"mix": run_mix, "bert": run_bert}[name](torch, args, dev, stream)

    # Table-1 analogue: R tenants x conv2_2 (256,128,1152) b1, L2 flushed between steps
    table1 = None
    if args.table1 and rank == 0 and world == 1:
        rs = [int(r) for r in args.table1.split(",")]
        table1 = run_table1(torch, rs, dev, stream)
        table1["other_presets"] = {p: run_table1(torch, rs, dev, stream, p) for p in ("rnn-matvec", "square-256")}

    # BASELINE configs[4]: the fixed tenant total placed across the job's GPUs
    c5 = None
    if args.total_tenants > 0 and args.serve_seconds > 0:
        try:
            c5 = run_c5(torch, args, dev, rank, world, dist if world > 1 else None)
        except Exception as e:  # reported in the line; the headline stands
            c5 = {"error": f"{type(e).__name__}: {e}"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    tf = lambda ms: world * flops_round / (ms / 1e3) / 1e12  # noqa: E731
    packed = results["packed"]
    value = tf(packed["ms_per_step"])
    p99 = nearest_rank(packed["per_step_ms"], 99.0)
    # Roofline of the dominant kernel (the round-program super-kernel, one
    # launch per round).  Algorithmic work per launch: FLOPs = sum 2*M*N*K over
    # every member; bytes = compulsory implicit-GEMM bf16 traffic (input +
    # weights + output per member).  At batch 8 the round's
    # intensity (FLOPs/bytes) is below the ridge point, so HBM is the binding
    # roof; the tensor view is reported beside it.
    round_s = sk_avg[0] / 1e3
    achieved_gbs = bytes_round / round_s / 1e9
    achieved = flops_round / round_s / 1e12
    traffic = None
    prof = os.path.join(HERE, "profiles", "superkernel_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    attain_s = sum(max(L.flops(args.batch) / (burst * 1e12), L.compulsory_bytes(args.batch) / (hbm * 1e9))
                   for L in layers) * T
    cpu = None
    graph = load_graph(args)
    if world == 1:
        port, cores = cpu_graph(args, graph)
        cpu_tf, reps_cpu, el = port.sample(args.cpu_seconds)
        cpu = {"value": cpu_tf, "unit": "TFLOP/s", "cores": cores, "kind": "port",
               "sample": f"{reps_cpu} x one {args.model}@{args.image} b{args.batch} tenant pass "
                         f"(numpy fp32 dataflow graph, im2col+BLAS, oracle/cpu_conv.py), {el:.1f} s"}
    line = {
        "metric": "packed multi-tenant conv TFLOP/s vs time-/space-only; p99 query latency",
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": packed["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (U(-1,1) inputs, Kaiming-normal weights, seed 42)",
        "config": {
            "workload": workload_desc(args, graph),
            "tenants_per_gpu": T, "batch": args.batch, "placement": "tenant-sharded, no collective",
            "planner": f"space-time form_batches (max_waves={args.max_waves}; 1 = reference plan parity); "
                       f"packed = round program (1 persistent launch/round), modes.packed_per_plan = 1 launch "
                       f"per formed super-kernel",
            "superkernels_per_round": len(rnd.kernels),
            "planner_tiles_per_round": sum(k.planned_cost.blocks for k in rnd.kernels),
            "tiles_executed_per_round": len(tile_info),
            "executed_tile_variants": {"tall_256_rows": sum(t["rows"] == 256 for t in tile_info),
                                       "narrow_n": sum(t["cols"] < 256 and not t["cuda_core"] for t in tile_info),
                                       "split_k": sum(t["splits"] > 1 for t in tile_info),
                                       "cuda_core": sum(t["cuda_core"] for t in tile_info)},
            "l2": f"inputs larger than L2 ({bytes_round / 1e6:.0f} MB compulsory/round)",
        },
        "modes": {
            name: {"tflops": tf(r["ms_per_step"]), "ms_per_step": r["ms_per_step"], "launches_per_step": r["launches"],
                   "p99_ms": nearest_rank(r["per_step_ms"], 99.0)}
            for name, r in results.items()
        },
        "packed_over_space_only": results["space_only"]["ms_per_step"] / packed["ms_per_step"],
        "packed_over_time_only": results["time_only"]["ms_per_step"] / packed["ms_per_step"],
        "p99_query_latency_ms": serving["poisson_50pct"]["p99_ms"] if serving else p99,
        "p99_note": ("real-clock serving, Poisson arrivals at 50% of saturated load, SLO-bound dynamic batching "
                     "(see serving)") if serving else "round-program step time",
        "roofline": {
            "bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": achieved_gbs / hbm,
            "traffic": traffic, "algorithmic_bytes_per_launch": bytes_round,
            "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "kernel": "gmb::dev::superkernel<256> (round program)", "launches_per_round": 1,
            "avg_launch_us": round_s * 1e6, "timing": f"CUDA events around the round kernel, {len(round_ms)} replays",
            "tensor_view": {"achieved_tflops": achieved, "peak_tflops": burst,
                            "frac_of_dense_bf16": achieved / burst,
                            "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops; the round "
                                           f"kernel is timed alone)"},
            "attainable_tflops": flops_round / attain_s / 1e12 if attain_s else None,
            "frac_of_attainable": achieved / (flops_round / attain_s / 1e12) if attain_s else None,
            "attainable_note": "per-layer max(F/P_burst, B/BW) summed over the round",
        },
        "e2e": {"value": world * flops_round / e2e_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                "api": "SpaceTimeEngine.serve_rounds: K back-to-back rounds from pinned host batches (two sets "
                       "alternating), double-buffered: a second registration of the tenants with its own query "
                       "inputs and results alternates with the first, so step i+1's H2D and step i-1's D2H (two "
                       "copy streams) overlap round i; every step's H2D, round program and D2H inside the timed "
                       "wall-clock region",
                "single_round": {"value": world * flops_round / e2e_sync_s / 1e12, "ms_per_step": e2e_sync_s * 1e3,
                                 "median_ms": sorted(e2e_times)[len(e2e_times) // 2] * 1e3,
                                 "min_ms": min(e2e_times) * 1e3,
                                 "api": "SpaceTimeEngine.serve_round, one synchronous round per call (one graph: "
                                        "per-tenant H2D gating its chain in the round kernel, D2H)"}},
        "gpu_launches": args.steps * g_packed.kernels,
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if table1 is not None:
        line["table1"] = table1
    if serving is not None:
        line["serving"] = serving
    for name, sec in extra.items():
        line["config_" + name] = sec
    if c5 is not None:
        line["config_c5"] = c5
    print(json.dumps(line), flush=True)
    if args.csv:
        from paper_1901_00041_b200 import report
        report.write_csv(args.csv, report.bench_rows(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


SERVE_KEEP = ("tflops", "qps", "p50_ms", "p99_ms", "max_ms", "slo_violation_frac", "queries", "rounds",
              "mean_queries_per_round", "mean_round_ms", "plan_hits", "plan_misses", "plan_fallbacks",
              "plan_evictions", "plan_padded", "plans_cached", "evicted", "h2d_bytes", "d2h_bytes")


def serve_session(eng, seconds, rank, world, dist, **kw):
    """One timed gm_serve run (after a short warm-up run that fills the plan
    cache and pages in the path); stats summed / latencies merged over ranks
    (one all-gather after the run, off the hot path; nearest-rank p99)."""
    eng.serve(duration=0.3, warmup=0.1, seed=1, **kw)
    if dist is not None:
        dist.barrier()
    r = eng.serve(duration=seconds, warmup=min(0.2, seconds / 4), seed=42 + rank, **kw)
    st = {k: r.stats[k] for k in SERVE_KEEP}
    lat = r.latencies_ms
    if dist is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, (lat, st))
        lat = [x for g, _ in gathered for x in g]
        per = [s2 for _, s2 in gathered]
        q = sum(s2["queries"] for s2 in per)
        st = dict(per[0], tflops=sum(s2["tflops"] for s2 in per), qps=sum(s2["qps"] for s2 in per), queries=q,
                  slo_violation_frac=sum(s2["slo_violation_frac"] * s2["queries"] for s2 in per) / q if q else None,
                  h2d_bytes=sum(s2["h2d_bytes"] for s2 in per), d2h_bytes=sum(s2["d2h_bytes"] for s2 in per))
        if lat:
            st.update(p50_ms=nearest_rank(lat, 50.0), p99_ms=nearest_rank(lat, 99.0), max_ms=max(lat))
    return st


def serve_points(factory, seconds, rank=0, world=1, dist=None, slo_mults=(2.0, 4.0), **kw):
    """Closed-loop saturation, Poisson at 50% / 80% of the saturated query
    rate under the tenants' own SLOs, and SLO-bound points: Poisson at 80%
    with every SLO set to each of ``slo_mults`` x the saturated mean round
    time (2x: about one round of queueing plus the query's own round, so the
    batcher's SLO trigger fires and violations are counted; 4x: a binding SLO
    the loop can hold).  Queries carry data (per-query H2D / D2H inside the
    serving loop)."""
    sat = serve_session(factory(None, None), seconds, rank, world, dist, **kw)
    pts = {"closed_loop": sat}
    for f in (0.5, 0.8):
        pts[f"poisson_{int(f * 100)}pct"] = dict(serve_session(factory(f * sat["qps"], None), seconds, rank, world,
                                                               dist, **kw), load=f)
    for i, mult in enumerate(slo_mults):
        slo = mult * sat["mean_round_ms"] / 1e3
        key = "slo_bound_80pct" if i == 0 else f"slo_bound_80pct_{mult:g}x"
        pts[key] = dict(serve_session(factory(0.8 * sat["qps"], slo), seconds, rank, world, dist, **kw),
                        load=0.8, slo_ms=slo * 1e3, slo_mult=mult)
    return pts


def run_serving(args, layers, local, rank, world, dist):
    """Real-clock serving of the headline tenants through gm_serve (the B200
    form of run_space_time) on every rank: closed loop at saturation, Poisson
    at 50% / 80% of that rate (SLO --slo), and an SLO-bound point (SLO = 2 x
    the saturated round time).  Query latency = completion - arrival
    (queueing + batching wait + input copy + execution + result copy)."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    T = args.tenants

    def factory(total_qps, slo):
        rate = 0.0 if total_qps is None else total_qps / (T * world)
        specs = [ServeTenant(layers, max_batch=args.batch, rate_qps=rate, concurrency=args.batch,
                             slo_latency=slo or args.slo, io_slots=2 * args.batch) for _ in range(T)]
        return ServingEngine(specs, device_index=local, tenant_offset=rank * T)

    pts = serve_points(factory, args.serve_seconds, rank, world, dist)
    return dict({"api": "ServingEngine.serve -> gm_serve (C++ real-clock loop: arrivals, dynamic batcher, "
                        "per-query H2D / D2H, round-program dispatch, CUDA-event completions)",
                 "slo_ms": args.slo * 1e3, "max_batch": args.batch, "seconds_per_point": args.serve_seconds},
                **pts)


def run_c5(torch, args, dev, rank, world, dist):
    """BASELINE configs[4]: --total-tenants ResNet-50 tenants placed across the
    job's GPUs (placement.place_tenants: LPT by FLOPs, tenant-sharded, no
    collective; strong scaling: the total is fixed), each GPU serving its
    shard through gm_serve with dynamic batching (variants 1/2/4/8, bounded
    plan cache, background planning of new member sets), Poisson arrivals at
    50% of the closed-loop saturated rate under an SLO of 2x the saturated
    round time.  p99 is the nearest rank over every GPU's queries."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    from paper_1901_00041_b200.placement import place_tenants, tenants_of
    layers = W.resnet50(224)
    total = args.total_tenants
    demand = [(sum(L.flops(args.batch) for L in layers), sum(L.compulsory_bytes(args.batch) for L in layers))] * total
    mine = tenants_of(rank, place_tenants(demand, world))

    def factory(total_qps, slo):
        rate = 0.0 if total_qps is None else total_qps / total
        specs = [ServeTenant(layers, max_batch=args.batch, batches=[1, 2, 4, 8], rate_qps=rate,
                             concurrency=args.batch, slo_latency=slo or args.slo, io_slots=2 * args.batch)
                 for _ in mine]
        return ServingEngine(specs, device_index=dev.index, tenant_offset=mine[0] if mine else 0)

    kw = dict(prewarm=1, plan_cache_cap=256, async_plan=True)
    sat = serve_session(factory(None, None), args.serve_seconds, rank, world, dist, **kw)
    slo = 2.0 * sat["mean_round_ms"] / 1e3
    half = serve_session(factory(0.5 * sat["qps"], slo), args.serve_seconds, rank, world, dist, **kw)
    return {"workload": f"{total} tenants x resnet50@224 placed across {world} GPU(s) (BASELINE configs[4]): "
                        f"tenant-sharded, {len(mine)} on GPU {rank}; dynamic batching up to {args.batch} "
                        "(variants 1/2/4/8); data-bearing queries",
            "scaling": "strong (total tenants fixed)", "tenants_per_gpu": len(mine),
            "closed_loop": sat, "poisson_50pct_slo_bound": dict(half, slo_ms=slo * 1e3, load=0.5),
            "p99_ms": half["p99_ms"]}


def round_modes(torch, eng, stream, steps, warmup=3):
    """Packed round program vs time-only vs space-only over one engine's tenants."""
    rnd = eng.plan_round()
    gs = {"packed": eng.capture_round(rnd), "time_only": eng.capture_serial("time_only"),
          "space_only": eng.capture_serial("space_only")}
    out = {"superkernels_per_round": len(rnd.kernels), "tiles_per_round": sum(k.planned_cost.blocks for k in rnd.kernels),
           "gflop_per_round": eng.flops_per_round() / 1e9}
    for name, g in gs.items():
        for _ in range(warmup):
            g.launch(stream.cuda_stream)
        per, span = time_graph(torch, g, stream, steps)
        ms = span / steps
        out[name] = {"tflops": eng.flops_per_round() / (ms / 1e3) / 1e12, "ms_per_step": ms,
                     "p99_ms": nearest_rank(per, 99.0), "launches_per_step": g.kernels}
    out["packed_over_space_only"] = out["space_only"]["ms_per_step"] / out["packed"]["ms_per_step"]
    out["packed_over_time_only"] = out["time_only"]["ms_per_step"] / out["packed"]["ms_per_step"]
    # the packed round against its rooflines (same definitions as the headline's)
    burst, _, hbm, _ = load_peaks()
    attain_s = sum(max(L.flops(m.batch) / (burst * 1e12), L.compulsory_bytes(m.batch) / (hbm * 1e9))
                   for m in eng.models for L in m.layers)
    tf = out["packed"]["tflops"]
    out["roofline"] = {"frac_of_dense_bf16_burst": tf / burst, "attainable_tflops": eng.flops_per_round() / attain_s / 1e12,
                       "frac_of_attainable": tf / (eng.flops_per_round() / attain_s / 1e12),
                       "hbm_gbs": eng.compulsory_bytes_per_round() / (out["packed"]["ms_per_step"] / 1e3) / 1e9,
                       "frac_of_hbm": eng.compulsory_bytes_per_round() / (out["packed"]["ms_per_step"] / 1e3) / 1e9 / hbm}
    return out


def run_mix(torch, args, dev, stream):
    """BASELINE configs[2]: ResNet-50 + VGG-16 + MobileNet-v2 tenants (two each)
    at 224, different layer lists in one round program (MobileNet's depthwise
    layers are the super-kernel's CUDA-core tile type); round modes at batch
    4, then real-clock serving with Poisson arrivals and dynamic batching
    (max batch 8 in variants 2 and 8, SLOs 40/60/20 ms)."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine, SpaceTimeEngine
    models = [("resnet50", W.resnet50(224), 0.040), ("vgg16", W.vgg16(224), 0.060),
              ("mobilenet_v2", W.mobilenet_v2(224), 0.020)] * 2
    eng = SpaceTimeEngine([m[1] for m in models], [4] * len(models), device_index=dev.index)
    rm = round_modes(torch, eng, stream, max(5, args.steps // 2))
    del eng

    def factory(total_qps, slo):
        specs = []
        for _, layers, own_slo in models:
            rate = 0.0 if total_qps is None else total_qps / len(models)
            specs.append(ServeTenant(layers, max_batch=8, rate_qps=rate, concurrency=8, slo_latency=slo or own_slo,
                                     batches=[2, 8], io_slots=16))
        return ServingEngine(specs, device_index=dev.index)

    sv = serve_points(factory, max(0.5, args.serve_seconds)) if args.serve_seconds > 0 else None
    return {"workload": "2x resnet50 + 2x vgg16 + 2x mobilenet_v2 @224 (BASELINE configs[2]); round modes at "
                        "batch 4; serving: max batch 8 (variants 2/8), SLO 40/60/20 ms, Poisson at 50%/80% of "
                        "closed-loop saturation (equal per-tenant rates), SLO-bound point (2x round time); "
                        "data-bearing queries",
            "round_b4": rm, "serving": sv}


def run_bert(torch, args, dev, stream):
    """BASELINE configs[3]: 16 tenants x BERT-base projection/FFN GEMMs (12
    encoder layers: qkv, attn-out, ffn1, ffn2), seq 128, batch 1 and 4."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    out = {"workload": "16 tenants x BERT-base 12-layer projection/FFN GEMMs, seq 128 (BASELINE configs[3])"}
    for b in (1, 4):
        eng = SpaceTimeEngine([W.bert_base_gemms(128, layers=12)] * 16, [b] * 16, device_index=dev.index)
        out[f"batch{b}"] = round_modes(torch, eng, stream, max(5, args.steps // 2))
        del eng
    if args.serve_seconds > 0:
        from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
        layers = W.bert_base_gemms(128, layers=12)

        def factory(total_qps, slo):
            rate = 0.0 if total_qps is None else total_qps / 16
            specs = [ServeTenant(layers, max_batch=4, batches=[1, 2, 4], rate_qps=rate, concurrency=4,
                                 slo_latency=slo or 0.020, io_slots=8) for _ in range(16)]
            return ServingEngine(specs, device_index=dev.index)

        out["serving"] = serve_points(factory, max(0.5, args.serve_seconds), prewarm=1, plan_cache_cap=256,
                                      async_plan=True)
        out["serving_note"] = ("16 tenants, dynamic batch 1-4 (variants 1/2/4; 4^16 member sets: bounded plan "
                               "cache, new sets planned in the background), SLO 20 ms, data-bearing queries")
    return out


def run_table1(torch, rs, dev, stream, preset="resnet18-conv2_2"):
    """Paper Table 1 analogue on B200: R tenants each issuing one preset
    operator (b1); conv2_2 is the headline column, rnn-matvec and square-256
    the paper's other two."""
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    from paper_1901_00041_b200 import workload as W
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    rows = []
    for r in rs:
        eng = SpaceTimeEngine([W.table1_layers(preset)] * r, [1] * r, device_index=dev.index)
        flops = W.table1_flops(preset) * r  # the reference shape's FLOPs (rnn-matvec: N = 1)
        rnd = eng.plan_round()
        gs = {"packed": eng.capture_round(rnd), "time_only": eng.capture_serial("time_only"),
              "space_only": eng.capture_serial("space_only")}
        row = {"R": r, "superkernels": len(rnd.kernels)}
        for name, g in gs.items():
            for _ in range(3):
                g.launch(stream.cuda_stream)
            # each step isolated (host synchronized before it): back-to-back
            # replays of the space-only graph (R parallel branches) made its
            # per-step times bimodal (20-30 vs 180-190 TFLOP/s at R >= 64)
            # depending on how far host submission ran ahead; median of 30
            per, _ = time_graph(torch, g, stream, 30, flush=flush, isolate=True)
            ms = sorted(per)[len(per) // 2]
            row[name + "_tflops"] = flops / (ms / 1e3) / 1e12
        row["over_space_only"] = row["packed_tflops"] / row["space_only_tflops"]
        row["over_time_only"] = row["packed_tflops"] / row["time_only_tflops"]
        rows.append(row)
        del eng, gs
    from paper_1901_00041_b200.scheduler import geomean
    shape = {"resnet18-conv2_2": "conv2_2 (256,128,1152) as a 3x3 conv", "square-256": "square-256 GEMM (256,256,256)",
             "rnn-matvec": "rnn-matvec (512,1,512), computed at N = 8, FLOPs counted at N = 1"}[preset]
    return {"workload": shape + " b1 per tenant, L2 flushed between steps; median of 30 host-isolated steps per mode",
            "rows": rows,
            "geomean_over_space_only": geomean([r["over_space_only"] for r in rows]),
            "geomean_over_time_only": geomean([r["over_time_only"] for r in rows])}


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
