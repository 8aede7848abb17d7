#!/usr/bin/env python
"""Benchmark of the B200 SFT/ASFT hot path (driver contract).

Default workload = BASELINE.json's headline: the Morlet wavelet transform, method 1
(direct, MDS5P6 ASFT, fp32), N=102400, sigma=8192, xi=10 — one step = one transform of
one signal. ``--workload`` selects the other BASELINE configs (1, 2, 4, 5).

Arms:
  --impl ours (default)   the product: libsftgpu (K4 tensor-core / K1 scan kernels) through the C ABI.
  --impl reference        the reference's CPU path on all host threads: the reference
                          library compiled from its own sources (oracle/_ref, built by
                          oracle/ref.mk with a mini-Eigen shim), Recursive2 fp64 (its
                          bench default); the restated port in oracle/ if that build is absent.
Multi-GPU: one process per GPU (torchrun); single-signal workloads run independent
replicas ("replicas only"); the scalogram shards scales across ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 * 1024 * 1024
PAPER_MS = 0.545  # PAPER.md:28-30, RTX 3090, N=102400, sigma=8192
METRIC = "Morlet transform ms @N=102400,σ=8192; Msamples·scales/s; HBM GB/s vs peak"
UNIT = "Msamples·scales/s"

WORKLOADS = {
    # BASELINE config 3 (headline)
    "morlet_direct": dict(abbrev="MDS5P6", sigma=8192.0, xi=10.0, n=102400, batch=1, precision=0,
                          desc="Morlet method 1 (direct, MDS5P6 ASFT, P_S auto=7, P_D=6) fp32, N=102400, sigma=8192, xi=10"),
    # BASELINE config 1
    "gauss_sft_fp64": dict(abbrev="GDP6", sigma=8192.0, xi=0.0, n=102400, batch=1, precision=1,
                           desc="Gaussian smoothing SFT (GDP6) fp64, N=102400, sigma=8192"),
    # BASELINE config 2 (the sigma=8192 member)
    "gauss_asft_fp32": dict(abbrev="GDS10P6", sigma=8192.0, xi=0.0, n=102400, batch=1, precision=0,
                            desc="Gaussian smoothing ASFT (GDS10P6) fp32, N=102400, sigma=8192"),
    # BASELINE config 4
    "morlet_multiply_batch": dict(abbrev="MMS5P3", sigma=8192.0, xi=10.0, n=102400, batch=4096, precision=0,
                                  desc="Morlet method 2 (multiply, MMS5P3 ASFT) fp32, 4096 x N=102400, sigma=8192, xi=10"),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ------------------------------------------------------------------ distributed helpers
def dist_init(args, local):
    """One process per GPU. NCCL by default; --dist-backend gloo lets a multi-rank run
    share one GPU (used to exercise the N>1 path when only one device is available)."""
    import torch
    import torch.distributed as dist

    world = env_int("WORLD_SIZE", 1)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world


def device_index(args, local):
    return 0 if args.share_device else local


def max_over_ranks(value: float, world: int) -> float:
    """Max of a host scalar over ranks (CPU tensor: works with NCCL and gloo)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        t = torch.tensor([value], dtype=torch.float64, device="cuda")
    else:
        t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_tensor(x, world: int):
    if world == 1:
        return x
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        dist.broadcast(x, src=0)
        return x
    h = x.cpu()
    dist.broadcast(h, src=0)
    x.copy_(h)
    return x


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                self.reasons |= self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def kernel_name(plan) -> str:
    """The dominant kernel of a plan: K4 (tensor cores) or K1 (CUDA-core scan)."""
    if plan.describe().get("tensor_cores"):
        return "sft_tc_kernel (K4: tcgen05 kind::tf32 3xTF32 chunked scan)"
    return "sft_scan_kernel (K1)"


def ncu_traffic(workload: str):
    """Per-launch dram bytes of K1 from the committed ncu --set full capture (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


# ------------------------------------------------------------------ reference arm (CPU)
def workload_config(args, w, abbrev, K):
    """The config object both arms print (identical keys and values)."""
    world = args.gpus
    return {"workload": args.workload, "desc": w["desc"], "abbreviation": abbrev, "K": K, "batch": w["batch"],
            "n": w["n"], "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def cpu_reference_measure(w, steps, warmup, sample_signals, strategy=None, precision=None, port=False):
    """Times the reference's own CPU transform: the library compiled from
    /root/reference/proj/src by oracle/ref.mk (oracle/_ref, kind "reference"); where that
    build is absent, the restated port in oracle/ (kind "port"). Spec built by the
    reference's own factory, untimed (as proj/src/eval.cpp:186-190); default engine =
    the reference bench's Recursive2 (eval.cpp:187) in fp64. Median of ``steps`` after
    ``warmup`` (eval.cpp:192-203), all host threads as workers. Returns a dict."""
    cores = os.cpu_count() or 1
    strategy = 2 if strategy is None else strategy
    precision = 1 if precision is None else precision
    try:
        if port:
            raise ImportError("port requested")
        import oracle.ref as R

        R.lib()
        kind = "reference"
    except Exception:  # noqa: BLE001  (no reference build on this box)
        R, kind = None, "port"
    import oracle as O

    xs = [O.make_test_signal(O.SEEDED_NOISE, w["n"], 1234 + i) for i in range(sample_signals)]
    if R is not None:
        spec = R.Spec(w["abbrev"], w["sigma"], w["xi"], strategy=strategy, precision=precision)
        K = spec.half_width
        run = lambda x: R.apply_transform(spec, x, 1, cores)  # noqa: E731
    else:
        spec = _port_spec(w)
        K = spec["K"]
        run = lambda x: _port_run(O, spec, x, strategy, precision, cores)  # noqa: E731
    for _ in range(warmup):
        run(xs[0])
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        for x in xs:
            run(x)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": sample_signals * w["n"] / t / 1e6, "seconds": t, "cores": cores, "kind": kind, "K": K,
            "strategy": ["KernelIntegral", "Recursive1", "Recursive2"][strategy],
            "precision": ["f32", "f64"][precision]}


def _port_spec(w):
    """Restated-oracle fallback: the spec fixture written beside the oracle by
    oracle/make_bench_specs.py (so this arm never loads the product library)."""
    with open(os.path.join(ROOT, "oracle", "bench_specs.json")) as f:
        return json.load(f)[w["abbrev"] + f"@{w['sigma']:g}"]


def _port_run(O, spec, x, strategy, precision, workers):
    import numpy as np

    k = spec["kind"]
    gamma = 1.0 / (2.0 * spec["sigma"] ** 2)
    if k <= 2:
        return O.gauss_smooth(x, 1, k, spec["K"], spec["beta"], spec["n0"], spec["alpha"], gamma, strategy, precision,
                              np.array(spec["a"]), np.array(spec["b"]), np.array(spec["d"]), workers)
    cc = np.array(spec["cos_coeffs"][0]) + 1j * np.array(spec["cos_coeffs"][1])
    if k == 3:
        sc = np.array(spec["sin_coeffs"][0]) + 1j * np.array(spec["sin_coeffs"][1])
        return O.morlet_direct(x, 1, spec["K"], spec["beta"], spec["n0"], spec["alpha"], gamma, strategy, precision,
                               spec["cos_orders"], cc, spec["sin_orders"], sc, workers)
    return O.morlet_multiply(x, 1, spec["K"], spec["beta"], spec["n0"], spec["alpha"], spec["sigma"], spec["xi"],
                             strategy, precision, cc.real, workers)


def run_reference(args, w):
    """--impl reference: the reference's CPU path on this box's host cores, rank 0 only
    (other ranks exit without work), same metric / unit / config as our arm."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    sample = 1 if w["batch"] == 1 else 2
    m = cpu_reference_measure(w, args.steps, max(2, args.warmup), sample)
    f32 = cpu_reference_measure(w, max(5, min(args.steps, 7)), 2, sample, precision=0)
    prt = cpu_reference_measure(w, max(5, min(args.steps, 7)), 2, sample, port=True)
    value = m["value"]
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": max(2, args.warmup), "ms_per_step": m["seconds"] * 1e3 / sample, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": m["precision"], "data": "synthetic (splitmix64 noise, seed 1234+i, make_test_signal)",
        "config": workload_config(args, w, w["abbrev"], m["K"]),
        "engine": f"{m['strategy']} {m['precision']} (the reference bench default, proj/src/eval.cpp:186-189)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": m["cores"], "kind": m["kind"],
                         "sample": f"{sample} signal(s) of N={w['n']} per step, median of {args.steps} steps after "
                                   f"{max(2, args.warmup)} warm-ups, {m['strategy']} {m['precision']}, "
                                   f"workers={m['cores']} (the reference parallelises over orders)"},
        "f32_recursive2": {"value": f32["value"], "unit": UNIT, "ms_per_signal": f32["seconds"] * 1e3 / sample},
        # the restated port (oracle/) of the same path, same engine, for comparison: the
        # compiled reference runs on a mini-Eigen shim
        "restated_port": {"value": prt["value"], "unit": UNIT, "ms_per_signal": prt["seconds"] * 1e3 / sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm (GPU)
def graph_upload(graph, stream) -> None:
    """cuGraphUpload of a captured torch CUDA graph's executable on `stream` (driver API:
    one driver instance, so the handle torch holds is valid here)."""
    import ctypes

    drv = ctypes.CDLL("libcuda.so.1")
    drv.cuGraphUpload.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    rc = drv.cuGraphUpload(ctypes.c_void_p(int(graph.raw_cuda_graph_exec())), ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cuGraphUpload failed ({rc})")


def run_ours(args, w, spec_of):
    import torch
    import torch.distributed as dist

    import paper_2110_11866_b200 as P

    rank, local = env_int("RANK", 0), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(device_index(args, local))
    world = dist_init(args, device_index(args, local))

    spec = spec_of()
    n, batch = w["n"], w["batch"]
    plan = P.TransformPlan(spec, n, batch)
    in_es = 4 if w["precision"] == 0 else 8
    out_es = in_es * (2 if plan.complex_out else 1)
    step_bytes = batch * n * (in_es + out_es)
    prec = P.Precision.Single if w["precision"] == 0 else P.Precision.Double
    K = args.steps
    # L2 state: every timed step reads inputs no earlier step (timed or warm-up) touched
    # since an L2 flush. Small steps get disjoint (input, output) buffer pairs, one per
    # timed step (cycling only beyond 3x L2 of buffers, i.e. after L2 turned over), the
    # untimed warm-up / graph-upload replay uses a separate pair, and 2x L2 is written
    # right before the timed region. Steps larger than L2 stream on their own.
    small = step_bytes < L2_BYTES
    R = min(K, max(2, math.ceil(3 * L2_BYTES / step_bytes))) if small else 1
    seeds = [1234 + rank * 7919 + 17 * i for i in range(min(R, 8))]
    base = [P.generate_signals(P.TestSignalKind.SeededNoise, n, sd, batch, prec) for sd in seeds]
    xs = [base[i] if i < len(base) else base[i % len(base)].clone() for i in range(R)]
    outs = [plan.empty_output() for _ in range(R)]
    warm_x, warm_o = (base[0].clone(), plan.empty_output()) if small else (xs[0], outs[0])
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            plan.execute(warm_x, warm_o)
        stream.synchronize()

        def steps_body(timed):
            for k in range(K):
                if timed:
                    plan.execute(xs[k % R], outs[k % R])
                else:
                    plan.execute(warm_x, warm_o)

        graph = None
        if not args.no_graph:
            # the graph is captured on the disjoint buffers; its upload replay runs a twin
            # graph on the warm-up pair so the timed buffers stay untouched
            graph, upload = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                steps_body(True)
            with torch.cuda.graph(upload, stream=stream):
                steps_body(False)
            upload.replay()
            # the timed graph's own one-time upload to the device (cuGraphUpload) happens
            # here, not at its first replay inside the timed region: uploading 200 kernel
            # nodes costs ~1 ms (~5 us per step at the headline size, measured by
            # tools/k1_protocols.py) and is setup, like plan creation
            try:
                graph_upload(graph, stream)
            except Exception as e:  # noqa: BLE001
                # no driver-API upload: one untimed replay uploads the graph instead; the
                # L2 flush right before the timed region still makes every input cold
                print(f"bench: cuGraphUpload unavailable ({e}); uploading by an untimed replay", file=sys.stderr)
                graph.replay()
            stream.synchronize()

        def timed_region():
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(1)  # 2x L2 written: nothing of the timed buffers is resident
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                steps_body(True)
            ev1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            return ev0.elapsed_time(ev1)

        with ClockSampler(device_index(args, local)) as clk:
            ms = timed_region()
            # keep the clock record meaningful for sub-second regions: sample a few more
            # identical replays (not part of the reported number) only if too few samples
            t_extra = time.perf_counter()
            while len(clk.samples) < 20 and time.perf_counter() - t_extra < 2.0 and graph is not None:
                upload.replay()
                stream.synchronize()
    ms = max_over_ranks(ms, world)
    ms_per_step = ms / K
    samples = n * batch * K * world
    value = samples / (ms * 1e-3) / 1e6

    # e2e through the C ABI with pinned host buffers: every step copies its input H2D and
    # its result D2H. Small steps use the pipelined entry point over a ring of distinct
    # host buffer pairs (copies of step k+-1 overlap the kernel of step k); steps too large
    # for a pinned ring run the synchronous call.
    host_step = batch * n * (in_es + out_es)
    pairs = 3 if 3 * host_step <= (2 << 30) else 1
    x_hosts, o_hosts = [], []
    for i in range(pairs):
        xh = torch.empty((batch, n), dtype=plan.dtype()).pin_memory()
        xh.copy_(xs[i % R].cpu())
        x_hosts.append(xh)
        o_hosts.append(torch.empty(outs[0].shape, dtype=plan.dtype()).pin_memory())
    e2e_steps = max(1, min(K * 10, 300)) if pairs > 1 else max(1, min(K, 3))

    def e2e_run(steps):
        for i in range(steps):
            if pairs > 1:
                plan.execute_host_async(x_hosts[i % pairs].numpy(), o_hosts[i % pairs].numpy(), stream.cuda_stream)
            else:
                plan.execute_host(x_hosts[0].numpy(), o_hosts[0].numpy(), stream.cuda_stream)
        stream.synchronize()

    with torch.cuda.stream(stream):
        e2e_run(max(3, args.warmup))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_run(e2e_steps)
        e2e_s = time.perf_counter() - t0
    e2e_value = n * batch * e2e_steps * world / max_over_ranks(e2e_s, world) / 1e6
    e2e_path = ("sftgpu_transform_execute_host_async (C ABI, pipelined over 3 pinned host buffer pairs; "
                "wall clock around all steps + final stream sync)" if pairs > 1 else
                "sftgpu_transform_execute_host (C ABI, pinned host buffers, one synchronous call per step; "
                "large tensor-core plans pipeline sub-batches inside the call)")

    peak, peak_src = measured_peaks()
    launches = plan.launches
    kernel_ms = ms_per_step / launches
    achieved = step_bytes / launches / (kernel_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.workload)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = 1 if batch == 1 else 2
        m = cpu_reference_measure(w, 5, 2, sample)
        cpu = {"value": m["value"], "unit": UNIT, "cores": m["cores"], "kind": m["kind"],
               "sample": f"{sample} signal(s) of N={n} per step ({'the reference compiled from its sources, oracle/_ref' if m['kind'] == 'reference' else 'restated port, oracle/'}; "
                         f"{m['strategy']} {m['precision']}, the reference bench default; workers={m['cores']}), "
                         f"median of 5 after 2 warm-ups",
               "ms_per_signal": m["seconds"] * 1e3 / sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": (value / world) / (n / (PAPER_MS * 1e-3) / 1e6) if (n == 102400 and batch == 1) else None,
            "dtype": "f32" if w["precision"] == 0 else "f64",
            "data": "synthetic (device splitmix64 noise, bit-identical to make_test_signal)",
            "config": workload_config(args, w, spec.abbreviation, spec.half_width),
            "timing": {"l2": (f"inputs larger than L2 in aggregate: {R} disjoint input/output buffer pairs "
                              f"({R * step_bytes / 2**20:.1f} MiB), every timed step reads a pair no earlier step "
                              f"touched, L2 flushed (2x L2 written) right before the timed region; warm-up and "
                              f"graph upload on a separate pair") if small else
                              "step working set larger than L2 (streams on its own); L2 flushed before the region",
                       "method": ("CUDA graph of K back-to-back steps, uploaded to the device (cuGraphUpload) "
                                  "before the region, CUDA events on the launch stream around its first replay, "
                                  "max over ranks") if graph is not None
                       else "K launches, CUDA events around them, max over ranks"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": step_bytes / launches,
                         "kernel": kernel_name(plan), "kernel_ms": kernel_ms},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": batch * n * in_es,
                    "d2h_bytes_per_step": batch * n * out_es, "steps": e2e_steps,
                    "path": e2e_path},
            "gpu_launches": K * launches,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_scalogram(args):
    """BASELINE config 5: 128-scale Morlet scalogram (direct, P_D=6, xi=10) on N=2^24,
    scales sharded across ranks, input broadcast once (NCCL), gather timed separately."""
    import torch
    import torch.distributed as dist

    import paper_2110_11866_b200 as P
    from paper_2110_11866_b200 import scalogram as SG

    rank, local = env_int("RANK", 0), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(device_index(args, local))
    world = dist_init(args, device_index(args, local))
    n, ns = args.scalogram_n, args.scalogram_scales
    cache = os.path.join(ROOT, "paper_2110_11866_b200", "data", f"scalogram{ns}_xi10_pd6.coef")
    specs = SG.build_specs(SG.scale_sigmas(ns), xi=10.0, pd=6, cache=cache)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    if rank == 0:
        x.copy_(P.generate_signals(P.TestSignalKind.SeededNoise, n, 1234, 1, P.Precision.Single)[0])
    broadcast_tensor(x, world)
    sc = SG.Scalogram(n, specs, world, rank, args.shard)
    out = sc.empty_output()
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            sc.run(x, out)
        stream.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(device_index(args, local)) as clk:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(args.steps):
                sc.run(x, out)
            ev1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
        ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, world)
    value = n * ns * args.steps / (ms * 1e-3) / 1e6
    # final gather to rank 0 (optional, timed separately)
    gather_ms = None
    if world > 1 and args.gather and dist.get_backend() == "nccl":
        torch.cuda.synchronize()
        dist.barrier()
        g0 = time.perf_counter()
        sc.gather(out)
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - g0) * 1e3
    # e2e: pinned host input -> H2D, all of this rank's scales, D2H of its rows
    xh = torch.empty(n, dtype=torch.float32).pin_memory()
    xh.copy_(x.cpu())
    oh = torch.empty(out.shape, dtype=torch.float32).pin_memory()
    if world > 1:
        dist.barrier()
    e0 = time.perf_counter()
    with torch.cuda.stream(stream):
        xd = torch.empty_like(x)
        xd.copy_(xh, non_blocking=True)
        sc.run(xd, out)
        oh.copy_(out, non_blocking=True)
        stream.synchronize()
    e2e_value = n * ns / max_over_ranks(time.perf_counter() - e0, world) / 1e6
    peak, peak_src = measured_peaks()
    launches_per_step = sc.launches
    kernel_ms = ms / args.steps / max(1, launches_per_step)
    # algorithmic bytes: the signal read once per launch (one
    # multi-scale launch produces all of a rank's scales) + complex64 outputs
    if sc.multi:
        step_bytes = sum(n * 4 + p.batch * sc.count * 8 for _, p in sc.multi)
        kname = f"sft_tc_kernel (K4), {len(sc.multi)} multi-scale launch(es) of <= 128 scales"
    else:
        step_bytes = len(sc.rows) * sc.count * 12
        kname = (kernel_name(sc.plans[0]) + ", one launch per scale") if sc.plans else "none"
    achieved = step_bytes / max(1, launches_per_step) / (kernel_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": "Morlet transform ms @N=102400,σ=8192; Msamples·scales/s; HBM GB/s vs peak",
            "value": value, "unit": "Msamples·scales/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device splitmix64 noise, seed 1234), broadcast from rank 0",
            "config": {"workload": "scalogram", "desc": f"Morlet direct scalogram, {ns} scales sigma 16..16384, "
                       f"N={n}, xi=10, P_D=6, n0=min(5, sigma/4), fp32", "shard": args.shard,
                       "parallelism": f"{args.shard}-sharded x{world}", "n": n, "scales": ns,
                       "l2": "step working set (>= 1 GiB of outputs) larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic("scalogram"), "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": step_bytes / max(1, launches_per_step),
                         "kernel": kname, "kernel_ms": kernel_ms},
            "e2e": {"value": e2e_value, "unit": "Msamples·scales/s", "h2d_bytes_per_step": n * 4,
                    "d2h_bytes_per_step": sc.output_bytes(), "steps": 1,
                    "path": "Scalogram.run (public API) with pinned host input/output"},
            "gpu_launches": args.steps * launches_per_step,
            "gather_ms": gather_ms,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["scalogram"], default="morlet_direct")
    ap.add_argument("--scalogram-n", type=int, default=1 << 24)
    ap.add_argument("--scalogram-scales", type=int, default=128)
    ap.add_argument("--shard", choices=["scale", "chunk"], default="scale")
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--share-device", action="store_true",
                    help="all ranks on cuda:0 (with --dist-backend gloo): exercises the N>1 path on one GPU")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload == "scalogram":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "scalogram CPU reference is hours of CPU time; "
                              "the reference arm times the headline workload"}))
            return
        return run_scalogram(args)
    w = WORKLOADS[args.workload]

    def spec_of():
        import paper_2110_11866_b200 as P

        return P.make_transform_spec(w["abbrev"], w["sigma"], w["xi"],
                                     P.TransformOptions(precision=P.Precision(w["precision"]),
                                                        strategy=P.Strategy.KernelIntegral))

    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w, spec_of)


if __name__ == "__main__":
    main()
