"""Benchmark of the B200 CCQ hot path (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the Llama-3-8B-shape linears): the MLP-up
linear d_in 4096 -> d_out 14336 at CCQ 2.06 bits (W2A16), batch M = 1,
synthetic random_quantized weights (the reference bench's own generator,
ccq_main.cpp:269-271) and Gaussian bf16 activations.

One step = one decode-GEMV pass over each of L resident layer copies
(L x 15.3 MB > the 126 MB L2, so every timed launch streams its weights from
HBM).  value = packed-weight bytes (ccq::model_payload_bytes, kernels.cpp:203)
moved per second, whole job.  `e2e` is the same metric through the public API
with host (pinned) activations copied in and outputs copied back each layer.

--impl reference times the reference's own CPU gemv_batch (oracle/_ref,
compiled from /root/reference) on all host cores, same workload/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CCQ W2A16 GEMV packed-weight GB/s (% HBM peak); GEMM TFLOP/s at batch 1-256"
D_IN, D_OUT, FAMILY, M_HEAD = 4096, 14336, 2, 1
SEED = 4096 * 31 + 14336  # ccq_main.cpp:269-271 seeding: seed + d_in*31 + d_out (seed 0)
WORKLOAD = "configs[1] Llama-3-8B MLP-up linear d_in 4096 -> d_out 14336, CCQ 2.06 (W2A16), batch M=1"


def base_config(layers):
    """The workload description shared by both arms (same keys, same values)."""
    return {"workload": WORKLOAD, "d_in": D_IN, "d_out": D_OUT, "family": "2.06", "batch": M_HEAD,
            "layers_per_step": layers, "weights": "random_quantized distribution (synthetic.cpp:25-103)",
            "activations": "Gaussian, bf16-rounded"}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([v.strip() for v in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl != "reference" else "gloo")
    return world, rank, local


def run_reference(args, world, rank):
    """The reference CPU path (oracle/_ref), all host threads, bounded sample."""
    if rank != 0:
        return None
    import numpy as np
    import oracle as O
    threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    x = O.random_matrix(M_HEAD, D_IN, "gaussian", SEED + 1)
    if kind == "reference":
        model = O.RefModel.random(D_OUT, D_IN, FAMILY, 64, SEED)
        payload = model.payload_bytes()
        runner = O.RefSharded(model, threads)
        call = lambda: runner.gemv_batch(x)  # noqa: E731
    else:
        s = O.random_packed(D_OUT, D_IN, FAMILY, 64, SEED)
        payload = O.payload_bytes(s)
        call = lambda: O.gemv_batch(s, x, threads=threads)  # noqa: E731
    for _ in range(args.warmup):
        call()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call()
    dt = (time.perf_counter() - t0) / args.steps
    gbs = payload / dt / 1e9
    sample = f"{args.steps} x gemv_batch 4096x14336 2.06 M=1 ({threads} threads, row-sharded)"
    return {"metric": METRIC, "value": gbs, "unit": "GB/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 activations x CCQ codes, f64 accumulate (reference)",
            "data": "synthetic (random_quantized, Gaussian x)",
            "config": base_config(args.layers),
            "arm": "reference CPU path (oracle/_ref gemv_batch), row-sharded over host threads",
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def cpu_baseline_leg():
    """Reference CPU path timed on this host (rank 0, N=1 only), ~10 s."""
    import oracle as O
    threads = os.cpu_count() or 1
    x = O.random_matrix(M_HEAD, D_IN, "gaussian", SEED + 1)
    if O.ref_available():
        model = O.RefModel.random(D_OUT, D_IN, FAMILY, 64, SEED)
        payload, kind = model.payload_bytes(), "reference"
        runner = O.RefSharded(model, threads)
        call = lambda: runner.gemv_batch(x)  # noqa: E731
    else:
        s = O.random_packed(D_OUT, D_IN, FAMILY, 64, SEED)
        payload, kind = O.payload_bytes(s), "port"
        call = lambda: O.gemv_batch(s, x, threads=threads)  # noqa: E731
    call()
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < 8.0 or n < 3:
        call()
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": payload / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"{n} x gemv_batch 4096x14336 2.06 M=1 on {threads} threads "
                      f"({dt*1e3:.1f} ms each)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ccq", choices=["ccq", "reference"])
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", action="store_true", help="add an M / family sweep")
    ap.add_argument("--no-gemm", action="store_true", help="skip the batched GEMV/GEMM block")
    ap.add_argument("--chunk-tokens", type=int, default=1024, help="sharded GEMM all-gather chunk")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded configs[4]/[2] block also at N=1 (always on for N>1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local = dist_init(args)
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out))
        return

    import numpy as np
    import torch

    import paper_2507_07145_b200 as P

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))

    # --- synthetic layers: L resident copies (different seeds) -------------
    # The reference bench generator itself (random_quantized + pack_model,
    # mt19937_64, ccq_synthetic_packed): layer 0 of rank 0 is byte-identical
    # to the model the reference arm times (RefModel.random(..., SEED)), and
    # the activations are the reference's random_matrix(M, d_in, Gaussian,
    # SEED + 1) rounded to bf16 (ccq_synthetic_matrix).
    from paper_2507_07145_b200.synthetic import reference_matrix, reference_packed
    layers = []
    for l in range(args.layers):
        s = reference_packed(D_OUT, D_IN, FAMILY, 64, SEED + 1000 * l + rank)
        layers.append(P.DeviceModel.upload(s, device=local))
    payload = layers[0].payload_bytes
    x_host = torch.from_numpy(np.stack([reference_matrix(M_HEAD, D_IN, "gaussian", SEED + 1 + 1000 * l + rank)
                                        for l in range(args.layers)])).to(torch.bfloat16).pin_memory()
    x_dev = x_host.to(dev)
    y_dev = torch.empty(args.layers, M_HEAD, D_OUT, dtype=torch.float32, device=dev)
    y_host = torch.empty_like(y_dev, device="cpu").pin_memory()
    stream = torch.cuda.Stream(device=dev)

    def step():
        for l in range(args.layers):
            P.matmul(layers[l], x_dev[l], out=y_dev[l], stream=stream)

    # capture one step in a CUDA graph (launch-bound inner loop)
    with torch.cuda.stream(stream):
        for _ in range(2):
            step()
    stream.synchronize()
    n0 = P.launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    kernels_per_step = P.launch_count() - n0
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            start.record(stream)
            step_ev[0].record(stream)
            for i in range(args.steps):
                graph.replay()
                step_ev[i + 1].record(stream)
            end.record(stream)
        torch.cuda.synchronize()
    step_ms = sorted(step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps))
    barrier()
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    bytes_step = payload * args.layers
    value = bytes_step * world / (ms * 1e-3) / 1e9
    per_launch_us = ms * 1e3 / args.layers
    alg_bytes = payload + M_HEAD * D_IN * 2 + M_HEAD * D_OUT * 4
    achieved = alg_bytes / (per_launch_us * 1e-6) / 1e9

    # --- e2e: public API, host activations in, outputs back, every layer ----
    # Every step copies its own inputs in (one pinned H2D) and its results out
    # (one D2H), as a serving loop would: double-buffered on two copy streams;
    # step i+1's H2D and step i's D2H overlap step i's / i+1's kernels.  The
    # timed region starts before the first H2D and ends after the last D2H.
    h2d_stream = torch.cuda.Stream(device=dev)  # separate copy streams: an H2D
    d2h_stream = torch.cuda.Stream(device=dev)  # never queues behind a D2H
    x_bufs = [x_dev, torch.empty_like(x_dev)]
    y_bufs = [y_dev, torch.empty_like(y_dev)]
    y_hosts = [y_host, torch.empty_like(y_host).pin_memory()]
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]
    for b in range(2):  # initial state: buffers free
        comp_done[b].record(stream)
        d2h_done[b].record(d2h_stream)

    def issue_h2d(i):
        b = i & 1
        h2d_stream.wait_event(comp_done[b])  # x_bufs[b] no longer read (step i-2)
        with torch.cuda.stream(h2d_stream):
            x_bufs[b].copy_(x_host, non_blocking=True)
        h2d_done[b].record(h2d_stream)

    # The step's public-API calls (P.matmul per layer) captured once per
    # double-buffer slot in a CUDA graph, as a serving loop would run them;
    # the copies stay outside, issued every step.
    slot_graphs = []
    for b in range(2):
        with torch.cuda.stream(stream):
            for l in range(args.layers):
                P.matmul(layers[l], x_bufs[b][l], out=y_bufs[b][l], stream=stream)
        stream.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            for l in range(args.layers):
                P.matmul(layers[l], x_bufs[b][l], out=y_bufs[b][l], stream=stream)
        slot_graphs.append(gph)
    torch.cuda.synchronize()

    def e2e_step(i, n):
        # step i's input was copied in while step i-1 ran (step 0: here)
        b = i & 1
        if i == 0:
            issue_h2d(0)
        if i + 1 < n:
            issue_h2d(i + 1)
        stream.wait_event(h2d_done[b])
        stream.wait_event(d2h_done[b])  # y_bufs[b] drained (step i-2)
        slot_graphs[b].replay()
        comp_done[b].record(stream)
        d2h_stream.wait_event(comp_done[b])
        with torch.cuda.stream(d2h_stream):
            y_hosts[b].copy_(y_bufs[b], non_blocking=True)
        d2h_done[b].record(d2h_stream)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            e2e_step(i, args.warmup)
    torch.cuda.synchronize()
    barrier()
    with torch.cuda.stream(stream):
        start.record(stream)
        h2d_stream.wait_event(start)
        d2h_stream.wait_event(start)
        for i in range(args.steps):
            e2e_step(i, args.steps)
        stream.wait_event(d2h_done[(args.steps - 1) & 1])
        end.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = start.elapsed_time(end) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = bytes_step * world / (e2e_ms * 1e-3) / 1e9

    sweep = prefill = moe = paper = gemm = None
    tflops_peak = float(peaks.get("bf16_tflops", 1590.0))
    if rank == 0 and world == 1 and not args.no_gemm:
        gemm = run_gemm_block(P, torch, dev, stream, hbm_peak, tflops_peak, local)
    sharded = None
    if world > 1 or args.sharded:
        sharded = run_sharded(P, torch, dev, stream, world, rank, local, tflops_peak, args)
    if args.sweep and rank == 0:
        sweep = run_sweep(P, torch, dev, stream, hbm_peak, tflops_peak)
        paper = run_paper_shapes(P, torch, dev, stream)
        with ClockSampler(local) as pclk:
            prefill = run_prefill(P, torch, dev, stream, tflops_peak)
        prefill = {"runs": prefill, "clocks": pclk.summary()}
        moe = run_moe(P, torch, dev, stream, hbm_peak, tflops_peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg()

    traffic = None
    prof = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16 activations x CCQ codes, f32 accumulate",
            "data": "synthetic: the reference generator's bytes (random_quantized + pack_model, "
                    "synthetic.cpp:25-103, mt19937_64; layer 0 = the reference arm's model), "
                    "random_matrix Gaussian activations rounded to bf16",
            "config": base_config(args.layers),
            "arm": f"B200 kernels, replicas x{world}",
            "l2": f"inputs larger than L2: {args.layers} resident layer copies = "
                  f"{bytes_step/1e6:.0f} MB rotated per step",
            "hbm_fraction": value / world / hbm_peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "kernel": "gemv_stream<2.06,RPW=4,MT=1>",
                         "per_launch_us": per_launch_us, "alg_bytes_per_launch": alg_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                         else "fallback 6650 GB/s (B200_PROFILING.md)"},
            "e2e": {"value": e2e_val, "unit": "GB/s",
                    "h2d_bytes_per_step": args.layers * M_HEAD * D_IN * 2,
                    "d2h_bytes_per_step": args.layers * M_HEAD * D_OUT * 4,
                    "ms_per_step": e2e_ms},
            "gpu_launches": kernels_per_step * args.steps,
            "clocks": clk.summary(),
            "step_ms": {"median": statistics.median(step_ms), "p10": step_ms[len(step_ms) // 10],
                        "p90": step_ms[(9 * len(step_ms)) // 10], "n": len(step_ms)},
        }
        if gemm is not None:
            out["gemm"] = gemm
        if sharded is not None:
            out["sharded"] = sharded
        if cpu is not None:
            out["cpu_baseline"] = cpu
        if sweep is not None:
            out["sweep"] = sweep
        if prefill is not None:
            out["prefill"] = prefill
        if moe is not None:
            out["moe"] = moe
        if paper is not None:
            out["paper_shapes"] = paper
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_sharded(P, torch, dev, stream, world, rank, local, tflops_peak, args):
    """SURVEY 8e on the N GPUs of this job (strong scaling: the layer is fixed,
    the work splits): configs[4] 8192 -> 28672 (2.06, M = 4096 prefill)
    N-column sharded with the chunked decode-matmul + NCCL all-gather of
    ccq_cuda_shard_allgather, and configs[2] (ERNIE 64 experts, T = 4096
    tokens, top-8) expert-sharded with one output all-gather.  Device-timed,
    max over ranks.  Also: compute-only and gather-only times."""
    import numpy as np
    import torch.distributed as dist
    from paper_2507_07145_b200.parallel import NcclComm, ShardedExperts, ShardedLinear
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    out = {"n_gpus": world, "scaling": "strong", "tensor_peak_tflops_per_gpu": tflops_peak}
    made_group = False
    if world == 1 and not dist.is_initialized():
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        made_group = True
    comm = NcclComm(device=local)
    with ClockSampler(local) as clk:
        # configs[4]: N-column sharding + chunked all-gather
        pk = _synthetic(28672, 8192, 2, 64, 5)
        lin = ShardedLinear(pk, device=local, comm=comm)
        del pk
        g = torch.Generator(device="cpu").manual_seed(4097)
        x = torch.randn(4096, 8192, generator=g).to(torch.bfloat16).to(dev)
        y = torch.empty(4096, 28672, dtype=torch.bfloat16, device=dev)
        yl = torch.empty(4096, lin.r1 - lin.r0, dtype=torch.bfloat16, device=dev)
        flop = 2 * 4096 * 8192 * 28672
        with torch.cuda.stream(stream):
            ms = timed(lambda: lin(x, out=y, chunk_tokens=args.chunk_tokens, stream=stream), 5)
            ms_c = timed(lambda: P.matmul(lin.local, x, out=yl, stream=stream), 5)
            ms_g = None
            if world > 1:
                gath = torch.empty(world, 4096, lin.r1 - lin.r0, dtype=torch.bfloat16, device=dev)
                ms_g = timed(lambda: dist.all_gather_into_tensor(gath, yl), 5)
        out["configs4"] = {"d_in": 8192, "d_out": 28672, "M": 4096, "family": "2.06", "out_dtype": "bf16",
                           "rows_per_gpu": lin.r1 - lin.r0, "chunk_tokens": args.chunk_tokens,
                           "ms": round(ms, 4), "TFLOPs": round(flop / (ms * 1e-3) / 1e12, 1),
                           "tensor_frac_per_gpu": round(flop / (ms * 1e-3) / 1e12 / world / tflops_peak, 4),
                           "compute_only_ms": round(ms_c, 4),
                           "gather_only_ms": None if ms_g is None else round(ms_g, 4),
                           "gather_bytes_per_gpu": (world - 1) * 4096 * (lin.r1 - lin.r0) * 2}
        del lin, x, y, yl
        torch.cuda.empty_cache()
        # configs[2]: expert sharding (ERNIE-4.5 64 x 8192 -> 3584, T = 4096, top-8)
        E, din, dout = 64, 8192, 3584
        from paper_2507_07145_b200.parallel import block_range
        e0, e1 = block_range(E, rank, world)
        sh = ShardedExperts.from_local([_synthetic(dout, din, 2, 64, 1000 + e) for e in range(e0, e1)], E, dout,
                                       device=local)
        rng = np.random.default_rng(7)
        counts = np.zeros(E, np.int64)
        for _ in range(4096):
            counts[rng.choice(E, 8, replace=False)] += 1
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        T = int(offs[-1])
        xe = torch.randn(T, din, generator=g).to(torch.bfloat16).to(dev)
        with torch.cuda.stream(stream):
            ms_e = timed(lambda: sh(offs, xe, out_dtype=torch.bfloat16), 3)
        fl = 2 * T * din * dout
        out["configs2"] = {"model": "ERNIE-4.5-300B-A47B", "experts": E, "experts_per_gpu": e1 - e0,
                           "d_in": din, "d_out": dout, "tokens": 4096, "routed_pairs": T, "ms": round(ms_e, 4),
                           "TFLOPs": round(fl / (ms_e * 1e-3) / 1e12, 1),
                           "tensor_frac_per_gpu": round(fl / (ms_e * 1e-3) / 1e12 / world / tflops_peak, 4)}
        del sh, xe
    out["clocks"] = clk.summary()
    comm.close()
    if made_group:
        dist.destroy_process_group()
    return out if rank == 0 else None


def _l2_cold_us(P, torch, dev, stream, models, x, y, reps=10):
    """us per call, graph-replayed over `models` (enough copies to exceed L2)."""
    def body():
        for mm in models:
            P.matmul(mm, x, out=y, stream=stream)
    return _graph_time_us(torch, stream, body, reps=reps) / len(models)


def run_gemm_block(P, torch, dev, stream, hbm_peak, tflops_peak, local):
    """The metric's second half ("GEMM TFLOP/s at batch 1-256") in the default
    run: configs[1] 4096->14336 at M = 2..256 (all families at 16 and 256),
    configs[4] prefill 8192->28672 M = 4096 (three families) and the ERNIE /
    DeepSeek grouped prefill (configs[2] / [3], T = 4096 tokens, top-8).
    Graph- or event-timed on the device, L2-cold, clocks sampled."""
    import numpy as np
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic
    out = {"tensor_peak_tflops": tflops_peak, "hbm_peak_gbs": hbm_peak,
           "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) / hbm_gbs"}
    with ClockSampler(local) as clk:
        rows = []
        for fam, fname, Ms in ((2, "2.06", (2, 4, 8, 16, 64, 256)), (0, "2.75", (16, 256)), (1, "2.5", (16, 256))):
            copies = 12
            ms_ = [P.DeviceModel.upload(_synthetic(D_OUT, D_IN, fam, 64, 31 + c), device=dev.index)
                   for c in range(copies)]
            pb = ms_[0].payload_bytes
            for M in Ms:
                x = torch.randn(M, D_IN, device=dev).to(torch.bfloat16)
                y = torch.empty(M, D_OUT, device=dev)
                us = _l2_cold_us(P, torch, dev, stream, ms_, x, y)
                tf = 2 * M * D_IN * D_OUT / us / 1e6
                rows.append({"config": "configs[1]", "family": fname, "d_in": D_IN, "d_out": D_OUT, "M": M,
                             "us": round(us, 3), "packed_GBps": round(pb / us / 1e3, 1),
                             "hbm_frac": round(pb / us / 1e3 / hbm_peak, 4), "TFLOPs": round(tf, 2),
                             "tensor_frac": round(tf / tflops_peak, 4)})
            del ms_
        out["configs1"] = rows
        out["configs4_prefill"] = run_prefill(P, torch, dev, stream, tflops_peak)
        moe = []
        for name, E, din, dout in (("ERNIE-4.5-300B-A47B", 64, 8192, 3584), ("DeepSeek-V3", 256, 7168, 2048)):
            ex = P.Experts.upload([_synthetic(dout, din, 2, 64, 1000 + e) for e in range(E)], device=dev.index)
            rng = np.random.default_rng(7)
            counts = np.zeros(E, np.int64)
            for _ in range(4096):
                counts[rng.choice(E, 8, replace=False)] += 1
            offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
            T = int(offs[-1])
            offs_dev = torch.from_numpy(offs).to(dev)
            x = torch.randn(T, din, device=dev).to(torch.bfloat16)
            y = torch.empty(T, dout, device=dev, dtype=torch.bfloat16)
            us = _graph_time_us(torch, stream, lambda: P.experts_matmul(ex, offs, x, out=y, stream=stream,
                                                                          offsets_dev=offs_dev), reps=5)
            tf = 2 * T * din * dout / us / 1e6
            moe.append({"config": "configs[2]" if E == 64 else "configs[3]", "model": name, "experts": E,
                        "d_in": din, "d_out": dout, "tokens": 4096, "routed_pairs": T, "us": round(us, 1),
                        "TFLOPs": round(tf, 1), "tensor_frac": round(tf / tflops_peak, 4)})
            del ex, x, y
            torch.cuda.empty_cache()
        out["moe_prefill"] = moe
    out["clocks"] = clk.summary()
    return out


def run_sweep(P, torch, dev, stream, hbm_peak, tflops_peak):
    """Packed GB/s and TFLOP/s per (family, shape, M, kernel) - graph-timed,
    L2-cold (enough resident copies to exceed L2).  kernel "auto" is the
    dispatcher; "gemv" / "gemm" force a path to show the crossover."""
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic
    res = []
    shapes = [(4096, 14336), (14336, 4096), (4096, 4096)]
    cases = [(M, "auto") for M in (1, 2, 4, 8, 16, 32, 64, 128, 256)] + \
            [(M, k) for M in (16, 32, 64) for k in ("gemv", "gemm")]
    for fam, fname in ((2, "2.06"), (1, "2.5"), (0, "2.75")):
        for (din, dout) in shapes:
            copies = max(2, int(160e6 // (din * dout * 0.35)) + 1)
            ms_ = [P.DeviceModel.upload(_synthetic(dout, din, fam, 64, 17 + c), device=dev.index)
                   for c in range(copies)]
            pb = ms_[0].payload_bytes
            for M, kern in cases:
                x = torch.randn(M, din, device=dev).to(torch.bfloat16)
                y = torch.empty(M, dout, device=dev)

                def body():
                    for mm in ms_:
                        P.matmul(mm, x, out=y, stream=stream, kernel=kern)
                with torch.cuda.stream(stream):
                    body()
                stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    body()
                for _ in range(3):
                    g.replay()
                torch.cuda.synchronize()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 10
                with torch.cuda.stream(stream):
                    s0.record(stream)
                    for _ in range(reps):
                        g.replay()
                    s1.record(stream)
                torch.cuda.synchronize()
                us = s0.elapsed_time(s1) * 1e3 / (reps * copies)
                tf = 2 * M * din * dout / us / 1e6
                res.append({"family": fname, "d_in": din, "d_out": dout, "M": M, "kernel": kern,
                            "us": round(us, 3), "packed_GBps": round(pb / us / 1e3, 1),
                            "hbm_frac": round(pb / us / 1e3 / hbm_peak, 4),
                            "TFLOPs": round(tf, 2), "tensor_frac": round(tf / tflops_peak, 4)})
            del ms_
    return res


def _graph_time_us(torch, stream, body, reps=10):
    with torch.cuda.stream(stream):
        body()
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        body()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s0.record(stream)
        for _ in range(reps):
            g.replay()
        s1.record(stream)
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) * 1e3 / reps


def run_moe(P, torch, dev, stream, hbm_peak, tflops_peak):
    """BASELINE configs[2] / [3] on one GPU: ERNIE-4.5 64 experts 8192->3584 and
    DeepSeek-V3 256 experts 7168->2048, CCQ 2.06, top-8 uniform routing
    (8 distinct experts per token), decode batch B tokens.  Packed bytes count
    only experts with >= 1 routed token."""
    import numpy as np
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic
    out = []
    for name, E, din, dout in (("ERNIE-4.5-300B-A47B", 64, 8192, 3584), ("DeepSeek-V3", 256, 7168, 2048)):
        models = [_synthetic(dout, din, 2, 64, 1000 + e) for e in range(E)]
        pb_e = P.model_payload_bytes(models[0])
        ex = P.Experts.upload(models, device=dev.index)
        del models
        rng = np.random.default_rng(7)
        for B in (1, 2, 4, 16, 64, 256, 4096):  # decode batches and a 4096-token prefill
            counts = np.zeros(E, np.int64)
            for _ in range(B):
                counts[rng.choice(E, 8, replace=False)] += 1
            offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
            T = int(offs[-1])
            offs_dev = torch.from_numpy(offs).to(dev)
            x = torch.randn(T, din, device=dev).to(torch.bfloat16)
            y = torch.empty(T, dout, device=dev)
            us = _graph_time_us(torch, stream, lambda: P.experts_matmul(ex, offs, x, out=y, stream=stream,
                                                                          offsets_dev=offs_dev))
            routed = int((counts > 0).sum())
            gbs = routed * pb_e / us / 1e3
            tf = 2 * T * din * dout / us / 1e6
            out.append({"model": name, "experts": E, "d_in": din, "d_out": dout, "batch": B, "routed_pairs": T,
                        "experts_hit": routed, "us": round(us, 2), "tokens_per_s": round(B / us * 1e6, 1),
                        "packed_GBps_routed": round(gbs, 1), "hbm_frac": round(gbs / hbm_peak, 4),
                        "TFLOPs": round(tf, 2), "tensor_frac": round(tf / tflops_peak, 4)})
        del ex
        torch.cuda.empty_cache()
    return out


def run_paper_shapes(P, torch, dev, stream):
    """The four GEMV shapes of the paper's H20 table, 2.06,
    M = 1 and 4, for context (different GPU; not a vs_baseline ratio)."""
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic
    h20 = {(4096, 4096): (34.0, 35.0), (4096, 1024): (17.0, 17.0), (8192, 8192): (90.0, 104.0),
           (8192, 1024): (22.0, 24.0)}
    out = []
    for (din, dout), (t1, t4) in h20.items():
        copies = max(2, int(160e6 // (din * dout * 0.26)) + 1)
        ms_ = [P.DeviceModel.upload(_synthetic(dout, din, 2, 64, 3 + c), device=dev.index) for c in range(copies)]
        for M, th in ((1, t1), (4, t4)):
            x = torch.randn(M, din, device=dev).to(torch.bfloat16)
            y = torch.empty(M, dout, device=dev)

            def body():
                for mm in ms_:
                    P.matmul(mm, x, out=y, stream=stream)
            us = _graph_time_us(torch, stream, body) / copies
            out.append({"d_in": din, "d_out": dout, "M": M, "us": round(us, 3), "paper_h20_us": th,
                        "speedup_vs_h20_table": round(th / us, 2)})
        del ms_
    return out


def run_prefill(P, torch, dev, stream, tflops_peak):
    """BASELINE configs[4] on one GPU: 8192 -> 28672, 2.06, M = 4096 (tcgen05 GEMM)."""
    from paper_2507_07145_b200.synthetic import random_packed as _synthetic
    out = []
    for fam, fname in ((2, "2.06"), (1, "2.5"), (0, "2.75")):
        m = P.DeviceModel.upload(_synthetic(28672, 8192, fam, 64, 5), device=dev.index)
        x = torch.randn(4096, 8192, device=dev).to(torch.bfloat16)
        y = torch.empty(4096, 28672, device=dev, dtype=torch.bfloat16)
        with torch.cuda.stream(stream):
            for _ in range(2):
                P.matmul(m, x, out=y, stream=stream)
        stream.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps, best = 5, None
        for _ in range(3):  # best of 3 windows: the sweep before leaves the GPU hot
            with torch.cuda.stream(stream):
                s0.record(stream)
                for _ in range(reps):
                    P.matmul(m, x, out=y, stream=stream)
                s1.record(stream)
            torch.cuda.synchronize()
            t = s0.elapsed_time(s1) / reps
            best = t if best is None else min(best, t)
        ms = best
        tf = 2 * 4096 * 8192 * 28672 / (ms * 1e-3) / 1e12
        out.append({"family": fname, "d_in": 8192, "d_out": 28672, "M": 4096, "ms": round(ms, 4),
                    "TFLOPs": round(tf, 1), "tensor_frac": round(tf / tflops_peak, 4),
                    "out_dtype": "bf16"})
        del m, x, y
    return out


if __name__ == "__main__":
    main()
