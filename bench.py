#!/usr/bin/env python
"""Benchmark of the DDF codelet executor on B200 (BASELINE.json metric:
SpMV/SpTRSV fp64 GFLOP/s and % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json configs[1] -- SpTRSV on the lower triangle of
the 3-D 7-point Laplacian, 100^3 grid (n = 1e6, nnz = 3.97e6), plan t=3,
groups=8. A step is one complete triangular solve (one kernel launch). The
solve does not shard, so N > 1 runs N independent replicas
("scaling": "weak"). SpMV configs (--config 1/3/5) shard the plan's partitions
across ranks with an NCCL all-gather of x per step ("scaling": "strong").

Timing: W untimed warm-up steps; K timed steps between a barrier +
cudaDeviceSynchronize on both sides; each step is bracketed by CUDA events
on the launching stream with an L2 flush before it, outside the events (a
2x-L2 write, then a 2x-L2 read of a second buffer, so no dirty flush lines are
written back during the step); ms_per_step is the mean device time, maxed
over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: ("spmv", "config1-spmv-2d5pt-1000^2"),
    2: ("sptrsv", "config2-sptrsv-3d7pt-lower-100^3"),
    3: ("spmv", "config3-spmv-27pt-3dof-80^3"),
    4: ("sptrsv", "config4-sptrsv-supernodal-400k"),
    5: ("spmv", "config5-spmv-powerlaw-20M"),
}
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                "clocks_event_reasons.sw_power_cap")
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--t", type=int, default=3)
    p.add_argument("--groups", type=int, default=8)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=6.0, help="bounded CPU-baseline sample length")
    p.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                   help="sharded SpMV x exchange: fused peer-memory pull (p2p) or NCCL all-gather")
    return p.parse_args()


def flops(kernel, n_rows, nnz):
    """theoretical_flops, bench.cpp:27-32."""
    return 2 * nnz if kernel == "spmv" else 2 * nnz - n_rows


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms."""

    def __init__(self, index):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [f.strip() for f in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        window = [s for ts, s in self.samples if t0 <= ts <= t1]
        scope = "timed_region"
        if not window:
            window = [s for _, s in self.samples]
            scope = "whole_run"
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "scope": "unavailable"}
        sm = [float(s[1]) for s in window if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in window if s[2].replace(".", "").isdigit()]
        reasons = sorted({REASONS[i] for s in window for i in range(4) if len(s) > 4 + i and s[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(window), "scope": scope}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


def cpu_baseline(kernel, a, plan_t, groups, vec, seconds):
    """The reference executor (oracle/_ref) on the host cores; bounded sample."""
    from oracle.oracle import Oracle, Ref

    n_flops = flops(kernel, a.n_rows, a.nnz())
    kind = "reference" if Ref.available() else "port"
    workers = 1 if kernel == "sptrsv" else (os.cpu_count() or 1)
    if kind == "reference":
        rc = Ref.csr(a.view())
        rplan, _ = Ref.time_inspect(0 if kernel == "spmv" else 1, rc, plan_t, groups)
        probe_fn = Ref.time_spmv if kernel == "spmv" else Ref.time_sptrsv
        t1, _ = probe_fn(rplan, rc, vec, workers, 1, 1)
        reps = int(max(3, min(1000, seconds / max(t1[0], 1e-6))))
        times, _ = probe_fn(rplan, rc, vec, workers, 0, reps)
    else:
        import paper_2111_12243_b200 as P

        plan = P.inspect(P.KernelKind.Spmv if kernel == "spmv" else P.KernelKind.Sptrsv, a, plan_t, groups)
        exp = plan.export_arrays()
        fn = (lambda: Oracle.run_spmv(exp, a.view(), vec)) if kernel == "spmv" else \
            (lambda: Oracle.run_sptrsv(exp, a.view(), vec))
        times = []
        t_end = time.time() + seconds
        while len(times) < 3 or time.time() < t_end:
            s = time.perf_counter()
            fn()
            times.append(time.perf_counter() - s)
        workers = 1
    med = float(np.median(times))
    return {"value": n_flops / med / 1e9, "unit": "GFLOP/s", "cores": workers, "kind": kind,
            "sample": f"{len(times)} complete run_{kernel} calls on the full matrix (median {med * 1e3:.2f} ms), "
                      f"plan t={plan_t} groups={groups}, workers={workers}"
                      + (" (the reference pool races on deep level-set solves, SURVEY.md §0.8; with 4 or 16 workers it segfaults 3/3 on config 2, tools/ref_workers_probe.py)"
                         if kernel == "sptrsv" and kind == "reference" else ""),
            "ms_median": med * 1e3}


def run_reference(args):
    """--impl reference: the reference's own CPU executor on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2111_12243_b200 as P
    from oracle.oracle import Oracle, Ref

    kernel, workload = CONFIGS[args.config]
    a = P.generate_config(args.config, args.scale)
    vec = P.uniform_vector(a.n_cols, 10 + args.config)
    n_flops = flops(kernel, a.n_rows, a.nnz())
    workers = 1 if kernel == "sptrsv" else (os.cpu_count() or 1)
    if Ref.available():
        kind = "reference"
        rc = Ref.csr(a.view())
        rplan, insp = Ref.time_inspect(0 if kernel == "spmv" else 1, rc, args.t, args.groups)
        fn = Ref.time_spmv if kernel == "spmv" else Ref.time_sptrsv
        times, _ = fn(rplan, rc, vec, workers, args.warmup, args.steps)
    else:
        kind, workers = "port", 1
        t0 = time.perf_counter()
        plan = P.inspect(P.KernelKind.Spmv if kernel == "spmv" else P.KernelKind.Sptrsv, a, args.t, args.groups)
        insp = time.perf_counter() - t0
        exp = plan.export_arrays()
        run = (lambda: Oracle.run_spmv(exp, a.view(), vec)) if kernel == "spmv" else \
            (lambda: Oracle.run_sptrsv(exp, a.view(), vec))
        for _ in range(args.warmup):
            run()
        times = []
        for _ in range(args.steps):
            s = time.perf_counter()
            run()
            times.append(time.perf_counter() - s)
    times = np.asarray(times)
    value = n_flops * len(times) / times.sum() / 1e9
    line = {
        "metric": "fp64 GFLOP/s of the codelet executor (2*nnz SpMV / 2*nnz-n SpTRSV)",
        "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus, "device": "host CPU", "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(times.mean() * 1e3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE.json config generator)",
        "impl": "reference",
        "config": {"workload": workload, "n": a.n_rows, "nnz": a.nnz(), "t": args.t, "groups": args.groups,
                   "kernel": kernel, "parallelism": f"cpu workers={workers}"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": workers, "kind": kind,
                         "sample": f"{len(times)} complete run_{kernel} calls on the full matrix"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "inspector_seconds": insp,
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    import paper_2111_12243_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    kernel, workload = CONFIGS[args.config]
    kk = P.KernelKind.Spmv if kernel == "spmv" else P.KernelKind.Sptrsv
    a = P.generate_config(args.config, args.scale)
    t0 = time.perf_counter()
    plan = P.inspect(kk, a, args.t, args.groups)
    inspector_s = time.perf_counter() - t0
    # the same inspection with the window mining on the GPU (same plan, bit for bit)
    t0 = time.perf_counter()
    plan_dev = P.inspect_device(kk, a, args.t, args.groups, local)
    inspector_dev_s = time.perf_counter() - t0
    inspector_dev_same = plan_dev.hash() == plan.hash()
    del plan_dev
    exe = P.Executor(1, local)
    n_parts = plan.counts().n_partitions
    sharded = kernel == "spmv" and world > 1
    if sharded:
        p0, p1 = rank * n_parts // world, (rank + 1) * n_parts // world
        bound = P.BoundPlan(exe, plan, a, partitions=(p0, p1))
    else:
        bound = P.BoundPlan(exe, plan, a)
    info = bound.info()
    dev = torch.device("cuda", local)
    vec_h = P.uniform_vector(a.n_cols, 10 + args.config)
    vec = torch.from_numpy(vec_h).to(dev)
    rows = bound.row_end - bound.row_begin
    out = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    exchange_kind = None
    peer_ex = None
    if sharded and args.exchange == "p2p":
        # fused exchange: one launch pulls the shard's remote columns from the
        # peers' IPC windows over NVLink and multiplies (dist.PeerExchange)
        from paper_2111_12243_b200.dist import PeerExchange, shard_row_ranges

        try:
            bound.x_runs()  # raises for shards the fused path does not take (segmented plans)
            peer_ex = PeerExchange(bound, shard_row_ranges(plan, world), rank, a.n_cols)
        except Exception as e:  # e.g. a segmented plan or no peer access: fall back to NCCL
            exchange_kind = f"nccl (p2p unavailable: {type(e).__name__}: {e})"
            peer_ex = None
        flag = torch.tensor([1 if peer_ex is not None else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() == 0 and peer_ex is not None:
            peer_ex.close()
            peer_ex = None
            exchange_kind = exchange_kind or "nccl (p2p unavailable on a peer)"
    if peer_ex is not None:
        exchange_kind = "p2p (fused peer-memory pull + multiply)"
        x_mine = vec[bound.row_begin:bound.row_end].clone()

        def step(ev_mid=None):
            if ev_mid is not None:
                ev_mid.record()
            peer_ex.multiply(x_mine, out)
    elif sharded:
        exchange_kind = exchange_kind or "nccl all-gather"
        # every rank owns the x slice of its rows; a step all-gathers x then multiplies
        sizes = torch.tensor([rows], device=dev)
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes)
        sizes_l = [int(s.item()) for s in all_sizes]
        pad = max(sizes_l)
        x_local = torch.zeros(pad, dtype=torch.float64, device=dev)
        x_local[:rows] = vec[bound.row_begin:bound.row_end]
        x_gathered = torch.empty(pad * world, dtype=torch.float64, device=dev)
        x_full = torch.empty(a.n_cols, dtype=torch.float64, device=dev)
        offs = np.concatenate([[0], np.cumsum(sizes_l)])

        def exchange():
            dist.all_gather_into_tensor(x_gathered, x_local)
            for r in range(world):
                x_full[offs[r]:offs[r + 1]] = x_gathered[r * pad:r * pad + sizes_l[r]]

        def step(ev_mid=None):
            exchange()
            if ev_mid is not None:
                ev_mid.record()
            bound.spmv(x_full, out)
    elif kernel == "spmv":
        def step(ev_mid=None):
            if ev_mid is not None:
                ev_mid.record()
            bound.spmv(vec, out)
    else:
        def step(ev_mid=None):
            if ev_mid is not None:
                ev_mid.record()
            bound.sptrsv(vec, out)

    # ---- parity against the C oracle, once, before timing ----
    parity = "unchecked"
    got = None
    try:
        from oracle.oracle import Oracle

        step()
        torch.cuda.synchronize()
        got = out[:rows].cpu().numpy()
        exp = plan.export_arrays()
        if kernel == "spmv":
            want = Oracle.run_spmv(exp, a.view(), vec_h)[bound.row_begin:bound.row_end]
        else:
            want = Oracle.run_sptrsv(exp, a.view(), vec_h)[0]
        parity = "bitwise" if np.array_equal(got.view(np.int64), want.view(np.int64)) else "MISMATCH"
        del exp
    except Exception as e:  # the oracle is a checker only; a failure here is reported, not hidden
        parity = f"unchecked ({type(e).__name__}: {e})"

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    # L2 flush between steps: write a 2x-L2 buffer, then read a second one, so
    # the step starts cold AND without dirty flush lines (their write-back
    # would otherwise be charged to the step's own HBM traffic)
    flush_buf = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    clean_buf = torch.ones(2 * l2 // 4, dtype=torch.float32, device=dev)
    clean_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush():
        flush_buf.zero_()
        torch.sum(clean_buf, 0, out=clean_sink)
    sampler = ClockSampler(local)

    for _ in range(args.warmup):
        flush()
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.time()
    for i in range(args.steps):
        flush()
        ev[i][0].record()
        step(ev[i][1])
        ev[i][2].record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    wall1 = time.time()
    step_ms = np.array([s.elapsed_time(e) for s, _, e in ev])
    kern_ms = np.array([m.elapsed_time(e) for _, m, e in ev])

    # ---- e2e: host buffers through the C ABI (H2D input, kernel, D2H result) ----
    e2e_parity = "unchecked"
    if sharded:
        e2e_ms = step_ms.copy()  # x already device-resident per rank; reported as the exchange+compute step
        h2d = d2h = 0
    else:
        host_in = torch.from_numpy(vec_h.copy()).pin_memory()
        host_out = torch.empty(max(rows, 1), dtype=torch.float64).pin_memory()
        hin, hout = host_in.numpy(), host_out.numpy()
        for _ in range(max(1, args.warmup)):
            (bound.spmv_host if kernel == "spmv" else bound.sptrsv_host)(hin, hout, stream=stream)
        torch.cuda.synchronize()
        e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
        for i in range(args.steps):
            e2e_ev[i][0].record()
            (bound.spmv_host if kernel == "spmv" else bound.sptrsv_host)(hin, hout, stream=stream)
            e2e_ev[i][1].record()
        torch.cuda.synchronize()
        e2e_ms = np.array([s.elapsed_time(e) for s, e in e2e_ev])
        h2d, d2h = 8 * a.n_cols, 8 * rows
        if got is not None and rows > 0:  # the host-buffer result against the device path's (oracle-checked) one
            e2e_parity = ("bitwise (equal to the device path)"
                          if np.array_equal(hout[:rows].view(np.int64), got.view(np.int64)) else "MISMATCH")
    sampler.stop()

    ms_step = float(step_ms.mean())
    ms_kern = float(kern_ms.mean())
    ms_e2e = float(e2e_ms.mean())
    if dist:
        t = torch.tensor([ms_step, ms_kern, ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, ms_kern, ms_e2e = [float(v) for v in t.tolist()]
    total_flops = flops(kernel, a.n_rows, a.nnz())
    units = total_flops if sharded else total_flops * world  # replicas: every rank does the whole job
    value = units / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    achieved = info["algorithmic_bytes"] / (ms_kern * 1e-3) / 1e9
    traffic = ncu_traffic(workload)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(kernel, a, args.t, args.groups, vec_h, args.cpu_seconds)
        except Exception as e:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "unavailable",
                   "sample": f"{type(e).__name__}: {e}"}
    clocks = sampler.summary(wall0, wall1)
    line = {
        "metric": "fp64 GFLOP/s of the codelet executor (2*nnz SpMV / 2*nnz-n SpTRSV)",
        "value": value,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config generator, DESIGN.md Inputs)",
        "config": {
            "workload": workload, "kernel": kernel, "n": a.n_rows, "nnz": a.nnz(), "t": args.t,
            "groups": args.groups, "partitions": n_parts, "scale": args.scale,
            "parallelism": (f"row-sharded x{world} (x exchange: {exchange_kind})" if sharded else
                            (f"replicas x{world}" if world > 1 else "single GPU")),
            "l2": "flushed before every timed step, outside the events: 2x-L2 write, then 2x-L2 read of a second buffer (cold, no dirty lines)",
            "mode": "parity (bitwise equal to the reference executor)",
            "bound": info,
        },
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": info["algorithmic_bytes"], "kernel_ms": ms_kern,
                     "peak_source": peak_src, "frac_of_nominal_8TBps": achieved / 8000.0},
        "cpu_baseline": cpu,
        "e2e": {"value": total_flops * (1 if sharded else world) / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                "path": "psc_bound_*_host (pinned host buffers; SpTRSV: b gathered from mapped host memory unit by unit in level order during the solve, x shipped per finished unit by bulk copies; column-split SpMV: x uploaded range by range ahead of its pass, y sent down per row slice of the last pass)",
                "parity": e2e_parity},
        "gpu_launches": args.steps * bound.launches(),
        "clocks": clocks,
        "inspector_seconds": inspector_s,
        "inspector_device_seconds": inspector_dev_s,
        "inspector_device_plan_equal": inspector_dev_same,
    }
    if kernel == "sptrsv":  # the solve is bound by its dependency chain, not by HBM
        line["roofline"]["critical_path"] = {
            "levels": n_parts, "ns_per_level": ms_kern * 1e6 / max(1, n_parts),
            "note": "sync-free solve: time ~ levels x per-level hop latency; HBM frac is not the binding limit"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
