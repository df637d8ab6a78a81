#!/usr/bin/env python
"""Benchmark of the DDF codelet executor on B200 (BASELINE.json metric:
SpMV/SpTRSV fp64 GFLOP/s and % of the HBM roofline at 1/2/4/8 B200 vs host CPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--mode fast|parity]
                    [--impl ours|reference]

Default workload: BASELINE.json configs[4] -- SpMV on the symmetric power-law
matrix, n = 20M, nnz = 401M (the largest single-GPU configuration, and the one
the 1/2/4/8-GPU metric is defined on), plan t=3, groups=8, fast mode
(reassociated sums, gated at 1e-12 normwise against the reference's naive
baseline); the parity mode (bitwise equal to the reference executor) is timed
on the same workload and reported beside it. A step is one complete
y = A x. With N > 1 the plan's partitions are sharded over the ranks (row
shards, scheduler.cpp:67-89) and each step all-gathers x over NCCL first
("scaling": "strong"); SpTRSV configs (2, 4) run N replicas ("weak").

--gpus N without torchrun re-launches this script under
torch.distributed.run with N ranks; under torchrun the world size must be N.

Timing: W untimed warm-up steps; K timed steps between a barrier +
cudaDeviceSynchronize on both sides; each step is bracketed by CUDA events on
the launching stream with an L2 flush before it, outside the events (a
2x-L2 write, then a 2x-L2 read of a second buffer, so no dirty flush lines are
written back during the step); ms_per_step is the mean device time, maxed
over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
METRIC = "fp64 GFLOP/s of the codelet executor (2*nnz SpMV / 2*nnz-n SpTRSV)"
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                "clocks_event_reasons.sw_power_cap")
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    p.add_argument("--mode", default="fast", choices=["fast", "parity"],
                   help="SpMV summation: fast (reassociated, 1e-12 normwise) or parity (bitwise the reference's)")
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--t", type=int, default=3)
    p.add_argument("--groups", type=int, default=8)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-repeats", type=int, default=3, help="reference run_bench repetitions (CPU baseline)")
    return p.parse_args()


def flops(kernel, n_rows, nnz):
    """theoretical_flops, bench.cpp:27-32."""
    return 2 * nnz if kernel == "spmv" else 2 * nnz - n_rows


def config_dict(args, kernel, workload, n, nnz, world):
    """The same dict from both arms (the driver compares them)."""
    sharded = kernel == "spmv" and world > 1
    return {"workload": workload, "kernel": kernel, "n": n, "nnz": nnz, "t": args.t, "groups": args.groups,
            "scale": args.scale, "mode": args.mode if kernel == "spmv" else "parity",
            "parallelism": (f"row shards x{world} (x exchanged every step)" if sharded else
                            (f"replicas x{world}" if world > 1 else "single device")),
            "l2": "flushed before every timed step (2x-L2 write, then 2x-L2 read of a second buffer)"}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms."""

    def __init__(self, index):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={CLOCK_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def ncu_traffic(workload, mode):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{workload}/{mode}")
    except Exception:
        return None


def cpu_baseline(kernel, csr_view, args, vec, results):
    """The reference's own run_bench (bench.cpp:118-187: inspect, then paired
    medians of the naive baseline and the executor) on the host cores: SpMV
    at every host thread and at 1 worker; SpTRSV at 1 worker (the reference
    pool races on deep level-set solves). As the checker (not
    timed), the reference executor and naive baseline also run once on the
    bench's input and every GPU mode's result is compared with them."""
    from oracle.oracle import Ref

    if not Ref.available():
        return ({"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "unavailable",
                 "sample": "oracle/_ref (the reference library) was not built"}, "unchecked (no reference library)")
    rc = Ref.csr(csr_view)
    k = 0 if kernel == "spmv" else 1
    nproc = os.cpu_count() or 1
    plan, insp = Ref.time_inspect(k, rc, args.t, args.groups)
    n_flops = flops(kernel, csr_view.n_rows, csr_view.nnz)
    runs = {}
    for w in ([nproc, 1] if kernel == "spmv" else [1]):
        runs[w] = Ref.paired_timing(plan, rc, k, vec, w, args.cpu_repeats if w > 1 else max(1, args.cpu_repeats - 1))
    top = max(runs)
    base_s = runs[top][0]
    cpu = {"value": n_flops / runs[top][1] / 1e9, "unit": "GFLOP/s", "cores": top, "kind": "reference",
           "sample": (f"the reference inspector once, then run_bench's paired protocol (bench.cpp:88-104: one "
                      f"warm-up, {args.cpu_repeats} alternating repetitions, medians) of the naive CSR baseline and "
                      f"psc::run_{kernel} on the full matrix at workers={top}"
                      + (f" and at workers=1 ({max(1, args.cpu_repeats - 1)} repetitions)" if len(runs) > 1 else "")),
           "cpu_model": cpu_model(),
           "executor_ms": {str(w): r[1] * 1e3 for w, r in runs.items()},
           "executor_gflops": {str(w): n_flops / r[1] / 1e9 for w, r in runs.items()},
           "naive_baseline_ms": base_s * 1e3,
           "naive_baseline_gflops": n_flops / base_s / 1e9,
           "reference_inspector_s": insp}
    # the checker: the reference executor and naive baseline on this input
    if kernel == "spmv":
        want, base = Ref.run_spmv(plan, rc, vec, nproc), Ref.spmv_baseline(rc, vec)
    else:
        want, base = Ref.run_sptrsv(plan, rc, vec, 1)[0], Ref.sptrsv_baseline(rc, vec)
    den = float(np.max(np.abs(base))) or 1.0
    tol = 1e-12 if kernel == "spmv" else 1e-10
    check = {"tolerance_normwise": tol}
    for mode, got in results.items():
        if mode is None or got is None:
            continue
        bitwise = bool(np.array_equal(got.view(np.int64), want.view(np.int64)))
        nw = float(np.max(np.abs(got - base)) / den)
        check[mode] = {"bitwise_vs_reference_executor": bitwise, "normwise_vs_reference_baseline": nw,
                       "ok": bitwise if mode == "parity" else nw <= tol}
    return cpu, check


def run_reference(args):
    """--impl reference: the reference's own CPU executor (oracle/_ref, built
    from /root/reference) on this box's host cores, every host thread; the
    inputs come from configs.cpp compiled into that same library, so no
    product library is loaded."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle.oracle import Ref

    kernel, workload = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpsc_ref.so was not built"}), flush=True)
        return
    a = Ref.generate_config(args.config, args.scale)
    v = a.view()
    vec = Ref.uniform_vector(v.n_cols, 10 + args.config)
    n_flops = flops(kernel, v.n_rows, v.nnz)
    workers = 1 if kernel == "sptrsv" else (os.cpu_count() or 1)
    rplan, insp = Ref.time_inspect(0 if kernel == "spmv" else 1, a, args.t, args.groups)
    fn = Ref.time_spmv if kernel == "spmv" else Ref.time_sptrsv
    times, _ = fn(rplan, a, vec, workers, args.warmup, args.steps)
    value = n_flops * len(times) / times.sum() / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(times.mean() * 1e3), "higher_is_better": True,
        "scaling": "strong" if kernel == "spmv" and world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config generator, DESIGN.md Inputs)", "impl": "reference",
        "config": config_dict(args, kernel, workload, v.n_rows, v.nnz, world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                         "sample": f"{len(times)} complete psc::run_{kernel} calls on the full matrix, "
                                   f"workers={workers}, after {args.warmup} untimed ones",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ms_median": float(np.median(times) * 1e3),
        "inspector_seconds": insp,
        "device": "host CPU",
        "native_libs": mapped_repo_libs(),
    }
    print(json.dumps(line), flush=True)


def mapped_repo_libs():
    """This repo's shared libraries mapped into this process (the reference arm must map only oracle/_ref)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {line.split()[-1] for line in f if line.rstrip().endswith(".so")}
        return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT))
    except Exception:
        return None


def spawn(args):
    """--gpus N without torchrun: re-launch under torch.distributed.run with N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def run_ours(args):
    import torch

    import paper_2111_12243_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    kernel, workload = CONFIGS[args.config]
    mode = args.mode if kernel == "spmv" else "parity"
    kk = P.KernelKind.Spmv if kernel == "spmv" else P.KernelKind.Sptrsv
    a = P.generate_config(args.config, args.scale)
    t0 = time.perf_counter()
    # (ranks share the host: each inspects with its share of the cores; the plan is the same)
    plan = P.inspect(kk, a, args.t, args.groups, max(1, (os.cpu_count() or 1) // world) if world > 1 else 0)
    inspector_s = time.perf_counter() - t0
    inspector_dev_s, inspector_dev_same = None, None
    if world == 1:  # the same inspection with the window mining on the GPU (same plan, bit for bit)
        t0 = time.perf_counter()
        plan_dev = P.inspect_device(kk, a, args.t, args.groups, local)
        inspector_dev_s = time.perf_counter() - t0
        inspector_dev_same = plan_dev.hash() == plan.hash()
        del plan_dev
    exe = P.Executor(1, local)
    n_parts = plan.counts().n_partitions
    sharded = kernel == "spmv" and world > 1
    parts = None
    if sharded:
        from paper_2111_12243_b200.dist import shard_partitions

        parts = shard_partitions(n_parts, world, rank)
    mode_id = 1 if mode == "fast" else 0
    bound = P.BoundPlan(exe, plan, a, mode=mode_id, partitions=parts)
    info = bound.info()
    dev = torch.device("cuda", local)
    vec_h = P.uniform_vector(a.n_cols, 10 + args.config)
    vec = torch.from_numpy(vec_h).to(dev)
    rows = bound.row_end - bound.row_begin
    out = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    exchange = None
    if sharded:
        # every rank owns the x slice of its rows. A step exchanges x and
        # multiplies: over peer memory (IPC windows; fast mode: copy-engine pulls
        # pass by pass, each pass waiting only for its column range), or, where
        # IPC is unavailable on any rank, an NCCL all-gather then the multiply
        from paper_2111_12243_b200.dist import PeerExchange, XExchange, shard_row_ranges

        ranges = shard_row_ranges(plan, world)
        x_mine = vec[bound.row_begin:bound.row_end].clone()
        pex, ok = None, 1
        try:
            pex = PeerExchange(bound, ranges, rank, a.n_cols)
        except Exception as err:  # every rank reaches the all-reduce below
            print(f"bench.py: peer exchange unavailable on rank {rank}: {err}", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0 and pex is not None:
            pex.close()
            pex = None
        if pex is not None:
            exchange = "peer pulls over NVLink (IPC windows)"

            def exchange_multiply(xs):
                pex.multiply(xs, out)
        else:
            exchange = "NCCL all-gather"
            xex = XExchange(ranges, a.n_cols, dev)

            def exchange_multiply(xs):
                bound.spmv(xex.exchange(xs), out)

        def step():
            exchange_multiply(x_mine)
    elif kernel == "spmv":
        def step(b=bound):
            b.spmv(vec, out)
    else:
        def step(b=bound):
            b.sptrsv(vec, out)

    step()
    torch.cuda.synchronize()
    got = out[:rows].cpu().numpy()

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    clean_buf = torch.ones(2 * l2 // 4, dtype=torch.float32, device=dev)
    clean_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush():
        flush_buf.zero_()
        torch.sum(clean_buf, 0, out=clean_sink)

    def timed(fn, steps, warmup, barrier):
        for _ in range(warmup):
            flush()
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        if barrier and dist:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.time()
        for i in range(steps):
            flush()
            ev[i][0].record()
            fn()
            ev[i][1].record()
        torch.cuda.synchronize()
        if barrier and dist:
            dist.barrier()
        w1 = time.time()
        return np.array([s.elapsed_time(e) for s, e in ev]), w0, w1

    sampler = ClockSampler(local)
    step_ms, wall0, wall1 = timed(step, args.steps, args.warmup, True)

    # ---- the other SpMV mode on the same workload (parity when the headline is fast) ----
    other, other_got = None, None
    if kernel == "spmv" and not sharded:
        other_mode = "parity" if mode == "fast" else "fast"
        ob = P.BoundPlan(exe, plan, a, mode=1 if other_mode == "fast" else 0)
        ob.spmv(vec, out)
        torch.cuda.synchronize()
        other_got = out[:rows].cpu().numpy()
        oms, _, _ = timed(lambda: ob.spmv(vec, out), max(3, args.steps // 5), 2, False)
        other = {"mode": other_mode, "ms_per_step": float(oms.mean()),
                 "value": flops(kernel, a.n_rows, a.nnz()) / (oms.mean() * 1e-3) / 1e9,
                 "frac_of_hbm_peak": info["algorithmic_bytes"] / (oms.mean() * 1e-3) / 1e9 / measured_peak()[0],
                 "launches_per_step": ob.launches()}
        ob.close()

    # ---- e2e: the public host-buffer API (H2D input, kernels, D2H result) ----
    e2e_check = None
    if sharded:
        # per rank: its x slice up from pinned host memory, the exchange and the
        # shard's multiply, its y rows back down
        host_in = torch.from_numpy(vec_h[bound.row_begin:bound.row_end].copy()).pin_memory()
        host_out = torch.empty(max(rows, 1), dtype=torch.float64).pin_memory()
        dev_in = torch.empty_like(x_mine)

        def e2e_step():
            dev_in.copy_(host_in, non_blocking=True)
            exchange_multiply(dev_in)
            host_out.copy_(out, non_blocking=True)

        e2e_ms, _, _ = timed(e2e_step, args.steps, args.warmup, True)
        h2d, d2h = 8 * rows, 8 * rows
        e2e_check = "bitwise equal to the device path" if np.array_equal(
            host_out.numpy()[:rows].view(np.int64), got.view(np.int64)) else "MISMATCH"
    else:
        host_in = torch.from_numpy(vec_h.copy()).pin_memory()
        host_out = torch.empty(max(rows, 1), dtype=torch.float64).pin_memory()
        hin, hout = host_in.numpy(), host_out.numpy()
        call = bound.spmv_host if kernel == "spmv" else bound.sptrsv_host
        for _ in range(max(1, args.warmup)):
            call(hin, hout, stream=stream)
        torch.cuda.synchronize()
        e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
        for i in range(args.steps):
            e2e_ev[i][0].record()
            call(hin, hout, stream=stream)
            e2e_ev[i][1].record()
        torch.cuda.synchronize()
        e2e_ms = np.array([s.elapsed_time(e) for s, e in e2e_ev])
        h2d, d2h = 8 * a.n_cols, 8 * rows
        e2e_check = "bitwise equal to the device path" if np.array_equal(hout[:rows].view(np.int64), got.view(np.int64)) \
            else "MISMATCH"
    sampler.stop()

    ms_step, ms_e2e = float(step_ms.mean()), float(e2e_ms.mean())
    if dist:
        t = torch.tensor([ms_step, ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, ms_e2e = [float(v) for v in t.tolist()]
    total_flops = flops(kernel, a.n_rows, a.nnz())
    units = total_flops if sharded else total_flops * world  # replicas: every rank does the whole job
    value = units / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    achieved = info["algorithmic_bytes"] / (ms_step * 1e-3) / 1e9
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu, parity = None, "unchecked (N > 1, or --no-cpu-baseline)"
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu, parity = cpu_baseline(kernel, a.view(), args, vec_h, {mode: got, other["mode"] if other else None: other_got})
        except Exception as e:  # reported, not hidden
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "unavailable", "sample": f"{type(e).__name__}: {e}"}
            parity = f"unchecked ({type(e).__name__}: {e})"
    line = {
        "metric": METRIC,
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
        "config": config_dict(args, kernel, workload, a.n_rows, a.nnz(), world),
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(workload, mode),
                     "algorithmic_bytes_per_step": info["algorithmic_bytes"],
                     "bytes_formula": ("12*nnz + 4*(n+1) + 8*n_cols + 8*n (SpMV)" if kernel == "spmv" else
                                       "12*nnz + 4*(n+1) + 16*n (SpTRSV)") + ", SURVEY.md §8d",
                     "timed": f"the whole step ({bound.launches()} launches of this repo's kernels) per CUDA events on the launching stream",
                     "peak_source": peak_src, "frac_of_nominal_8TBps": achieved / 8000.0},
        "other_mode": other,
        "cpu_baseline": cpu,
        "e2e": {"value": total_flops * (1 if sharded else world) / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                "path": ("per rank: its x slice up from pinned host memory, the exchange and the shard's multiply, "
                         "its rows back down" if sharded else
                         "psc_bound_*_host with pinned host buffers (the C ABI's host-buffer entry points)"),
                "check": e2e_check},
        "exchange": exchange,
        "gpu_launches": args.steps * bound.launches(),
        "clocks": sampler.summary(wall0, wall1),
        "inspector_seconds": inspector_s,
        "inspector_device_seconds": inspector_dev_s,
        "inspector_device_plan_equal": inspector_dev_same,
        "bound": info,
    }
    if kernel == "sptrsv":  # the solve is bound by its dependency chain
        # a bitwise solve carries each x into the next level through 7 dependent FP64 operations
        # (multiply, add, 0 + partial, subtract, three division steps, 8-9 cycles each) plus the hop
        # between lanes: ~100 cycles per level at best
        sm_ghz = float(line["clocks"].get("sm_max_mhz") or 1965.0) / 1e3
        floor_ms = n_parts * 100.0 / sm_ghz * 1e-6
        line["roofline"]["critical_path"] = {
            "levels": n_parts, "ns_per_level": ms_step * 1e6 / max(1, n_parts),
            "parity_floor_ms": floor_ms,
            "target_0p30_ms": info["algorithmic_bytes"] / (0.30 * peak * 1e9) * 1e3,
            "note": "sync-free solve: time ~ levels x per-level hop latency; parity_floor_ms = levels x ~100 cycles "
                    "(the dependent FP64 chain of one row), the least any bitwise-equal solve can take"}
        if args.config != 4:  # (config 4's long rows take the streaming kernel: no records)
            line["roofline"]["record_pack"] = "the per-row record pack (trsv_pack_kernel) runs at bind and after a value change, outside the timed step"
    if args.config == 5 and mode == "fast":  # uniformly random columns: the gathers, not HBM, bound the step
        line["roofline"]["gather_bound"] = {
            "note": "each entry gathers one x value at a random column (config 5); the L1/L2 path serves ~1 such gather "
                    "per SM-cycle (tools/gather_probe.cu on this B200: 255 G gathers/s beside a 12 B/entry stream), "
                    "so 401M gathers take >= ~1.57 ms whatever the HBM bandwidth (DESIGN.md)",
            "gathers_per_step": a.nnz(),
            "gathers_per_s_measured": 255e9,
            "bound_ms": a.nnz() / 255e9 * 1e3,
            "frac": (a.nnz() / 255e9 * 1e3) / ms_step}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
