#!/usr/bin/env python
"""Benchmark: simulated workload traces/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

`--gpus N` without a launcher (WORLD_SIZE unset) re-executes itself under
torch.distributed.run with N ranks (one process per GPU, NCCL), so both
launch forms measure N GPUs.

A "step" simulates the configuration's whole per-GPU trace batch (default C2:
1M traces x 64 apps) under every policy of the configuration (C2: all four),
i.e. one K1 trace_sim (on the lane engine: the main launch + the 64-bit-key
retry launch, which finds nothing to do on C2) + one K2 stats_reduce (+ the
cross-GPU aggregate all-gather for N > 1).  The unit is one trace simulated under one
policy.  Scaling is weak: every rank simulates its own contiguous trace-id
shard of the configured size, generated on its GPU before timing.

`value` is device-timed (CUDA events, max over ranks) with inputs resident
in HBM (1 GiB of T0 records per GPU, larger than L2).  `e2e` is the same
metric through the C ABI host-buffer call (sg_simulate_batch_host) with
pinned host inputs/outputs and all copies inside the timed region.
`cpu_baseline` times the reference's own simulate() (memshare, installed in
oracle/_ref) on the host cores over a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import multiprocessing as mp
import os
import platform
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_DIR = os.path.join(ROOT, "oracle", "_ref")
TIME_SCALE_DYADIC = 1000.0 / 1024.0
FALLBACK_HBM_GBS = 6650.0


# ------------------------------------------------------------- CPU reference

def _ref_worker(args):
    """Time the reference's simulate() on traces [t0, t1) of cfg under every
    policy until `budget_s` elapses.  Profiles are built before the timer."""
    cfg_name, n_traces_override, t0, t1, budget_s = args
    sys.path.insert(0, REF_DIR)
    sys.path.insert(0, ROOT)
    import memshare.device as rdev
    import memshare.harness as rh
    import memshare.policy as rp
    from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate

    cfg = CONFIGS[cfg_name]
    apps = as_u32x4(generate(cfg.gen, t0, t1 - t0))
    ndev = cfg.ndev
    specs = []
    for t in range(t1 - t0):
        for pol in cfg.policies:
            kind = rp.PolicyKind.parse(pol)
            for d in range(ndev):
                rows = [r for r in apps[t] if ((int(r[3]) >> 8) & 0xFF) == d] if ndev > 1 else apps[t]
                insts = [rh.AppProfile(f"a{i}", [rh.Phase(cpu_ms=int(a)),
                                                 rh.Phase(alloc_mib=int(m), busy_ms=int(b),
                                                          free_mib=int(m))], priority=int(at) & 0xFF)
                         for i, (a, m, b, at) in enumerate(rows)]
                specs.append((t, rh.WorkloadSpec(
                    instances=insts, policy=kind,
                    devices=rdev.parse_device_config({"devices": [{"mib": cfg.cap_mib[d]}]}),
                    time_scale=TIME_SCALE_DYADIC)))
    per_trace = len(cfg.policies) * ndev
    done = 0
    start = time.perf_counter()
    for i, (_, spec) in enumerate(specs):
        rh.simulate(spec)
        if (i + 1) % per_trace == 0:
            done += len(cfg.policies)
            if time.perf_counter() - start >= budget_s:
                break
    return done, time.perf_counter() - start


def cpu_reference_rate(cfg_name: str, budget_s: float, pool=None, cores=None, seed_base=10_000_000):
    """traces/s (trace x policy simulations) of the reference simulate() over
    all host cores, each core on its own contiguous trace range."""
    cores = cores or os.cpu_count() or 1
    from paper_1712_04495_b200.tracegen import CONFIGS
    cfg = CONFIGS[cfg_name]
    # enough traces per worker for the budget (reference ~1e3 traces/s/core at 64 apps)
    per = max(8, int(budget_s * 2000 * 64 / cfg.gen.apps_per_trace / len(cfg.policies)) + 1)
    jobs = [(cfg_name, None, seed_base + w * per, seed_base + (w + 1) * per, budget_s)
            for w in range(cores)]
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    try:
        res = pool.map(_ref_worker, jobs, chunksize=1)
    finally:
        if own:
            pool.close()
            pool.join()
    total = sum(d for d, _ in res)
    wall = max(t for _, t in res)
    return total / wall, total, wall, cores


def cpu_port_rate(cfg_name: str, n_traces: int):
    """The C restatement (oracle/, OpenMP over all cores) on a sample: a
    second, faster CPU point of comparison."""
    from oracle import oracle as O
    from paper_1712_04495_b200.tracegen import CONFIGS, as_u32x4, generate
    cfg = CONFIGS[cfg_name]
    apps = as_u32x4(generate(cfg.gen, 20_000_000, n_traces))
    t0 = time.perf_counter()
    for pol in cfg.policies:
        O.simulate_burst(apps, cfg.cap_mib, pol, threads=0)
    dt = time.perf_counter() - t0
    return n_traces * len(cfg.policies) / dt, dt


# ------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks and throttle reasons during the timed region, polled through
    NVML from a thread every 50 ms (an nvidia-smi child process was seen to
    stall single kernel launches when its queries land inside them); falls
    back to `nvidia-smi -lms 200` when pynvml is missing."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.thread = None
        self.rows = []
        self.out = ""
        self.window = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            sm_max = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            import threading
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), sm_max,
                                          ["Active" if r & b else "Not Active" for b in bits],
                                          time.perf_counter()))
                    except pynvml.NVMLError:
                        pass
                    self.stop.wait(0.05)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()
            for line in (self.out or "").splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    self.rows.append((float(f[1]), float(f[2]), f[5:9], None))
                except ValueError:
                    continue

    def mark(self, t0, t1):
        """The timed region (host perf_counter): summary() keeps its samples."""
        self.window = (t0, t1)

    def summary(self):
        rows = self.rows
        if self.window is not None:
            inside = [r for r in rows if r[3] is not None and self.window[0] <= r[3] <= self.window[1]]
            rows = inside or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted({self.NAMES[i] for _, _, r, _ in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons, "samples": len(rows),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


# ------------------------------------------------------------- helpers

def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "k1_traffic.json")
TRAFFIC_SOURCE = "dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full launch (profiles/k1_traffic.json)"


def measured_traffic(config, traces_per_gpu):
    """DRAM bytes per K1 launch from the committed ncu capture, when it was
    taken on this configuration and batch size (else None)."""
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    from paper_1712_04495_b200.tracegen import CONFIGS
    if t.get("config") != config or traces_per_gpu != CONFIGS[config].n_traces:
        return None
    return int(t["dram_bytes_read"]) + int(t["dram_bytes_write"]), t.get("issue_active_pct")


def cpu_model() -> str:
    """lscpu's model name (reported with every CPU number)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


def relaunch_distributed(args) -> int:
    """--gpus N > 1 outside a launcher: run this script as N ranks under
    torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------- reference arm

def run_reference_arm(args, ws, rank):
    from paper_1712_04495_b200.tracegen import CONFIGS
    cfg = CONFIGS[args.config]
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    pool = mp.get_context("fork").Pool(cores)
    try:
        budget = args.ref_step_s
        for _ in range(args.warmup):
            cpu_reference_rate(args.config, min(budget, 1.0), pool, cores, seed_base=30_000_000)
        rates, totals, walls = [], 0, 0.0
        for k in range(args.steps):
            r, tot, wall, _ = cpu_reference_rate(args.config, budget, pool, cores,
                                                 seed_base=40_000_000 + k * 1_000_000)
            rates.append(r)
            totals += tot
            walls += wall
    finally:
        pool.close()
        pool.join()
    value = totals / walls
    line = {
        "impl": "reference", "metric": "simulated workload traces/s",
        "value": value, "unit": "traces/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * walls / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": config_block(cfg, args, ws),
        "cpu_baseline": {"value": value, "unit": "traces/s", "cores": cores, "kind": "reference",
                         "sample": f"{totals} trace-policy simulations of {args.config} "
                                   f"(memshare.harness.simulate, {args.steps} steps of "
                                   f"~{budget:.1f} s on {cores} processes)",
                         "cpu": cpu_model(), "python": platform.python_version()},
        "e2e": {"value": value, "unit": "traces/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(cfg, args, ws):
    return {"workload": f"{cfg.name}: {cfg.description}", "traces_per_gpu": args.traces,
            "apps_per_trace": cfg.gen.apps_per_trace, "policies": list(cfg.policies),
            "devices_per_trace": cfg.ndev, "cap_mib": list(cfg.cap_mib), "seed": cfg.gen.seed,
            "unit": "one trace simulated under one policy",
            "l2": "inputs (16 B/app, >= 1 GiB per GPU at C2) exceed the 126 MB L2",
            "parallelism": f"trace shards x{ws}"}


# ------------------------------------------------------------- our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--traces", type=int, default=0, help="traces per GPU (default: config)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: check the multi-rank flow with several ranks on one GPU")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    ws, rank, local = dist_env()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    from paper_1712_04495_b200.tracegen import CONFIGS
    cfg = CONFIGS[args.config]
    if args.traces <= 0:
        args.traces = cfg.n_traces // max(cfg.gpus, 1) if cfg.gpus > 1 else cfg.n_traces

    if args.impl == "reference":
        return run_reference_arm(args, ws, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1712_04495_b200 import batch as B
    from paper_1712_04495_b200 import parallel as PAR
    from paper_1712_04495_b200.policy import policy_mask

    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    n = args.traces
    t_begin = rank * n
    napp = cfg.gen.apps_per_trace
    _, pols = policy_mask(cfg.policies)
    npol = len(pols)
    apps = B.generate_traces(cfg.gen, t_begin, n, device=local)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches = 0
    # K1 (lane engine: main pass + 64-bit-key retry pass) + K2 stats_reduce
    k1_launches = B.k1_launches(cfg.gen.apps_per_trace, npol, cfg.ndev)
    k1_kernel = B.K1_KERNELS[B.k1_engine(cfg.gen.apps_per_trace, npol, cfg.ndev)]

    def step(i=None):
        nonlocal launches
        if i is not None:
            ev[i][0].record(stream)
        res = B.simulate_batch(apps, pols, cfg.cap_mib, stream=stream)
        if i is not None:
            ev[i][1].record(stream)
        agg = B.reduce_stats(res.stats_raw, stream=stream)
        launches += k1_launches + 1
        if ws > 1:
            agg = PAR.allreduce_aggregate(agg)
        return res, agg

    # the clock sampler (an nvidia-smi child) starts before the warm-up: its
    # start-up must not land inside the timed steps; it keeps sampling
    # through them
    with ClockSampler(local) as clk:
        time.sleep(0.2)
        # warm-up keeps the previous step's outputs alive exactly like the
        # timed loop, so both output buffer sets are already in torch's
        # caching allocator (a cudaMalloc inside the timed region would
        # stall the stream between two steps)
        res = None
        for _ in range(args.warmup):
            res, agg = step()
        torch.cuda.synchronize()
        launches = 0
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        # a Python garbage-collection pass between two launches would leave
        # the stream idle (the host feeds the queue step by step)
        gc.collect()
        gc.disable()
        w0 = time.perf_counter()
        t_start.record(stream)
        for i in range(args.steps):
            res, agg = step(i)
        t_end.record(stream)
        torch.cuda.synchronize()
        clk.mark(w0, time.perf_counter())
        gc.enable()
    if ws > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    print(f"[bench] K1 per-step ms: {' '.join(f'{x:.2f}' for x in kern_ms)}", file=sys.stderr)
    tt = torch.tensor([elapsed_ms, max(kern_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tt[0])
    aggd = B.aggr_to_dict(agg)
    units_per_step = n * npol * ws
    value = units_per_step * args.steps / (elapsed_ms / 1000.0)
    ms_per_step = elapsed_ms / args.steps

    # roofline of K1: algorithmic bytes per launch / mean launch duration
    # (16 B/app in; per policy 8 B/app grant + end and, per (trace, device),
    # the 32 B record + 16 B percentages + 8 B speed-up out)
    in_b = n * napp * 16
    out_b = n * npol * (napp * 8 + cfg.ndev * (32 + 16 + 8))
    alg_bytes = in_b + out_b
    mean_k = statistics.mean(kern_ms) / 1000.0
    peak, peak_src = hbm_peak()
    achieved = alg_bytes / mean_k / 1e9
    traffic, issue_pct = measured_traffic(args.config, n) or (None, None)

    # e2e through the C ABI host-buffer pipeline
    e2e = None
    if not args.no_e2e:
        host_apps = B.pinned_apps(n, napp)
        host_apps[...] = apps.cpu().numpy().view(np.uint32)
        outb = B.HostBuffers(npol, n, napp, cfg.ndev)
        for _ in range(1):
            B.simulate_batch_host(host_apps, pols, cfg.cap_mib, device=local, out=outb,
                                  chunk_traces=args.chunk)
        e2e_steps = max(1, min(args.steps, 5))
        if ws > 1:
            dist.barrier()
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            hr = B.simulate_batch_host(host_apps, pols, cfg.cap_mib, device=local, out=outb,
                                       chunk_traces=args.chunk)
            _ = float(outb.stats["makespan"][0, 0, 0])
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        gc.enable()
        if ws > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": units_per_step * e2e_steps / float(dt[0]), "unit": "traces/s",
               "h2d_bytes_per_step": hr.h2d_bytes, "d2h_bytes_per_step": hr.d2h_bytes,
               "api": "sg_simulate_batch_host (C ABI, pinned host buffers, 4-stream pipeline; "
                      "end and busy ticks cross PCIe as u16 (K5 pack16) and host threads write "
                      "the grant and end arrays)",
               "steps": e2e_steps}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            r, tot, wall, cores = cpu_reference_rate(args.config, args.cpu_budget)
            cpu = {"value": r, "unit": "traces/s", "cores": cores, "kind": "reference",
                   "sample": f"{tot} trace-policy simulations of {args.config} traces "
                             f"[10M, ...) in {wall:.1f} s: memshare.harness.simulate "
                             f"(oracle/_ref) on {cores} processes",
                   "cpu": cpu_model(), "python": platform.python_version()}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": "traces/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc!r}"}
        try:
            pr, pdt = cpu_port_rate(args.config, 20_000 if napp <= 64 else 5_000)
            cpu["port"] = {"value": pr, "unit": "traces/s", "cores": os.cpu_count(),
                           "kind": "port", "sample": f"oracle/ C restatement, OpenMP, {pdt:.1f} s",
                           "cpu": cpu_model()}
        except Exception as exc:  # pragma: no cover
            cpu["port"] = {"value": None, "sample": f"unavailable: {exc!r}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "simulated workload traces/s", "value": value, "unit": "traces/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (counter-based SplitMix64 generator, generated on-GPU before timing)",
            "config": config_block(cfg, args, ws),
            "decisions_per_s": aggd["sum_grants"] / (ms_per_step / 1000.0),
            "events_per_s": aggd["sum_pops"] / (ms_per_step / 1000.0),
            "aggregate": aggd,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per launch",
                         "traffic_source": TRAFFIC_SOURCE if traffic else None, "peak_source": peak_src,
                         "kernel": k1_kernel, "alg_bytes_per_launch": alg_bytes,
                         "mean_launch_ms": mean_k * 1000.0,
                         # outputs only (the inputs are generated on the device
                         # before timing)
                         "alg_bytes_outputs_only": out_b,
                         "frac_outputs_only": out_b / mean_k / 1e9 / peak,
                         # what bounds this kernel instead: issue slots (the ncu capture above)
                         "issue_active_frac": issue_pct / 100.0 if issue_pct else None},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
