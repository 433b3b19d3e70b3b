#!/usr/bin/env python
"""Benchmark of the Q-less tall-skinny QR hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n COLS] [--m ROWS] [--no-sweep]
    python bench.py --config c4 [--gpus N]    # BASELINE configs[3]: 1e9 x 16 [A b] least squares, strong scaling
    python bench.py --impl reference ...      # the reference's CPU implementation, host cores

Metric: Q-less QR effective HBM GB/s = 8*m*n / t (one logical read of X).  One "step" is one
Q-less TSQR factorisation (sqb_tsqr_qless_dev: the streaming kernel + the R-factor combine) of
an m x n FP64 Gaussian matrix that is already resident in HBM.  Workload = BASELINE.json
configs[1] (single-B200 column sweep at m = 2^27): the headline is the n = 8 point of the sweep,
the whole sweep (n = 1..64, TSQR / CholQR2 / SVQB2) is attached as "sweep".  X (n GiB) is far
larger than the 126 MB L2, so every step streams from HBM.

`value` is the SUSTAINED figure: K steps timed after 300 ms of untimed back-to-back steps, i.e.
with the board on its power cap; `burst` is the same K steps on a settled (idle) board.

N > 1: `--gpus N` without a torchrun environment re-executes this script under
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU); under the driver's own
torchrun the ranks are used as given.  Rows are sharded: each rank factors its own 2^27-row slab and
the n x n triangles are combined with an NCCL all-gather inside the library (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Q-less QR effective HBM GB/s (8*m*n bytes / time-to-solution), FP64"
NOMINAL_HBM_GBS = 8000.0
FP64_PEAK_TFLOPS = 36.9   # measured DFMA / DMMA peak at 1.965 GHz (tools/probe_fp64.cu, profiles/probes/)
READ_CEILING_GBS = 7400.0  # measured read-only stream (tools/probe.cu)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def spawn_command(n_gpus, argv, port):
    """The command `--gpus N` re-executes when no torchrun environment is present."""
    # the launcher's own argument parser prefix-matches options placed after the script name (`--m` and `--n` are
    # ambiguous prefixes of its `--master-addr`, `--nnodes`, ...): only the contract's three flags go on the
    # command line, the full argument list travels in SQB_BENCH_ARGV (see main)
    os.environ["SQB_BENCH_ARGV"] = json.dumps(list(argv))
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", str(n_gpus)]


def rows_label(m):
    return f"2^{m.bit_length() - 1}" if m > 0 and m & (m - 1) == 0 else str(m)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    BAD = {0x08: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown"}
    NOTE = {0x04: "sw_power_cap"}

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self._stop_evt = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def run(self):
        if self.nv is None:
            return
        while not self._stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in {**self.BAD, **self.NOTE}.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.004)

    def stop(self):
        self._stop_evt.set()
        self.join(timeout=2)
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def roofline_bound(method, m, n, hbm_peak_gbs):
    """Which roofline binds one streaming pass: 8mn bytes over HBM against the pass's FP64 flops at
    the measured FP64 peak (TSQR 2mn^2; Gram mn(n+1) executed, gram.cpp:118-119)."""
    t_hbm = 8.0 * m * n / (hbm_peak_gbs * 1e9)
    flops = 2.0 * m * n * n if method == "tsqr" else float(m) * n * (n + 1)
    t_fp = flops / (FP64_PEAK_TFLOPS * 1e12)
    return ("hbm", t_hbm, flops) if t_hbm >= t_fp else ("fp64", t_fp, flops)


def cpu_reference_run(m, n, steps, warmup, method="tsqr", x_host=None):
    """Times the reference's own CPU implementation (oracle/_ref when built, else the C port) on
    the host cores.  Returns (best GB/s, mean GB/s, description dict)."""
    import numpy as np
    import oracle

    nbytes = 8.0 * m * n
    if oracle.ref is not None:
        ref = oracle.ref
        h, view = ref.matrix_handle(m, n)
        if x_host is not None:
            view[:, :] = x_host
            gen = "rows of the GPU arm's matrix"
        elif m * n <= (1 << 24):
            view[:, :] = oracle.gaussian(m, n, 1234)
            gen = "counter-based Gaussian, seed 1234"
        else:  # large samples: numpy's generator straight into the reference's buffer, column by column
            rng = np.random.default_rng(1234)
            for j in range(n):
                rng.standard_normal(m, out=view[:, j])
            gen = "numpy standard_normal, seed 1234"
        for _ in range(warmup):
            ref.timed(h, method, n)
        ts = [ref.timed(h, method, n)[0] for _ in range(steps)]
        ts_nv = [ref.timed(h, "tsqr_novalidate", n)[0] for _ in range(min(steps, 3))] if method == "tsqr" else []
        ref.matrix_destroy(h)
        info = {"kind": "reference", "cores": ref.threads, "kernel_table": ref.kernel_table()}
        if ts_nv:
            info["value_without_validation_scan"] = nbytes / min(ts_nv) / 1e9
    else:
        x = x_host if x_host is not None else oracle.gaussian(m, n, 1234)
        gen = "counter-based Gaussian, seed 1234"
        fn = {"tsqr": oracle.port.tsqr_qless, "cholqr2": oracle.port.cholqr2}[method]
        for _ in range(warmup):
            fn(x)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn(x)
            ts.append(time.perf_counter() - t0)
        info = {"kind": "port", "cores": 1}
    info["sample"] = (f"{method} of a {m} x {n} FP64 Gaussian ({nbytes / 2**30:.2f} GiB; {gen}), "
                      f"{steps} timed calls after {warmup} warm-ups")
    return nbytes / min(ts) / 1e9, nbytes * len(ts) / sum(ts) / 1e9, info


def reference_rows(m, n, requested):
    """Rows of the reference arm's matrix: the GPU arm's own m when the host has room for it
    (matrix + the reference's workspaces + slack), otherwise the largest power of two that fits."""
    if requested:
        return int(requested)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 8 << 30
    rows = m
    while rows > 1024 and 8 * rows * n * 1.5 + (2 << 30) > avail:
        rows //= 2
    return rows


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.n
    m = reference_rows(args.m, n, args.cpu_rows)
    best, mean, info = cpu_reference_run(m, n, args.steps, args.warmup)
    t_ms = 8.0 * m * n / (mean * 1e9) * 1e3
    info["value"] = mean
    info["unit"] = "GB/s"
    same = m == args.m
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": mean, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"tsqr_qless m=2^27 n={n} (BASELINE configs[1]); reference CPU path "
                               + ("at the GPU arm's full size" if same else f"on a bounded {m}-row sample of it"),
                   "m": m, "n": n, "same_config": same},
        "cpu_baseline": info, "best_gbs": best,
        "e2e": {"value": mean, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


class Rig:
    """One rank's device, context and process group."""

    def __init__(self):
        import torch
        import paper_2603_20889_b200 as sq
        from paper_2603_20889_b200 import sharding
        self.torch, self.sq, self.sharding = torch, sq, sharding
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # flow check on a one-GPU box (--share-gpu): every rank on cuda:0, gloo process group, the library's
        # exchange hook instead of NCCL (which refuses two ranks on one device) - never a scaling number
        share = os.environ.get("SQB_BENCH_SHARE_GPU") == "1"
        if share:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device(f"cuda:{self.local}")
        self.dist = None
        self.transport = None
        self.nccl_log = None
        self.ctx = sq.Context(self.local)
        self.ctx.use_torch_stream()
        if self.world > 1:
            import torch.distributed as dist
            # the communicator log stays on, but NCCL writes INFO lines to stdout by default, where the one
            # JSON line belongs: send them to a file and replay it on stderr when the run is over
            os.environ.setdefault("NCCL_DEBUG", "INFO" if self.rank == 0 else "WARN")
            if "NCCL_DEBUG_FILE" not in os.environ:
                self.nccl_log = os.path.join(tempfile.gettempdir(), f"sqb_nccl_{os.getpid()}.log")
                os.environ["NCCL_DEBUG_FILE"] = self.nccl_log
            if share:
                dist.init_process_group("gloo")
                self.transport = sharding.attach(self.ctx, dist) + " over gloo, ranks share cuda:0 (flow check only)"
            else:
                dist.init_process_group("nccl", device_id=self.dev)
                self.transport = sharding.attach(self.ctx, dist)  # the library's own NCCL communicator
            self.dist = dist

    def sync_all(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
            self.torch.cuda.synchronize()

    def max_ranks(self, v):
        return self.sharding.max_over_ranks(v, self.dist) if self.dist is not None else float(v)

    def timed(self, fn, steps, warmup, spinup_ms=0.0):
        """W warm-ups, then exactly K steps between CUDA events on the launching stream, bracketed by
        barrier + synchronize; max over ranks.  spinup_ms > 0 first runs untimed back-to-back steps so
        that the timed region starts with the board already on its sustained clocks."""
        torch, ctx = self.torch, self.ctx
        if spinup_ms > 0.0:
            t_end = time.perf_counter() + spinup_ms * 1e-3
            while time.perf_counter() < t_end:
                for _ in range(8):
                    fn()
                torch.cuda.synchronize()
        for _ in range(warmup):
            fn()
        self.sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ctx.launch_count
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        self.sync_all()
        ctx.synchronize("bench")  # surfaces device-side numerical failures
        return self.max_ranks(e0.elapsed_time(e1)) / steps, ctx.launch_count - l0

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()
        if self.nccl_log and os.path.exists(self.nccl_log):
            with open(self.nccl_log, errors="replace") as f:
                sys.stderr.write(f.read())
            os.unlink(self.nccl_log)


def traffic_per_launch(method, n, m):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full captures
    (profiles/traffic.json: bytes measured at `m` rows), scaled to this run's row count."""
    tfile = ROOT / "profiles" / "traffic.json"
    try:
        ent = json.loads(tfile.read_text()).get(f"{method}_n{n}")
        return float(ent["bytes"]) * m / float(ent["m"]) if ent else None
    except Exception:
        return None


def run_headline(rig, args):
    import numpy as np
    torch, sq, ctx = rig.torch, rig.sq, rig.ctx
    rank, world, local, dev = rig.rank, rig.world, rig.local, rig.dev
    m, n = args.m, args.n

    def run_method(x, method):
        if method == "tsqr":
            return ctx.tsqr_qless_sharded(x) if world > 1 else ctx.tsqr_qless(x)
        if method == "cholqr2":
            return ctx.cholqr2_sharded(x) if world > 1 else ctx.cholqr2(x)
        return ctx.svqb2_sharded(x) if world > 1 else ctx.svqb2(x)

    # ---- burst: K steps on a settled board, inputs resident in HBM ---------------------------------
    x = ctx.fill_gaussian(m, n, seed=1234, row_offset=rank * m, m_total=world * m)
    # the generator kernel (log/cos heavy) runs into the 1 kW power cap; let the board settle first
    torch.cuda.synchronize()
    time.sleep(1.0)
    sampler = ClockSampler(local)
    sampler.start()
    ms_burst, _ = rig.timed(lambda: run_method(x, args.method), args.steps, args.warmup)
    clocks_burst = sampler.stop()
    total_bytes = 8.0 * m * n * world
    burst = total_bytes / (ms_burst * 1e-3) / 1e9

    # ---- dominant kernel (the streaming launch that reads X once) timed IN SITU for the roofline:
    # the same step issued as its two launches, CUDA events bracketing the first one only
    peak, peak_src = measured_peaks()
    plan = ctx.default_tsqr_plan(m, n) if args.method == "tsqr" else ctx.default_gram_plan(m, n)
    lib, I64, vp = ctx.lib, sq.I64, ctx._ptr
    k = plan.num_blocks
    if args.method == "tsqr":
        y = ctx.empty_matrix(k * n, n)
        r_out = ctx.empty_matrix(n, n)

        def stream_launch():
            ctx._check(lib.sqb_tsqr_stage1_dev(ctx.handle, vp(x), I64(m), I64(n), I64(m), I64(0), I64(0),
                                               vp(y)), "stage1")

        def rest_of_step():  # stage 2: one block over the k stacked triangles, sign-normalised
            ctx._check(lib.sqb_tsqr_qless_dev(ctx.handle, vp(y), I64(k * n), I64(n), I64(k * n), I64(1),
                                              I64(k * n), vp(r_out)), "stage2")
        kname = ("tsqr_thread_kernel" if n <= 2 else "tsqr_fold_kernel" if n <= 28 else "tsqr_mma_kernel") + \
                " (stage 1: one launch streams X once)"
    else:
        c_out = ctx.empty_matrix(n, n)

        def stream_launch():
            ctx._check(lib.sqb_tsmttsm_dev(ctx.handle, vp(x), I64(m), I64(n), I64(m), I64(0), I64(0),
                                           vp(c_out)), "tsmttsm")

        def rest_of_step():
            ctx.cholesky(c_out)
        kname = "gram kernel (first streaming pass) + gram_reduce_kernel"
    time.sleep(0.5)  # settled board, like the burst figure
    for _ in range(args.warmup):
        stream_launch()
        rest_of_step()
    rig.sync_all()
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    for e0, e1 in pairs:
        e0.record()
        stream_launch()
        e1.record()
        rest_of_step()
    rig.sync_all()
    try:
        ctx.synchronize("bench")
    except sq.Error:
        pass
    ms_kernel = rig.max_ranks(sum(a.elapsed_time(b) for a, b in pairs) / len(pairs))
    bound, t_floor, flops = roofline_bound("tsqr" if args.method == "tsqr" else "gram", m, n, peak)
    achieved_gbs = 8.0 * m * n / (ms_kernel * 1e-3) / 1e9
    if bound == "hbm":
        roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                    "frac": achieved_gbs / peak, "peak_source": peak_src}
    else:  # FP64 pipe (DFMA and DMMA share it): algorithmic flops of the pass against the measured FP64 peak
        ach = flops / (ms_kernel * 1e-3) / 1e12
        roofline = {"bound": "fp64", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP64_PEAK_TFLOPS,
                    "peak_source": "measured FP64 DFMA/DMMA peak at 1.965 GHz (profiles/probes/probe_fp64.txt); "
                                   "the HBM roofline is not the binding one at this column count",
                    "achieved_gbs": achieved_gbs, "frac_of_hbm_copy_peak": achieved_gbs / peak}
    roofline.update({"traffic": traffic_per_launch(args.method, n, m), "kernel": kname, "kernel_ms": ms_kernel,
                     "frac_of_nominal_8TBs": achieved_gbs / NOMINAL_HBM_GBS,
                     "frac_of_measured_read_ceiling": achieved_gbs / READ_CEILING_GBS,
                     "algorithmic_bytes_per_launch": 8.0 * m * n, "algorithmic_flops_per_launch": flops,
                     "binding_floor_ms": t_floor * 1e3, "timed_on": "settled board (burst clocks)"})

    # ---- headline: the same K steps after 300 ms of back-to-back steps (sustained, on the power cap) --
    time.sleep(0.5)
    sampler2 = ClockSampler(local)
    sampler2.start()
    ms_step, launches = rig.timed(lambda: run_method(x, args.method), args.steps, args.warmup, spinup_ms=300.0)
    clocks = sampler2.stop()
    value = total_bytes / (ms_step * 1e-3) / 1e9

    out = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.method} m={rows_label(m)} n={n} Gaussian (BASELINE configs[1], headline point of the "
                               f"column sweep); value = SUSTAINED (K steps after 300 ms of untimed back-to-back "
                               f"steps, board on its power cap), burst = the same K steps on a settled board",
                   "m_per_gpu": m, "n": n, "method": args.method,
                   "l2": "inputs (>= 1 GiB) larger than the 126 MB L2; no flush needed",
                   "plan": {"num_blocks": plan.num_blocks, "panel_rows": plan.panel_rows},
                   "transport": rig.transport},
        "clocks": clocks, "gpu_launches": launches, "roofline": roofline,
        "burst": {"value": burst, "unit": "GB/s", "ms_per_step": ms_burst, "clocks": clocks_burst,
                  "frac_of_nominal_8TBs": burst / (NOMINAL_HBM_GBS * world)},
        "frac_of_nominal_8TBs": value / (NOMINAL_HBM_GBS * world),
    }

    # ---- end to end through the host-pointer API (H2D of X and D2H of R inside the timed region) --
    if not args.no_e2e:
        xh_t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        xh_t.copy_(x.t())
        xh = xh_t.numpy().T  # F-ordered m x n view of pinned memory
        if world > 1:
            fn = {"tsqr": ctx.tsqr_qless_sharded_host}.get(args.method)
        else:
            fn = {"tsqr": ctx.tsqr_qless, "cholqr2": ctx.cholqr2, "svqb2": ctx.svqb2}[args.method]
        if fn is not None:
            e2e_steps = max(3, min(args.steps, 10))
            fn(xh)
            rig.sync_all()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                fn(xh)
            rig.sync_all()
            dt = rig.max_ranks((time.perf_counter() - t0) / e2e_steps)
            out["e2e"] = {"value": total_bytes / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 8 * m * n,
                          "d2h_bytes_per_step": 8 * n * n, "ms_per_step": dt * 1e3, "steps": e2e_steps,
                          "api": f"paper_2603_20889_b200.{fn.__name__}(numpy pinned host array) -> sqb_*_host "
                                 f"(X streamed through a 3-slab ring, {ctx.host_slab_bytes >> 20} MiB slabs)"}
        del xh, xh_t

    # ---- the reference's CPU path on this box's host cores, bounded sample --------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            mc = args.cpu_rows or (1 << 27) // max(n, 8)
            xs = np.asfortranarray(x[:mc].cpu().numpy())
            best, mean, info = cpu_reference_run(mc, n, 5, 1, args.method, xs)
            info.update({"value": mean, "unit": "GB/s", "best": best})
            out["cpu_baseline"] = info
            # parity of the headline run against the reference on that sample
            import oracle
            r_gpu = run_method(x[:mc], args.method)
            ctx.synchronize()
            if args.method != "svqb2":
                o = oracle.ref or oracle.port
                r_cpu = o.tsqr_qless(xs) if args.method == "tsqr" else o.cholqr2(xs)
                err = float(np.linalg.norm(r_gpu.cpu().numpy() - r_cpu))
                out["parity"] = {"abs_err_F": err, "bound_64_n_eps_normX": float(64 * n * 2.22e-16 * np.linalg.norm(xs)),
                                 "rows": mc, "oracle": "reference" if oracle.ref else "port"}
        except Exception as exc:  # the baseline must never sink the bench line
            out["cpu_baseline"] = {"error": repr(exc)}

    # ---- column sweep (BASELINE configs[1]) ----------------------------------------------------------
    if world == 1 and not args.no_sweep:
        del x
        torch.cuda.empty_cache()
        # the reference's Roofline model (perf_model.hpp) with this box's measured copy bandwidth
        from paper_2603_20889_b200 import perf_model as pmod
        hw = pmod.find_hardware("B200")
        hw.mem_bandwidth = peak * 1e9
        out["model_hardware"] = {"name": hw.name, "mem_bandwidth": hw.mem_bandwidth, "peak_fp64": hw.peak_fp64,
                                 "machine_balance": pmod.machine_balance(hw)}
        out["sweep_protocol"] = f"{args.sweep_reps} timed reps after 3 warm-ups per point (reference PAPER.md:305-307)"
        sweep = []
        for nn in (1, 2, 4, 8, 16, 32, 64):
            xs = ctx.fill_gaussian(m, nn, seed=1234)
            row = {"n": nn, "gib": 8.0 * m * nn / 2**30}
            for meth in ("tsqr", "cholqr2", "svqb2"):
                try:
                    ms, _ = rig.timed(lambda: run_method(xs, meth), args.sweep_reps, 3)
                    gbs = 8.0 * m * nn / (ms * 1e-3) / 1e9
                    model_s = pmod.composite_time(hw, meth, m, nn)
                    bnd, t_fl, _ = roofline_bound("tsqr" if meth == "tsqr" else "gram", m, nn, peak)
                    passes = 1 if meth == "tsqr" else 2
                    row[meth] = {"ms": ms, "gbs": gbs, "frac_8TBs": gbs / NOMINAL_HBM_GBS, "frac_measured": gbs / peak,
                                 "bound": bnd, "frac_of_binding_roofline": passes * t_fl * 1e3 / ms,
                                 "model_time_s": model_s, "model_ratio": ms * 1e-3 / model_s}
                    if meth == "tsqr":
                        row[meth]["fp64_tflops_2mn2"] = 2.0 * m * nn * nn / (ms * 1e-3) / 1e12
                        # north_star "sustains": the same reps after 300 ms of back-to-back steps (power cap)
                        ms_s, _ = rig.timed(lambda: run_method(xs, meth), args.sweep_reps, 3, spinup_ms=300.0)
                        row[meth]["sustained_gbs"] = 8.0 * m * nn / (ms_s * 1e-3) / 1e9
                        row[meth]["sustained_frac_8TBs"] = row[meth]["sustained_gbs"] / NOMINAL_HBM_GBS
                        time.sleep(0.3)
                except sq.Error as exc:
                    row[meth] = {"error": type(exc).__name__}
            sweep.append(row)
            del xs
            torch.cuda.empty_cache()
        out["sweep"] = sweep
    return out


def run_c4(rig, args):
    """BASELINE configs[3]: single-pass least squares via Q-less QR of [A b], 1e9 x 16 FP64 (A: 15
    columns + b), rows sharded over the ranks (strong scaling: the total row count is fixed), n x n
    combine over NCCL.  The right-hand side is b = A x_true + 1e-3 * noise, so the solution is known."""
    import numpy as np
    torch, ctx = rig.torch, rig.ctx
    rank, world = rig.rank, rig.world
    m_total, ncols = args.c4_rows, 16
    n = ncols - 1
    lo, hi = rig.sharding.slab_bounds(m_total, world, rank)
    ml = hi - lo
    xl = ctx.fill_gaussian(ml, ncols, seed=1234, row_offset=lo, m_total=m_total)  # [A noise]
    a, rhs = xl[:, :n], xl[:, n]
    x_true = torch.linspace(-1.0, 1.0, n, dtype=torch.float64, device=rig.dev)
    rhs.mul_(1e-3)
    for j in range(n):  # harness only: b = A x_true + 1e-3 noise, one column at a time (no m x n temporary)
        rhs.add_(a[:, j], alpha=float(x_true[j]))
    torch.cuda.synchronize()
    time.sleep(1.0)

    def step():
        return ctx.solve_lstsq_sharded(a, rhs) if world > 1 else ctx.solve_lstsq(a, rhs, "tsqr")

    sampler = ClockSampler(rig.local)
    sampler.start()
    ms_step, launches = rig.timed(step, args.steps, args.warmup, spinup_ms=300.0)
    clocks = sampler.stop()
    xs, res = step()
    ctx.synchronize("c4")
    xs_h = xs.cpu().numpy()
    err = float(np.max(np.abs(xs_h - x_true.cpu().numpy())))
    # every rank must hold the same bits
    same = True
    if rig.dist is not None:
        ref = xs.clone()
        rig.dist.broadcast(ref, src=0)
        same = bool(torch.equal(ref, xs))
        flag = torch.tensor([1.0 if same else 0.0], device=rig.dev, dtype=torch.float64)
        rig.dist.all_reduce(flag, op=rig.dist.ReduceOp.MIN)
        same = bool(flag.item() == 1.0)
    total_bytes = 8.0 * m_total * ncols
    value = total_bytes / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    return {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"solve_lstsq via Q-less TSQR of [A b], {m_total} x {ncols} FP64 (A {n} columns + b), "
                               f"rows sharded over {world} GPU(s) (BASELINE configs[3]); sustained (300 ms spin-up)",
                   "m_total": m_total, "rows_per_gpu": ml, "n": n, "transport": rig.transport,
                   "l2": "slab (>= 16 GB per GPU) larger than the 126 MB L2"},
        "clocks": clocks, "gpu_launches": launches,
        "solution": {"max_abs_err_vs_x_true": err, "noise_over_sqrt_m": 1e-3 / np.sqrt(m_total),
                     "residual": float(res.item()), "identical_on_all_ranks": same},
        "roofline": {"bound": "hbm" if ncols <= 12 else "fp64", "achieved": value / world, "peak": peak, "unit": "GB/s",
                     "frac": value / world / peak, "traffic": None, "peak_source": peak_src,
                     "note": "whole step per GPU (streaming kernel + combine + exchange) against the copy bandwidth; "
                             "16 columns is past the HBM-bound range of the Householder kernels (FP64 floor "
                             f"{2.0 * ml * ncols * ncols / (FP64_PEAK_TFLOPS * 1e12) * 1e3:.2f} ms per GPU)"},
        "frac_of_nominal_8TBs": value / (NOMINAL_HBM_GBS * world),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="sweep", choices=["sweep", "c4"])
    ap.add_argument("--n", type=int, default=8, help="columns of the headline workload")
    ap.add_argument("--m", type=int, default=1 << 27, help="rows per GPU")
    ap.add_argument("--c4-rows", type=int, default=10**9, help="total rows of the c4 least-squares problem")
    ap.add_argument("--method", default="tsqr", choices=["tsqr", "cholqr2", "svqb2"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep-reps", type=int, default=50)
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--share-gpu", action="store_true",
                    help="flow check on a one-GPU box: all ranks on cuda:0 over gloo (not a scaling number)")
    forwarded = os.environ.get("SQB_BENCH_ARGV") if "WORLD_SIZE" in os.environ else None
    args = ap.parse_args(json.loads(forwarded)) if forwarded else ap.parse_args()
    if args.share_gpu:
        os.environ["SQB_BENCH_SHARE_GPU"] = "1"
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        return run_reference_arm(args)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher around us: start one process per GPU ourselves
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and not args.share_gpu:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
        return sys.exit(subprocess.call(spawn_command(args.gpus, sys.argv[1:], free_port())))

    rig = Rig()
    if rig.world != args.gpus and rig.rank == 0:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {rig.world} rank(s); reporting n_gpus = "
              f"{rig.world}", file=sys.stderr)
    out = run_c4(rig, args) if args.config == "c4" else run_headline(rig, args)
    if rig.rank == 0:
        print(json.dumps(out))
    rig.close()


if __name__ == "__main__":
    main()
