#!/usr/bin/env python
"""Benchmark of the Q-less tall-skinny QR hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n COLS] [--m ROWS] [--no-sweep]
    python bench.py --impl reference ...      # the reference's CPU implementation, host cores

Metric: Q-less QR effective HBM GB/s = 8*m*n / t (one logical read of X).  One "step" is one
Q-less TSQR factorisation (sqb_tsqr_qless_dev: the streaming kernel + the R-factor combine) of
an m x n FP64 Gaussian matrix that is already resident in HBM.  Workload = BASELINE.json
configs[1] (single-B200 column sweep at m = 2^27): the headline `value` is the n = 8 point of the
sweep, the whole sweep (n = 1..64, TSQR / CholQR2 / SVQB2) is attached as "sweep".  X (n GiB) is
far larger than the 126 MB L2, so every step streams from HBM.

N > 1 (torchrun, one process per GPU): rows are sharded, each rank factors its own 2^27-row slab
and the n x n triangles are combined with an NCCL all-gather (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Q-less QR effective HBM GB/s (8*m*n bytes / time-to-solution), FP64"
NOMINAL_HBM_GBS = 8000.0


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def cpu_reference_run(m, n, steps, warmup, method="tsqr", x_host=None):
    """Times the reference's own CPU implementation (oracle/_ref when built, else the C port) on
    the host cores.  Returns (best GB/s, mean GB/s, description dict)."""
    import numpy as np
    import oracle

    nbytes = 8.0 * m * n
    if oracle.ref is not None:
        ref = oracle.ref
        h, view = ref.matrix_handle(m, n)
        view[:, :] = x_host if x_host is not None else oracle.gaussian(m, n, 1234)
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
        fn = {"tsqr": oracle.port.tsqr_qless, "cholqr2": oracle.port.cholqr2}[method]
        for _ in range(warmup):
            fn(x)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn(x)
            ts.append(time.perf_counter() - t0)
        info = {"kind": "port", "cores": 1}
    info["sample"] = f"{method} of a {m} x {n} FP64 Gaussian ({nbytes / 2**30:.2f} GiB), {steps} timed calls"
    return nbytes / min(ts) / 1e9, nbytes * len(ts) / sum(ts) / 1e9, info


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.n
    m = args.cpu_rows or (1 << 27) // max(n, 8)
    best, mean, info = cpu_reference_run(m, n, args.steps, args.warmup)
    t_ms = 8.0 * m * n / (mean * 1e9) * 1e3
    info["value"] = mean
    info["unit"] = "GB/s"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": mean, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"tsqr_qless m=2^27 n={n} (BASELINE configs[1]); reference CPU path on a "
                               f"bounded {m}-row sample of it", "m": m, "n": n},
        "cpu_baseline": info, "best_gbs": best,
        "e2e": {"value": mean, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=8, help="columns of the headline workload")
    ap.add_argument("--m", type=int, default=1 << 27, help="rows per GPU")
    ap.add_argument("--method", default="tsqr", choices=["tsqr", "cholqr2", "svqb2"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sweep-reps", type=int, default=5)
    ap.add_argument("--cpu-rows", type=int, default=0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import paper_2603_20889_b200 as sq

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = sq.Context(local)
    ctx.use_torch_stream()
    if world > 1:
        box = [ctx.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ctx.init_nccl(box[0], rank, world)

    m, n = args.m, args.n
    dev = torch.device(f"cuda:{local}")

    def sync_all():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    def run_method(x, method):
        if method == "tsqr":
            return ctx.tsqr_qless_sharded(x) if world > 1 else ctx.tsqr_qless(x)
        if method == "cholqr2":
            return ctx.cholqr2_sharded(x) if world > 1 else ctx.cholqr2(x)
        return ctx.svqb2_sharded(x) if world > 1 else ctx.svqb2(x)

    def timed(fn, steps, warmup, spinup_ms=0.0):
        # optional untimed spin-up so that the timed region starts at steady clocks (a 1.4 ms step
        # times 3 warm-ups is over before the SM clock has ramped), then the W warm-up steps proper
        if spinup_ms > 0.0:
            t_end = time.perf_counter() + spinup_ms * 1e-3
            while time.perf_counter() < t_end:
                for _ in range(8):
                    fn()
                torch.cuda.synchronize()
        for _ in range(warmup):
            fn()
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ctx.launch_count
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        sync_all()
        ctx.synchronize("bench")  # surfaces device-side numerical failures
        ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps, ctx.launch_count - l0

    # ---- headline: whole-job throughput, inputs resident in HBM ------------------------------
    x = ctx.fill_gaussian(m, n, seed=1234, row_offset=rank * m, m_total=world * m)
    # the generator kernel (log/cos heavy) runs into the 1 kW power cap; let the board settle so the
    # timed region measures the TSQR step, not the generator's thermal tail
    torch.cuda.synchronize()
    time.sleep(1.0)
    sampler = ClockSampler(local)
    sampler.start()
    ms_step, launches = timed(lambda: run_method(x, args.method), args.steps, args.warmup)
    clocks = sampler.stop()
    total_bytes = 8.0 * m * n * world
    value = total_bytes / (ms_step * 1e-3) / 1e9
    # ---- dominant kernel (the streaming launch that reads X once) timed IN SITU for the roofline:
    # the same step as above issued as its two launches, CUDA events bracketing the first one only
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
        kname = ("tsqr_thread_kernel" if n <= 4 else "tsqr_fold_kernel" if n <= 28 else "tsqr_mma_kernel") + \
                " (stage 1: one launch streams X once)"
    else:
        c_out = ctx.empty_matrix(n, n)

        def stream_launch():
            ctx._check(lib.sqb_tsmttsm_dev(ctx.handle, vp(x), I64(m), I64(n), I64(m), I64(0), I64(0),
                                           vp(c_out)), "tsmttsm")

        def rest_of_step():
            ctx.cholesky(c_out)
        kname = "gram kernel (first streaming pass) + gram_reduce_kernel"
    time.sleep(0.5)  # same board state as the headline: settled, not on the power cap
    for _ in range(args.warmup):
        stream_launch()
        rest_of_step()
    sync_all()
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    for e0, e1 in pairs:
        e0.record()
        stream_launch()
        e1.record()
        rest_of_step()
    sync_all()
    try:
        ctx.synchronize("bench")
    except sq.Error:
        pass
    ms_kernel = sum(a.elapsed_time(b) for a, b in pairs) / len(pairs)
    if dist is not None:
        t = torch.tensor([ms_kernel], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_kernel = float(t.item())
    achieved = 8.0 * m * n / (ms_kernel * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get(f"{args.method}_n{n}")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname, "kernel_ms": ms_kernel, "peak_source": peak_src,
                "frac_of_nominal_8TBs": achieved / NOMINAL_HBM_GBS,
                "frac_of_measured_read_ceiling_7400": achieved / 7400.0,
                "algorithmic_bytes_per_launch": 8.0 * m * n}

    time.sleep(0.5)
    # the same K steps after 300 ms of back-to-back steps: the sustained figure under the power cap
    sampler2 = ClockSampler(local)
    sampler2.start()
    ms_sus, _ = timed(lambda: run_method(x, args.method), args.steps, args.warmup, spinup_ms=300.0)
    clocks_sus = sampler2.stop()
    sustained = {"value": total_bytes / (ms_sus * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms_sus,
                 "clocks": clocks_sus, "note": "same K steps after 300 ms of untimed back-to-back steps"}

    out = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.method} m=2^27 n={n} Gaussian (BASELINE configs[1], headline point "
                               f"of the column sweep)", "m_per_gpu": m, "n": n, "method": args.method,
                   "l2": "inputs (>= 1 GiB) larger than the 126 MB L2; no flush needed",
                   "plan": {"num_blocks": plan.num_blocks, "panel_rows": plan.panel_rows}},
        "clocks": clocks, "gpu_launches": launches, "roofline": roofline, "sustained": sustained,
        "frac_of_nominal_8TBs": value / (NOMINAL_HBM_GBS * world),
    }

    # ---- end to end through the host-pointer API (H2D of X and D2H of R inside the timed region) --
    if not args.no_e2e:
        xh_t = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        xh_t.copy_(x.t())
        xh = xh_t.numpy().T  # F-ordered m x n view of pinned memory
        fn = {"tsqr": ctx.tsqr_qless, "cholqr2": ctx.cholqr2, "svqb2": ctx.svqb2}[args.method]
        e2e_steps = max(3, min(args.steps, 10))
        fn(xh)
        sync_all()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r_host = fn(xh)
        sync_all()
        dt = (time.perf_counter() - t0) / e2e_steps
        if dist is not None:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        out["e2e"] = {"value": total_bytes / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 8 * m * n,
                      "d2h_bytes_per_step": 8 * n * n, "ms_per_step": dt * 1e3, "steps": e2e_steps,
                      "api": f"paper_2603_20889_b200.{fn.__name__}(numpy pinned host array) -> sqb_*_host"}
        del xh, xh_t

    # ---- the reference's CPU path on this box's host cores, bounded sample --------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            mc = args.cpu_rows or (1 << 27) // max(n, 8)
            xs = np.asfortranarray(x[:mc].cpu().numpy())
            best, mean, info = cpu_reference_run(mc, n, 5, 1, args.method if args.method != "svqb2" else "svqb2", xs)
            info.update({"value": mean, "unit": "GB/s", "best": best})
            out["cpu_baseline"] = info
            # parity of the headline run against the reference on that sample
            import oracle
            r_gpu = run_method(x[:mc], args.method)
            ctx.synchronize()
            if args.method != "svqb2":
                r_cpu = (oracle.ref or oracle.port).tsqr_qless(xs) if args.method == "tsqr" else (oracle.ref or oracle.port).cholqr2(xs)
                err = float(np.linalg.norm(r_gpu.cpu().numpy() - r_cpu))
                out["parity"] = {"abs_err_F": err, "bound_64_n_eps_normX": float(64 * n * 2.22e-16 * np.linalg.norm(xs)),
                                 "rows": mc}
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
        sweep = []
        for nn in (1, 2, 4, 8, 16, 32, 64):
            xs = ctx.fill_gaussian(m, nn, seed=1234)
            row = {"n": nn, "gib": 8.0 * m * nn / 2**30}
            for meth in ("tsqr", "cholqr2", "svqb2"):
                try:
                    ms, _ = timed(lambda: run_method(xs, meth), args.sweep_reps, 2)
                    gbs = 8.0 * m * nn / (ms * 1e-3) / 1e9
                    model_s = pmod.composite_time(hw, meth, m, nn)
                    row[meth] = {"ms": ms, "gbs": gbs, "frac_8TBs": gbs / NOMINAL_HBM_GBS, "frac_measured": gbs / peak,
                                 "model_time_s": model_s, "model_ratio": ms * 1e-3 / model_s}
                    if meth == "tsqr":
                        row[meth]["fp64_tflops_2mn2"] = 2.0 * m * nn * nn / (ms * 1e-3) / 1e12
                except sq.Error as exc:
                    row[meth] = {"error": type(exc).__name__}
            sweep.append(row)
            del xs
            torch.cuda.empty_cache()
        out["sweep"] = sweep

    if rank == 0:
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
