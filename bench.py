#!/usr/bin/env python
"""SymmSpMV benchmark (BASELINE.json metric: SymmSpMV GFLOP/s and % of HBM roofline).

One "step" = one SymmSpMV y := A x (the whole hot path) over
one synthetic matrix of a BASELINE.json config, inputs resident in HBM.
Default workload: configs[4], the 7-point 512^3 Laplacian (the largest
single-GPU configuration and BASELINE.md's primary one).  The same run also
times configs[1..3] and configs[0] and reports them under `per_config`, each
with its own roofline, cpu_baseline, e2e and sampled parity.  x and y rotate
through ring buffers whose total size exceeds twice the L2 (PAPER.md:2045
protocol), and the matrix stream itself exceeds L2 every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--variant V]
    python bench.py --impl reference ...     # the CPU oracle arm (rank 0 only)

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU).  Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SymmSpMV GFLOP/s and % of HBM roofline (1/2/4/8 B200) vs host-core oracle"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="lap3d_512")
    ap.add_argument("--no-per-config", action="store_true", help="time only --config (no per_config block)")
    ap.add_argument("--soak-ms", type=float, default=250.0,
                    help="untimed steps right before the timed region (clock sampler running) [ms]")
    ap.add_argument("--variant", default="auto", choices=["tiled", "tiled_atomic", "atomic", "colored", "colored_smem", "spmv", "tree", "tiled_colored", "auto"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweep", default=None, choices=["gs", "kacz"],
                    help="NEXT-4: time symmetric Gauss-Seidel / Kaczmarz sweeps instead of SymmSpMV (own JSON line)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--all-variants", action="store_true", help="also time the other variants (extra key)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--tile-nnz", type=int, default=0, help="race_config.max_tile_nnz override")
    ap.add_argument("--tile-window", type=int, default=0, help="race_config.max_tile_window override")
    ap.add_argument("--tile-work", type=int, default=0, help="race_config.tile_work override")
    ap.add_argument("--vec", type=int, default=0, help="lanes per row override")
    ap.add_argument("--sched", action="append", default=[], help="race_config override key=value (repeatable)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="multi-rank: receive the x halo before the whole run (no interior/boundary overlap)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-rank path (row blocks + halo) even with one rank (tests the glue)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, variant: str):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(f"{workload}:{variant}")
    return None if e is None else e.get("dram_bytes_per_launch")


class ClockSampler:
    """Samples SM clocks + throttle reasons with NVML during the timed region."""

    def __init__(self, dev=0, period=0.02):
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    _NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
              0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
              0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in self._NAMES.items():
                    if r & bit and nm != "gpu_idle":
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def mark(self):
        """Start of the timed region (samples before it were taken during the soak)."""
        self.mark_at = len(self.samples)

    def report(self):
        m = getattr(self, "mark_at", 0)
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        timed = self.samples[m:]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "samples_timed": len(timed), "sm_mhz_timed": statistics.median(timed) if timed else None,
                "window": "soak (untimed steps, same kernels) + timed region"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def spmv_min_bytes(n: int, nnz_full: int) -> int:
    """Eq. 2 at alpha = 1/NNZR: 12 B per full nonzero, row pointers, x once, y written."""
    return 12 * nnz_full + 4 * (n + 1) + 16 * n


def nnz_full_of(U):
    rows = np.repeat(np.arange(U.n, dtype=np.int64), np.diff(U.row_ptr))
    return 2 * int(U.nnz) - int(np.count_nonzero(U.col == rows))


def cpu_baseline(U, x, seconds: float, nnz_full: int, label: str):
    """The oracle as it stands (serial Alg. 2, 1 core) on repeated full multiplies."""
    import oracle

    t0 = time.perf_counter()
    reps = 0
    while True:
        y = oracle.symmspmv(U, x)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or (reps >= 1 and el * (reps + 1) / reps > 3 * seconds):
            break
    per = el / reps
    return {"value": 2.0 * nnz_full / per / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
            "sample": f"{reps} full serial oracle SymmSpMV multiplies of {label} ({el:.1f} s, 1 host core)",
            "seconds_per_step": per, "y": y}


def cpu_baseline_omp(U, x, seconds: float, nnz_full: int, label: str):
    """The OpenMP oracle (Alg. 2 with thread-private target arrays) on all host cores."""
    import oracle

    oracle.symmspmv_omp(U, x)  # first touch of the private arrays
    t0 = time.perf_counter()
    reps = 0
    while True:
        _, nt = oracle.symmspmv_omp(U, x)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    per = el / reps
    return {"value": 2.0 * nnz_full / per / 1e9, "unit": "GFLOP/s", "cores": nt, "kind": "oracle_openmp",
            "sample": f"{reps} full OpenMP oracle SymmSpMV multiplies of {label} ({el:.1f} s, {nt} threads)",
            "seconds_per_step": per}


def run_reference(a):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import gen

    U, x = gen.make_config(a.config)
    nf = nnz_full_of(U)
    import oracle

    # each step: one full serial oracle multiply (bounded sample of the workload)
    for _ in range(max(0, min(a.warmup, 1))):
        oracle.symmspmv(U, x)
    times = []
    steps = max(1, a.steps)
    budget = 120.0
    t_all = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.symmspmv(U, x)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget:
            break
    per = sum(times) / len(times)
    val = 2.0 * nf / per / 1e9
    line = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": ws, "steps": len(times), "warmup": a.warmup,
            "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": a.config, "n": U.n, "nnz_upper": int(U.nnz), "nnz_full": nf},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                             "sample": f"{len(times)} serial oracle multiplies of {a.config} (capped at {budget:.0f} s)",
                             "openmp": {k: v for k, v in cpu_baseline_omp(U, x, 5.0, nf, a.config).items()
                                        if k != "seconds_per_step"}},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_multi(a, U, x, s, perm, inv, nf, ws, rank, local, dist, t_gen, t_sched):
    """N ranks, one per GPU: contiguous row blocks + halo (strong scaling)."""
    import torch

    import paper_1907_06487_b200 as P
    from paper_1907_06487_b200.dist import DistSymmSpMV

    t0 = time.perf_counter()
    D = DistSymmSpMV(s, U, overlap=not a.no_overlap)
    t_plan = time.perf_counter() - t0
    parts = D.parts()
    r0, r1 = D.row_begin, D.own_end
    xp = x[inv]
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    R = max(2, min(64, int(np.ceil(2 * l2 / (16.0 * max(D.n_local, 1))))))
    xs = []
    for _ in range(R):
        xl = D.empty_local()
        xl[:D.n_own].copy_(torch.from_numpy(xp[r0:r1].copy()))
        xs.append(xl)
    ys = [D.empty_local() for _ in range(R)]
    stream = torch.cuda.current_stream()
    for i in range(max(3, a.warmup)):
        D.run(xs[i % R], ys[i % R])
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, period=0.005) as clk:
        t_s = time.perf_counter()
        i = 0
        while (time.perf_counter() - t_s) * 1e3 < a.soak_ms:
            D.run(xs[i % R], ys[i % R])
            i += 1
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        ev0.record(stream)
        for i in range(a.steps):
            D.run(xs[i % R], ys[i % R])
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / a.steps
    # correctness of the timed configuration: gather own rows to rank 0, compare there
    y_own = ys[(a.steps - 1) % R][:D.n_own].contiguous()
    sizes = torch.tensor([D.n_own], device="cuda")
    all_sizes = [torch.zeros_like(sizes) for _ in range(ws)]
    dist.all_gather(all_sizes, sizes)
    mx = int(max(v.item() for v in all_sizes))
    pad = torch.zeros(mx, dtype=torch.float64, device="cuda")
    pad[:D.n_own] = y_own
    gathered = [torch.zeros_like(pad) for _ in range(ws)]
    dist.all_gather(gathered, pad)
    hb = torch.tensor([D.hx.halo_bytes()], device="cuda")
    dist.all_reduce(hb, op=dist.ReduceOp.MAX)
    bfrac = torch.tensor([parts["boundary_nnz"] / max(1, parts["boundary_nnz"] + parts["interior_nnz"])],
                         device="cuda", dtype=torch.float64)
    dist.all_reduce(bfrac, op=dist.ReduceOp.MAX)
    # e2e: every step copies this rank's x slice in from pinned host memory and
    # its y rows back out (device-timed, max over ranks)
    xh = torch.from_numpy(xp[r0:r1].copy()).pin_memory()
    yh = torch.empty(D.n_own, dtype=torch.float64).pin_memory()
    xe, ye = D.empty_local(), D.empty_local()
    e2e_steps = max(5, min(50, a.steps // 20))
    dist.barrier()
    torch.cuda.synchronize()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2.record(stream)
    for _ in range(e2e_steps):
        xe[:D.n_own].copy_(xh, non_blocking=True)
        D.run(xe, ye)
        yh.copy_(ye[:D.n_own], non_blocking=True)
    ev3.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([ev2.elapsed_time(ev3) / e2e_steps], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    if rank == 0:
        yperm = np.concatenate([gathered[r][:int(all_sizes[r].item())].cpu().numpy() for r in range(ws)])
        y = yperm[perm]
        n = U.n
        # parity of the timed multi-rank configuration against the full oracle,
        # and the host-core baseline (rank 0)
        cpu = None
        if not a.no_cpu_baseline:
            cb = cpu_baseline(U, x, min(3.0, a.cpu_seconds), nf, a.config)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["cpu_model"] = cpu_model()
            y_ref = cb["y"]
        else:
            import oracle

            y_ref = oracle.symmspmv(U, x)
        relerr = float(np.max(np.abs(y - y_ref)) / np.max(np.abs(y_ref)))
        bytes_min = P.min_bytes(n, int(U.nnz))
        peak, peak_src = peaks()
        achieved = bytes_min / (ms_step / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": 2.0 * nf / (ms_step / 1e3) / 1e9, "unit": "GFLOP/s", "n_gpus": ws,
            "steps": a.steps, "warmup": max(3, a.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "ours",
            "variant": "tiled_atomic+halo" + ("+overlap" if not a.no_overlap else ""),
            "gpu_launches": a.steps * (3 if not a.no_overlap else 2) * ws,
            "config": {"workload": a.config, "n": n, "nnz_upper": int(U.nnz), "nnz_full": nf,
                       "parallelism": f"rowblock{ws}", "max_halo_bytes_per_rank": int(hb.item()),
                       "max_boundary_nnz_frac": float(bfrac.item()),
                       "l2_policy": "inputs larger than L2 (matrix streamed once per step)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ws, "unit": "GB/s",
                         "frac": achieved / (peak * ws), "traffic": None, "bytes_per_launch": bytes_min,
                         "peak_source": peak_src + f" x {ws} GPUs"},
            "cpu_baseline": cpu,
            "parity_relinf": relerr,
            "e2e": {"value": 2.0 * nf / (float(te.item()) / 1e3) / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n, "ms_per_step": float(te.item())},
            "clocks": clk.report(),
            "schedule": {"build_s": t_sched, "plan_s": t_plan, "gen_s": t_gen},
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def run_sweep(a, U, x, s, nf, t_sched):
    """NEXT-4: symmetric GS / Kaczmarz sweeps (forward + backward), phase by
    phase on the schedule's level groups; device-timed; one JSON line."""
    import torch

    import oracle  # parity of the timed configuration on a sample is the oracle's job (tests); here: one check
    import paper_1907_06487_b200 as P

    n = U.n
    perm, inv = s.permutation()
    t0 = time.perf_counter()
    sw = P.Sweep(s, a.sweep)
    t_plan = time.perf_counter() - t0
    rows, ptr = sw.order()
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, n)
    bd = torch.from_numpy(b[inv].copy()).cuda()
    x0 = torch.from_numpy(x[inv].copy()).cuda()
    xd = x0.clone()
    for _ in range(max(3, a.warmup)):
        sw.run(xd, bd, symmetric=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xd.copy_(x0)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        sw.run(xd, bd, symmetric=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    # one symmetric sweep from x0 against the serial oracle in the plan's order
    xd.copy_(x0)
    sw.run(xd, bd, symmetric=True)
    torch.cuda.synchronize()
    x_ref = oracle.sweep(a.sweep, U, b, x, inv[rows].astype(np.int32), symmetric=True)
    err = float(np.max(np.abs(xd.cpu().numpy()[perm] - x_ref)) / max(np.max(np.abs(x_ref)), 1e-300))
    # algorithmic bytes of a symmetric sweep: 2 x (full matrix 12 B/nnz + row
    # order / pointers 8 B/row + b 8 B/row + x read + write 16 B/row)
    byts = 2 * (12 * nf + 32 * n)
    peak, peak_src = peaks()
    achieved = byts / (ms * 1e-3) / 1e9
    line = {"metric": f"symmetric {a.sweep.upper()} sweep (NEXT-4)", "value": 1e3 / ms, "unit": "sweeps/s",
            "ms_per_step": ms, "steps": a.steps, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": a.config, "n": n, "nnz_full": nf, "phases_per_sweep": int(len(ptr) - 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_launch": byts, "peak_source": peak_src,
                         "bytes_model": "2 x (12 nnz_full + 32 n): matrix, pointers + order, b, x read + write"},
            "parity_relinf_vs_serial_oracle": err, "gpu_launches": 2 * int(len(ptr) - 1) * a.steps,
            "schedule": {"build_s": t_sched, "plan_s": t_plan}}
    print(json.dumps(line), flush=True)
    return 0


PER_CONFIG = ("st27_128", "fem_knn_4M", "spin_22", "lap2d_64")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def probes(local):
    """K5 (symm_bw_probe): load-only and copy bandwidth measured in this run."""
    import paper_1907_06487_b200 as P

    out = {}
    for mode in ("load", "copy"):
        try:
            out[mode] = P.bw_probe(mode, 4 << 30, 5, device=local)
        except Exception as e:  # noqa: BLE001
            out[mode + "_error"] = str(e)
    return out


def denominators(achieved, peak, bw):
    """Fractions of the three roofline denominators."""
    d = {"copy_measured_peaks_json": {"gbs": peak, "frac": achieved / peak},
         "nominal_8TBs": {"gbs": 8000.0, "frac": achieved / 8000.0}}
    if "load" in bw:
        d["load_only_measured_here"] = {"gbs": bw["load"], "frac": achieved / bw["load"]}
    if "copy" in bw:
        d["copy_measured_here"] = {"gbs": bw["copy"], "frac": achieved / bw["copy"]}
    return d


def bench_single(a, name, local, bw, headline, cpu_seconds):
    """Gen + schedule + plan + timed steps of one config on this GPU; returns
    the JSON fields of that config (the headline line or a per_config entry)."""
    import torch

    import gen
    import paper_1907_06487_b200 as P

    t0 = time.perf_counter()
    U, x = gen.make_config(name)
    t_gen = time.perf_counter() - t0
    nf = nnz_full_of(U)
    sched_kw = {}
    if headline:
        if a.tile_nnz:
            sched_kw["max_tile_nnz"] = a.tile_nnz
        if a.tile_window:
            sched_kw["max_tile_window"] = a.tile_window
            sched_kw["max_tile_rows"] = a.tile_window
        if a.tile_work:
            sched_kw["tile_work"] = a.tile_work
        for kv in a.sched:
            k_, v_ = kv.split("=")
            sched_kw[k_] = int(v_)
    t0 = time.perf_counter()
    s = P.build_schedule(U, **sched_kw)
    t_sched = time.perf_counter() - t0
    st = s.stats
    perm, inv = s.permutation()
    all_v = headline and a.all_variants
    t0 = time.perf_counter()
    plan = P.Plan(s, U, variant=a.variant if not all_v else "auto", build_all=all_v, vec_width=a.vec if headline else 0)
    t_plan = time.perf_counter() - t0
    dev_bytes, bytes_min = plan.bytes()
    n = U.n
    # ring buffers: x, y rings larger than 2x L2 in total
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    R = max(2, int(np.ceil(2 * l2 / (16.0 * max(n, 1)))))
    R = min(R, 64)
    xp = torch.from_numpy(x[inv].copy()).cuda()
    xs = [xp.clone() for _ in range(R)]
    ys = [torch.empty_like(xp) for _ in range(R)]
    stream = torch.cuda.current_stream()

    def step(i, variant):
        plan.run(xs[i % R], ys[i % R], stream=stream, variant=variant)
        return plan.last_launches

    def timed(variant, steps, warmup, soak_ms):
        for i in range(warmup):
            step(i, variant)
        torch.cuda.synchronize()
        launches = 0
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local, period=0.005) as clk:
            # soak: untimed steps so the clock record covers a loaded GPU
            t_s = time.perf_counter()
            i = 0
            while soak_ms > 0 and (time.perf_counter() - t_s) * 1e3 < soak_ms:
                for _ in range(8):
                    step(i, variant)
                    i += 1
                torch.cuda.synchronize()
            torch.cuda.synchronize()
            clk.mark()
            ev0.record(stream)
            for i in range(steps):
                launches += step(i, variant)
            ev1.record(stream)
            torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / steps, launches, clk.report()

    variant = a.variant if a.variant != "auto" else "tiled_atomic"  # what AUTO runs (symmspmv.h)
    ms_step, launches, clocks = timed(variant, a.steps, max(3, a.warmup), a.soak_ms)

    # per-step distribution (mean, median, min/max spread, flag > 5%),
    # from a separate pass with one event per step (not the timed number)
    nst = max(10, min(a.steps, 200))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)]
    evs[0].record(stream)
    for i in range(nst):
        step(i, variant)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    per = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(nst)])
    med = float(np.median(per))
    step_stats = {"steps": nst, "mean_ms": float(per.mean()), "median_ms": med, "min_ms": float(per.min()),
                  "max_ms": float(per.max()), "spread": float((per.max() - per.min()) / med),
                  "spread_over_5pct": bool((per.max() - per.min()) / med > 0.05)}
    t_s = ms_step / 1e3
    peak, peak_src = peaks()
    if variant == "spmv":  # the yardstick streams the full matrix (Eq. 2)
        bytes_min = spmv_min_bytes(n, nf)
    achieved = bytes_min / t_s / 1e9
    y_timed = ys[(a.steps - 1) % R].cpu().numpy()[perm]

    extra = {}
    if all_v:
        for v in ("atomic", "colored", "tiled", "tiled_atomic", "colored_smem", "spmv", "tiled_colored"):
            try:
                m, l, _ = timed(v, max(50, a.steps // 4), 5, 0)
                extra[v] = {"ms_per_step": m, "gflops": 2.0 * nf / (m / 1e3) / 1e9,
                            "hbm_frac": bytes_min / (m / 1e3) / 1e9 / peak, "launches_per_step": l / max(50, a.steps // 4)}
                if v == "spmv":  # the yardstick against its own Eq. 2 bytes (alpha = 1/NNZR)
                    sb = spmv_min_bytes(n, nf)
                    extra[v].update({"spmv_bytes_min": sb, "hbm_frac_spmv_model": sb / (m / 1e3) / 1e9 / peak,
                                     "symmspmv_speedup": m / ms_step})
            except Exception as e:  # noqa: BLE001
                extra[v] = {"error": str(e)}

    # e2e: host buffers through the C ABI (H2D x, permute, run, unpermute, D2H y)
    xh = torch.from_numpy(x.copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    e2e_steps = max(5, min(50, a.steps // 4))
    for _ in range(2):
        plan.run_host(xh.numpy(), yh.numpy(), stream=stream)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.run_host(xh.numpy(), yh.numpy(), stream=stream)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": 2.0 * nf / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n, "ms_per_step": e2e_s * 1e3,
           "path": "symmspmv_run_host: pinned host x -> H2D, permute, run, unpermute, D2H y (wall clock)"}
    del plan, xs, ys

    cpu, err = None, None
    if cpu_seconds > 0:
        # cpu_baseline leg: the oracle timed on the host, and its result compared
        # with the last timed GPU output on sampled rows
        cb = cpu_baseline(U, x, cpu_seconds, nf, name)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu["cpu_model"] = cpu_model()
        cpu["openmp"] = {k: v for k, v in cpu_baseline_omp(U, x, max(1.0, cpu_seconds / 2), nf, name).items()
                         if k != "seconds_per_step"}
        cpu["openmp"]["cpu_model"] = cpu["cpu_model"]
        y_ref = cb["y"]
        sample = np.random.default_rng(0).choice(n, size=min(n, 4096), replace=False)
        err = float(np.max(np.abs(y_timed[sample] - y_ref[sample])) / np.max(np.abs(y_ref)))

    l2_resident = 24 * n + 12 * int(U.nnz) < l2 // 2
    out = {
        "value": 2.0 * nf / t_s / 1e9, "ms_per_step": ms_step, "variant": variant, "gpu_launches": launches,
        "step_stats": step_stats,
        "config": {"workload": name, "n": n, "nnz_upper": int(U.nnz), "nnz_full": nf,
                   "l2_policy": f"inputs larger than L2: matrix {dev_bytes / 1e6:.0f} MB streamed per step; "
                                f"x/y ring of {R} vectors each ({2 * R * 8 * n / 1e6:.0f} MB)"
                   if not l2_resident else "L2-resident working set (latency-bound config; no HBM fraction claimed)"},
        "roofline": {"bound": "hbm" if not l2_resident else "latency (L2-resident)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(name, variant), "bytes_per_launch": bytes_min, "peak_source": peak_src,
                     "bytes_model": "12 nnz_u + 4 (n+1) + 24 n (Eq. 3 at alpha = 1/SymmNNZR)",
                     "denominators": denominators(achieved, peak, bw)},
        "frac_of_nominal_8TBs": achieved / 8000.0,
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "parity_sampled_relinf": err,
        "schedule": {"build_s": t_sched, "plan_s": t_plan, "gen_s": t_gen, "tiles": st["n_tiles"],
                     "phases": st["n_phases"], "levels": st["total_levels"], "eta": st["eta"],
                     "max_subcolors": st["max_subcolors"], "mean_subcolors": st["mean_subcolors"],
                     "bw_before": st["bandwidth_before"], "bw_after": st["bandwidth_after"],
                     "spill_entries": st["spill_entries"], "device_bytes": dev_bytes},
    }
    if extra:
        out["variants"] = extra
    del U, x, s
    torch.cuda.empty_cache()
    return out


def relaunch_under_torchrun(a):
    """--gpus N > 1 without a torchrun environment: re-run this command as N
    ranks (one per GPU) under torch.distributed.run."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < a.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus} but only {have} CUDA devices"}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    a = parse()
    ws, rank, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(a)
    if ws > 1 and a.gpus not in (1, ws):
        print(json.dumps({"metric": METRIC, "error": f"--gpus {a.gpus} but WORLD_SIZE={ws}"}), flush=True)
        return 2
    if a.impl == "reference":
        return run_reference(a)
    import torch

    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}), flush=True)
        return 1
    torch.cuda.set_device(local)
    if ws > 1 or a.force_dist:
        import torch.distributed as dist

        if a.force_dist and "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29531", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        import gen
        import paper_1907_06487_b200 as P

        t0 = time.perf_counter()
        U, x = gen.make_config(a.config)
        t_gen = time.perf_counter() - t0
        nf = nnz_full_of(U)
        t0 = time.perf_counter()
        s = P.build_schedule(U)
        t_sched = time.perf_counter() - t0
        perm, inv = s.permutation()
        return run_multi(a, U, x, s, perm, inv, nf, ws, rank, local, dist, t_gen, t_sched)
    if a.sweep:
        import gen
        import paper_1907_06487_b200 as P

        U, x = gen.make_config(a.config)
        nf = nnz_full_of(U)
        t0 = time.perf_counter()
        s = P.build_schedule(U)
        return run_sweep(a, U, x, s, nf, time.perf_counter() - t0)

    bw = probes(local)
    head = bench_single(a, a.config, local, bw, True, 0.0 if a.no_cpu_baseline else a.cpu_seconds)
    peak, peak_src = peaks()
    line = {"metric": METRIC, "value": head.pop("value"), "unit": "GFLOP/s", "n_gpus": 1, "steps": a.steps,
            "warmup": max(3, a.warmup), "ms_per_step": head.pop("ms_per_step"), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "ours"}
    line.update(head)
    line["config"]["parallelism"] = "single"
    line["bw_probe_gbs"] = bw
    if not a.no_per_config and a.variant in ("auto", "tiled_atomic") and not a.all_variants:
        pc = {}
        for name in PER_CONFIG:
            if name == a.config:
                continue
            try:
                pc[name] = bench_single(a, name, local, bw, False,
                                        0.0 if a.no_cpu_baseline else min(3.0, a.cpu_seconds))
            except Exception as e:  # noqa: BLE001
                pc[name] = {"error": str(e)}
        line["per_config"] = pc
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
