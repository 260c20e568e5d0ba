#!/usr/bin/env python
"""Benchmark of the spectral point-mass filter hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl cuda|reference]

A STEP is one filter epoch over the whole batch, i.e. every row of SURVEY
§8(a): (re-centre grid + multilinear resample, R12) -> forward DFT per axis
-> s*Psi over l Euler substeps -> inverse DFT -> normalise (Alg. 1-6) ->
likelihood, normaliser and moments (eq:filt).

Default workload C4 (BASELINE configs[3]): one 4-D CV filter on 96^4 (85 M
points, fp64, l = 10) -- the largest single-GPU configuration (the tier rule's
N = 1 headline). Under torchrun (N > 1) its grid is slab-sharded over the ranks
(strong scaling, two all-to-all per predict). --workload C5 runs BASELINE
configs[4]: 4096 independent 2-D filters on 128^2, sharded by filter index,
4096/N per rank (strong scaling, no data-path collective).

Metric (BASELINE.json): grid-point FPE updates/sec = filters * points / t_step.
Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize, CUDA events on the library's stream (one per step: median and
p10/p90 reported), max over ranks. Workloads whose weights exceed the 126 MB L2
(C4, C5) need no flush; the L2-resident ones (C1-C3, C6) are timed with an L2
flush before every step (and without, reported beside).

Roofline: achieved = the method's algorithmic bytes
(read + write every weight once: 16 B per grid point in fp64, 8 B in fp32) /
the whole epoch (or predict) time, against MEASURED_PEAKS.json's copy bandwidth;
per-kernel figures (live CUDA-event time of the dominant kernel, ncu shares,
DRAM bytes) go to roofline.kernels. ALU fractions use the FP64/FP32 peaks
measured on this pool's B200 (profiles/r2/fp64_peaks.json).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import make_config, simulate  # noqa: E402

WORKLOADS = {
    "C4": dict(cid="C4", over={}),
    "C5": dict(cid="C5", over={}),
    "C5f32": dict(cid="C5", over={"dtype": "f32"}),
    "C3": dict(cid="C3", over={}),
    "C2": dict(cid="C2", over={}),
    "C1": dict(cid="C1", over={}),
    "C5l1": dict(cid="C5", over={"l": 1}),      # report l = 1 next to l = 10
    # NEXT-1: the paper's FDM baseline (eq:FST) on the C5 batch, DST-I on FP64 tensor cores
    "C5fdm": dict(cid="C5", over={}, diff_mode=2),
    # NEXT-4: Crank-Nicolson substeps (R27) and eigenvector-aligned grids (R28) on the C5 batch
    "C5cn": dict(cid="C5", over={}, step=1),
    "C5eig": dict(cid="C5", over={}, grid=1),
    # NEXT-3: the paper's §VI scenario (coordinated turn, terrain altitude + GM noise, N_pa = 34)
    "C6": dict(cid="C6", over={}),
}
L2_BYTES = 126e6


def peaks():
    """(HBM GB/s, source, max SM MHz) from MEASURED_PEAKS.json (driver-written)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)", d.get("sm_max_mhz", 1965.0)
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", 1965.0


def alu_peaks():
    """Measured FP64 / FP32 FMA and FP64 DMMA peaks of this pool's B200 (tools/micro/peaks_fp64.cu):
    TFLOP/s, an FMA counting 2. Issue slots per second = TFLOP/s / 2."""
    p = os.path.join(ROOT, "profiles", "r2", "fp64_peaks.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    g = lambda k, v: d.get(k, {}).get("tflops", v)  # noqa: E731
    return {"fp64": g("fp64_fma", 36.6), "fp32": g("fp32_fma", 71.9), "dmma": g("fp64_dmma", 37.1),
            "source": "profiles/r2/fp64_peaks.json (measured)" if d else "nominal"}


class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region (the
    B200_PROFILING.md clocks line), via NVML from a background thread every 2 ms."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        import threading
        self.samples, self.reasons, self.power = [], 0, []
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _run(self):
        nv, h = self.nv, self.h
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(h))
                self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
            except Exception:
                pass
            self.stop_ev.wait(0.002)

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_ev.set()
        self.th.join()
        rs = sorted(name for bit, name in self.REASONS.items() if self.reasons & bit)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": rs, "samples": len(self.samples),
                "power_w_max": max(self.power) if self.power else None, "source": "nvml, 2 ms"}


def dist_env():
    from paper_2412_07240_b200.dist import env
    return env()


def kernel_metrics(kernel: str):
    """ncu numbers for `kernel` committed under profiles/ (dram traffic per launch,
    FP64-pipe utilisation), written by tools/ncu_to_json.py from a --set full capture."""
    p = os.path.join(ROOT, "profiles", "kernel_metrics.json")
    if not os.path.exists(p):
        return {}
    return json.load(open(p)).get(kernel, {})


def launch_shares(workload: str):
    """Per-kernel ncu launch list of one epoch of `workload` (cold-cache, serialised: the
    SHARES are comparable with the live step, not the absolute times); tools/ncu_epoch_json.py."""
    p = os.path.join(ROOT, "profiles", "r2", "launch_shares.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(workload)


def cpu_info():
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        nproc = len(os.sched_getaffinity(0))
    except AttributeError:
        nproc = os.cpu_count() or 1
    return nproc, model


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count() or 1


def oracle_sample_cfg(cfg):
    """The bounded oracle sample of a workload: batched workloads run their first filters;
    a single grid above 4 M points (C4's 96^4) runs the same model on a 32^4 sub-grid --
    the oracle's dense O(N^2) DFT costs N MACs per point per axis and direction, so its
    per-point rate at 96^4 is about a third of the sub-grid's (stated with the number)."""
    if cfg.batch == 1 and cfg.points > 4_000_000:
        sub = cfg.replace(n=(32,) * cfg.nx)
        return sub, f"{{nf}} successive epochs of the {cfg.name} model on a 32^{cfg.nx} sub-grid (at 96^{cfg.nx} the oracle needs " \
                    f"{cfg.points / 32 ** cfg.nx:.0f}x the points at ~3x the per-point work: minutes per epoch)"
    return cfg, None


def oracle_sample(cfg, zs, budget_s: float, max_filters: int, threads=None):
    """Time the CPU oracle (as it stands) on a bounded sample: one epoch (predict + update +
    moments + regrid) per filter, filters 0.. until the budget is used. Returns
    (points_per_s, filter_epochs, seconds)."""
    from threadpoolctl import threadpool_limits
    from oracle import pmf_oracle as O
    n = tuple(cfg.n)
    done, t_tot = 0, 0.0
    nb = min(cfg.batch, max_filters)
    with threadpool_limits(threads):
        # batched: filters 0, 1, .. one epoch each; one filter (batch 1): its successive
        # epochs, until the budget is used
        b, w = 0, None
        while True:
            if w is None or nb > 1:
                w, c, B = O.initial_density(cfg.prior_mean[b], cfg.prior_cov, n, cfg.k_sigma)
            t0 = time.perf_counter()
            w, c, B = O.predict(w, c, B, cfg.A, cfg.Q, cfg.tau, cfg.l)
            w, _ = O.update(w, c, B, O.make_likelihood(cfg, O.grid_points(c, B, n), zs[1, b]))
            mean, cov = O.moments(w, c, B)
            c2, B2 = O.regrid_target(mean, cov, n, cfg.k_sigma)
            w = O.regrid(w, c, B, c2, B2)
            c, B = c2, B2
            t_tot += time.perf_counter() - t0
            done += 1
            if t_tot >= budget_s or (nb > 1 and done >= nb):
                break
            b = (b + 1) % nb
    return done * cfg.points / t_tot, done, t_tot


def cpu_baseline(cfg, budget_s: float):
    """The oracle on the host cores at all threads (the reported value) and at 1 thread."""
    scfg, note = oracle_sample_cfg(cfg)
    zs = simulate(scfg.replace(batch=min(scfg.batch, 256)), T=1)["z"]
    scfg = scfg.replace(batch=min(scfg.batch, 256))
    nproc, model = cpu_info()
    v, nf, ts = oracle_sample(scfg, zs, budget_s=0.5 * budget_s, max_filters=scfg.batch)
    v1, nf1, ts1 = oracle_sample(scfg, zs, budget_s=0.5 * budget_s, max_filters=scfg.batch, threads=1)
    what = note or f"{{nf}} of {cfg.batch} filters x 1 epoch"
    return {"value": v, "unit": "grid-point updates/s", "cores": threads_used(), "kind": "oracle",
            "sample": what.format(nf=nf) + f" ({ts:.1f} s of CPU time)", "nproc": nproc, "cpu_model": model,
            "single_thread": {"value": v1, "sample": what.format(nf=nf1) + f" ({ts1:.1f} s)", "cores": 1}}


def step_stats(ms):
    q = np.percentile(np.asarray(ms), [10, 50, 90])
    return {"reps": len(ms), "median_ms": float(q[1]), "p10_ms": float(q[0]), "p90_ms": float(q[2])}


def workload_name(workload, cfg, world=1, strong_batch=None):
    """config.workload, identical on both arms."""
    b = cfg.batch if strong_batch is None else strong_batch
    return (f"{workload}: {b} x {'x'.join(map(str, cfg.n))} {cfg.nx}-D filters, "
            f"l={cfg.l}, tau={cfg.tau}, k_sigma={cfg.k_sigma}")


def metric_name(dtype):
    return "grid-point FPE updates/sec (fp64)" if dtype == "f64" else "grid-point FPE updates/sec (fp32)"


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, timed as the reference arm (rank 0 only);
    each step is a bounded sample of the workload; ms_per_step is the measured time of the
    sampled work of one step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    cfg = make_config(wl["cid"], **wl["over"])
    scfg, note = oracle_sample_cfg(cfg)
    scfg = scfg.replace(batch=min(scfg.batch, 64))
    zs = simulate(scfg, T=1)["z"]
    per_step = []
    for _ in range(args.warmup + args.steps):
        v, nf, t = oracle_sample(scfg, zs, budget_s=args.ref_budget, max_filters=64)
        per_step.append((v, nf, t))
    timed = per_step[args.warmup:]
    val = statistics.median(v for v, _, _ in timed)
    nf = timed[0][1]
    sample = (note.format(nf=nf) if note else f"{nf} of {cfg.batch} filters x 1 epoch") + \
        " per step (the oracle is an O(N^2) naive DFT)"
    nproc, model = cpu_info()
    line = {"impl": "reference", "metric": metric_name(cfg.dtype), "value": val,
            "unit": "grid-point updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(t for _, _, t in timed), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.workload, cfg), "sample": sample},
            "cpu_baseline": {"value": val, "unit": "grid-point updates/s", "cores": threads_used(), "kind": "oracle",
                             "sample": sample, "nproc": nproc, "cpu_model": model},
            "e2e": {"value": val, "unit": "grid-point updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def make_filter(pmf, cfg, wl, args, local, stream, fkw):
    f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, dtype=cfg.dtype, path=args.path,
                   device=local, stream=stream.cuda_stream, diff_mode=wl.get("diff_mode", 0),
                   step=wl.get("step", 0), grid=wl.get("grid", 0), **fkw)
    if cfg.lik_kind == 2:
        from workloads import terrain_table
        lik = pmf.make_likelihood(pmf.LIK_TERRAIN_GM, cfg.nx, gm=cfg.extra["gm"])
        f.set_terrain(*terrain_table(cfg))
    else:
        lik = (pmf.make_likelihood(pmf.LIK_RANGE_GAUSS, cfg.nx, sigma=cfg.sigma) if cfg.lik_kind == 1
               else pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, cfg.nx, H=cfg.H, R=cfg.R))
    f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
    return f, lik


def run_workload(args, workload, rank, world, local, secondary=False):
    """One bench measurement of `workload`; returns the JSON-line dict (rank 0 prints it)."""
    import torch
    import torch.distributed as dist
    from paper_2412_07240_b200 import pmf
    from paper_2412_07240_b200.dist import max_over_ranks, shard
    wl = WORKLOADS[workload]
    cfg = make_config(wl["cid"], **wl["over"])
    if args.l:
        cfg = cfg.replace(l=args.l)
    # One large filter (batch 1) with N > 1 GPUs (or --virtual-ranks): its grid is split into
    # slabs along the last axis (strong scaling, all-to-all transposes). Batched filters (C5):
    # filter index sharded, 4096/N per rank (strong scaling, no data-path collective).
    real_nccl = world > 1 or args.nccl_self          # --nccl-self: a 1-rank NCCL communicator at N = 1
    sharded = cfg.batch == 1 and cfg.nx >= 2 and (real_nccl or args.virtual_ranks > 1)

    def nccl_kw():
        obj = [pmf.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return dict(world=world, rank=rank, unique_id=obj[0], sharded=True)
    T = args.warmup + 2 * args.steps + 3
    glob_batch = cfg.batch
    zs = simulate(cfg, T=T)["z"]                        # (T+1, batch, nz)
    if cfg.batch > 1 and world > 1:
        lo, hi = shard(cfg.batch, rank, world)
        cfg = cfg.replace(batch=hi - lo, prior_mean=cfg.prior_mean[lo:hi])
        zs = np.ascontiguousarray(zs[:, lo:hi])
    stream = torch.cuda.Stream()
    fkw = {}
    if sharded and real_nccl:
        fkw = nccl_kw()
    elif sharded:
        fkw = dict(world=args.virtual_ranks, sharded=True)
    f, lik = make_filter(pmf, cfg, wl, args, local, stream, fkw)
    dtype = cfg.dtype
    esize = 8 if dtype == "f64" else 4
    z_dev = torch.tensor(zs, dtype=torch.float64, device=f"cuda:{local}")   # inputs resident in HBM
    dt = cfg.tau / cfg.l
    f.update(z_dev[0], lik)
    f.regrid(cfg.k_sigma)
    k = 1
    for _ in range(args.warmup):
        f.step(dt, cfg.l, z_dev[k], lik, cfg.k_sigma)
        k += 1
    torch.cuda.synchronize()      # (not f.sync(): that would flush the pending regrid outside the timed region)
    points_step = cfg.batch * cfg.points                # this rank's grid points per step
    l2_resident = esize * points_step <= L2_BYTES
    flush_buf = torch.empty(int(2 * L2_BYTES) // 4, dtype=torch.float32, device=f"cuda:{local}") \
        if l2_resident else None

    def timed_steps(kk, flush):
        """K steps, one CUDA-event pair per step on the library's stream; returns per-step ms."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                if flush:
                    flush_buf.fill_(float(i))               # > L2: evicts the grid (outside the event pair)
                evs[i][0].record(stream)
                f.step(dt, cfg.l, z_dev[kk + i], lik, cfg.k_sigma)
                evs[i][1].record(stream)
        evs[-1][1].synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    launches0 = f.launches
    f.profile(True)
    torch.cuda.synchronize()
    ms_steps = timed_steps(k, flush=l2_resident)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = f.launches - launches0
    k += args.steps
    epoch_kernel = f.epoch_kernel                    # kernel family of the timed epochs
    kern_total_ms, kern_n = f.profile_read()
    f.profile(False)
    t_ms = sum(ms_steps)
    t_max = max_over_ranks(t_ms, device=f"cuda:{local}")
    ranks_work = 1 if sharded else world             # all ranks' points (filter-sharded) vs one grid
    value = ranks_work * points_step * args.steps / (t_max * 1e-3)
    ms_step = t_max / args.steps
    stats = step_stats(ms_steps)
    unflushed = None
    if l2_resident:
        ms_nf = timed_steps(k, flush=False)
        k += args.steps
        unflushed = {"value": ranks_work * points_step * len(ms_nf) / (sum(ms_nf) * 1e-3), **step_stats(ms_nf),
                     "what": "same steps without the L2 flush (the grid stays L2-resident between epochs)"}

    # ---------------------------------------------------------------- FPE time update alone (Alg. 1-6)
    # north_star's "FPE time update at >= 60% of the HBM roofline": predict-only steps
    # (no likelihood, no regrid) on the same resident state; 16 B/point algorithmic, over the
    # WHOLE predict (every kernel of it), event-timed per step.
    hbm_gbs, hbm_src, sm_max = peaks()
    ap = alu_peaks()
    tu = None
    if not args.no_time_update:
        for _ in range(2):
            f.predict(dt, cfg.l)
            f.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f.profile(True)
        tms = []
        for _ in range(args.steps):
            if l2_resident:
                with torch.cuda.stream(stream):
                    flush_buf.fill_(0.5)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            f.predict(dt, cfg.l)
            f.sync()
            t1.record(stream)
            t1.synchronize()
            tms.append(t0.elapsed_time(t1))
        km_ms, km_n = f.profile_read()
        f.profile(False)
        tt = max_over_ranks(statistics.median(tms), device=f"cuda:{local}")
        pts = ranks_work * points_step
        tu = {"ms_per_step": tt, "value": pts / (tt * 1e-3), "unit": "grid-point updates/s", **step_stats(tms),
              "hbm_frac": 2 * esize * points_step / (tt * 1e-3) / 1e9 / hbm_gbs,
              "hbm_frac_what": f"{2 * esize} B per grid point / the whole predict (event-timed) / {hbm_gbs} GB/s",
              "dominant_kernel_ms": km_ms / max(km_n, 1),
              "what": "predict only (prep + every transform/Psi kernel + closed-form normalisation)"}
        if f.path == pmf.PATH_RESIDENT:
            # the predict's algorithmic issue slots against the measured FP64 (FP32) peak
            spp = 0.5 * 4 * 3.5 * math.log2(cfg.n[0]) + psi_slots(cfg, wl) * (cfg.n[1] // 2 + 1) / cfg.n[1]
            peak_slots = (ap["fp64"] if dtype == "f64" else ap["fp32"]) / 2 * 1e12
            tu["alu_frac"] = spp * points_step / (tt * 1e-3) / peak_slots

    # ---------------------------------------------------------------- e2e: host buffers through the C ABI
    e2e = None
    if not args.no_e2e:
        Te = min(args.steps, 10)
        zs_e = zs[:Te + 3]
        z_pin = torch.tensor(zs_e, dtype=torch.float64).pin_memory()
        if sharded and real_nccl:
            fkw = nccl_kw()
        fe, _ = make_filter(pmf, cfg, wl, args, local, stream, fkw)
        mean = np.empty((cfg.batch, cfg.nx))
        cov = np.empty((cfg.batch, cfg.nx, cfg.nx))
        logc = np.empty(cfg.batch)
        zp = z_pin.data_ptr()
        zstride = cfg.batch * cfg.nz * 8
        import ctypes as C
        fe._check(fe.lib.pmf_update(fe.h, C.c_void_p(zp), 0, C.byref(lik)))
        fe.regrid(cfg.k_sigma)
        fe.moments_into(mean, cov, logc)
        for i in range(2):                                    # warm-up (graph capture happens here)
            fe._check(fe.lib.pmf_step(fe.h, dt, cfg.l, C.c_void_p(zp + (i + 1) * zstride), 0, C.byref(lik),
                                      cfg.k_sigma))
            fe.moments_into(mean, cov, logc)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # every step: H2D of the step's measurements from pinned host memory (the library stages
        # them), and the step's result (moments of every filter) read back into pinned host memory
        # asynchronously on the library's stream (pmf_moments_async): no host stall between steps;
        # all reads complete inside the timed region (e1 follows them)
        async_ok = not (sharded and real_nccl) and args.virtual_ranks == 1
        mom_pin = torch.empty(fe.moments_bytes // 8, dtype=torch.float64).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(Te):
            fe._check(fe.lib.pmf_step(fe.h, dt, cfg.l, C.c_void_p(zp + (i + 3) * zstride), 0, C.byref(lik),
                                      cfg.k_sigma))
            if async_ok:
                fe.moments_async(mom_pin)                     # D2H read of the step's result
            else:
                fe.moments_into(mean, cov, logc)
        e1.record(stream)
        e1.synchronize()
        if async_ok:
            rec = mom_pin.numpy().reshape(cfg.batch, -1)
            assert np.all(rec[:, -1] == 0.0), "a filter's update failed in the e2e run"
        te = max_over_ranks(e0.elapsed_time(e1), device=f"cuda:{local}")
        e2e = {"value": ranks_work * points_step * Te / (te * 1e-3), "unit": "grid-point updates/s",
               "h2d_bytes_per_step": cfg.batch * cfg.nz * 8,
               "d2h_bytes_per_step": fe.moments_bytes, "steps": Te}
        fe.close()

    # ---------------------------------------------------------------- roofline
    # The method's algorithmic bytes per epoch: read + write every weight once (16 B per grid
    # point fp64, 8 B fp32), over the whole event-timed epoch. kernels[]: the dominant
    # kernel's live event time (the library brackets it on its stream) and the ncu launch-list
    # shares of every kernel of one epoch (committed under profiles/r2).
    kern_ms = kern_total_ms / max(kern_n, 1)
    alg_bytes = 2 * esize * points_step
    achieved = alg_bytes / (ms_step * 1e-3) / 1e9
    dom = dominant_kernel(cfg, f, pmf, wl, epoch_kernel, esize, points_step)
    km = kernel_metrics(dom["name"])
    kernels = [{"name": dom["name"], "live_ms": kern_ms, "timed_launches": kern_n,
                "share_of_step_live": kern_ms / ms_step, "alg_bytes_per_launch": dom["bytes"],
                "alg_bytes_per_unit": dom["per"],
                "achieved_GBps": dom["bytes"] / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else None,
                "dram_bytes_ncu": km.get("dram_bytes"), "fp64_pipe_frac_ncu":
                    (km["fp64_pipe_pct"] / 100.0) if "fp64_pipe_pct" in km else None,
                # the co-bottleneck of the FFT passes: shared-memory wavefronts (% of peak, ncu)
                "smem_wavefronts_frac_ncu": (km["smem_wavefronts_pct"] / 100.0) if "smem_wavefronts_pct" in km else None,
                "ncu_source": km.get("source")}]
    ls = launch_shares(workload)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs,
            "traffic": (ls or {}).get("dram_bytes_per_epoch"), "kernel": "whole epoch (every kernel of the step)",
            "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_unit": f"{2 * esize} B per grid point per epoch",
            "peak_source": hbm_src, "kernels": kernels,
            "ncu_epoch": ls}
    if wl.get("diff_mode", 0) == 2:
        # FDM: the last-axis DST kernel = two dense GEMMs (forward, inverse) per pencil on the FP64
        # tensor cores: 2 x 2 x N_L flops per grid point (FMA = 2 flops), against the measured DMMA peak
        NL = cfg.n[-1]
        flops = 2 * 2 * NL * points_step
        ach_t = flops / (kern_ms * 1e-3) / 1e12
        roof["tensor"] = {"achieved": ach_t, "peak": ap["dmma"], "unit": "TFLOP/s", "frac": ach_t / ap["dmma"],
                          "kernel": dom["name"], "peak_source": ap["source"] + " fp64_dmma",
                          "alg_flops_per_unit": f"{4 * NL} flop per grid point"}
    if f.path == pmf.PATH_RESIDENT:
        # The fused epoch kernel's FP64 (FP32) issue: the predict's algorithmic slots (SURVEY
        # §8(d): 3.5 log2 N per complex point per axis and direction, halved for real data, and
        # 3 l + 10 per spectral point) / the kernel's live time / the MEASURED FMA issue peak
        slots_pp = 0.5 * 4 * 3.5 * math.log2(cfg.n[0]) + psi_slots(cfg, wl) * (cfg.n[1] // 2 + 1) / cfg.n[1]
        pname = "FP64" if dtype == "f64" else "FP32"
        peak_alu = (ap["fp64"] if dtype == "f64" else ap["fp32"]) / 2
        ach = slots_pp * points_step / (kern_ms * 1e-3) / 1e12
        roof["alu"] = {"achieved": ach, "peak": peak_alu, "unit": f"T {pname} issue slots/s", "frac": ach / peak_alu,
                       "kernel": dom["name"], "peak_source": ap["source"] + f" ({pname} FMA TFLOP/s / 2)",
                       "alg_units_per_unit": f"{slots_pp:.1f} {pname} issue slots per grid point"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_budget)
    l2txt = (f"inputs larger than L2 ({esize * points_step / 1e6:.0f} MB of weights per GPU): no flush" if not l2_resident
             else f"weights ({esize * points_step / 1e6:.1f} MB) fit in the 126 MB L2: a 252 MB buffer is written "
                  f"before every timed step (flushed); unflushed numbers under steps_unflushed")
    line = {"metric": metric_name(dtype), "value": value, "unit": "grid-point updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": workload_name(workload, cfg, world, glob_batch),
                       "step": "regrid + predict (Alg. 1-6) + update + moments, every filter",
                       "substeps": "crank-nicolson (R27)" if wl.get("step", 0) else "semi-implicit euler (P:313-318)",
                       "grid": "eigenvector-aligned (R28)" if wl.get("grid", 0) else "axis-aligned (R12)",
                       "l2": l2txt,
                       "path": ("fdm: DST-I GEMMs on FP64 tensor cores" if wl.get("diff_mode", 0) == 2 else epoch_kernel),
                       "parallelism": (f"slab-sharded x{world if real_nccl else args.virtual_ranks}"
                                       f"{' (NCCL)' if real_nccl else ' (virtual ranks)'} along the last "
                                       "axis (2 all-to-all per predict, all-reduce per update)" if sharded
                                       else f"filter-sharded x{world}: {cfg.batch} of {glob_batch} filters on this "
                                            "rank (no data-path collective)" if glob_batch > 1
                                       else "one GPU")},
            "steps_timing": stats, "steps_unflushed": unflushed,
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
            "time_update": tu}
    f.close()
    return line


def psi_slots(cfg, wl):
    """Issue slots of the spectral multiplier per half-spectrum point: Euler
    3 l + 10 (per substep one factor, two FMA + one multiply); Crank-Nicolson (R27) 5 l + 12
    (l + 1 factors, each also entering the numerator product as 2 - f)."""
    return 5 * cfg.l + 12 if wl.get("step", 0) else 3 * cfg.l + 10


def dominant_kernel(cfg, f, pmf, wl, epoch_kernel, esize, points_step):
    """Name and algorithmic bytes per launch of the kernel the library's profiling events bracket."""
    tname = "double" if cfg.dtype == "f64" else "float"
    nspec = points_step // cfg.n[1] * (cfg.n[1] // 2 + 1) if cfg.nx > 1 else points_step
    if wl.get("diff_mode", 0) == 2:
        return {"name": f"k_dst<{cfg.n[-1]}, {'true' if cfg.nx == 1 else 'false'}, 2>",
                "bytes": 2 * esize * points_step, "per": f"{2 * esize} B per grid point"}
    if f.path == pmf.PATH_RESIDENT:
        cn = 1 if wl.get("step", 0) else 0                # template <T, RG, UPDATE, CN>
        return {"name": f"k_resident_epoch<{tname}, 1, 1, {cn}>", "bytes": 2 * esize * points_step,
                "per": f"{2 * esize} B per grid point"}
    if f.path == pmf.PATH_PLANE and cfg.nx == 4 and cfg.dtype == "f64" and cfg.n[2] == cfg.n[3]:
        # K2: reads and writes the half spectrum once
        tm = 48 if cfg.n[2] == 96 else (32 if cfg.n[2] >= 64 else cfg.n[2] // 2)   # Q2<NQ>::TEAMS
        return {"name": f"k_q_mid<{cfg.n[2]}, {tm}>", "bytes": 2 * 2 * esize * nspec,
                "per": f"{4 * esize} B per half-spectrum point (read + write of the spectrum)"}
    if f.path == pmf.PATH_PLANE:
        return {"name": f"k_plane_mid<{tname}, {cfg.n[-1]}, 2, {cfg.nx}, {1 if cfg.n[-1] == 96 else 3}>",
                "bytes": 2 * 2 * esize * nspec, "per": f"{4 * esize} B per half-spectrum point"}
    if epoch_kernel == "cluster":
        return {"name": "k_cluster_epoch<true, true, 16>", "bytes": 2 * esize * points_step,
                "per": f"{2 * esize} B per grid point (whole epoch)"}
    if epoch_kernel == "line":
        return {"name": f"k_line_epoch<{tname}, true, true, {cfg.n[0]}>", "bytes": 2 * esize * points_step,
                "per": f"{2 * esize} B per grid point (whole epoch)"}
    return {"name": "pencil predict (prep .. finalize)", "bytes": 2 * esize * points_step,
            "per": f"{2 * esize} B per grid point (whole predict)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--l", type=int, default=None, help="override Euler substeps")
    ap.add_argument("--path", type=int, default=0, help="0 auto, 1 pencil, 2 resident, 3 plane")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-time-update", action="store_true")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="split one filter into this many slabs on one GPU (exercises the sharded path)")
    ap.add_argument("--nccl-self", action="store_true",
                    help="N = 1 only: run the one-filter workload on the real NCCL sharded path with a "
                         "1-rank communicator (send/recv to itself): checks the multi-process code path on one GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=16.0)
    ap.add_argument("--ref-budget", type=float, default=4.0)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--also", default="auto",
                    help="comma list of further workloads measured compactly into the line's 'also' (N=1); "
                         "auto: the other BASELINE configs and NEXT rows with the default C4 workload")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    # stdout carries exactly ONE line, the JSON: anything a library prints there during the run
    # (NCCL's "NCCL version ..." banner goes to stdout) is sent to stderr instead
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = run_workload(args, args.workload, rank, world, local)
    also_list = ("C5,C5l1,C5f32,C5cn,C3,C2,C1,C5fdm,C6" if args.workload == "C4" else "") \
        if args.also == "auto" else args.also
    if also_list and world == 1:
        # the other configurations, measured the same way (compact: no e2e, no oracle)
        also = {}
        for w in also_list.split(","):
            sub = argparse.Namespace(**{**vars(args), "steps": 20, "warmup": 3, "no_e2e": w != "C5",
                                        "no_cpu": w != "C5", "path": 0, "virtual_ranks": 1, "nccl_self": False, "cpu_budget": 8.0})
            r = run_workload(sub, w, rank, world, local, secondary=True)
            also[w] = {k: r[k] for k in ("value", "unit", "ms_per_step", "dtype", "steps_timing", "steps_unflushed",
                                         "roofline", "time_update", "gpu_launches", "clocks", "e2e", "cpu_baseline")}
            also[w].update(workload=r["config"]["workload"], path=r["config"]["path"], l2=r["config"]["l2"])
        line["also"] = also
    if rank == 0:
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())
        if args.json_out:
            with open(args.json_out, "w") as fh:
                json.dump(line, fh, indent=1)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
