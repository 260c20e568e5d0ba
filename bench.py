#!/usr/bin/env python
"""Benchmark of the spectral point-mass filter hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl cuda|reference]

A STEP is one filter epoch over the whole batch, i.e. every row of SURVEY
§8(a): (re-centre grid + multilinear resample, R12) -> forward DFT per axis
-> s*Psi over l Euler substeps -> inverse DFT -> normalise (Alg. 1-6) ->
likelihood, normaliser and moments (eq:filt). Default workload C5 (BASELINE
configs[4]): 4096 independent 2-D CV filters on 128x128, fp64, l = 10 -- the
largest single-GPU configuration whose per-GPU work is fixed, sharded by filter
index across ranks (weak scaling: every rank runs its own 4096 filters; no
collective on the data path).

Metric (BASELINE.json): grid-point FPE updates/sec = filters * 128^2 / t_step.
Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize, CUDA events on the library's stream, max over ranks.
The weights (537 MB fp64) exceed the 126 MB L2, so no flush is needed.
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
    "C5": dict(cid="C5", over={}),
    "C5f32": dict(cid="C5", over={"dtype": "f32"}),
    "C4": dict(cid="C4", over={}),
    "C3": dict(cid="C3", over={}),
    "C2": dict(cid="C2", over={}),
    "C1": dict(cid="C1", over={}),
    # NEXT-1: the paper's FDM baseline (eq:FST) on the C5 batch, DST-I on FP64 tensor cores
    "C5l1": dict(cid="C5", over={"l": 1}),      # report l = 1 next to l = 10
    "C5fdm": dict(cid="C5", over={}, diff_mode=2),
    # NEXT-4: Crank-Nicolson substeps (R27) and eigenvector-aligned grids (R28) on the C5 batch
    "C5cn": dict(cid="C5", over={}, step=1),
    "C5eig": dict(cid="C5", over={}, grid=1),
    # NEXT-3: the paper's §VI scenario (coordinated turn, terrain altitude + GM noise, N_pa = 34)
    "C6": dict(cid="C6", over={}),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)", d.get("sm_max_mhz", 1965.0)
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", 1965.0


# B200: 148 SMs x 64 FP64 FMA/clk (the FP64 pipe is half the FP32 rate on B200);
# one FMA counts as 2 flops. See DESIGN.md §5.
def fp64_peak_tflops(mhz):
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region (the
    B200_PROFILING.md clocks line), via NVML from a background thread every 2 ms
    (the timed region is only tens of ms, too short for `nvidia-smi -lms`)."""
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


def oracle_sample(cfg, zs, budget_s: float, max_filters: int):
    """Time the CPU oracle (as it stands) on a bounded sample: one epoch
    (predict + update + moments + regrid) per filter, filters 0.. until the
    budget is used. Returns (points_per_s, filter_epochs, seconds)."""
    from oracle import pmf_oracle as O
    n = tuple(cfg.n)
    done, t_tot = 0, 0.0
    for b in range(min(cfg.batch, max_filters)):
        w, c, B = O.initial_density(cfg.prior_mean[b], cfg.prior_cov, n, cfg.k_sigma)
        t0 = time.perf_counter()
        w, c, B = O.predict(w, c, B, cfg.A, cfg.Q, cfg.tau, cfg.l)
        w, _ = O.update(w, c, B, O.make_likelihood(cfg, O.grid_points(c, B, n), zs[1, b]))
        mean, cov = O.moments(w, c, B)
        c2, B2 = O.regrid_target(mean, cov, n, cfg.k_sigma)
        w = O.regrid(w, c, B, c2, B2)
        t_tot += time.perf_counter() - t0
        done += 1
        if t_tot >= budget_s:
            break
    return done * cfg.points / t_tot, done, t_tot


def psi_slots(cfg, wl):
    """Issue slots of the spectral multiplier per half-spectrum point: Euler
    3 l + 10 (per substep one factor, two FMA + one multiply); Crank-Nicolson (R27) 5 l + 12
    (l + 1 factors, each also entering the numerator product as 2 - f)."""
    return 5 * cfg.l + 12 if wl.get("step", 0) else 3 * cfg.l + 10


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count() or 1


def workload_name(workload, cfg):
    """config.workload, identical on both arms."""
    return (f"{workload}: {cfg.batch} x {'x'.join(map(str, cfg.n))} {cfg.nx}-D filters per GPU, "
            f"l={cfg.l}, tau={cfg.tau}, k_sigma={cfg.k_sigma}")


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    cfg = make_config(wl["cid"], **wl["over"])
    zs = simulate(cfg.replace(batch=min(cfg.batch, 64)), T=1)["z"]
    cfgs = cfg.replace(batch=min(cfg.batch, 64))
    per_step = []
    for _ in range(args.warmup + args.steps):
        v, nf, t = oracle_sample(cfgs, zs, budget_s=args.ref_budget, max_filters=64)
        per_step.append((v, nf, t))
    timed = per_step[args.warmup:]
    val = statistics.median(v for v, _, _ in timed)
    nf = timed[0][1]
    # the arm's metric name (the oracle itself always computes in fp64)
    metric = "grid-point FPE updates/sec (fp64)" if cfg.dtype == "f64" else "grid-point FPE updates/sec (fp32)"
    line = {"impl": "reference", "metric": metric, "value": val,
            "unit": "grid-point updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * cfg.batch * cfg.points / val, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.workload, cfg),
                       "sample": f"{nf} filter-epochs per step (oracle is O(N^2) naive DFT)"},
            "cpu_baseline": {"value": val, "unit": "grid-point updates/s", "cores": threads_used(), "kind": "oracle",
                             "sample": f"{nf} of {cfg.batch} filters x 1 epoch per step"},
            "e2e": {"value": val, "unit": "grid-point updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_workload(args, workload, rank, world, local, secondary=False):
    """One bench measurement of `workload`; returns the JSON-line dict (rank 0 prints it)."""
    import torch
    import torch.distributed as dist
    from paper_2412_07240_b200 import pmf
    wl = WORKLOADS[workload]
    cfg = make_config(wl["cid"], **wl["over"])
    if args.l:
        cfg = cfg.replace(l=args.l)
    from paper_2412_07240_b200.dist import max_over_ranks, rank_seed
    # One large filter (batch 1, C2-C4) with N > 1 GPUs (or --virtual-ranks): its grid is
    # split into slabs along the last axis (strong scaling, all-to-all transposes).
    # Batched filters (C5): every rank runs its own batch (weak scaling, no collective).
    sharded = cfg.batch == 1 and cfg.nx >= 2 and (world > 1 or args.virtual_ranks > 1)
    if not sharded:
        cfg = make_config(wl["cid"], **{**wl["over"], "seed": rank_seed(cfg.seed, rank), "l": cfg.l})
    dtype = cfg.dtype
    T = args.warmup + args.steps + 1
    zs = simulate(cfg, T=T)["z"]                       # (T+1, batch, nz)
    stream = torch.cuda.Stream()
    fkw = {}
    if sharded and world > 1:
        obj = [pmf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        fkw = dict(world=world, rank=rank, unique_id=obj[0])
    elif sharded:
        fkw = dict(world=args.virtual_ranks, sharded=True)
    diff_mode = wl.get("diff_mode", 0)
    fkw.update(step=wl.get("step", 0), grid=wl.get("grid", 0))
    f = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, dtype=dtype, path=args.path,
                   device=local, stream=stream.cuda_stream, diff_mode=diff_mode, **fkw)
    if cfg.lik_kind == 2:
        from workloads import terrain_table
        lik = pmf.make_likelihood(pmf.LIK_TERRAIN_GM, cfg.nx, gm=cfg.extra["gm"])
        f.set_terrain(*terrain_table(cfg))
    else:
        lik = (pmf.make_likelihood(pmf.LIK_RANGE_GAUSS, cfg.nx, sigma=cfg.sigma) if cfg.lik_kind == 1
               else pmf.make_likelihood(pmf.LIK_LINEAR_GAUSS, cfg.nx, H=cfg.H, R=cfg.R))
    f.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
    z_dev = torch.tensor(zs, dtype=torch.float64, device=f"cuda:{local}")   # inputs resident in HBM
    dt = cfg.tau / cfg.l
    f.update(z_dev[0], lik)
    f.regrid(cfg.k_sigma)
    k = 1
    for _ in range(args.warmup):
        f.step(dt, cfg.l, z_dev[k], lik, cfg.k_sigma)
        k += 1
    torch.cuda.synchronize()      # (not f.sync(): that would flush the pending regrid outside the timed region)
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    launches0 = f.launches
    f.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0 = k
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(args.steps):
            f.step(dt, cfg.l, z_dev[k0 + i], lik, cfg.k_sigma)
        ev1.record(stream)
    ev1.synchronize()
    clk = clocks.stop()
    launches = f.launches - launches0
    epoch_kernel = f.epoch_kernel                    # kernel family of the timed epochs
    kern_total_ms, kern_n = f.profile_read()
    f.profile(False)
    t_ms = ev0.elapsed_time(ev1)
    torch.cuda.synchronize()
    t_max = max_over_ranks(t_ms, device=f"cuda:{local}")
    points_step = cfg.batch * cfg.points
    ranks_work = 1 if sharded else world             # strong (sharded) vs weak scaling
    value = ranks_work * points_step * args.steps / (t_max * 1e-3)
    ms_step = t_max / args.steps

    # ---------------------------------------------------------------- FPE time update alone (Alg. 1-6)
    # north_star's "FPE time update at >= 60% of the HBM roofline": predict-only steps
    # (no likelihood, no regrid) on the same resident state; 16 B/point algorithmic.
    tu = None
    if not args.no_time_update:
        for _ in range(2):
            f.predict(dt, cfg.l)
            f.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f.profile(True)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            f.predict(dt, cfg.l)
            f.sync()
        t1.record(stream)
        t1.synchronize()
        km_ms, km_n = f.profile_read()
        f.profile(False)
        tt = max_over_ranks(t0.elapsed_time(t1), device=f"cuda:{local}") / args.steps
        hbm_gbs = peaks()[0]
        esz = 8 if dtype == "f64" else 4
        pts = (1 if sharded else world) * cfg.batch * cfg.points
        tu = {"ms_per_step": tt, "value": pts / (tt * 1e-3), "unit": "grid-point updates/s",
              "kernel_ms": km_ms / max(km_n, 1),
              "hbm_frac": 2 * esz * cfg.batch * cfg.points / (km_ms / max(km_n, 1) * 1e-3) / 1e9 / hbm_gbs,
              "what": "predict only (prep + transform/Psi kernel + closed-form normalisation), same filters"}
        if f.path == pmf.PATH_RESIDENT:
            # the predict's algorithmic issue slots against the FP64 (FP32) issue peak
            spp = 0.5 * 4 * 3.5 * math.log2(cfg.n[0]) + psi_slots(cfg, wl) * (cfg.n[1] // 2 + 1) / cfg.n[1]
            tu["alu_frac"] = (spp * cfg.batch * cfg.points / (km_ms / max(km_n, 1) * 1e-3)) / \
                (148 * (64 if dtype == "f64" else 128) * peaks()[2] * 1e6)

    # ---------------------------------------------------------------- e2e: host buffers through the C ABI
    e2e = None
    if not args.no_e2e:
        Te = min(args.steps, 10)
        zs_e = simulate(cfg, T=Te + 3)["z"]
        z_pin = torch.tensor(zs_e, dtype=torch.float64).pin_memory()
        if sharded and world > 1:
            obj = [pmf.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            fkw = dict(world=world, rank=rank, unique_id=obj[0])
        fkw.update(step=wl.get("step", 0), grid=wl.get("grid", 0))
        fe = pmf.Filter(cfg.nx, cfg.n, cfg.A, cfg.Q, batch=cfg.batch, dtype=dtype, path=args.path,
                        device=local, stream=stream.cuda_stream, diff_mode=diff_mode, **fkw)
        if cfg.lik_kind == 2:
            fe.set_terrain(*terrain_table(cfg))
        fe.set_gaussian(cfg.prior_mean, np.broadcast_to(cfg.prior_cov, (cfg.batch, cfg.nx, cfg.nx)), cfg.k_sigma)
        mean = np.empty((cfg.batch, cfg.nx))
        cov = np.empty((cfg.batch, cfg.nx, cfg.nx))
        logc = np.empty(cfg.batch)
        zp = z_pin.data_ptr()
        zstride = cfg.batch * cfg.nz * 8
        import ctypes as C
        fe.lib.pmf_update(fe.h, C.c_void_p(zp), 0, C.byref(lik))
        fe.regrid(cfg.k_sigma)
        fe.moments_into(mean, cov, logc)
        for i in range(2):                                    # warm-up (graph capture happens here)
            rc = fe.lib.pmf_step(fe.h, dt, cfg.l, C.c_void_p(zp + (i + 1) * zstride), 0, C.byref(lik), cfg.k_sigma)
            assert rc == 0, fe.lib.pmf_last_error(fe.h)
            fe.moments_into(mean, cov, logc)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # the step's result (moments of every filter) is read back every step into pinned host
        # memory, asynchronously on the library's stream (pmf_moments_async): no host stall
        # between steps; all reads complete inside the timed region (e1 follows them)
        async_ok = not (sharded and world > 1) and args.virtual_ranks == 1
        mom_pin = torch.empty(fe.moments_bytes // 8, dtype=torch.float64).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(Te):
            rc = fe.lib.pmf_step(fe.h, dt, cfg.l, C.c_void_p(zp + (i + 3) * zstride), 0, C.byref(lik), cfg.k_sigma)
            assert rc == 0, fe.lib.pmf_last_error(fe.h)
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

    # ---------------------------------------------------------------- roofline (dominant kernel)
    # algorithmic bytes: read + write every weight once per epoch; the kernel's
    # average duration comes from CUDA events the library records around it on its stream.
    hbm, hbm_src, sm_max = peaks()
    esize = 8 if dtype == "f64" else 4
    kern_ms = kern_total_ms / max(kern_n, 1)
    tname = "double" if dtype == "f64" else "float"
    roof_extra = None
    if diff_mode == 2:
        # FDM: the last-axis DST kernel = two dense GEMMs (forward, inverse) per pencil on the
        # FP64 tensor cores: 2 x 2 x N_L flops per grid point (FMA = 2 flops)
        NL = cfg.n[-1]
        kname = f"k_dst<{NL}, {'true' if cfg.nx == 1 else 'false'}, 2>"
        flops = 2 * 2 * NL * points_step
        bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 1648.2) \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1648.2
        peak_t = bf16 * 45.0 / 2250.0     # FP64 tensor: measured bf16 x the nominal ratio 45/2250 TF
        ach_t = flops / (kern_ms * 1e-3) / 1e12
        roof_extra = {"bound": "tensor", "achieved": ach_t, "peak": peak_t, "unit": "TFLOP/s",
                      "frac": ach_t / peak_t, "traffic": None, "kernel": kname, "kernel_ms": kern_ms,
                      "timed_launches": kern_n, "share_of_step": kern_ms / ms_step,
                      "peak_source": "MEASURED_PEAKS.json bf16_tflops x nominal FP64-tensor/bf16 ratio 45/2250",
                      "alg_flops_per_launch": flops, "alg_flops_per_unit": f"{4 * NL} flop per grid point"}
    if f.path == pmf.PATH_RESIDENT:
        # the fused epoch kernel: read + write every weight once
        kname = f"k_resident_epoch<{tname}, 1, 1>"
        alg_bytes, per = 2 * esize * points_step, f"{2 * esize} B per grid point"
    elif f.path == pmf.PATH_PLANE:
        # the last-axis pass (forward DFT x s Psi x inverse DFT, Alg. 3-5): read + write the
        # half spectrum once, nspec = (N1/2+1) N0 N2 (N3) complex points per filter
        nspec = cfg.batch * cfg.points // cfg.n[1] * (cfg.n[1] // 2 + 1)
        kname = f"k_plane_mid<{tname}, {cfg.n[-1]}, 2, {cfg.nx}, {1 if cfg.n[-1] == 96 else 3}>"
        alg_bytes, per = 2 * 2 * esize * nspec, f"{4 * esize} B per half-spectrum point"
    elif epoch_kernel == "cluster":
        kname = "k_cluster_epoch<true, true, 16>"
        alg_bytes, per = 2 * esize * points_step, f"{2 * esize} B per grid point (whole epoch)"
    elif epoch_kernel == "line":
        kname = f"k_line_epoch<{tname}, true, true, {cfg.n[0]}>"
        alg_bytes, per = 2 * esize * points_step, f"{2 * esize} B per grid point (whole epoch)"
    else:
        kname = "pencil predict (prep .. finalize)"
        alg_bytes, per = 2 * esize * points_step, f"{2 * esize} B per grid point (whole predict)"
    km = kernel_metrics(kname)
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": km.get("dram_bytes"), "kernel": kname, "kernel_ms": kern_ms, "timed_launches": kern_n,
            "share_of_step": kern_ms / ms_step, "peak_source": hbm_src, "alg_bytes_per_launch": alg_bytes,
            "alg_bytes_per_unit": per,
            "fp64_pipe_frac_ncu": (km["fp64_pipe_pct"] / 100.0) if "fp64_pipe_pct" in km else None,
            "ncu_source": km.get("source")}
    if roof_extra is not None:
        roof = roof_extra
    elif f.path == pmf.PATH_RESIDENT:
        # The fused epoch kernel is FP64-issue bound (ALU roofline below the HBM one): per
        # grid point the predict alone needs ~70 FP64 issue slots (FFT 3.3e9 +
        # Psi 1.4e9 slots for 4096 x 128^2, i.e. 3.5 log2 N per complex point per axis and
        # direction, halved for real data, and 3 l + 10 per spectral point) against 16 B of
        # HBM traffic, while B200 issues 148 x 64 FP64 lanes per clock. Peak = that issue
        # rate at the max SM clock; the HBM fraction is kept alongside.
        # fp32: the same slots on the FP32 pipe (128 lanes per SM per clock)
        slots_pp = 0.5 * 4 * 3.5 * math.log2(cfg.n[0]) + psi_slots(cfg, wl) * (cfg.n[1] // 2 + 1) / cfg.n[1]
        slots = slots_pp * points_step
        lanes, pname = (64, "FP64") if dtype == "f64" else (128, "FP32")
        peak_alu = 148 * lanes * sm_max * 1e6 / 1e12
        ach = slots / (kern_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": ach, "peak": peak_alu, "unit": f"T {pname} issue slots/s",
                "frac": ach / peak_alu, "traffic": km.get("dram_bytes"), "kernel": kname, "kernel_ms": kern_ms,
                "timed_launches": kern_n, "share_of_step": kern_ms / ms_step,
                "peak_source": f"148 SMs x {lanes} {pname} lanes x max SM clock (B200_PROFILING / B300 guide unit counts)",
                "alg_units_per_launch": slots, "alg_units_per_unit": f"{slots_pp:.1f} {pname} issue slots per grid point",
                "fp64_pipe_frac_ncu": (km["fp64_pipe_pct"] / 100.0) if "fp64_pipe_pct" in km else None,
                "ncu_source": km.get("source"),
                "hbm": {"achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                        "alg_bytes_per_launch": alg_bytes, "alg_bytes_per_unit": per, "peak_source": hbm_src}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, nf, ts = oracle_sample(cfg, zs, budget_s=args.cpu_budget, max_filters=cfg.batch)
        cpu = {"value": v, "unit": "grid-point updates/s", "cores": threads_used(), "kind": "oracle",
               "sample": f"{nf} of {cfg.batch} filters x 1 epoch ({ts:.1f} s of CPU time)"}

    line = {"metric": "grid-point FPE updates/sec (fp64)" if dtype == "f64" else "grid-point FPE updates/sec (fp32)",
            "value": value, "unit": "grid-point updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": workload_name(workload, cfg),
                       "step": "regrid + predict (Alg. 1-6) + update + moments, every filter",
                       "substeps": "crank-nicolson (R27)" if wl.get("step", 0) else "semi-implicit euler (P:313-318)",
                       "grid": "eigenvector-aligned (R28)" if wl.get("grid", 0) else "axis-aligned (R12)",
                       "l2": (f"inputs larger than L2 ({esize * points_step / 1e6:.0f} MB of weights per GPU)"
                              if esize * points_step > 126e6 else
                              f"weights ({esize * points_step / 1e6:.0f} MB) fit in the 126 MB L2: L2-resident workload"),
                       "path": ("fdm: DST-I GEMMs on FP64 tensor cores" if diff_mode == 2 else epoch_kernel),
                       "parallelism": (f"slab-sharded x{world if world > 1 else args.virtual_ranks} along the last "
                                       "axis (2 all-to-all per predict, all-reduce per update)" if sharded
                                       else f"filter-sharded x{world} (no data-path collective)")},
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
            "time_update": tu}
    f.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--l", type=int, default=None, help="override Euler substeps")
    ap.add_argument("--path", type=int, default=0, help="0 auto, 1 pencil, 2 resident, 3 plane")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-time-update", action="store_true")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="split one filter into this many slabs on one GPU (exercises the sharded path)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=8.0)
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--also", default="auto",
                    help="comma list of further workloads measured compactly into the line's 'also' (N=1); "
                         "auto: C4,C3 with the default C5 workload")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2412_07240_b200 import pmf

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = run_workload(args, args.workload, rank, world, local)
    also_list = ("C5l1,C5f32,C5cn,C4,C3,C2,C1,C5fdm,C6" if args.workload == "C5" else "") if args.also == "auto" else args.also
    if also_list and world == 1:
        # the other large single-GPU configurations, measured the same way (compact)
        also = {}
        for w in also_list.split(","):
            sub = argparse.Namespace(**{**vars(args), "steps": max(5, min(args.steps, 10)), "warmup": 3,
                                        "no_e2e": True, "no_cpu": True, "path": 0, "virtual_ranks": 1})
            r = run_workload(sub, w, rank, world, local, secondary=True)
            also[w] = {k: r[k] for k in ("value", "unit", "ms_per_step", "dtype")}
            also[w].update(workload=r["config"]["workload"], path=r["config"]["path"],
                           roofline=r["roofline"], time_update=r["time_update"], gpu_launches=r["gpu_launches"],
                           clocks=r["clocks"])
        line["also"] = also
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                json.dump(line, fh, indent=1)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
