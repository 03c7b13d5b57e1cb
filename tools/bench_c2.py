#!/usr/bin/env python
"""tools/bench_c2.py -- the round-1 headline (C2 step, kept as a tool): BASELINE.json metric: Toeplitz rows x orders / s for the
p = 1..p_max order sweep, plus the fused-pass roofline fraction.

Workload (configs[1], "C2"): synthetic AR(50) series, n = 1e7, fp64, roots
|r| ~ U[1.2, 3] (seeded, cascade-form simulation, N(0,1) innovations), p_max =
200; LSAR and Repeated-Halving sweeps side by side at s in {1e4, 1e5}.  One
step = every sweep of that list once; rows x orders per sweep = p_max (n -
p_max).  Data is synthetic (no dataset is named).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): independent replicas of the workload per
rank ("replicas only" -- the row-sharded multi-GPU sweep is future work),
barrier + max-over-ranks device time.  --impl reference times the CPU port of
the reference (oracle/, single-threaded like the reference) on a bounded lag
sample of the same workload, extrapolated per lag (labelled as such).
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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRIC = "Toeplitz rows x orders / s for the p=1..p_max sweep"
UNIT = "rows*orders/s"
WORKLOAD = ("C2: AR(50) n=1e7 fp64, p_max=200, LSAR and Repeated-Halving side by side "
            "at s in {1e4, 1e5}")
SEED = 2112_12994


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=None, help="override series length (debug)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--sequential", action="store_true",
                    help="run the step's sweeps one after another instead of concurrently")
    ap.add_argument("--profile-step", action="store_true",
                    help="wrap one extra step in cudaProfilerStart/Stop (ncu --profile-from-start off)")
    return ap.parse_args()


def sweeps_for(cs):
    """The C2 step: LSAR and Repeated Halving side by side at every sample size."""
    return [("lsar", c) for c in cs] + [("rh", c) for c in cs]


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU port
def cpu_sweep_estimate(y, p_bar, sweeps, n_pass=1_000_000, c_cap=5_000, rh_rows=60_000):
    """Single-threaded oracle port timed on a bounded sample, extrapolated per part.

    A lag body of the reference splits into parts with known size scaling:
      * O(w) + O(w p): leverage update + distribution + c draws (lsar.cpp:83-93,
        sketch.cpp:20-59) and the per-tap residual (toeplitz.cpp:84-98) -- timed
        on a prefix of n_pass rows at p in {1, p_bar/2, p_bar}, fitted a + b p and
        scaled by w / w';
      * O(c p^2): sampled gather + CPQR solve (sketch.cpp:61-79,
        toeplitz.cpp:57-71) -- timed on c' = min(c, c_cap) rows at p in
        {p_bar/4, p_bar/2, p_bar}, fitted as a quadratic in p and scaled by c / c'.
    LSAR = sum over p of all parts; RH = the upfront phase (repeated_halving.cpp:
    126-189, timed on two prefixes, linear in rows) + per lag one sampling
    draw from the fixed distribution and the solve part (repeated_halving.cpp:
    205-231).  Returns (total seconds, per-sweep detail, description).
    """
    from oracle import oracle as orc
    orc.lib()
    n = y.size
    w = n - p_bar
    yp = np.ascontiguousarray(y[: min(n, n_pass + p_bar)])
    wp = yp.size - p_bar
    rng = np.random.default_rng(7)
    pp = np.arange(1, p_bar + 1, dtype=float)
    # O(w p) residual, per row
    P1 = sorted({1, max(1, p_bar // 2), p_bar})
    t_res = []
    for p in P1:
        phi = rng.standard_normal(p) * 0.01
        t0 = time.perf_counter()
        orc.residuals(yp[p_bar - p:], wp + p, p, phi)
        t_res.append(time.perf_counter() - t0)
    cr = np.polyfit(np.array(P1, float), np.array(t_res), 1) if len(P1) > 1 else [0.0, t_res[0]]
    res_sweep = float(np.sum(np.maximum(np.polyval(cr, pp), 0.0))) * (w / wp)
    # O(w) leverage update + distribution (+ draws, per c)
    s0 = orc.init_leverage_p1(yp[:wp])
    r0 = rng.standard_normal(wp)
    t0 = time.perf_counter()
    s1 = orc.leverage_update(s0, r0)
    dist = orc.leverage_to_distribution(s1)
    t_upd = (time.perf_counter() - t0) * (w / wp)
    solve_fit, samp, solve_fit_cp = {}, {}, {}
    P2 = sorted({max(1, p_bar // 4), max(1, p_bar // 2), p_bar})
    for c in sorted({c for _, c in sweeps}):
        t0 = time.perf_counter()
        orc.sample_rows(dist, c, 11)
        samp[c] = (time.perf_counter() - t0) * (w / wp)
        cp = min(c, c_cap)
        if cp in solve_fit_cp:
            solve_fit[c] = solve_fit_cp[cp] * (c / cp)
            continue
        ts = []
        for p in P2:
            idx = rng.integers(0, wp - 1, cp)
            wt = np.ones(cp)
            t0 = time.perf_counter()
            a, b = orc.apply_sample(yp, wp + p, p, idx, wt)
            orc.solve_exact(a, b)
            ts.append(time.perf_counter() - t0)
        deg = min(2, len(P2) - 1)
        cs_ = np.polyfit(np.array(P2, float), np.array(ts), deg)
        solve_fit_cp[cp] = float(np.sum(np.maximum(np.polyval(cs_, pp), 0.0)))
        solve_fit[c] = solve_fit_cp[cp] * (c / cp)
    # RH upfront (halving + upward sampling + final unsketched scores) at c' = c_cap:
    # linear in rows from two prefixes; for c > c' add the extra CPQR of the c x k
    # level matrices (the solve part at p_bar scaled by c) once per level.
    k = p_bar + 1

    def depth(c, m):
        base = max(c, 10 * k * int(np.ceil(np.log(k + 1.0))))
        d = 0
        while m > base:
            m //= 2
            d += 1
        return d

    up = None
    if any(m_ == "rh" for m_, _ in sweeps):
        cu = min(c_cap, min(c for m_, c in sweeps if m_ == "rh"))
        r1, r2 = rh_rows // 2, rh_rows
        t1 = orc.rh_time_upfront(np.ascontiguousarray(y[: r1 + p_bar]), p_bar, cu, 7)
        t2 = orc.rh_time_upfront(np.ascontiguousarray(y[: r2 + p_bar]), p_bar, cu, 7)
        slope = (t2 - t1) / (r2 - r1)
        up = {"c0": cu, "t0": t1 + slope * (w - r1)}
    qr_pbar = {}
    for c in solve_fit:
        # single-lag CPQR at p = p_bar for c rows (for the RH level-factor correction)
        qr_pbar[c] = solve_fit[c] / max(1.0, float(np.sum((pp / p_bar) ** 2)))
    total = 0.0
    detail = []
    for method, c in sweeps:
        if method == "lsar":
            est = res_sweep + p_bar * (t_upd + samp[c]) + solve_fit[c]
        else:
            upc = up["t0"]
            if c > up["c0"]:
                upc += depth(c, w) * max(0.0, qr_pbar[c] - qr_pbar[c] * up["c0"] / c)
            est = upc + p_bar * samp[c] + solve_fit[c]
        total += est
        detail.append({"method": method, "c": c, "sweep_s": est})
    desc = (f"oracle port, 1 thread, bounded sample extrapolated per part: residual pass and "
            f"leverage/draws on a {wp}-row prefix at p in {P1} (scaled by rows), gather+CPQR on "
            f"min(c,{c_cap}) rows at p in {P2} (scaled by c), RH upfront at c={c_cap} on "
            f"{rh_rows // 2}/{rh_rows}-row prefixes (linear in rows; + level CPQR for larger c)")
    return total, detail, desc


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    y, _, p_bar, cs = gen.make_config_series(args.config, seed=SEED, n=args.n)
    n = y.size
    eng = tf.Engine(local)
    series = tf.TimeSeries(y)
    eng.upload(series)
    sweeps = sweeps_for(cs)
    ro_sweep = p_bar * (n - p_bar)
    ro_step = ro_sweep * len(sweeps)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB > L2

    # one context (device buffers + stream) per sweep: the four sweeps of a step
    # are independent fits and run concurrently, each on its own
    # stream; the step's device time is the span from the earliest sweep start
    # to the latest sweep end (CUDA events, tf_sweep_span)
    engs = [eng] + [tf.Engine(local) for _ in sweeps[1:]]
    for e in engs:
        e.upload(series)

    def run_sweep(k, seed0, want_diag, fits, ser):
        method, c = sweeps[k]
        if method == "lsar":
            fits[k] = tf.lsar_fit(ser, p_bar, c, seed0 + k, engine=engs[k], want_diag=want_diag)
        else:
            fits[k] = tf.rh_fit(ser, p_bar, c, None, seed0 + k, engine=engs[k], want_diag=want_diag)

    def one_step(seed0, want_diag=False, concurrent=not args.sequential, ser=None):
        ser = ser or series
        fits = [None] * len(sweeps)
        if concurrent:
            th = [threading.Thread(target=run_sweep, args=(k, seed0, want_diag, fits, ser))
                  for k in range(len(sweeps))]
            for t in th:
                t.start()
            for t in th:
                t.join()
        else:
            for k in range(len(sweeps)):
                run_sweep(k, seed0, want_diag, fits, ser)
        if any(f is None for f in fits):
            raise RuntimeError("a sweep failed")
        spans = [e.sweep_span(engs[0]) for e in engs]
        if concurrent:
            dev = (max(b for _, b in spans) - min(a for a, _ in spans)) * 1e-3
        else:
            dev = sum(b - a for a, b in spans) * 1e-3
        diags, launches = [], 0
        for k, f in enumerate(fits):
            if want_diag and f.diag is not None:
                diags.append((sweeps[k][0], sweeps[k][1], f.diag))
                launches += int(f.diag["launches"][0]) if "launches" in f.diag else 0
        return dev, diags, launches

    for w in range(args.warmup):
        flush.fill_(float(w))
        one_step(100 + 10 * w)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    dev_times = []
    with ClockSampler(local) as clk:
        wall0 = time.time()
        for s in range(args.steps):
            flush.fill_(float(s))
            torch.cuda.synchronize()
            d, _, _ = one_step(1000 + 10 * s)
            dev_times.append(d)
        torch.cuda.synchronize()
        wall = time.time() - wall0
    T = float(sum(dev_times))
    if dist:
        t = torch.tensor([T], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        T = float(t.item())
    value = world * args.steps * ro_step / T

    if args.profile_step:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        one_step(7000)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()

    # ---- instrumented step (sweeps one after another, so per-kernel event
    #      times are the kernels' own): phases, launches, roofline of the pass ----
    _, diags, launches = one_step(5000, want_diag=True, concurrent=False)
    fp64_peak = eng.probe_fp64_peak()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    w_rows = n - p_bar
    t_pass = 0.0
    bytes_alg = 0.0
    flops_alg = 0.0
    t_roof = 0.0
    n_pass = 0
    phase_tot = np.zeros(3)
    for method, c, dg in diags:
        if method != "lsar" or "phases" not in dg:
            continue
        ph = dg["phases"]
        phase_tot += ph.sum(0)
        for p in range(1, p_bar + 1):
            tp = float(ph[p - 1, 2])
            b = 24.0 * w_rows                # read y, read s_p, write s_{p+1}
            f = (2.0 * p + 4.0) * w_rows     # p FMAs + square, scale, add, reduce
            t_pass += tp
            bytes_alg += b
            flops_alg += f
            t_roof += max(b / (hbm_peak * 1e9), f / (fp64_peak * 1e12))
            n_pass += 1
    traffic = None
    tp_path = os.path.join(ROOT, "profiles", "ncu_pass_traffic.json")
    if os.path.exists(tp_path):
        try:
            tj = json.load(open(tp_path))
            if tj.get("n") == n and tj.get("p_bar") == p_bar:
                traffic = tj.get("dram_bytes_per_launch_avg")
        except Exception:
            traffic = None
    # The sweep's roofline time is dominated by the fp64 FIR (lags p >~ 60 are
    # DMMA-bound, the rest HBM-bound): the headline bound is the fp64 tensor
    # pipe; the HBM view and the per-lag max(HBM, fp64) composite sit beside it.
    fp64_ach = flops_alg / t_pass / 1e12 if t_pass > 0 else None
    hbm_ach = bytes_alg / t_pass / 1e9 if t_pass > 0 else None
    roofline = {
        "kernel": "k_lsar_pass_pst (fused FIR residual on fp64 tensor cores + leverage update + CDF partials)",
        "bound": "tensor",
        "achieved": fp64_ach,
        "peak": fp64_peak,
        "unit": "TFLOP/s",
        "frac": (fp64_ach / fp64_peak) if fp64_ach else None,
        "traffic": traffic,
        "peak_source": "fp64 DFMA/DMMA peak measured in this run (tf_probe_fp64_peak; MEASURED_PEAKS.json "
                       "and B200_PROFILING.md state no fp64 figure)",
        "algorithmic_per_row": "2p+4 flop and 24 B per row per lag (y, s in, s out)",
        "hbm_achieved_gbs": hbm_ach,
        "hbm_peak_gbs": hbm_peak,
        "hbm_frac": (hbm_ach / hbm_peak) if hbm_ach else None,
        "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
        "sweep_roofline_frac": (t_roof / t_pass) if t_pass > 0 else None,
        "sweep_roofline_note": "sum over lags of max(24 B/row at hbm peak, (2p+4) flop/row at fp64 peak) / "
                               "sum of measured pass times",
        "pass_ms_per_lsar_sweep": 1e3 * t_pass / max(1, sum(1 for d in diags if d[0] == "lsar")),
        "phase_ms_lsar": {"sample": 1e3 * phase_tot[0], "solve": 1e3 * phase_tot[1],
                          "pass": 1e3 * phase_tot[2]},
    }

    # ---- e2e: public API with host buffers, H2D upload + sweeps + D2H inside the timer ----
    e2e_steps = max(1, min(args.steps, 3))
    pinned = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pinned[:] = y
    h2d = 8 * n * len(engs)  # every context uploads the series from the pinned host buffer
    d2h = 8 * len(sweeps) * (p_bar + p_bar * (p_bar + 1) // 2 + p_bar)  # taus, coefs, lag times
    torch.cuda.synchronize()
    t0 = time.time()
    for s in range(e2e_steps):
        fresh = tf.TimeSeries(pinned, copy=False)  # pinned host buffer; each context uploads it (H2D)
        one_step(7000 + 10 * s, ser=fresh)
    torch.cuda.synchronize()
    t_e2e = (time.time() - t0) / e2e_steps
    if dist:
        t = torch.tensor([t_e2e], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e = {"value": world * ro_step / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t0 = time.time()
        est, detail, desc = cpu_sweep_estimate(y, p_bar, sweeps)
        cpu = {"value": ro_step / est, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{desc}; wall {time.time() - t0:.1f}s", "sweeps": detail}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": n, "p_max": p_bar, "sweeps": [f"{m}:s={c}" for m, c in sweeps],
                   "rows_orders_per_step": ro_step, "parallelism": f"replicas x{world}",
                   "l2": "flushed between steps (256 MiB write); series 80 MB + 2 x 80 MB state > L2",
                   "timing": ("device time: CUDA events (span from the earliest sweep start to the latest "
                              "sweep end; the four sweeps run concurrently, one context and stream each)"
                              if not args.sequential else
                              "device time: CUDA events around each sweep, sweeps one after another"),
                   "roofline_timing": "k_lsar_pass_pst per-launch CUDA events in an instrumented step "
                                      "with the sweeps run one after another"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches) * args.steps if launches else None,
        "clocks": clk.summary(), "wall_s_timed_region": wall,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


_REF_Y = None
_REF_PBAR = 0


def _ref_sweep_worker(sweep):
    est, detail, desc = cpu_sweep_estimate(_REF_Y, _REF_PBAR, [sweep])
    return est, detail, desc


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2112_12994_b200 import gen
    y, _, p_bar, cs = gen.make_config_series(args.config, seed=SEED, n=args.n)
    n = y.size
    sweeps = sweeps_for(cs)
    ro_step = p_bar * (n - p_bar) * len(sweeps)
    # each step: the four sweeps are independent fits; the reference is
    # single-threaded, so with all host cores it runs them side by side, one
    # process each -- each process times the bounded per-part
    # sample of its sweep, and the step ends with the slowest sweep
    for _ in range(args.warmup):  # small warm-up (page-in, library load)
        cpu_sweep_estimate(y[: 20 * p_bar + 4000], p_bar, sweeps[:1], n_pass=10_000, c_cap=2 * p_bar,
                           rh_rows=4000)
    import multiprocessing as mp
    global _REF_Y, _REF_PBAR
    _REF_Y, _REF_PBAR = y, p_bar
    ctx = mp.get_context("fork")
    ncores = os.cpu_count() or 1
    procs = min(len(sweeps), ncores)
    ests, details = [], None
    t0 = time.time()
    with ctx.Pool(procs) as pool:
        for _ in range(max(1, args.steps)):
            res = pool.map(_ref_sweep_worker, sweeps)
            ests.append(max(r[0] for r in res))
            details = [r[1][0] for r in res]
            desc = res[0][2]
    wall = time.time() - t0
    est = float(np.median(ests))
    value = ro_step / est
    detail = details
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(ests),
        "warmup": args.warmup, "ms_per_step": 1e3 * est, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD, "n": n, "p_max": p_bar,
                   "sweeps": [f"{m}:s={c}" for m, c in sweeps], "rows_orders_per_step": ro_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": (f"oracle port of the reference (Eigen absent, reference not "
                                    f"buildable); the {len(sweeps)} sweeps run side by side, one "
                                    f"single-threaded process each on {procs} of {ncores} host cores; "
                                    f"step = slowest sweep; per sweep: {desc}; median of {len(ests)} "
                                    f"steps, wall {wall:.1f}s"),
                         "sweeps": detail},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
