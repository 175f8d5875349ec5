#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: fp64 matrix-free A.u GDoF/s vs roofline
for p = 1..16; Chebyshev-Jacobi step time).

Default (N=1): BASELINE config 2 (configs[1]) -- 16^3 deformed hexes, p = 8, mu = exp(3S),
u uniform in [-1,1] from seed 1.  One step = one A_D u apply + one degree-4 Chebyshev-Jacobi
application (b = 0, x0 = u, R16) = 5 operator applies.  `value` = N / (mean apply time) in GDoF/s.
Between timed steps the L2 is flushed: a 512 MB write, then a read of the same buffer, so the L2 holds
no data of the workload and no dirty flush lines are written back inside the timed region (the
write-only flush's write-back costs the config-2 apply ~3 us; that number is reported too).  Extra keys report the config-3 p-sweep,
config 4 (135 M dofs) and the config-5 p-MG preconditioned CG solve measured in the same run.

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
(N > 1 under torch.distributed.run: independent replicas, one per GPU -- DESIGN.md "replicas only").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1402_5938_b200 import inputs  # noqa: E402

METRIC = "fp64 matrix-free A.u GDoF/s (BASELINE config 2: 16^3 deformed hexes, p=8, mu=exp(3S))"
UNIT = "GDoF/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic(d):
    """apply bytes = 48 E n^3 (G) + 16 N (u read once, v written once);
    Chebyshev step bytes = 48 E n^3 + 40 N; apply flops = E (12 n^4 + 15 n^3)."""
    n = d["p"] + 1
    E = d["nex"] * d["ney"] * d["nez"]
    N = inputs.ndofs(d)
    return dict(N=N, E=E, n=n, apply_bytes=48 * E * n ** 3 + 16 * N, step_bytes=48 * E * n ** 3 + 40 * N,
                apply_flops=E * (12 * n ** 4 + 15 * n ** 3))


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", "sfmg_clocks_%d.csv" % os.getpid())

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            t0 = time.time()   # wait for the first sample so the timed region is covered
            while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(rows), "reasons": reasons}


def fp64_peak():
    """FP64 vector (DFMA) peak measured on this GPU by tools/fp64_peak; None if unavailable."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    try:
        if not os.path.exists(exe):
            from paper_1402_5938_b200 import _build
            _build.build_tools()
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout.strip().splitlines()
        return json.loads(out[-1])
    except Exception as ex:  # measurement tool only; the bench line does not depend on it
        return {"error": str(ex)[:200]}


# ------------------------------------------------------------------------------------------ multi-rank
def reduce_max(x: float, world: int, device) -> float:
    """Max over ranks of a per-rank time (the contract's max-over-ranks timing); identity at N=1."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(n_dofs: int, world: int, t_max: float) -> float:
    """Whole-job throughput of `world` independent replicas (weak scaling): all dofs / slowest rank."""
    return world * n_dofs / t_max / 1e9


# ------------------------------------------------------------------------------------------ oracle (CPU)
def cpu_model():
    """Host CPU model name (lscpu) reported beside every oracle time."""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_config5_solve():
    """Config-5 p-MG PCG solve on the oracle (O3 sum-factorised tier, as it stands), measured end to end:
    hierarchy setup (geometry, diagonals, 10 power iterations per level) and the whole solve."""
    import oracle
    oracle.build()
    d = inputs.CONFIG5
    t0 = time.perf_counter()
    H = oracle.Hier(d["nex"], d["ney"], d["nez"], d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0),
                    d.get("c0", 1.0), d.get("c1", 0.0))
    t1 = time.perf_counter()
    b = H.levels[0].load_vector(1)
    r = H.solve(b, mode=1, rtol=1e-8, maxit=200)
    t2 = time.perf_counter()
    return {"solve_ms": (t2 - t1) * 1e3, "setup_s": t1 - t0, "pcg_iterations": r["iterations"],
            "converged": r["converged"], "cores": oracle.get_threads(), "cpu": cpu_model(), "kind": "oracle",
            "sample": "whole config-5 MG-PCG solve to 1e-8 (O3 tier), measured"}


def oracle_cheb_sample(d, seed, ne=4):
    """The oracle's degree-4 Chebyshev application (O2 direct-quadrature applies, as it stands) on a
    bounded sample: the workload's order, warp and coefficient on ne^3 elements; GDoF/s per step =
    sample dofs / (time / 4)."""
    import oracle
    oracle.build()
    L = oracle.Level(ne, ne, ne, d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0), d.get("c0", 1.0),
                     d.get("c1", 0.0), eager=True, geom_tier=2, tier=2)
    u = inputs.uniform_pm1(seed, L.N)
    lam = L.lambda_max(10, inputs.POWER_SEED)
    L.cheb(np.zeros(L.N), u, 4, 0.1 * lam, 1.1 * lam)
    t0 = time.perf_counter()
    L.cheb(np.zeros(L.N), u, 4, 0.1 * lam, 1.1 * lam)
    dt = time.perf_counter() - t0
    return {"value": L.N / (dt / 4) / 1e9, "unit": UNIT, "cores": oracle.get_threads(), "cpu": cpu_model(),
            "kind": "oracle", "sample": "degree-4 Chebyshev (O2 applies) on %d^3 elements at p=%d, N=%d" % (
                ne, d["p"], L.N)}


def oracle_apply_sample(d, seed, target_s=10.0):
    """Time the oracle's O2 direct-quadrature apply (as it stands) over a bounded, evenly spaced sample
    of the workload's elements with geometric factors precomputed; returns GDoF/s-equivalent
    (N/E dofs per element), cores used and a description of the sample."""
    import oracle
    oracle.build()
    L = oracle.Level(d["nex"], d["ney"], d["nez"], d["p"], d.get("warp", 0), d.get("amp", 0.0), d.get("coeff", 0),
                     d.get("c0", 1.0), d.get("c1", 0.0), eager=False, geom_tier=2, tier=2)
    u = inputs.uniform_pm1(seed, L.N)
    ne = 16
    while True:     # grow the sample until one pass costs ~target_s / 4 wall seconds
        el = (np.arange(ne, dtype=np.int64) * max(1, L.E // ne)) % L.E
        L.cache_elements(el)
        t0 = time.perf_counter()
        L.apply_elements(u, el, tier=2)
        dt = time.perf_counter() - t0
        if dt > target_s / 4 or ne >= L.E:
            break
        ne = min(L.E, ne * 4)
    reps, tot = 0, 0.0
    while tot < target_s * 0.75 and reps < 50:
        t0 = time.perf_counter()
        L.apply_elements(u, el, tier=2)
        tot += time.perf_counter() - t0
        reps += 1
    per_elem = tot / reps / ne
    gdofs = (L.N / L.E) / per_elem / 1e9
    return gdofs, oracle.get_threads(), ("O2 apply over %d of %d elements (evenly spaced), %d reps, G precomputed; "
                                         "GDoF/s scaled by N/E dofs per element" % (ne, L.E, reps))


def run_reference(args, rank, world):
    """--impl reference: the oracle as the reference arm (tier: no reference implementation exists)."""
    if rank != 0:
        return 0
    d = inputs.CONFIG2
    import oracle
    oracle.build()
    L = oracle.Level(d["nex"], d["ney"], d["nez"], d["p"], d["warp"], d["amp"], d["coeff"], d["c0"], d["c1"],
                     eager=False, geom_tier=2, tier=2)
    u = inputs.uniform_pm1(1, L.N)
    ne = 64
    el = (np.arange(ne, dtype=np.int64) * (L.E // ne)) % L.E
    L.cache_elements(el)
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        L.apply_elements(u, el, tier=2)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
    per_step = sum(times) / len(times)
    value = (L.N / L.E) * ne / per_step / 1e9
    sample = "per step: O2 apply over %d of %d config-2 elements, G precomputed; GDoF/s scaled by N/E" % (ne, L.E)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "BASELINE config 2 (16^3 deformed hexes, p=8, mu=exp(3S), seed 1)",
                      "sample": sample},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ GPU arm
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    from paper_1402_5938_b200 import sfmg

    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream()
    hbm_peak, peak_kind = peaks()
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return reduce_max(x, world, dev)

    # ---------------- main workload: config 2
    d = inputs.CONFIG2
    alg = algorithmic(d)
    lv = sfmg.Level(sfmg.Problem.from_dict(d), device=dev)
    N = lv.N
    u_host = torch.from_numpy(inputs.uniform_pm1(inputs.SEEDS[2], N)).pin_memory()
    u = u_host.to(dev, non_blocking=True)
    v = torch.empty_like(u)
    b = torch.zeros_like(u)
    x = torch.empty_like(u)
    lam = lv.lambda_max(10, inputs.POWER_SEED)
    lo, hi = 0.1 * lam, 1.1 * lam
    launches_per_step = 2 + 9         # apply: init + element kernel; cheb(4): init + 4 element + 4 update

    def step(ev):
        ev[0].record(stream)
        lv.apply(u, v)
        ev[1].record(stream)
        x.copy_(u)
        ev[2].record(stream)
        lv.cheb(b, x, 4, lo, hi)
        ev[3].record(stream)

    for _ in range(max(3, args.warmup)):
        step([torch.cuda.Event(enable_timing=True) for _ in range(4)])
    barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            l2_flush(flush, k)              # L2 flush between timed steps (not in the step time)
            step(evs[k])
        t_end.record(stream)
        barrier()
    t_apply = sum(e[0].elapsed_time(e[1]) for e in evs) * 1e-3 / args.steps
    t_cheb = sum(e[2].elapsed_time(e[3]) for e in evs) * 1e-3 / args.steps
    t_step = sum(e[0].elapsed_time(e[3]) - e[1].elapsed_time(e[2]) for e in evs) * 1e-3 / args.steps
    t_apply, t_cheb, t_step = (max_over_ranks(t_apply), max_over_ranks(t_cheb), max_over_ranks(t_step))
    value = replica_value(N, world, t_apply)

    # ---------------- dominant kernel: the element (operator) kernel k_apply_v4<8>, timed by the
    # library with CUDA events around each of its launches on the launching stream (separate pass:
    # the events stop the kernel from overlapping its predecessor)
    lv.profile(True)
    kreps = max(3, min(args.steps, 50))
    for k in range(kreps):   # one element-kernel launch per L2 flush: every timed launch is cold
        l2_flush(flush, k)
        lv.apply(u, v)
    torch.cuda.synchronize()
    k_ms, k_launches = lv.profile_read(reset=True)
    lv.profile(False)
    t_kernel = max_over_ranks(k_ms * 1e-3 / k_launches)
    traffic, traffic_src = None, None
    for tf in ("r02_traffic.json", "r01_traffic.json"):   # dram read + write bytes per launch of this kernel
        try:                                                 # from the committed ncu --set full capture
            with open(os.path.join(ROOT, "profiles", tf)) as fh:
                tj = json.load(fh)
            traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
            traffic_src = "profiles/%s (ncu --set full, dram__bytes_read.sum + write.sum)" % tf
            break
        except Exception:
            pass
    roof = {"bound": "hbm", "achieved": alg["apply_bytes"] / t_kernel / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": alg["apply_bytes"] / t_kernel / 1e9 / hbm_peak, "traffic": traffic,
            "traffic_source": traffic_src,
            "kernel": "k_apply_v4<8,DIR,GS> element kernel (%d launches, each right after an L2 flush, %.2f us mean)"
                      % (k_launches, t_kernel * 1e6),
            "peak_kind": peak_kind, "algorithmic_bytes_per_launch": alg["apply_bytes"],
            "abi_apply_us": t_apply * 1e6, "abi_apply_frac": alg["apply_bytes"] / t_apply / 1e9 / hbm_peak}

    # the same ABI apply after a write-only flush (the flush's dirty lines are written back inside the
    # timed region): reported next to `value` for transparency
    t_apply_dirty = max_over_ranks(time_events(lambda: lv.apply(u, v), stream, None, 20, warm=3,
                                               flush_fn=lambda k: l2_flush(flush, k, read=False)))

    # ---------------- end to end through the host-buffer ABI (pinned host in, host out)
    v_host = torch.empty(N, dtype=torch.float64).pin_memory()
    un, vn = u_host.numpy(), v_host.numpy()
    for _ in range(3):
        lv.apply_host(un, vn)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(e2e_steps):
        lv.apply_host(un, vn)
    t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e = {"value": world * N / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
           "call": "sfmg_apply_host (pinned host u -> device -> A_D u -> host), wall clock per call (syncs)"}

    extras = {}
    if not args.quick:
        extras = run_extras(args, sfmg, dev, stream, flush, hbm_peak)

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "BASELINE config 2: 16^3 deformed hexes (x+0.1 sin sin sin), p=8, "
                                  "mu=exp(3 sin2pix sin2piy sin2piz), N=129^3, u~U[-1,1] seed 1; step = A_D u + "
                                  "one degree-4 Chebyshev-Jacobi application (b=0, x0=u)",
                      "l2": "flushed between timed steps (512 MB write, then a read of it: clean lines)",
                      "parallelism": "replicas" if world > 1
                      else "single GPU"},
           "apply_ms": t_apply * 1e3, "apply_ms_write_only_flush": t_apply_dirty * 1e3, "cheb_step_ms": t_cheb / 4 * 1e3,
           "cheb_step_gdofs": world * N / (t_cheb / 4) / 1e9,
           "cheb_step_hbm_frac": alg["step_bytes"] / (t_cheb / 4) / 1e9 / hbm_peak,
           "apply_tflops": alg["apply_flops"] / t_apply / 1e12,
           "roofline": roof, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
           "clocks": clk.summary()}
    out.update(extras)
    cpu_extra = {}
    if rank == 0 and world == 1 and not args.no_cpu:
        gd, cores, sample = oracle_apply_sample(d, inputs.SEEDS[2])
        out["cpu_baseline"] = {"value": gd, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                               "cpu": cpu_model()}
        if not args.quick:   # the oracle also at T=1, its Chebyshev step, configs 3-5
            import oracle
            oracle.set_threads(1)
            g1, c1, s1 = oracle_apply_sample(d, inputs.SEEDS[2], target_s=4.0)
            oracle.set_threads(cores)
            cpu_extra["cpu_baseline_t1"] = {"value": g1, "unit": UNIT, "cores": c1, "kind": "oracle", "sample": s1}
            cpu_extra["cpu_baseline_cheb_step"] = oracle_cheb_sample(d, inputs.SEEDS[2])
            cpu_extra["cpu_baseline_config3"] = {}
            for p in (1, 2, 4, 8, 16):
                gp, cp_, sp = oracle_apply_sample(inputs.CONFIG3[p], inputs.SEEDS[3], target_s=3.0)
                cpu_extra["cpu_baseline_config3"]["p%d" % p] = {"value": gp, "unit": UNIT, "cores": cp_, "sample": sp}
            g4, c4, s4 = oracle_apply_sample(inputs.CONFIG4, inputs.SEEDS[4], target_s=3.0)
            cpu_extra["cpu_baseline_config4"] = {"value": g4, "unit": UNIT, "cores": c4, "kind": "oracle", "sample": s4}
            cpu_extra["cpu_baseline_config5"] = oracle_config5_solve()
    if rank == 0:
        # key order: the contract keys, the CPU baselines, the detailed extras, and last the compact
        # config-3 p-sweep (the metric's p = 1..16 roofline fractions), so a stdout tail keeps it
        sweep = out.pop("sweep_config3", None)
        final = dict(out)
        final.update(cpu_extra)
        if sweep is not None:
            final["sweep_config3"] = sweep
            final["sweep_frac"] = {"p%d" % r["p"]: {"apply": round(r["apply_hbm_frac"], 3),
                                                    "kernel": round(r["apply_kernel_hbm_frac"], 3),
                                                    "cheb_step": round(r["cheb_step_hbm_frac"], 3)} for r in sweep}
        print(json.dumps(final), flush=True)


def l2_flush(flush, k, read=True):
    """Evict the workload from L2 between timed steps: write a buffer larger than L2, then read it
    back so the lines left in L2 are clean (no write-back of flush data inside the timed region)."""
    flush.fill_(float(k))
    if read:
        flush.sum()


def time_events(fn, stream, flush, reps, warm=3, flush_fn=None):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for k in range(reps):
        if flush_fn is not None:
            flush_fn(k)
        elif flush is not None:
            l2_flush(flush, k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def run_extras(args, sfmg, dev, stream, flush, hbm_peak):
    import torch
    out = {}
    pk = fp64_peak()
    out["fp64_peak"] = pk
    fp64_tf = pk.get("fp64_dfma_tflops") if isinstance(pk, dict) else None
    sweep = []
    for p in (1, 2, 4, 8, 16):
        d = inputs.CONFIG3[p]
        alg = algorithmic(d)
        lv = sfmg.Level(sfmg.Problem.from_dict(d), device=dev)
        u = torch.from_numpy(inputs.uniform_pm1(inputs.SEEDS[3], lv.N)).to(dev)
        v, b, x = torch.empty_like(u), torch.zeros_like(u), u.clone()
        lam = lv.lambda_max(10, inputs.POWER_SEED)
        ta = time_events(lambda: lv.apply(u, v), stream, flush, 20)
        tw = time_events(lambda: lv.apply(u, v), stream, None, 20)
        tc = time_events(lambda: lv.cheb(b, x, 4, 0.1 * lam, 1.1 * lam), stream, flush, 10) / 4
        # the element kernel alone (library events around each launch, L2 flushed between applies)
        lv.profile(True)
        for k in range(10):
            l2_flush(flush, k)
            lv.apply(u, v)
        torch.cuda.synchronize()
        k_ms, k_n = lv.profile_read(reset=True)
        lv.profile(False)
        tk = k_ms * 1e-3 / max(k_n, 1)
        sweep.append({"p": p, "ne": d["nex"], "apply_us": ta * 1e6, "apply_gdofs": lv.N / ta / 1e9,
                      "apply_kernel_us": tk * 1e6, "apply_kernel_hbm_frac": alg["apply_bytes"] / tk / 1e9 / hbm_peak,
                      "apply_hbm_frac": alg["apply_bytes"] / ta / 1e9 / hbm_peak,
                      "apply_tflops": alg["apply_flops"] / ta / 1e12,
                      "apply_fp64_frac": (alg["apply_flops"] / ta / 1e12 / fp64_tf) if fp64_tf else None,
                      "apply_warm_us": tw * 1e6, "apply_warm_gdofs": lv.N / tw / 1e9,
                      "cheb_step_us": tc * 1e6, "cheb_step_gdofs": lv.N / tc / 1e9,
                      "cheb_step_hbm_frac": alg["step_bytes"] / tc / 1e9 / hbm_peak})
        del lv, u, v, b, x
    out["sweep_config3"] = sweep
    if not args.no_config4:
        d = inputs.CONFIG4
        alg = algorithmic(d)
        lv = sfmg.Level(sfmg.Problem.from_dict(d), device=dev)
        u = torch.from_numpy(inputs.uniform_pm1(inputs.SEEDS[4], lv.N)).to(dev)
        v, b, x = torch.empty_like(u), torch.zeros_like(u), u.clone()
        lam = lv.lambda_max(10, inputs.POWER_SEED)
        ta = time_events(lambda: lv.apply(u, v), stream, flush, 10)
        tc = time_events(lambda: lv.cheb(b, x, 4, 0.1 * lam, 1.1 * lam), stream, flush, 5) / 4
        out["config4"] = {"N": lv.N, "apply_ms": ta * 1e3, "apply_gdofs": lv.N / ta / 1e9,
                          "apply_hbm_frac": alg["apply_bytes"] / ta / 1e9 / hbm_peak,
                          "cheb_step_ms": tc * 1e3, "cheb_step_gdofs": lv.N / tc / 1e9,
                          "cheb_step_hbm_frac": alg["step_bytes"] / tc / 1e9 / hbm_peak}
        del lv, u, v, b, x
        torch.cuda.empty_cache()
        if int(os.environ.get("WORLD_SIZE", "1")) == 1:
            out["config4"]["fused_step_opt_in"] = fused_config4()
    # config 5: p-MG 16 -> 1, V(2,2) degree-4 Chebyshev, coarse CG 1e-10, PCG to 1e-8
    d = inputs.CONFIG5
    t0 = time.perf_counter()
    H = sfmg.Hierarchy(sfmg.Problem.from_dict(d), sfmg.MgParams(), device=dev)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    bvec = H.levels[0].load_vector(1)
    H.solve(bvec, mode=1, rtol=1e-8)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    xs, rep = H.solve(bvec, mode=1, rtol=1e-8)
    e.record(stream)
    e.synchronize()
    t_solve = a.elapsed_time(e) * 1e-3
    tv = time_events(lambda: H.vcycle(bvec, xs), stream, flush, 5, warm=1)
    out["config5_pmg_pcg"] = {"N": H.N, "levels": H.nlevels, "setup_s": t_setup, "pcg_iterations": rep["iterations"],
                              "converged": rep["converged"], "rel_residual": rep["r_norm"] / rep["r0_norm"],
                              "solve_ms": t_solve * 1e3, "vcycle_ms": tv * 1e3, "fine_applies": rep["fine_applies"]}
    del H
    # NEXT-1: the paper's own settings on its 3d-const problem (8^3, p = 16, unit cube, mu = 1):
    # Jacobi(3,3) / Cheb(3,3) on [lambda/4, lambda] (10 Arnoldi), p -> 1 then 8^3 -> 4^3 -> 2^3
    d = inputs.problem(8, 16)
    nx = {}
    for sm in ("jacobi", "cheb"):
        H = sfmg.Hierarchy(sfmg.Problem.from_dict(d), sfmg.MgParams.paper(sm, h_levels=2), device=dev)
        bvec = H.levels[0].load_vector(1)
        for mode, mname in ((0, "mg_solver"), (1, "pcg")):
            H.solve(bvec, mode=mode, rtol=1e-8, max_iter=300)
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, rep = H.solve(bvec, mode=mode, rtol=1e-8, max_iter=300)
            e.record(stream)
            e.synchronize()
            nx["%s_%s33" % (mname, sm)] = {"iterations": rep["iterations"], "converged": rep["converged"],
                                            "solve_ms": a.elapsed_time(e), "fine_applies": rep["fine_applies"]}
        del H
    out["next1_3dconst_p16_paper_settings"] = nx
    # NEXT-3: Gauss-Legendre quadrature variant of the apply (config-3 meshes)
    gq = []
    for p in (4, 8, 16):
        d = dict(inputs.CONFIG3[p], quadrature=1)
        alg = algorithmic(d)
        lv = sfmg.Level(sfmg.Problem.from_dict(d), device=dev)
        u = torch.from_numpy(inputs.uniform_pm1(inputs.SEEDS[3], lv.N)).to(dev)
        v = torch.empty_like(u)
        ta = time_events(lambda: lv.apply(u, v), stream, flush, 10)
        gq.append({"p": p, "apply_us": ta * 1e6, "apply_gdofs": lv.N / ta / 1e9,
                   "apply_hbm_frac": alg["apply_bytes"] / ta / 1e9 / hbm_peak})
        del lv, u, v
    out["next3_gauss_apply_config3"] = gq

    def timed_solve(prob, mg, mode):
        H = sfmg.Hierarchy(sfmg.Problem.from_dict(prob), mg, device=dev)
        bvec = H.levels[0].load_vector(1)
        H.solve(bvec, mode=mode, rtol=1e-8, max_iter=300)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _, rep = H.solve(bvec, mode=mode, rtol=1e-8, max_iter=300)
        e.record(stream)
        e.synchronize()
        r = {"N": H.N, "levels": H.nlevels, "iterations": rep["iterations"], "converged": rep["converged"],
             "solve_ms": a.elapsed_time(e)}
        del H
        return r
    # NEXT-4: high-order h-multigrid, tab:box / tab:3d-box settings (three meshes at the fine order),
    # Cheb(3,3) pCG, Gauss quadrature (the paper's) and collocated LGL
    out["next4_3dconst_hmg_pcg_cheb33"] = {
        "p%d_%s" % (p, "gauss" if q else "lgl"): timed_solve(dict(inputs.problem(8, p), quadrature=q),
                                                           sfmg.MgParams.paper_h("cheb", 2), 1)
        for p in (4, 8) for q in (1, 0)}
    # NEXT-2: 2d-const 32^2 (tab:box), p-multigrid and h-multigrid Cheb(3,3) pCG, Gauss quadrature
    out["next2_2dconst_pcg_cheb33"] = {
        "p%d_%s" % (p, name): timed_solve(dict(nex=32, ney=32, nez=1, p=p, dim=2, quadrature=1), mk("cheb", 2), 1)
        for p in (4, 16) for name, mk in (("pmg", sfmg.MgParams.paper), ("hmg", sfmg.MgParams.paper_h))}
    return out


def fused_config4():
    """The opt-in fused Chebyshev step / apply (one persistent kernel per step, y in an L2-resident plane
    ring) on config 4, timed by tools/quick_bench.py in a subprocess: the library reads
    SFMG_FUSED once per process."""
    import subprocess
    env = dict(os.environ, SFMG_FUSED="1", SFMG_L2_PERSIST_MB="64")
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_bench.py"), "4"], env=env,
                           capture_output=True, text=True, timeout=600)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
        return {"apply_ms": d["t_apply_us"] * 1e-3, "apply_hbm_frac": d["frac_hbm_apply"],
                "cheb_step_ms": d["t_step_us"] * 1e-3, "cheb_step_hbm_frac": d["frac_hbm_step"],
                "env": "SFMG_FUSED=1 SFMG_L2_PERSIST_MB=64", "timer": "tools/quick_bench.py (CUDA events, L2 flushed)"}
    except Exception as ex:   # noqa: BLE001  (a measurement key, never the bench's result)
        return {"error": str(ex)[:200]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sfmg", choices=["sfmg", "reference"])
    ap.add_argument("--quick", action="store_true", help="main workload only (no sweep / config 4 / config 5)")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
