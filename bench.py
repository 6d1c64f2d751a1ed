#!/usr/bin/env python3
"""Benchmark of the B200 restarted-PDHG LP engine (contract in the task prompt;
workload choice and roofline arithmetic in DESIGN.md §6).

Headline workload (BASELINE.json metric "LPs solved/sec to 1e-4 KKT (batched)",
configs[1]): C2 = a batch of 1024 PyEPO-style 5x5 shortest-path LPs sharing K
with varying costs, raPDHG (headline; r2HPDHG reported as "secondary") to 1e-4
relative KKT.  One step = one pass of the
whole hot path: lp_create_batch (upload, validate, transpose, precondition),
lp_solve_batch (every instance to OPTIMAL), lp_get_solutions, lp_destroy.

  value : LPs/s with inputs resident in HBM (device pointers), per-step CUDA
          events on the solve stream, L2 flushed between steps, max over ranks.
  e2e   : the same through the C ABI with pinned HOST buffers: H2D of the
          problem + costs and D2H of every solution inside the timed region.
  --impl reference : the CPU oracle (oracle/) on the host cores, same metric.

Multi-GPU (torchrun): every rank solves its own batch (independent LPs, no
data-path collective) -> "scaling": "weak".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# NCCL's version banner would land on stdout next to the one JSON line rank 0 prints
os.environ.setdefault("NCCL_DEBUG", "WARN")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lpgen  # noqa: E402

METRIC = "LPs solved/sec to 1e-4 KKT (batched)"
UNIT = "LPs/s"
WORKLOAD = ("C2: batch of 1024 PyEPO-style 5x5 shortest-path LPs (40 arcs, 25 flow rows, shared K, "
            "varying c), to 1e-4 relative KKT, every instance OPTIMAL")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--alg", default="ra", choices=["r2", "ra"])
    ap.add_argument("--secondary-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the C4 whole-GPU leg")
    ap.add_argument("--large-m", type=int, default=100_000)
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (1e8 nnz) whole-GPU leg")
    ap.add_argument("--no-dense", action="store_true", help="skip the C3 shared-dense-K (DMMA) leg")
    ap.add_argument("--no-spo", action="store_true", help="skip the SPO+ (Warcraft-shaped) leg")
    ap.add_argument("--c5-sharded", action="store_true",
                    help="run the C5 leg on the row-sharded NCCL engine even at one rank (it is used for N > 1)")
    ap.add_argument("--no-c5-sharded", action="store_true",
                    help="at one rank, skip the sharded-engine C5 run that follows the grid-path C5 leg")
    ap.add_argument("--c5-axis", default="auto", choices=["rows", "cols", "auto"],
                    help="sharding axis of the C5 sharded leg; auto = the axis whose exchanged vector is "
                         "shorter (lp_shard_axis, DESIGN reading 33): columns for C5 (m < n)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def log(msg):
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------- clocks -----

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("BENCH_CLOCK_MS", "50")], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ workload -----

def make_workload(batch: int, seed: int):
    lp, C = lpgen.g_grid(batch=batch, seed=seed)
    return lp, C


def cpu_baseline(lp, C, alg, seconds):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    workload: whole-batch solves repeated until ~`seconds` of CPU time."""
    import oracle
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads)
    done, t0 = 0, time.perf_counter()
    reps = 0
    while True:
        _, _, res = oracle.solve_batch(lp, C, None, alg, threads=threads)
        assert all(r["status"] == oracle.OPTIMAL for r in res)
        done += len(res)
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{reps} x the full {len(C)}-LP C2 batch ({done} LPs, {dt:.1f} s wall)",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------ reference -----

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    lp, C = make_workload(args.batch, seed=2)
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads)
    # bounded sample per step so that warmup + steps end within a few minutes
    t0 = time.perf_counter()
    oracle.solve_batch(lp, C[:64], None, args.alg, threads=threads)
    per_lp = (time.perf_counter() - t0) / 64
    budget = 150.0 / max(args.steps + args.warmup, 1)
    sample = int(max(8, min(args.batch, budget / max(per_lp, 1e-9))))
    for w in range(args.warmup):
        oracle.solve_batch(lp, C[:sample], None, args.alg, threads=threads)
    times = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        _, _, res = oracle.solve_batch(lp, C[:sample], None, args.alg, threads=threads)
        times.append(time.perf_counter() - t0)
        assert all(r["status"] == oracle.OPTIMAL for r in res)
    total = sum(times)
    value = sample * args.steps / total
    desc = f"{sample} of the {args.batch} C2 instances per step, oracle solve_batch on {threads} threads"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "batch": args.batch, "sample_per_step": sample,
                       "algorithm": "r2hpdhg" if args.alg == "r2" else "rapdhg", "eps": 1e-4},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- ours -----

def run_ours(args):
    import torch
    import paper_2412_09734_b200 as mp

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    lp, C = make_workload(args.batch, seed=2 + rank)
    prob_h = mp.Problem.from_lp(lp)
    prob_d = prob_h.to(dev)
    C_d = torch.as_tensor(C, device=dev)
    # pinned host copies for the end-to-end leg
    pin = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).pin_memory()
    prob_p = mp.Problem(lp.n, lp.m1, lp.m2, pin(lp.row_ptr, torch.int64), pin(lp.col_idx, torch.int32),
                        pin(lp.val, torch.float64), pin(lp.c, torch.float64), pin(lp.q, torch.float64),
                        pin(lp.l, torch.float64), pin(lp.u, torch.float64))
    C_p = pin(C, torch.float64)
    X_p = torch.empty((args.batch, lp.n), dtype=torch.float64).pin_memory()
    Y_p = torch.empty((args.batch, lp.m), dtype=torch.float64).pin_memory()
    X_d = torch.empty((args.batch, lp.n), dtype=torch.float64, device=dev)
    Y_d = torch.empty((args.batch, lp.m), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    def step(prob, Cx, X, Y, mem, alg=args.alg, rule="adaptive", rho=1.0, opts=None):
        bs = mp.BatchSolver(prob, Cx)
        # iteration_limit: safety net; every instance must be OPTIMAL
        res = bs.solve(algorithm=alg, iteration_limit=200_000, step_rule=rule, reflection=rho, **(opts or {}))
        bs.solutions(memory=mem, X=X, Y=Y)
        bs.close()
        return res

    def timed(prob, Cx, X, Y, mem, steps, collect, alg=args.alg, rule="adaptive", rho=1.0, opts=None):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        # per step, after its end event: every instance's status and the library's solve time;
        # the last step's full results (no step's result array is retained past the next step)
        summary = {"all_optimal": True, "solve_s": [], "last": None}
        for s in range(steps):
            flush.zero_()                       # evict L2 between steps (outside the event pair)
            ev[s][0].record(stream)
            res = step(prob, Cx, X, Y, mem, alg, rule, rho, opts)
            ev[s][1].record(stream)
            if collect:
                summary["all_optimal"] &= bool(np.all(res["status"] == mp.LP_OPTIMAL))
                summary["solve_s"].append(float(res["solve_seconds"][0]))
                summary["last"] = res
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev), summary

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    log("warm-up")
    for _ in range(max(args.warmup, 3)):
        step(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE)
        step(prob_p, C_p, X_p, Y_p, mp.LP_HOST)
    # ---- device-resident timed region ----
    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                           if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit() else local)
    barrier()
    sampler.start()
    n0 = mp.launch_count()
    barrier()
    log("timed region (device-resident)")
    ms, results = timed(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE, args.steps, True)
    barrier()
    launches = mp.launch_count() - n0
    clocks = sampler.stop()
    # ---- end-to-end timed region (host buffers through the C ABI) ----
    barrier()
    log("timed region (end to end)")
    ms_e2e, _ = timed(prob_p, C_p, X_p, Y_p, mp.LP_HOST, args.steps, False)
    barrier()
    # ---- secondary: the other algorithm on the same workload (context, not the headline) ----
    alg2 = "r2" if args.alg == "ra" else "ra"
    log("secondary algorithm")
    step(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE, alg2)
    barrier()
    ms2, res2 = timed(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE, args.secondary_steps, True, alg2)
    barrier()
    # ---- constant-step variants (reading 34), same workload ----
    log("constant-step variants")
    var_ms, var_res = {}, {}
    # (name, algorithm, step rule, reflection, options): SURVEY §8(f) rows 2 and 4, DESIGN.md
    # readings 34, 36 and 38
    POLISH = {"feasibility_polishing": 1}
    VARIANTS = (("r2hpdhg_constant_step", "r2", "constant", 1.0, None),
                ("rapdhg_constant_step", "ra", "constant", 1.0, None),
                ("r2hpdhg_partial_reflection_0.8", "r2", "adaptive", 0.8, None),
                ("rapdhg_feasibility_polishing", "ra", "adaptive", 1.0, POLISH))
    for name, va, rule, rho, opts in VARIANTS:
        step(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE, va, rule, rho, opts)
        barrier()
        var_ms[name], var_res[name] = timed(prob_d, C_d, X_d, Y_d, mp.LP_DEVICE, args.secondary_steps, True, va,
                                            rule, rho, opts)
        barrier()
    t = torch.tensor([ms, ms_e2e, ms2] + [var_ms[v[0]] for v in VARIANTS], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, ms_e2e, ms2 = float(t[0]), float(t[1]), float(t[2])
    var_ms = {v[0]: float(t[3 + i]) for i, v in enumerate(VARIANTS)}
    variants = {}
    for name, va, rule, rho, opts in VARIANTS:
        itv = np.asarray(var_res[name]["last"]["iterations"])
        variants[name] = {
            "algorithm": "r2hpdhg" if va == "r2" else "rapdhg", "step_rule": rule, "reflection": rho,
            "value": args.batch * args.secondary_steps * ws / (var_ms[name] * 1e-3), "unit": UNIT,
            "ms_per_step": var_ms[name] / args.secondary_steps,
            "all_optimal": var_res[name]["all_optimal"],
            "iterations": {"p50": float(np.median(itv)), "p99": float(np.percentile(itv, 99)), "max": int(itv.max())}}
        if rule == "constant":
            variants[name]["step"] = "eta = 0.998 / sigma_max(K~), 200 power iterations (inside the timed step)"
        if opts is POLISH:
            variants[name]["polished"] = int(np.sum(var_res[name]["last"]["polish"] == 1))
            variants[name]["polish"] = ("after the 1e-4 solve, primal (c = 0) and dual (q = 0) sub-solves to "
                                        "eps_feas_polish = 1e-6 on the same kernel (inside the timed step)")
    it2 = np.asarray(res2["last"]["iterations"])
    secondary = {"algorithm": "r2hpdhg" if alg2 == "r2" else "rapdhg",
                 "value": args.batch * args.secondary_steps * ws / (ms2 * 1e-3), "unit": UNIT,
                 "ms_per_step": ms2 / args.secondary_steps,
                 "all_optimal": res2["all_optimal"],
                 "iterations": {"p50": float(np.median(it2)), "p99": float(np.percentile(it2, 99)),
                                "max": int(it2.max())}}
    # correctness of every timed instance
    assert results["all_optimal"], "non-optimal instance in the timed region"
    lps = args.batch * args.steps * ws
    value = lps / (ms * 1e-3)
    e2e = lps / (ms_e2e * 1e-3)
    last = results["last"]
    iters = np.asarray(last["iterations"])
    atts = np.asarray(last["attempts"])
    kern_ms = statistics.mean(results["solve_s"]) * 1e3
    # roofline of the dominant kernel (the per-instance solver kernel): fp64 ALU bound
    nnz, n, m = lp.nnz, lp.n, lp.m
    flop_attempt = 4 * nnz + 25 * (n + m)          # SURVEY §8(d) d.2 per-attempt flops
    flops = float(atts.sum()) * flop_attempt
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp64_peak, peak_src = _fp64_peak("fp64_dfma_tflops", sm_max)
    achieved = flops / (kern_ms * 1e-3) / 1e12
    h2d = (lp.row_ptr.nbytes + lp.col_idx.nbytes + lp.val.nbytes + lp.c.nbytes + lp.q.nbytes + lp.l.nbytes +
           lp.u.nbytes + C.nbytes)
    d2h = X_p.numel() * 8 + Y_p.numel() * 8 + args.batch * 96
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "batch": args.batch, "algorithm": "r2hpdhg" if args.alg == "r2" else "rapdhg",
                   "eps": 1e-4, "l2": "flushed between steps (256 MiB write outside the event pair)",
                   "parallelism": f"instances x{ws} ranks (weak)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": ms_e2e / args.steps},
        "gpu_launches": int(launches),
        "roofline": {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": _traffic("tiny_kernel_c2", "bytes_per_launch"),
                     "traffic_source": "profiles/traffic.json (ncu --set full capture, per launch)",
                     "kernel": "tiny_kernel<raPDHG, adaptive, RPT=1, CPT=2, W=4, WT=2> (register-resident warp per LP)", "kernel_ms": kern_ms,
                     "flops_per_launch": flops,
                     "peak_source": peak_src,
                     "note": "per-instance solves are latency-bound, see DESIGN.md §6",
                     # the batch time is the slowest instance's attempts x one warp's attempt latency
                     "critical_path": {"attempts_slowest": int(atts.max()),
                                       "us_per_attempt": kern_ms * 1e3 / max(1, int(atts.max())),
                                       "cycles_per_attempt": kern_ms * 1e-3 / max(1, int(atts.max())) * sm_max * 1e6,
                                       "attempts_mean": float(atts.mean()),
                                       "alu_headroom": fp64_peak / achieved if achieved > 0 else None}},
        "iterations": {"p50": float(np.median(iters)), "p99": float(np.percentile(iters, 99)),
                       "max": int(iters.max()), "attempts_total": int(atts.sum())},
        "clocks": clocks,
        "secondary": secondary,
        "variants": variants,
    }
    if rank == 0:
        log("C1 leg (one small LP, r2HPDHG)")
        line["c1"] = c1_leg(mp, torch, dev)
    if not args.no_large:
        log("large-LP leg (C4)")
        line["large_lp"] = large_lp_leg(mp, torch, dev, stream, peaks, args, cpu=rank == 0 and not args.no_cpu_baseline)
    if not args.no_c5 and (ws > 1 or args.c5_sharded):
        log(f"large-LP leg (C5, 1e8 nnz), sharded over the ranks (NCCL, axis {args.c5_axis})")
        try:
            c5 = c5_sharded_leg(mp, torch, dev, ws, rank, args)
        except Exception as e:   # a context leg: its failure is recorded, the headline line still prints
            c5 = {"error": f"{type(e).__name__}: {e}"[:400]}
        if rank == 0:
            line["c5_sharded"] = c5
    elif not args.no_c5 and rank == 0:
        log("large-LP leg (C5, 1e8 nnz)")
        line["c5"] = large_lp_leg(mp, torch, dev, stream, peaks, args, m=5_000_000, seed=5, label="C5", reps=1,
                                  cpu=not args.no_cpu_baseline)
        if not args.no_c5_sharded:   # the multi-GPU engine on the same LP at one NCCL rank (context)
            log(f"large-LP leg (C5) on the sharded engine, one rank (axis {args.c5_axis})")
            try:
                line["c5_sharded"] = c5_sharded_leg(mp, torch, dev, 1, 0, args)
            except Exception as e:
                line["c5_sharded"] = {"error": f"{type(e).__name__}: {e}"[:400]}
    if not args.no_dense:
        log("dense shared-K leg (C3)")
        line["dense_batch"] = dense_leg(mp, torch, dev, peaks, args.no_cpu_baseline or rank != 0)
    if not args.no_spo and rank == 0:
        log("SPO+ leg (Warcraft-shaped batches)")
        line["spo"] = spo_leg(mp, torch, dev)
    if rank == 0:
        log("infeasibility-detection leg (mixed-status batch)")
        line["infeasibility"] = infeasibility_leg(mp, torch, dev)
    if rank == 0:
        log("batch-size scaling leg (C2 shape)")
        line["batch_scaling"] = batch_scaling_leg(mp, torch, dev)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        log("cpu baseline")
        line["cpu_baseline"] = cpu_baseline(lp, C, args.alg, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def spmv_pair_leg(mp, torch, dev, prob, lp, hbm, reps=20):
    """The SpMV pair alone (BASELINE metric "SpMV-pair GB/s vs HBM peak"): K~ v and K~' w with the
    library's standalone SpMV kernels (lp_spmv_scaled) on device-resident vectors; algorithmic
    B_pair = 24 nnz + 4(m+1) + 4(n+1) + 8n + 8m bytes per pair."""
    with mp.Solver(prob) as s:
        v = torch.rand(lp.n, dtype=torch.float64, device=dev)
        w = torch.rand(lp.m, dtype=torch.float64, device=dev)
        outs = (torch.empty(lp.m, dtype=torch.float64, device=dev), torch.empty(lp.n, dtype=torch.float64, device=dev))
        for _ in range(3):
            s.spmv_scaled(v, w, out=outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        for _ in range(reps):
            s.spmv_scaled(v, w, out=outs)
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        t_pair = e0.elapsed_time(e1) / reps * 1e-3
    b_pair = 24 * lp.nnz + 4 * (lp.m + 1) + 4 * (lp.n + 1) + 8 * lp.n + 8 * lp.m
    gf = gather_floor_us(lp.n, lp.m, lp.nnz, "ra", hbm)
    cus = cusparse_pair_us(torch, dev, lp, reps)
    return {"us": t_pair * 1e6, "algorithmic_bytes": b_pair, "gbs": b_pair / t_pair / 1e9,
            "cusparse_yardstick": cus,
            "gather_floor_us": gf[1] if gf else None, "frac_of_gather_floor": gf[1] / (t_pair * 1e6) if gf else None,
            "frac_of_hbm": b_pair / t_pair / 1e9 / hbm, "kernel": "spmv_kernel (standalone; K~x over the two column halves when split, K~'w)",
            "note": "random-column gathers move 32-byte sectors for 8 useful bytes (DESIGN.md §6)"}


def cusparse_pair_us(torch, dev, lp, reps=20):
    """Library yardstick for the SpMV pair: the same sparsity pattern as
    two fp64 CSR matrices (K and its explicit transpose, int32 indices) multiplied by torch's
    sparse CSR matvec, which calls cuSPARSE SpMV. Not on the product path; None if torch's
    sparse build refuses."""
    try:
        rp = torch.from_numpy(lp.row_ptr.astype(np.int32)).to(dev)
        ci = torch.from_numpy(lp.col_idx.astype(np.int32)).to(dev)
        va = torch.from_numpy(lp.val).to(dev)
        K = torch.sparse_csr_tensor(rp, ci, va, size=(lp.m, lp.n))
        Kt = K.to_sparse_csc()   # CSC of K = CSR of K'
        Kt = torch.sparse_csr_tensor(Kt.ccol_indices().to(torch.int32), Kt.row_indices().to(torch.int32),
                                     Kt.values(), size=(lp.n, lp.m))
        v = torch.rand(lp.n, 1, dtype=torch.float64, device=dev)
        w = torch.rand(lp.m, 1, dtype=torch.float64, device=dev)
        for _ in range(3):
            K @ v, Kt @ w
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            K @ v
            Kt @ w
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        del K, Kt, rp, ci, va
        torch.cuda.empty_cache()
        return {"us": us, "library": "cuSPARSE SpMV via torch.sparse_csr_tensor @ dense (fp64, int32 CSR, "
                "unscaled K and an explicit K' CSR; output allocation included)"}
    except (RuntimeError, TypeError) as e:
        return {"us": None, "error": str(e).splitlines()[0][:160]}


def _fp64_peak(key, sm_max):
    """Measured fp64 DFMA / DMMA TFLOP/s (profiles/fp64_peaks.json, scripts/micro/fp64_peak.cu on
    this pool's B200), else the derived 148 SMs x 64 FMA/clk x 2 flop x sm_max."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))[key])
        return v, "measured: profiles/fp64_peaks.json (scripts/micro/fp64_peak.cu)"
    except (OSError, KeyError, ValueError):
        return 148 * 64 * 2 * sm_max * 1e6 / 1e12, "derived: 148 SMs x 64 FP64 FMA/clk x 2 flop x sm_max"


def _traffic(key, field):
    """DRAM bytes (per launch, or per attempt for the grid kernel, like `achieved`) of a kernel from
    the committed ncu captures (profiles/traffic.json), or None."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[key][field])
    except (OSError, KeyError, ValueError):
        return None


def gather_floor_us(n, m, nnz, alg, hbm):
    """Gather-bound floor of one accepted grid-path attempt: every nonzero gathers
    one fp64 at a random column, and B200 serves random 8-byte gathers at a rate set by the
    gathered array's size (L2-resident below ~72 MB, then DRAM sectors): the SpMV-like sweep of
    profiles/gather_rates.json (12 B/nnz stream + gather, measured) gives each SpMV's floor by
    linear interpolation in the target's size (y': 8m bytes for K~'y', x': 8n bytes for K~x',
    each optionally split into column parts), plus the fused vector updates at HBM peak.
    Returns (floor_us, pair_floor_us) or None."""
    try:
        sw = json.load(open(os.path.join(ROOT, "profiles", "gather_rates.json")))["spmv_like_sweep"]
    except (OSError, KeyError, ValueError):
        return None
    pts = sorted((d["array_mb"], d["ms_per_1e8"]) for d in sw)

    def ms_per_1e8(mb):
        if mb <= pts[0][0]:
            return pts[0][1]
        for (a, ta), (b, tb) in zip(pts, pts[1:]):
            if mb <= b:
                return ta + (tb - ta) * (mb - a) / (b - a)
        (a, ta), (b, tb) = pts[-2], pts[-1]
        return tb + (tb - ta) * (mb - b) / (b - a)
    def spmv_us(rows, target_elems):
        # a target past the L2 knee may be split into k column parts (k passes, each gathering
        # from 1/k of the vector; the row partials cost 16 B per row per extra pass at HBM peak):
        # the floor takes the best k, as the grid kernel's two-pass phase B does with k = 2
        best = None
        for k in (1, 2, 3, 4):
            t = nnz / 1e8 * ms_per_1e8(8 * target_elems / k / 1e6) * 1e3 + (k - 1) * 16 * rows / (hbm * 1e9) * 1e6
            best = t if best is None else min(best, t)
        return best
    pair = spmv_us(m, n) + spmv_us(n, m)
    upd = (64 * n + 56 * m if alg == "ra" else 88 * n + 88 * m) / (hbm * 1e9) * 1e6
    return pair + upd, pair


def attempt_bytes(n, m, nnz, alg, elem=8):
    """Algorithmic bytes of one accepted attempt of the grid path (DESIGN.md §6,
    SURVEY §8(d) d.2): the SpMV pair streams K~ and K~' once (4-byte index + elem-byte value
    per entry each) plus their int32 row pointers and gathers x' and y' once; the fused updates
    move 8n + 7m (raPDHG) or 11n + 11m (r2HPDHG) vector elements.  elem = 8 (fp64) or 4 (fp32
    storage, reading 39)."""
    pair = 2 * (4 + elem) * nnz + 4 * (m + 1) + 4 * (n + 1) + elem * (n + m)
    upd = elem * (8 * n + 7 * m if alg == "ra" else 11 * n + 11 * m)
    return pair, pair + upd


def oracle_cores():
    return len(os.sched_getaffinity(0))


def c1_leg(mp, torch, dev, reps=200, oracle_reps=20):
    """C1 (BASELINE configs[0]): one random sparse LP G-RAND(50, 100, 10, seed 1), r2HPDHG to 1e-4
    relative KKT.  Time of the whole path for one LP through the C ABI with device-resident
    inputs (lp_create: validate, transpose, precondition; lp_solve; lp_get_solution; lp_destroy),
    CUDA events on the solve stream, median of `reps`; the solve's own kernel time; the counts.
    Beside it the CPU oracle on one host core (a single LP: the oracle's OpenMP loops only split
    SpMV rows, so one thread is its natural setting here)."""
    import oracle
    lp = lpgen.g_rand(50, 100, 10, seed=1)
    prob = mp.Problem.from_lp(lp).to(dev)
    st = torch.cuda.current_stream()
    ts, ks = [], []
    for rep in range(reps + 5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with mp.Solver(prob) as s:
            r = s.solve(algorithm="r2")
            x, y, lam = s.solution(memory=mp.LP_DEVICE)
        e1.record(st)
        torch.cuda.synchronize()
        if rep >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
            ks.append(r["solve_seconds"] * 1e6)
    oracle.set_threads(1)
    to = []
    for _ in range(oracle_reps):
        t0 = time.perf_counter()
        ro = oracle.solve(lp, "r2")
        to.append((time.perf_counter() - t0) * 1e6)
    oracle.set_threads(oracle_cores())
    return {"workload": "C1: G-RAND(50, 100, 10, seed 1), one LP, r2HPDHG to 1e-4 relative KKT",
            "metric": "time to 1e-4 KKT (one LP, whole path)", "unit": "us", "higher_is_better": False,
            "time_us": float(np.median(ts)), "solve_kernel_us": float(np.median(ks)),
            "status_optimal": r["status"] == mp.LP_OPTIMAL, "iterations": int(r["iterations"]),
            "attempts": int(r["attempts"]), "restarts": int(r["restarts"]), "rel_kkt": float(r["rel_kkt"]),
            "objective_rel_err": abs(r["primal_objective"] - lp.obj_star) / (1 + abs(lp.obj_star)),
            "path": "create + solve + get_solution + destroy, device inputs; the solve runs the CTA-per-LP kernel",
            "cpu_baseline": {"value": float(np.median(to)), "unit": "us", "cores": 1, "kind": "oracle",
                             "sample": f"median of {oracle_reps} full oracle solves of the same LP (one thread)",
                             "iterations": int(ro["iterations"]), "cpu_model": _cpu_model()}}


def oracle_large_baseline(lp, alg, full, label):
    """The CPU oracle beside a large-LP leg, on every host core: a full solve (C4) or, for C5, the
    per-attempt time from two short solves (3 and 1 accepted steps; the setup cancels) times the
    GPU's attempt count -- labelled extrapolated."""
    import oracle
    cores = oracle_cores()
    oracle.set_threads(cores)
    if full:
        t0 = time.perf_counter()
        r = oracle.solve(lp, alg, iteration_limit=20_000)
        t = time.perf_counter() - t0
        return {"kind": "oracle", "cores": cores, "unit": "ms", "value": t * 1e3, "cpu_model": _cpu_model(),
                "sample": f"one full {label} solve ({r['iterations']} iterations, {r['attempts']} attempts), "
                          f"setup included", "iterations": int(r["iterations"]), "attempts": int(r["attempts"]),
                "us_per_attempt_incl_setup": t * 1e6 / max(1, r["attempts"])}
    r = oracle.solve(lp, alg, iteration_limit=3, eps_abs=0.0, eps_rel=0.0)
    setup_s, solve_s = oracle.last_timing()
    per = solve_s / max(1, r["attempts"])
    return {"kind": "oracle", "cores": cores, "unit": "us_per_attempt", "value": per * 1e6,
            "setup_s": setup_s, "cpu_model": _cpu_model(),
            "sample": f"{label}: one oracle solve of 3 accepted steps ({r['attempts']} attempts); per-attempt time = "
                      "its iteration phase / attempts (the oracle's setup timed apart)"}


def large_lp_leg(mp, torch, dev, stream, peaks, args, m=None, seed=4, label="C4", reps=3, cpu=False, fp32=True):
    """One large random sparse LP (C4 = G-RAND(1e5, 2e5, 20, seed 4); C5 = G-RAND(5e6, 1e7,
    20, seed 5)) solved to 1e-4 on the whole-GPU grid path: time to tolerance and the
    achieved algorithmic GB/s of the fused SpMV-pair + update loop."""
    m = args.large_m if m is None else m
    t0 = time.time()
    lp = lpgen.g_rand(m, 2 * m, 20, seed=seed)
    gen_s = time.time() - t0
    prob = mp.Problem.from_lp(lp).to(dev)
    torch.cuda.synchronize()
    t0 = time.time()
    s_setup = mp.Solver(prob)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    s_setup.close()
    out = {"workload": f"{label}: G-RAND({m}, {2 * m}, 20, seed {seed}), one LP on the whole GPU (grid path), to 1e-4",
           "nnz": lp.nnz, "generate_s": gen_s, "create_s_wall": setup_s}
    hbm = peaks.get("hbm_gbs", 6546.6)
    if lp.m >= 1_000_000:   # at C4 a pair is ~10 us of GPU time, below the binding's per-call host cost
        out["spmv_pair"] = spmv_pair_leg(mp, torch, dev, prob, lp, hbm)
    runs = [(a, "fp64") for a in ("ra", "r2")] + ([(a, "fp32") for a in ("ra", "r2")] if fp32 else [])
    for alg, prec in runs:
        key = alg if prec == "fp64" else f"{alg}_fp32"
        with mp.Solver(prob) as s:
            log(f"large leg {key}: warm-up")
            s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=20_000, precision=prec)   # warm-up
            best = None
            for _ in range(reps):
                r = s.solve(algorithm=alg, path=mp.PATH_GRID, iteration_limit=20_000, precision=prec)
                best = r if best is None or r["solve_seconds"] < best["solve_seconds"] else best
        pair, acc = attempt_bytes(lp.n, lp.m, lp.nnz, alg, 8 if prec == "fp64" else 4)
        rej = best["attempts"] - best["iterations"]
        byts = best["iterations"] * acc + rej * (pair // 2)
        t = best["solve_seconds"]
        gbs = byts / t / 1e9
        out[key] = {"status_optimal": best["status"] == mp.LP_OPTIMAL, "time_ms": t * 1e3,
                    "iterations": best["iterations"], "attempts": best["attempts"], "restarts": best["restarts"],
                    "rel_kkt": best["rel_kkt"], "objective_rel_err": abs(best["primal_objective"] - lp.obj_star)
                    / (1 + abs(lp.obj_star)), "us_per_attempt": t * 1e6 / best["attempts"],
                    "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                 "traffic": _traffic(("grid_kernel_c5" if lp.m >= 1_000_000 else "grid_kernel_c4")
                                                     + ("" if prec == "fp64" else "_fp32"), "bytes_per_attempt"),
                                 "kernel": "grid_kernel", "storage": prec,
                                 "traffic_source": "profiles/traffic.json (ncu --set full capture, per attempt)",
                                 "algorithmic_bytes_per_accepted_attempt": acc,
                                 "note": "working set (~70 MB) is L2-resident at C4; achieved may exceed HBM"}}
        if prec == "fp32":
            out[key]["objective_rel_err_vs_fp64"] = abs(best["primal_objective"] - out[alg]["objective"]) / (
                1 + abs(out[alg]["objective"]))
            out[key]["speedup_vs_fp64"] = out[alg]["time_ms"] / (t * 1e3)
            continue
        out[key]["objective"] = best["primal_objective"]
        if cpu and (lp.m < 1_000_000 or alg == "ra"):   # C5: one oracle solve (its setup is ~50 s)
            log(f"large leg {alg}: CPU oracle beside it")
            cb = oracle_large_baseline(lp, alg, full=lp.m < 1_000_000, label=label)
            if cb["unit"] == "us_per_attempt":   # C5: extrapolated to the GPU's attempts
                cb["extrapolated_ms"] = cb["value"] * best["attempts"] * 1e-3 + cb["setup_s"] * 1e3
                cb["note"] = "extrapolated: oracle per-attempt time x the GPU solve's attempts + the oracle's setup"
                cb["gpu_speedup_extrapolated"] = cb["extrapolated_ms"] / (t * 1e3)
            else:
                cb["gpu_speedup"] = cb["value"] / (t * 1e3)
            out[alg]["cpu_baseline"] = cb
        gf = gather_floor_us(lp.n, lp.m, lp.nnz, alg, hbm)
        if gf is not None:
            out[alg]["roofline"]["gather_floor"] = {
                "us_per_attempt": gf[0], "spmv_pair_us": gf[1],
                "frac": gf[0] / out[alg]["us_per_attempt"],
                "source": "profiles/gather_rates.json (scripts/micro/gather_bench.cu, measured random-gather rates)",
                "model": "per SpMV: nnz x measured time per random gather at the target's size (12 B/nnz stream "
                         "included; a target past the L2 knee may be split into column parts, best of 1-4) + "
                         "fused vector updates at HBM peak (DESIGN.md section 6)"}
    return out


def c5_sharded_leg(mp, torch, dev, ws, rank, args, m=5_000_000, seed=5):
    """C5 = G-RAND(5e6, 1e7, 20, seed 5) sharded over the job's ranks: by rows
    (each rank an nnz-balanced row block, the n-long K~'y partials all-reduced every attempt) or
    by columns (reading 33: column blocks, the m-long K~x' partials all-reduced) -- `--c5-axis`,
    default the axis whose exchanged vector is shorter.  Time to 1e-4 = max over ranks of the
    library's device-timed solve (strong scaling: the LP is fixed)."""
    import torch.distributed as tdist
    t0 = time.time()
    lp = lpgen.g_rand(m, 2 * m, 20, seed=seed)
    gen_s = time.time() - t0
    axis = args.c5_axis
    if axis == "auto":
        axis = "cols" if mp.shard_axis(lp.m, lp.n) == mp.SHARD_COLS else "rows"
    full = mp.Problem.from_lp(lp)
    if axis == "cols":
        cuts = mp.col_partition(full, ws)
        c0, c1 = cuts[rank], cuts[rank + 1]
        loc = mp.local_cols(full, c0, c1).to(dev)
        kw = dict(axis="cols", global_col_offset=c0, n_global=lp.n)
        what = "column-sharded", "K~x' partials (m-long)"
    else:
        cuts = mp.row_partition(lp.row_ptr, ws)
        r0, r1 = cuts[rank], cuts[rank + 1]
        loc = mp.local_rows(full, r0, r1).to(dev)
        kw = dict(global_row_offset=r0, m1_global=lp.m1, m2_global=lp.m2)
        what = "row-sharded", "K~'y partials (n-long)"
    del full
    uid = [mp.nccl_unique_id() if rank == 0 else None]
    if ws > 1:
        tdist.broadcast_object_list(uid, src=0)
    comm = mp.nccl_comm_init(ws, uid[0], rank)
    out = {"workload": f"C5: G-RAND({m}, {2 * m}, 20, seed {seed}), one LP {what[0]} over {ws} GPU(s) "
                       f"(NCCL all-reduce of the {what[1]}), to 1e-4",
           "nnz": lp.nnz, "ranks": ws, "axis": axis, "block_max": int(max(np.diff(cuts))), "generate_s": gen_s,
           "scaling": "strong"}
    try:
        with mp.ShardedSolver(loc, comm=comm, rank=rank, nranks=ws, **kw) as s:
            for alg in ("ra",):
                s.solve(algorithm=alg, iteration_limit=20_000)                 # warm-up
                if ws > 1:
                    tdist.barrier()
                r = s.solve(algorithm=alg, iteration_limit=20_000)
                t = torch.tensor([r["solve_seconds"]], dtype=torch.float64, device=dev)
                if ws > 1:
                    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
                pair, acc = attempt_bytes(lp.n, lp.m, lp.nnz, alg)
                out[alg] = {"status_optimal": r["status"] == mp.LP_OPTIMAL, "time_ms": float(t[0]) * 1e3,
                            "iterations": r["iterations"], "attempts": r["attempts"], "restarts": r["restarts"],
                            "rel_kkt": r["rel_kkt"],
                            "objective_rel_err": abs(r["primal_objective"] - lp.obj_star) / (1 + abs(lp.obj_star)),
                            "us_per_attempt": float(t[0]) * 1e6 / r["attempts"],
                            "algorithmic_gbs_per_gpu": r["iterations"] * acc / ws / float(t[0]) / 1e9}
    finally:
        mp.nccl_comm_destroy(comm)
    return out


def dense_leg(mp, torch, dev, peaks, no_cpu_baseline=False):
    """C3: 256 dense 200x400 LPs sharing K: LPs/s on the fp64 tensor-core (DMMA)
    path and on the per-instance path, with the DMMA path's achieved fp64 rate."""
    lp, C, Q, obj = lpgen.g_dense(200, 400, batch=256, seed=3)
    prob = mp.Problem.from_lp(lp).to(dev)
    Cd, Qd = torch.as_tensor(C, device=dev), torch.as_tensor(Q, device=dev)
    out = {"workload": "C3: 256 dense 200x400 LPs sharing K (c, q vary), raPDHG to 1e-4"}
    for name, path in (("dmma", mp.PATH_DMMA), ("per_instance", mp.PATH_INSTANCE)):
        bs = mp.BatchSolver(prob, Cd, Qd)
        bs.solve(algorithm="ra", path=path, iteration_limit=100_000)
        res = bs.solve(algorithm="ra", path=path, iteration_limit=100_000)
        bs.close()
        t = float(res[0]["solve_seconds"])
        d = {"value": 256 / t, "unit": UNIT, "solve_ms": t * 1e3,
             "all_optimal": bool((res["status"] == mp.LP_OPTIMAL).all()),
             "max_obj_rel_err": float(np.max(np.abs(res["primal_objective"] - obj) / (1 + np.abs(obj))))}
        if name == "dmma":
            # the method's own work: every instance's attempts, two m x n matvecs (2*m*n flops each)
            # per attempt; the kernel executes more -- each group of 8 runs in lock-step until its
            # slowest instance is done (reported beside it as "executed")
            att_i = np.asarray(res["attempts"], dtype=np.float64)
            flops = float(att_i.sum()) * 2 * 2 * 200 * 400
            att = att_i.reshape(-1, 8).max(axis=1)
            flops_ex = float(att.sum()) * 2 * 2 * 200 * 400 * 8
            peak, peak_src = _fp64_peak("fp64_dmma_tflops", peaks.get("sm_max_mhz", 1965.0))
            d["roofline"] = {"bound": "tensor", "achieved": flops / t / 1e12, "peak": peak, "unit": "TFLOP/s",
                             "frac": flops / t / 1e12 / peak,
                             "executed": {"achieved": flops_ex / t / 1e12, "frac": flops_ex / t / 1e12 / peak,
                                          "note": "lock-step groups of 8: each group runs its slowest "
                                                  "instance's attempts"},
                             "traffic": _traffic("dmma_kernel_c3", "bytes_per_launch"),
                            "traffic_source": "profiles/traffic.json (ncu --set full capture, per launch)",
                            "kernel": "dmma_kernel<4>",
                             "peak_source": peak_src}
        out[name] = d
    out["speedup_dmma_vs_per_instance"] = out["dmma"]["value"] / out["per_instance"]["value"]
    if not no_cpu_baseline:
        import oracle
        cores = oracle_cores()
        oracle.set_threads(cores)
        k = 32
        t0 = time.perf_counter()
        _, _, ro = oracle.solve_batch(lp, C[:k], Q[:k], "ra", iteration_limit=100_000, threads=cores)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": k / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"the first {k} of the 256 C3 instances, oracle solve_batch (one LP per "
                                         "thread)", "cpu_model": _cpu_model(),
                               "all_optimal": all(r["status"] == 1 for r in ro)}
    return out


def infeasibility_workload(batch):
    """The infeasibility leg's batch: one planted LP (lpgen.g_infeasible("dual"): column j has
    G[:, j] >= 0, A[:, j] = 0, u_j = +inf) with perturbed costs; c_j > 0 on even instances
    (bounded) and c_j < 0 on odd ones (unbounded along e_j).  Returns (lp, C, unbounded mask)."""
    for seed in range(200):   # the first planted LP whose K fits the register-resident kernel
        lp = lpgen.g_infeasible("dual", seed, m1=10, m2=3, n=20, density=0.15)
        if np.diff(lp.row_ptr).max() <= 8 and np.bincount(lp.col_idx, minlength=lp.n).max() <= 8:
            break
    j = int(np.nonzero(~np.isfinite(lp.u))[0][0])
    rng = np.random.default_rng(5)
    C = lp.c + 0.1 * rng.normal(size=(batch, lp.n))
    C[::2, j] = np.abs(C[::2, j]) + 1.0
    C[1::2, j] = -np.abs(C[1::2, j]) - 0.5
    return lp, C, np.arange(batch) % 2 == 1

def infeasibility_leg(mp, torch, dev, batch=1024, reps=5):
    """SURVEY §8(f) row 1 on a batch: 1024 LPs sharing K (lpgen.g_infeasible("dual")), half of
    the cost vectors bounded (OPTIMAL), half unbounded (DUAL_INFEASIBLE, certified by the primal
    ray of P:530-531); the C2 step (create + solve + get + destroy, device-resident)."""
    lp, C, unbounded = infeasibility_workload(batch)
    want = np.where(unbounded, mp.LP_DUAL_INFEASIBLE, mp.LP_OPTIMAL)
    prob = mp.Problem.from_lp(lp).to(dev)
    Cd = torch.as_tensor(C, device=dev)
    X = torch.empty((batch, lp.n), dtype=torch.float64, device=dev)
    Y = torch.empty((batch, lp.m), dtype=torch.float64, device=dev)
    best, ok = None, True
    for rep in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        bs = mp.BatchSolver(prob, Cd)
        res = bs.solve(algorithm="ra", iteration_limit=200_000)
        bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
        bs.close()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ok &= bool((np.asarray(res["status"]) == want).all())
        if rep:
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
    it = np.asarray(res["iterations"])
    return {"workload": f"{batch} sparse LPs sharing K ({lp.m} x {lp.n}), half unbounded, raPDHG, 1e-4 / "
                        "infeasibility tolerance 1e-8", "unit": UNIT, "ms_per_step": best,
            "value": batch / (best * 1e-3), "statuses_as_planted": ok,
            "iterations": {"p50_optimal": float(np.median(it[::2])), "p50_infeasible": float(np.median(it[1::2])),
                           "max": int(it.max())}}


def batch_scaling_leg(mp, torch, dev, sizes=(4096, 16384, 65536), reps=3):
    """Context for serving: the C2 step (create + solve + get + destroy, device-resident) at larger
    batches of the same LP shape; the headline stays at BASELINE's 1024."""
    out = {"workload": "C2-shaped batches (5x5 grid LPs, raPDHG, 1e-4), batch size varied", "unit": UNIT}
    for B in sizes:
        lp, C = lpgen.g_grid(batch=B, seed=2)
        prob = mp.Problem.from_lp(lp).to(dev)
        Cd = torch.as_tensor(C, device=dev)
        X = torch.empty((B, lp.n), dtype=torch.float64, device=dev)
        Y = torch.empty((B, lp.m), dtype=torch.float64, device=dev)
        best, ok = None, True
        for rep in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            bs = mp.BatchSolver(prob, Cd)
            res = bs.solve(algorithm="ra", iteration_limit=200_000)
            bs.solutions(memory=mp.LP_DEVICE, X=X, Y=Y)
            bs.close()
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            ok &= bool((res["status"] == mp.LP_OPTIMAL).all())
            if rep:
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
        out[str(B)] = {"ms_per_step": best, "value": B / (best * 1e-3), "all_optimal": ok,
                       "max_iterations": int(res["iterations"].max())}
    return out


def spo_leg(mp, torch, dev, steps=10, ks=(12, 30), batch=70):
    """SPO+ training-step shape of P:198-215 / P:330-345: Warcraft-shaped
    8-connected k x k grid LPs, batch 70, synthetic terrain costs and a synthetic
    predictor whose output moves a little every step (as between optimiser steps).  One step =
    lp_spo_plus: inner costs 2c^ - c, the batch solve (warm-started from the previous step's
    inner solutions after the first), loss and subgradient.  Context: the paper's Table 1 average
    iteration counts at 1e-4."""
    out = {"workload": "Warcraft-shaped SPO+ steps: 8-connected k x k grid LPs, batch 70, 1e-4",
           "steps": steps}
    rng = np.random.default_rng(11)
    for k in ks:
        lp = lpgen.warcraft_lp(k)
        Ct = lpgen.warcraft_costs(k, batch, seed=k)
        prob = mp.Problem.from_lp(lp).to(dev)
        T = lambda a: torch.as_tensor(a, device=dev)
        # x*(c) of the dataset: precomputed once (outside the timed region) at a tight tolerance
        bs0 = mp.BatchSolver(prob, T(Ct))
        bs0.solve(algorithm="r2", step_rule="constant", eps_abs=1e-9, eps_rel=1e-9)
        Xt, _ = bs0.solutions(memory=mp.LP_DEVICE)
        bs0.close()
        Ct_d = T(Ct)
        ot = (Ct_d * Xt).sum(dim=1)
        base = Ct * rng.uniform(0.5, 1.5, size=Ct.shape)
        preds = [T(base * rng.uniform(0.97, 1.03, size=Ct.shape)) for _ in range(steps)]
        row = {"m": lp.m, "n": lp.n, "nnz": lp.nnz}
        for name, kw in (("rapdhg", dict(algorithm="ra")), ("r2hpdhg_constant_step",
                                                             dict(algorithm="r2", step_rule="constant"))):
            bs = mp.BatchSolver(prob, Ct_d)
            bs.spo_plus(preds[0], Ct_d, Xt, ot, **kw)                # warm-up (cold)
            stream = torch.cuda.current_stream()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            its, ok = [], True
            e0.record(stream)
            for s in range(steps):
                loss, grad, res = bs.spo_plus(preds[s], Ct_d, Xt, ot, warm=s > 0, **kw)
                its.append(float(np.mean(res["iterations"])))
                ok &= bool((res["status"] == mp.LP_OPTIMAL).all())
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            bs.close()
            row[name] = {"ms_per_step": ms, "value": batch / (ms * 1e-3), "unit": UNIT, "all_optimal": ok,
                         "mean_iterations_cold": its[0], "mean_iterations_warm": float(np.mean(its[1:])),
                         "lp_seconds_per_epoch_143_steps": ms * 143 / 1e3}
        out[f"k{k}"] = row
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
