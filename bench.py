#!/usr/bin/env python
"""bench.py -- time-to-certify (0 gap) and BnB nodes/sec on B200.

One "step" = one full certified solve (bnbglm::solve, bnb_engine.hpp:299-309)
of the BASELINE.json configs[1] workload (c2: synthetic sparse logistic
regression n=2000, p=500, k=8, rho=0.7, seed 0, M=2, lambda2=1; the other
configs are parity-test cases).  value = nodes processed / second over the
timed steps (whole job: all ranks); ms_per_step = time-to-certify.

With N > 1 ranks (torchrun) the same instance is certified by the
node-sharded solve (bnbg_solve_sharded over NCCL: X replicated, open nodes
dealt over the GPUs, incumbent / termination / node exchange per pass), so
the total work is fixed ("scaling": "strong").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the reference algorithm's CPU implementation (the C
restatement in oracle/, OpenBLAS DGEMM, all host threads) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, p, k, rho, loss, description)
    "c1": (1000, 100, 5, 0.5, 0, "synthetic sparse linear regression n=1000 p=100 k=5 rho=0.5"),
    "c2": (2000, 500, 8, 0.7, 1, "synthetic sparse logistic regression n=2000 p=500 k=8 rho=0.7"),
    "c3": (5000, 2000, 10, 0.9, 0, "synthetic sparse linear regression n=5000 p=2000 k=10 rho=0.9"),
    "c4": (20000, 5000, 15, 0.9, 1,
           "synthetic sparse logistic regression n=20000 p=5000 k=15 rho=0.9 (rho per PAPER.md:1199)"),
    "c5": (2000, 500, 8, 0.7, 0, "Rashomon set (epsilon 0.01, all supports within 1% of the optimum)"
                                 " for n=2000 p=500 k=8 rho=0.7 linear regression"),
}
METRIC = "BnB nodes/sec at time-to-certify (0 gap)"
FP64_PEAK_TFLOPS = 37.0  # measured DMMA.8x8x4 issue rate on this pool (profiles/r01_fp64_peak.txt)


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def _load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def _ncu_traffic(kernel_class, config):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary, when that capture was taken on this config (its report is named
    after it, e.g. ncu_gemm_big_c3w.ncu-rep); None otherwise."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None
    ent = d.get(f"{kernel_class}@{config}") or d.get(kernel_class, {})
    src = ent.get("source", "")
    if f"_{config}." not in src and f"_{config}w." not in src:
        return None
    return ent.get("dram_bytes_per_launch")


def run_reference(args, spec, rank):
    """Reference arm: the CPU implementation of the path on the host cores."""
    if rank != 0:
        return
    from oracle import oracle as O
    n, p, k, rho, loss, desc = spec
    O.build()
    threads = os.cpu_count() or 1
    blas = O.use_openblas(threads)
    inst = O.generate(n, p, k, rho, loss, 5.0, 0, 2.0, 1.0)
    cfg_full = O.solver_cfg(workers=threads)
    # untimed warm-up: bounded 1 s samples
    for _ in range(args.warmup):
        O.solve(inst, O.solver_cfg(workers=threads, time_limit=1.0))
    # one probe run decides whether K full certifies fit in ~4 minutes
    t0 = time.perf_counter()
    first = O.solve(inst, cfg_full)
    t_full = time.perf_counter() - t0
    results = [(first.nodes_processed, t_full, first.status)]
    budget = 240.0
    limit = math.inf if t_full * args.steps <= budget else budget / args.steps
    for _ in range(args.steps - 1):
        t0 = time.perf_counter()
        c = O.solve(inst, O.solver_cfg(workers=threads, time_limit=limit))
        results.append((c.nodes_processed, time.perf_counter() - t0, c.status))
    nodes = sum(r[0] for r in results)
    secs = sum(r[1] for r in results)
    value = nodes / secs
    sample = (f"{args.steps} x full certify of {args.config} ({first.nodes_processed} nodes, "
              f"{t_full:.1f} s each)" if limit == math.inf else
              f"1 full certify ({t_full:.1f} s) + {args.steps - 1} samples capped at {limit:.0f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (generate_synthetic, seed 0)",
        "config": {"workload": f"{args.config}: {desc}, certify to 0 gap", "batch_size": "auto",
                   "time_to_certify_s": t_full},
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": threads, "kind": "port",
                         "sample": sample + ("; OpenBLAS DGEMM" if blas else "; C loops")},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(spec, args):
    from oracle import oracle as O
    n, p, k, rho, loss, desc = spec
    O.build()
    threads = os.cpu_count() or 1
    blas = O.use_openblas(threads)
    inst = O.generate(n, p, k, rho, loss, 5.0, 0, 2.0, 1.0)
    limit = args.cpu_seconds
    t0 = time.perf_counter()
    c = O.solve(inst, O.solver_cfg(workers=threads, time_limit=limit))
    secs = time.perf_counter() - t0
    return {"value": c.nodes_processed / secs, "unit": "nodes/s", "cores": threads, "kind": "port",
            "sample": (f"one certify of {args.config} on {threads} threads"
                       + (" (OpenBLAS DGEMM)" if blas else "") +
                       f": {c.nodes_processed} nodes in {secs:.1f} s, status {c.status}"),
            "time_to_certify_s": secs if c.status == "optimal" else None,
            "optimal_value": c.optimal_value, "support": c.support}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=120.0)
    ap.add_argument("--cpu-baseline-only", action="store_true",
                    help="only the cpu_baseline leg for --config (bounded by --cpu-seconds)")
    ap.add_argument("--time-limit", type=float, default=float("inf"),
                    help="per-certify time limit (c3/c4: nodes/s at a stated limit)")
    args = ap.parse_args()
    spec = CONFIGS[args.config]
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        run_reference(args, spec, rank)
        return
    if args.cpu_baseline_only:
        if rank == 0:
            print(json.dumps({"config": args.config, "cpu_baseline": cpu_baseline(spec, args)}),
                  flush=True)
        return

    import torch
    import paper_2605_22188_b200 as P

    torch.cuda.set_device(local)
    # BNBG_BENCH_SHARDED=1 runs the node-sharded path even at one rank (under
    # torchrun, NCCL world size 1) -- a check of the N > 1 code path on one GPU
    sharded = world > 1 or os.environ.get("BNBG_BENCH_SHARDED") == "1"
    dist = None
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, p, k, rho, loss, desc = spec
    inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                   seed=0, M=2.0, lambda2=1.0))
    cfg = P.SolverConfig(time_limit=args.time_limit)
    eng = P.Engine(inst, device=local)  # X, y resident in HBM before timing
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2

    def certify(engine):
        if args.config == "c5":  # collect_rashomon (rashomon.hpp:149-218): same hot path
            return engine.collect_rashomon(cfg, P.RashomonConfig(epsilon=0.01)).certificate
        return engine.solve_sharded(cfg, transport="nccl") if sharded else engine.solve(cfg)

    for _ in range(args.warmup):
        certify(eng)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    launches0 = eng.kernel_launches()
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    total_ms, nodes, certs = 0.0, 0, []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cert = certify(eng)
        e1.record()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
        nodes += cert.nodes_processed
        certs.append(cert)
    barrier()
    clocks = sampler.stop()
    launches = eng.kernel_launches() - launches0

    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # the sharded certificate already reports the nodes of all ranks
    total_ms_max, nodes_all = float(t[0]), float(nodes)
    value = nodes_all / (total_ms_max / 1e3)

    # roofline: one extra (untimed) certify with per-launch CUDA events on the engine stream
    eng.set_timing(True)
    before = eng.kernel_stats()
    prof_cert = certify(eng)
    after = eng.kernel_stats()
    eng.set_timing(False)
    delta = {kc: tuple(a - b for a, b in zip(after[kc], before[kc])) for kc in after}
    dom = max(delta, key=lambda kc: delta[kc][0])
    ms, fl, ln = delta[dom]
    peaks = _load_peaks()
    algorithmic = {
        "gemm_xv": "2*n*p flops per active column per launch",
        "gemm_xtr": "2*n*p flops per active column per launch",
        "pass": "4*n*p flops per node-iteration (X*V and X'*R; bound evaluations not counted)",
        "reopt": "4*q*n flops per support-iteration of the reference's projected gradient",
    }
    if dom in algorithmic:
        achieved = fl / (ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                "peak_source": "measured FP64 DMMA issue rate (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json has no fp64 entry",
                "algorithmic": algorithmic[dom]}
    else:
        node_its = prof_cert.node_iterations
        bytes_ = 41.0 * p * node_its if dom == "prox_fista" else float("nan")
        achieved = bytes_ / (ms / 1e3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic": "41*p bytes per node-iteration"}
    roof["traffic"] = _ncu_traffic(dom, args.config)
    roof["avg_launch_us"] = 1e3 * ms / max(ln, 1)
    roof["share_of_step"] = ms / max(1e-9, 1e3 * prof_cert.profile.total_seconds)
    roof["kernel_ms"] = {kc: round(v[0], 3) for kc, v in delta.items()}

    # e2e: the public API from host arrays (instance upload, solve, certificate readback)
    e2e_ms, e2e_nodes, h2d, d2h = 0.0, 0, 0, 0
    e2e_parts = [0.0, 0.0, 0.0]  # create (upload + L), solve, destroy
    # W untimed warm-up rounds first, as for the device-timed steps (the first
    # create of a process grows the stream-ordered memory pool)
    for it in range(args.warmup + args.steps):
        timed = it >= args.warmup
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2 = P.Engine(inst, device=local)
        t1 = time.perf_counter()
        c2 = certify(e2)
        bi, bo = e2.transfer_bytes()
        t2 = time.perf_counter()
        e2.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if not timed:
            continue
        e2e_parts[0] += t1 - t0
        e2e_parts[1] += t2 - t1
        e2e_parts[2] += t3 - t2
        e2e_ms += 1e3 * (t3 - t0)
        e2e_nodes += c2.nodes_processed
        h2d += bi
        d2h += bo + 8 * (2 * len(c2.support) + 16)
    if dist:
        te = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0])
    e2e_value = e2e_nodes / (e2e_ms / 1e3)

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(spec, args)
        if base.get("support") is not None and base["support"] != certs[0].support:
            base["support_mismatch"] = True

    if rank == 0:
        c0 = certs[0]
        line = {
            "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_synthetic, seed 0, problem.hpp:70-132)",
            "config": {"workload": f"{args.config}: {desc}, " + (
                           "certify to 0 gap" if math.isinf(args.time_limit)
                           else f"nodes/s within a {args.time_limit:g} s time limit"),
                       "n": n, "p": p, "k": k, "rho": rho, "loss": "logistic" if loss else "squared",
                       "batch_size": c0.batch_size_used,
                       "parallelism": f"node-sharded over {world} GPUs (NCCL)" if sharded
                       else "single GPU",
                       "l2": "flushed (256 MiB write) before every step",
                       "time_to_certify_s": total_ms_max / args.steps / 1e3,
                       "nodes_per_certify": c0.nodes_processed, "lb_batches": c0.lb_batches,
                       "relax_iterations": c0.relax_iterations,
                       "node_iterations": c0.node_iterations,
                       "optimal_value": c0.optimal_value, "support": c0.support,
                       "profile": {"lower_bound_s": c0.profile.lower_bound_seconds,
                                   "reoptimization_s": c0.profile.reoptimization_seconds,
                                   "transfer_s": c0.profile.transfer_seconds,
                                   "branch_generate_s": c0.profile.branch_generate_seconds}},
            "gpu_launches": launches,
            "clocks": clocks,
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "nodes/s",
                    "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                    "time_to_certify_s": e2e_ms / args.steps / 1e3,
                    "create_solve_destroy_s": [round(x / args.steps, 5) for x in e2e_parts]},
            "cpu_baseline": base,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
