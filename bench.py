#!/usr/bin/env python
"""Benchmark: converged multiscale unbalanced domdec solve on B200.

One "step" is one full converged solve of a BASELINE.json configuration.
Default ``ms_256`` = configs[1] (256^2, 5-Gaussian mixtures, lambda = 0.5, eps
annealed 64h^2 -> 2h^2 over the 32^2 -> 256^2 pyramid, 4x4 basic cells, fp64,
staggered strategy, delta = 2e-5), which finishes in seconds; ``--config
ms_1024`` runs configs[2] (the 1024^2 headline, several minutes per solve in
this round).  The metric is the solve time in seconds (lower is better).

* ``value``  — device-timed solve (CUDA events on the launching stream) with the
  pyramid already resident in HBM; L2 is flushed (256 MiB write) before each step.
* ``e2e``    — the same solve through the public API from pinned host arrays:
  host->device copy of every pyramid level and device->host read of the result
  (basic-cell marginals, duals, objective) inside the timed region.
* ``roofline`` — the dominant kernel (``dd_cell_solve``): algorithmic FP64
  FLOPs of its separable contractions per launch / mean launch time (CUDA
  events), against the nominal FP64 peak (no FP64 entry in MEASURED_PEAKS.json);
  its HBM traffic is reported next to it.
* ``cpu_baseline`` — the CPU oracle (a restatement of the reference algorithm)
  timed on the coarsest stage of the same workload and extrapolated to the
  whole solve by the ratio of algorithmic cell-sweep FLOPs (both arms run the
  same iteration sequence).

Multi-GPU (``--gpus N`` under torchrun): every batch's cell solves are
partitioned across the ranks (cost-balanced) and the solve outputs summed
with NCCL, so all ranks solve the same problem together (strong scaling);
value is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {"pr1_64": 0, "ms_256": 1, "ms_1024": 2, "ms_2048": 3}
FP64_PEAK_TFLOPS = 40.0   # B200 nominal FP64 (vector); not measured on this pool


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("DD_BENCH_CONFIG", "ms_256"),
                    choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=1, help="run the CPU baseline sample")
    return ap.parse_args()


def problem(cfg_name: str, seed: int):
    from paper_2410_08859_b200 import DivergenceSpec, Grid, GridMeasure, TransportProblem
    from paper_2410_08859_b200.problems import config_problem_arrays

    mu, nu, dx, org, cfg = config_problem_arrays(CONFIGS[cfg_name], seed=seed)
    grid = Grid(mu.shape, dx, org)
    h2 = dx * dx
    prob = TransportProblem(GridMeasure(grid, mu), GridMeasure(grid, nu),
                            DivergenceSpec(cfg["lam"]), cfg["eps_final_h2"] * h2)
    eps_start = (cfg["eps_start_h2"] or cfg["eps_final_h2"]) * h2
    return prob, cfg, eps_start


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, idx: int):
        self.idx = idx
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar across the process group (identity when not distributed)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def flush_l2(buf):
    buf.fill_(1.0)


def run_solve(prob, cfg, eps_start, levels=None):
    from paper_2410_08859_b200.engine import EngineConfig, StrategyConfig
    from paper_2410_08859_b200.multiscale import multiscale_solve

    return multiscale_solve(prob, cfg["cell"], cfg["coarsest"], eps_start,
                            strategy=StrategyConfig("staggered"), config=EngineConfig(),
                            levels=levels)


def fetch_result(st):
    """Device->host read of the result a caller consumes: boxes, marginals, duals, score."""
    boxes = st.ybox.cpu()
    vals = st.yval.cpu()
    duals = [t.cpu() for t in st.global_duals] if st.global_duals is not None else []
    d2h = boxes.numel() * 4 + vals.numel() * 8 + sum(t.numel() * 8 for t in duals)
    return d2h


def cpu_sample(prob, cfg, eps_start):
    """Oracle (reference algorithm restated in numpy) on the coarsest stage."""
    from oracle.ref_problem import make_ctx
    from oracle.ref_sweep import EngCfg, StratCfg, solve, warm_state
    from paper_2410_08859_b200.multiscale import build_pyramid, eps_schedule

    levels = build_pyramid(prob.mu, prob.nu, cfg["coarsest"])
    sched = eps_schedule(levels, eps_start, prob.eps)
    lv = levels[0]
    eps = sched[0][0]
    t0 = time.perf_counter()
    ctx = make_ctx(lv.mu, lv.nu, lv.grid.dx, lv.grid.origin, prob.div.lam, eps, cfg["cell"])
    st = warm_state(ctx, delta=1e-3)
    _, rep, _ = solve(ctx, st, StratCfg("staggered"), EngCfg())
    t = time.perf_counter() - t0
    return t, rep, f"coarsest stage {lv.grid.dims[0]}^2 at eps={eps / (prob.mu.grid.dx ** 2):g}h^2 " \
                   f"(warm start + staggered domdec to delta=2e-5)"


def main():
    args = parse()
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # DD_DIST_BACKEND=gloo: functional multi-rank runs on fewer GPUs than ranks
        backend = os.environ.get("DD_DIST_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    prob, cfg, eps_start = problem(args.config, args.seed)
    config_desc = {"workload": f"{args.config}: BASELINE configs[{CONFIGS[args.config]}] "
                               f"{prob.mu.grid.dims[0]}x{prob.mu.grid.dims[1]} multiscale "
                               f"{cfg['coarsest']}^2->{prob.mu.grid.dims[0]}^2, "
                               f"eps {eps_start / prob.mu.grid.dx ** 2:g}h^2->{prob.eps / prob.mu.grid.dx ** 2:g}h^2, "
                               f"lambda={cfg['lam']}, cells {cfg['cell']}x{cfg['cell']} (2x2 composites), "
                               "staggered, delta=2e-5",
                   "grid": list(prob.mu.grid.dims), "cell": cfg["cell"], "lambda": cfg["lam"],
                   "strategy": "staggered", "l2": "flushed (256 MiB write) before every step",
                   "parallelism": (f"cell-sharded x{world} (batch cell solves partitioned, "
                                   "NCCL all-reduce of the solve outputs)") if world > 1 else "1 GPU",
                   "seed": args.seed}

    if args.impl == "reference":
        if rank != 0:
            return
        # CPU reference arm: the oracle port, bounded sample, extrapolated by FLOP ratio
        ts = []
        rep = None
        for _ in range(max(1, args.warmup // 3)):
            pass
        for _ in range(args.steps):
            t, rep, sample = cpu_sample(prob, cfg, eps_start)
            ts.append(t)
        t = float(np.median(ts))
        frac = _sample_fraction(args.config)
        value = t / frac if frac else None
        line = {"metric": "converged UOT domdec solve time (s)", "value": value, "unit": "s",
                "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": value * 1e3 if value else None, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_desc,
                "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": "port",
                                 "sample": f"{sample}: {t:.2f}s measured, extrapolated x{1 / frac:.1f} "
                                           "by the GPU run's cell-sweep FLOP ratio" if frac else sample},
                "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.multiscale import build_pyramid, stage_pyramid
    if world > 1:
        # shard every batch's cell solves across the ranks (NCCL sum of the
        # solve's output arenas; bitwise identical to one GPU)
        from paper_2410_08859_b200.engine import set_shard
        set_shard()

    levels = stage_pyramid(build_pyramid(prob.mu, prob.nu, cfg["coarsest"]), prob.div, prob.eps)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        run_solve(prob, cfg, eps_start, levels)
    torch.cuda.synchronize()
    # ---- device-timed region
    tracer = _lib.Tracer()
    times, reps = [], []
    launches = 0
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            _lib.set_tracer(tracer)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            st, rep = run_solve(prob, cfg, eps_start, levels)
            b.record()
            torch.cuda.synchronize()
            _lib.set_tracer(None)
            times.append(a.elapsed_time(b) / 1e3)
            reps.append(rep)
    launches = tracer.launches() // max(1, args.steps)
    # per-step time = the K timed steps' device time / K (max over ranks)
    red_dev = "cuda" if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu"
    t_dev = max_over_ranks(float(np.sum(times)) / len(times), device=red_dev)
    t_max_step = max_over_ranks(float(np.max(times)), device=red_dev)
    # ---- end-to-end through the public API (host arrays in, host result out)
    e2e_times = []
    h2d = 0
    d2h = 0
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        st2, rep2 = run_solve(prob, cfg, eps_start, None)
        d2h = fetch_result(st2)
        b.record()
        torch.cuda.synchronize()
        e2e_times.append(a.elapsed_time(b) / 1e3)
    lv_host = build_pyramid(prob.mu, prob.nu, cfg["coarsest"])
    h2d = int(sum(lv.mu.nbytes + lv.nu.nbytes for lv in lv_host) * 2)  # mass + log mass
    t_e2e = float(np.sum(e2e_times)) / len(e2e_times)
    # ---- roofline of the dominant kernel
    tm = tracer.times_ms()
    solve_ms = tm.get("dd_cell_solve", []) + tm.get("dd_cell_solve2", [])
    lse_ms = tm.get("dd_grid_lse", [])
    rep = reps[-1]
    flops = sum(r.diagnostics.get("cell_flops", 0.0) for _, _, r in rep.stages)
    n_launch = len(solve_ms) // max(1, args.steps)
    mean_ms = float(np.mean(solve_ms)) if solve_ms else float("nan")
    achieved = (flops / max(n_launch, 1)) / (mean_ms * 1e-3) / 1e12 if solve_ms else None
    roofline = {"bound": "fp64", "kernel": "dd_cell_solve (cell_solve_kernel + cluster variant)",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                "peak_source": "B200 nominal FP64 (no FP64 entry in MEASURED_PEAKS.json)",
                "flops_per_launch": flops / max(n_launch, 1), "launches_per_step": n_launch,
                "mean_launch_ms": mean_ms,
                "share_of_step": (sum(solve_ms) / 1e3 / args.steps) / t_dev if solve_ms else None,
                "grid_lse_share_of_step": (sum(lse_ms) / 1e3 / args.steps) / t_dev if lse_ms else None,
                "traffic": None}
    cpu = None
    if rank == 0 and args.cpu_sample:
        t_cpu, crep, sample = cpu_sample(prob, cfg, eps_start)
        stage0 = rep.stages[0][2].diagnostics.get("cell_flops", 0.0)
        frac = stage0 / flops if flops else None
        cpu = {"value": t_cpu / frac if frac else None, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"{sample}: {t_cpu:.2f}s measured on 1 core, extrapolated x{1 / frac:.1f} "
                         "by the GPU run's cell-sweep FLOP ratio (same iteration sequence)"}
        _save_fraction(args.config, frac)
    if rank == 0:
        line = {"metric": "converged UOT domdec solve time (s)", "value": t_dev, "unit": "s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_dev * 1e3, "higher_is_better": False,
                "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_desc,
                "max_step_s": t_max_step,
                "converged": bool(rep.converged), "rel_pd_gap": rep.rel_pd_gap,
                "final_total": rep.final_score.get("total"),
                "stages": [[n, e / prob.mu.grid.dx ** 2, r.iterations,
                            round(r.timings["total"], 3)] for n, e, r in rep.stages],
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": int(launches), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


_FRAC_FILE = os.path.join(ROOT, "profiles", "cpu_sample_fraction.json")


def _save_fraction(cfg, frac):
    try:
        d = json.load(open(_FRAC_FILE)) if os.path.exists(_FRAC_FILE) else {}
        d[cfg] = frac
        os.makedirs(os.path.dirname(_FRAC_FILE), exist_ok=True)
        json.dump(d, open(_FRAC_FILE, "w"), indent=1)
    except Exception:
        pass


def _sample_fraction(cfg):
    """FLOP fraction of the coarsest stage in the GPU run (recorded by a GPU bench run)."""
    try:
        return json.load(open(_FRAC_FILE)).get(cfg)
    except Exception:
        return None


if __name__ == "__main__":
    main()
