#!/usr/bin/env python
"""Benchmark: converged multiscale unbalanced domdec solve on B200.

One "step" is one full converged solve of a BASELINE.json configuration.
Default ``ms_1024`` = configs[2], the metric's own config (1024^2, 8-Gaussian
mixtures + 1e-5 floor, masses 1.0 / 1.5, lambda = 1, eps annealed 256h^2 ->
2h^2 over the 64^2 -> 1024^2 pyramid, 8x8 basic cells with 2x2 composites,
fp64, staggered strategy, delta = 2e-5), solved with the SPEC / paper §4.3.1
multiscale protocol (global Sinkhorn at delta/4 below layer 8, domdec from
512^2).  ``--config ms_256`` runs configs[1].  The metric is the solve time in
seconds (lower is better).

* ``value``  — device-timed solve (CUDA events on the launching stream) with the
  pyramid already resident in HBM; L2 is flushed (256 MiB write) before each step.
* ``e2e``    — the same solve through the public API from host arrays: the
  host->device copy of every pyramid level and the device->host read of the
  result (basic-cell marginals, duals) inside the timed region.
* ``roofline`` — the dominant kernel (``dd_cell_solve``): algorithmic FP64
  FLOPs of its separable contractions per launch / mean launch time (CUDA
  events), against the FP64 DFMA peak measured on B200
  (``profiles/fp64_peak.json``, scripts/micro/fp64_peak.cu); DRAM traffic per
  launch and FP64-pipe utilisation from the committed ncu capture.
* ``cpu_baseline`` — the reference algorithm (the CPU oracle restatement) on a
  bounded sample of the same workload: complete composite-cell subproblems
  recorded from the 1024^2 stage (``tests/golden/ms1024_cells.npz``), solved
  process-parallel over all host cores with a bounded cell iteration cap; the
  measured time is reported together with its scaling to the whole solve by
  algorithmic cell-sweep work (labelled as a scaled estimate).
* ``--impl reference`` — that same CPU sample, timed per step on the host
  cores; ``value`` is the measured seconds of one sample (what ran), the scaled
  whole-solve estimate is a separate labelled field.

Multi-GPU (``--gpus N`` under torchrun): row-slab sharding (slab.py) — each
rank owns a contiguous slab of block rows and solves its composites; the Y
snapshot and blend sums are all-reduced per batch and the boundary block row
moves between neighbours at every A/B switch (strong scaling: the whole job
solves one problem); value is the max over ranks.
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

CONFIGS = {"pr1_64": 0, "ms_256": 1, "ms_1024": 2, "ms_2048": 3, "vol_128": 4}
FP64_NOMINAL_TFLOPS = 40.0   # B200 datasheet FP64 (fallback when no measurement is committed)
SAMPLE_CAP = 100             # cell iteration cap of the CPU sample


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("DD_BENCH_CONFIG", "ms_1024"),
                    choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=1, help="run the CPU baseline sample")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="fp32: north_star fp32 mode (cell sweeps in fp32, 1e-4 parity)")
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


PRECISION = "fp64"


def run_solve(prob, cfg, eps_start, levels=None):
    from paper_2410_08859_b200.engine import CellSolverConfig, EngineConfig, StrategyConfig
    from paper_2410_08859_b200.multiscale import multiscale_solve

    return multiscale_solve(prob, cfg["cell"], cfg["coarsest"], eps_start,
                            strategy=StrategyConfig("staggered"),
                            config=EngineConfig(cell=CellSolverConfig(precision=PRECISION)),
                            levels=levels)


def fetch_result(st):
    """Device->host read of the result a caller consumes: boxes, marginals, duals, score."""
    boxes, vals, _ = st.download_marginals()    # compacted on the device
    duals = [t.cpu() for t in st.global_duals] if st.global_duals is not None else []
    d2h = boxes.nbytes + vals.nbytes + sum(t.numel() * 8 for t in duals)
    return d2h


def cpu_sample(workers=None):
    """Oracle solves of the recorded 1024^2 cell sample (bounded cap), all host cores."""
    from oracle.cell_sample import run_sample, sample_flops

    wall, iters, cores, d, probs = run_sample(SAMPLE_CAP, workers)
    fl = sample_flops(probs, iters, int(d["nw0"]), int(d["nw1"]))
    desc = (f"{len(probs)} complete composite-cell subproblems of the first staggered batch of "
            f"the 1024^2 stage (tests/golden/ms1024_cells.npz), oracle cell solver (reference "
            f"cells.py restated), cell cap {SAMPLE_CAP}: {int(iters.sum())} cell iterations, "
            f"{fl:.3e} algorithmic FLOPs, {wall:.2f} s on {cores} processes")
    return wall, fl, cores, desc, d


def _peak():
    """Measured FP64 DFMA peak (profiles/fp64_peak.json) or the datasheet fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return float(d["tflops"]), f"measured FP64 DFMA peak on B200 ({d.get('how', '')})"
    except Exception:
        return FP64_NOMINAL_TFLOPS, "B200 datasheet FP64 (no measured FP64 peak committed)"


def _ncu_profile(nd=2, precision="fp64"):
    """Committed ncu --set full summary of the dominant kernel of this path (2D / three-axis,
    fp64 / fp32 mode): DRAM bytes per launch and pipe utilisation for roofline.traffic."""
    name = "r02_ncu_cell_solve" + ("3" if nd == 3 else "") + ("_fp32" if precision == "fp32" else "")
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name + ".json")))
    except Exception:
        return None


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
    global PRECISION
    PRECISION = args.precision
    dtype = "f64" if args.precision == "fp64" else "f32 cell sweeps / f64 state"
    prob, cfg, eps_start = problem(args.config, args.seed)
    dims = prob.mu.grid.dims
    nd = len(dims)
    xs = "x".join(str(n) for n in dims)
    cellx = "x".join([str(cfg["cell"])] * nd)
    comp = "x".join(["2"] * nd)
    config_desc = {"workload": f"{args.config}: BASELINE configs[{CONFIGS[args.config]}] "
                               f"{xs} multiscale "
                               f"{cfg['coarsest']}^{nd}->{dims[0]}^{nd}, "
                               f"eps {eps_start / prob.mu.grid.dx ** 2:g}h^2->{prob.eps / prob.mu.grid.dx ** 2:g}h^2, "
                               f"lambda={cfg['lam']}, cells {cellx} ({comp} composites), "
                               "staggered, delta=2e-5, SPEC multiscale (global Sinkhorn at delta/4 below "
                               "layer 8 / the finest layer, domdec above)"
                               + (", three-axis path (volume.py, csrc/vol.cu)" if nd == 3 else ""),
                   "grid": list(prob.mu.grid.dims), "cell": cfg["cell"], "lambda": cfg["lam"],
                   "strategy": "staggered", "l2": "flushed (256 MiB write) before every step",
                   "parallelism": (f"row-slab x{world} (each rank solves the composites of its "
                                   "block-row slab; NCCL all-reduce of the Y snapshot and blend "
                                   "sums per batch, halo exchange of the boundary block row "
                                   "at each A/B switch)") if world > 1 else "1 GPU",
                   "seed": args.seed, "precision": args.precision}

    if args.impl == "reference":
        if rank != 0:
            return
        # CPU reference arm: the oracle (reference algorithm restated) on the
        # recorded cell sample, process-parallel over the host cores
        from oracle.cell_sample import run_sample
        run_sample(2, None)          # warm-up: process pool and numpy paths
        ts = []
        for _ in range(args.steps):
            t, fl, cores, sample, d = cpu_sample()
            ts.append(t)
        t = float(np.median(ts))
        full = float(d["full_solve_cell_flops"])
        line = {"metric": "converged UOT domdec solve time (s)", "value": t, "unit": "s",
                "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": 1,
                "ms_per_step": t * 1e3, "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": config_desc,
                "cpu_baseline": {"value": t, "unit": "s", "cores": cores, "kind": "port",
                                 "sample": sample},
                "scaled_full_solve_s": {"value": t * full / fl, "how":
                                        "measured sample seconds x (algorithmic cell-sweep FLOPs "
                                        "of one whole converged GPU solve / the sample's); an "
                                        "estimate, not a measurement"},
                "e2e": {"value": t, "unit": "s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    from paper_2410_08859_b200 import _lib
    from paper_2410_08859_b200.multiscale import build_pyramid, stage_pyramid
    if world > 1:
        # row-slab sharding of every domdec solve (slab.py)
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
    solve_ms = (tm.get("dd_cell_solve", []) + tm.get("dd_cell_solve2", [])
                + tm.get("dd3_cell_solve", []))
    lse_ms = tm.get("dd_grid_lse", []) + tm.get("dd3_grid_lse", [])
    rep = reps[-1]
    flops = sum(r.diagnostics.get("cell_flops", 0.0) for _, _, r in rep.stages)
    n_launch = len(solve_ms) // max(1, args.steps)
    mean_ms = float(np.mean(solve_ms)) if solve_ms else float("nan")
    achieved = (flops / max(n_launch, 1)) / (mean_ms * 1e-3) / 1e12 if solve_ms else None
    peak, peak_src = _peak()
    prof = _ncu_profile(nd, args.precision)
    traffic = None
    if prof is not None:
        traffic = {"dram_bytes_per_launch": prof.get("dram_bytes"),
                   "achieved_gbs": prof.get("dram_gbs"),
                   "fp64_pipe_pct": prof.get("fp64_pipe_pct"),
                   "source": prof.get("source")}
    kname = ("dd3_cell_solve (cell_solve3_kernel)" if nd == 3 else
             "dd_cell_solve (cell_solve_kernel + cluster variant)")
    roofline = {"bound": "fp64", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if achieved else None, "peak_source": peak_src,
                "flops_per_launch": flops / max(n_launch, 1), "launches_per_step": n_launch,
                "mean_launch_ms": mean_ms,
                "share_of_step": (sum(solve_ms) / 1e3 / args.steps) / t_dev if solve_ms else None,
                "grid_lse_share_of_step": (sum(lse_ms) / 1e3 / args.steps) / t_dev if lse_ms else None,
                "traffic": traffic}
    cpu = None
    if rank == 0 and args.cpu_sample and world == 1 and args.config == "ms_1024":
        t_cpu, fl_cpu, cores, sample, _ = cpu_sample()
        cpu = {"value": t_cpu, "unit": "s", "cores": cores, "kind": "port", "sample": sample,
               "scaled_full_solve_s": t_cpu * flops / fl_cpu,
               "scaling": "measured sample seconds x (this run's algorithmic cell-sweep FLOPs per "
                          "solve / the sample's): an estimate of one whole solve on these cores"}
    if rank == 0:
        line = {"metric": "converged UOT domdec solve time (s)", "value": t_dev, "unit": "s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_dev * 1e3, "higher_is_better": False,
                "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic", "config": config_desc,
                "max_step_s": t_max_step,
                "converged": bool(rep.converged), "rel_pd_gap": rep.rel_pd_gap,
                "final_total": rep.final_score.get("total"),
                "stages": [[n, e / prob.mu.grid.dx ** 2, r.diagnostics.get("solver", "domdec"),
                            r.iterations, round(r.timings["total"], 3),
                            r.diagnostics.get("nonconverged_cells", 0)] for n, e, r in rep.stages],
                "stage_fields": ["grid n", "eps/h^2", "solver", "iterations", "seconds",
                                 "capped cell solves"],
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": int(launches), "clocks": clk.summary()}
        if args.precision == "fp32" and any("sweep_fallbacks" in r.diagnostics
                                            for _, _, r in rep.stages):
            line["fp32_sweeps"] = {
                "cell_sweeps": int(sum(2 * r.diagnostics.get("cell_iterations", 0)
                                       for _, _, r in rep.stages)),
                "redone_in_fp64": int(sum(r.diagnostics.get("sweep_fallbacks", 0)
                                          for _, _, r in rep.stages))}
        if world > 1:
            from paper_2410_08859_b200.engine import _SHARD as sh
            if sh is not None:
                line["slab"] = {"halo_and_replicate_bytes_sent_rank0": int(sh.bytes_exchanged),
                                "note": "point-to-point payload of rank 0 over all timed and "
                                        "untimed solves; per-batch dense all-reduces (Y snapshot, "
                                        "blend sums) are ny doubles each"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
