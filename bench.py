"""TT-GBF throughput bench (BASELINE.json metric: filter steps/s at d=6, N_pa=64 -> 65, rank <= 20).

Workload (BASELINE config 5 = config 3 batched): the 4096 seeded Monte Carlo
runs of the d=6 constant-velocity model, split evenly across the GPUs
(strong scaling; ``--batch B`` instead fixes B filters per GPU).  One bench
*step* = one ``tt_fft_pmf_step`` for every filter; all K timed steps of all
filters run in ONE persistent ``ttgbf_filter_run`` launch (device geometry,
per-step work claiming).  Filters that raise DegenerateDensityError restart
from the prior inside the timed region; only completed steps count.

  python bench.py [--gpus N --steps K --warmup W]
  python bench.py --impl reference ...   # the reference algorithm on the host cores
                                          # (oracle port; the Python reference cannot travel)

Multi-GPU: one process per GPU (``--gpus N`` re-launches itself under
torch.distributed.run when WORLD_SIZE is unset); runs are sharded by rank
with no data-path collective; the per-run squared-error sums are gathered
with one NCCL all_gather at the end.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2501_07942_b200.configs import BASELINE_CONFIGS, simulate  # noqa: E402

PROF_NAMES = ["miss_sort", "evaluator", "cache_eval", "core_lstsq", "hunt", "accept", "cache_check", "tt_round",
              "svd", "qr", "rng_choice", "snapshot", "chain_eval", "inject", "fft_conv", "neg_mass",
              "qr_panel", "qr_update", "round_rmul", "round_applyq", "fft_product", "svd_rrqr"]
METRIC = "TT-GBF filter steps/s (d=6, N_pa=64, rank<=20)"
WORKLOAD = "C5: d=6 CV, N_pa=64 (run as 65), rank cap 20, round tol 1e-8, cross tol 1e-2/max_rank 40, sigma 6"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--runs", type=int, default=0)     # total Monte Carlo runs (0: the config's, C5 = 4096)
    p.add_argument("--batch", type=int, default=0)    # filters per GPU (0: runs / GPUs, BASELINE config 5)
    p.add_argument("--slots", type=int, default=0)     # resident CTAs (0: SMs x ttgbf_ctas_per_sm)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C5")
    p.add_argument("--ws-mb", type=int, default=0)        # per resident CTA slot (0: split free HBM)
    # overflow workspaces for oversized FFT products: 64 x 800 MB (products with
    # 50 % headroom) + 24 x 1280 MB (the rest); measured: CTA time waiting for a
    # buffer 800 -> 73 CTA-s per launch vs one class of 56 x 1280 MB
    p.add_argument("--big-slots", type=int, default=64)
    p.add_argument("--big-mb", type=int, default=800)
    p.add_argument("--big2-slots", type=int, default=24)
    p.add_argument("--big2-mb", type=int, default=1280)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-s", type=float, default=20.0)
    p.add_argument("--dump", default=None, help="save the timed run's step records (npz) for analysis")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def trajectories(cfg, runs):
    spec = cfg["spec"]
    st, ms = [], []
    for r in runs:
        s, m = simulate(spec, cfg["x0_mean"], cfg["x0_cov"], cfg["steps"], np.random.SeedSequence((2024, int(r), 0)))
        st.append(s)
        ms.append(m)
    return np.stack(st), np.stack(ms)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.index),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
               "utilization.gpu,utilization.memory",
               "--format=csv,noheader,nounits", "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if len(s) > 2 and s[2].replace(".", "").isdigit()]
        mem = [float(s[9]) for s in self.samples if len(s) > 9 and s[9].isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": float(np.median(pw)) if pw else None,
                "mem_util_pct_median": float(np.median(mem)) if mem else None}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------
_W = {}   # per-process oracle filter state of the CPU reference arm


def _oracle_init(cfg_name, worker, stride):
    """Worker state: runs worker, worker + stride, ... of the config, each from
    the prior with its own SeedSequence((2024, run, 0)) trajectory."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _W.update(cfg=cfg_name, run=worker - stride, stride=stride, state=None)


def _oracle_new_run():
    from oracle import pmf
    cfg = BASELINE_CONFIGS[_W["cfg"]]
    _W["run"] += _W["stride"]
    _, meas = simulate(cfg["spec"], cfg["x0_mean"], cfg["x0_cov"], cfg["steps"],
                       np.random.SeedSequence((2024, _W["run"], 0)))
    g = _W["g"] = {"n_per_axis": cfg["grid"]["n_per_axis"], "sigma_mult": cfg["grid"]["sigma_mult"],
                   "round_tol": cfg["grid"]["round_tol"], "round_max_rank": cfg["grid"]["round_max_rank"]}
    axes, cores, _ = pmf.initial(cfg["x0_mean"], cfg["x0_cov"], g, cfg["cross"])
    _W["state"] = [axes, cores, 0, meas]


def _oracle_restart():
    from oracle import pmf
    cfg = BASELINE_CONFIGS[_W["cfg"]]
    axes, cores, _ = pmf.initial(cfg["x0_mean"], cfg["x0_cov"], _W["g"], cfg["cross"])
    _W["state"][:3] = [axes, cores, 0]


def _oracle_advance(arg):
    """Run this worker's filters for ~budget_s (or exactly `steps` attempted
    steps): the GPU arm's policy -- a failed step restarts its filter from the
    prior, a finished trajectory moves to the worker's next run.  Returns
    (completed steps, seconds)."""
    budget_s, steps = arg
    from oracle import pmf
    cfg = BASELINE_CONFIGS[_W["cfg"]]
    done = att = 0
    t0 = time.perf_counter()
    if _W["state"] is None:
        _oracle_new_run()
    while (steps and att < steps) or (not steps and time.perf_counter() - t0 < budget_s):
        axes, cores, k, meas = _W["state"]
        att += 1
        try:
            axes, cores, _ = pmf.step(axes, cores, cfg["spec"], meas[k], _W["g"], cfg["cross"])
            done += 1
            _W["state"][:3] = [axes, cores, k + 1]
            if k + 1 >= cfg["steps"]:
                _oracle_new_run()
        except pmf.Degenerate:
            _oracle_restart()
    return done, time.perf_counter() - t0


class CpuReference:
    """The reference algorithm (oracle port) on `cores` host processes, one
    filter stream each (runs interleaved across workers), state kept across
    samples so successive samples walk through the run set instead of
    re-timing the same first steps."""

    def __init__(self, cfg_name, cores):
        import multiprocessing as mp
        self.cores = cores
        self.pools = [mp.get_context("spawn").Pool(1, _oracle_init, (cfg_name, w, cores)) for w in range(cores)]

    def sample(self, budget_s=0.0, steps=0):
        res = [p.apply_async(_oracle_advance, ((budget_s, steps),)) for p in self.pools]
        out = [r.get() for r in res]
        done = sum(o[0] for o in out)
        wall = max(o[1] for o in out)
        # aggregate rate = sum of the workers' own rates (a worker finishing a
        # long step late does not idle the others in the count)
        return sum(o[0] / o[1] for o in out if o[1] > 0), done, wall

    def close(self):
        for p in self.pools:
            p.terminate()


def cpu_reference(cfg_name, cores, budget_s):
    """Completed oracle steps/s over `cores` worker processes, each for ~budget_s."""
    ref = CpuReference(cfg_name, cores)
    try:
        return ref.sample(budget_s)
    finally:
        ref.close()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    budget = max(5.0, min(60.0, 150.0 / max(1, args.steps + args.warmup)))
    ref = CpuReference(args.config, cores)
    try:
        # warm-up: every worker advances its first filter (the GPU arm's W warm-up steps)
        ref.sample(steps=args.warmup)
        vals = []
        t0 = time.perf_counter()
        done_total = 0
        for _ in range(args.steps):
            v, done, wall = ref.sample(budget)
            vals.append(v)
            done_total += done
        elapsed = time.perf_counter() - t0
    finally:
        ref.close()
    value = float(np.mean(vals))
    sample = (f"{args.steps} samples x {cores} processes x ~{budget:.0f}s of {args.config} oracle steps; "
              f"{done_total} completed steps; each process walks its own runs (run = worker + {cores} j) "
              f"after {args.warmup} untimed warm-up steps, restarting failed filters from the prior")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded trajectories)",
        "config": {"workload": WORKLOAD, "parallelism": "host processes"},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def dram_traffic_per_step():
    """DRAM bytes per attempted filter step of ttgbf_filter_run, from the newest
    committed ncu capture (dram__bytes_read.sum + dram__bytes_write.sum of a
    296-filter one-step launch, profiles/rNN_ncu_dram_c5.json)."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_dram_c5.json")))
    if not paths:
        return None, None
    rec = json.load(open(paths[-1]))
    return (float(rec["dram_bytes_per_attempted_step"]),
            f"profiles/{os.path.basename(paths[-1])} ({rec['kernel']}) x attempted steps")


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    from paper_2501_07942_b200 import build as pbuild
    if not pbuild.up_to_date():
        pbuild.build()
    from paper_2501_07942_b200 import roofline as rl
    from paper_2501_07942_b200.bank import BankConfig, FilterBank

    cfg = BASELINE_CONFIGS[args.config]
    g, x = cfg["grid"], cfg["cross"]
    from paper_2501_07942_b200.mc import shard
    total_runs = args.batch * world if args.batch > 0 else (args.runs or int(cfg["runs"]))
    runs = shard(total_runs, world, rank)          # strong scaling: the fixed C5 run set split across GPUs
    B = len(runs)
    from paper_2501_07942_b200 import _abi
    lib = _abi.load_library()
    if args.slots <= 0:
        args.slots = torch.cuda.get_device_properties(local).multi_processor_count * int(lib.ttgbf_ctas_per_sm())
    if args.ws_mb <= 0:
        free = torch.cuda.mem_get_info(local)[0]
        reserve = ((args.big_slots * args.big_mb + args.big2_slots * args.big2_mb) << 20) + B * (1 << 17) * 8 + (8 << 30)
        args.ws_mb = int(max(128, min(512, (free - reserve) // args.slots >> 20)))
    bcfg = BankConfig(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                      round_max_rank=g["round_max_rank"], tol=x["tol"], max_rank=x["max_rank"],
                      rng_seed=x["rng_seed"], ws_bytes=args.ws_mb << 20, state_doubles=1 << 17,
                      cache_cap=1 << 20, ws_slots=args.slots, big_slots=args.big_slots,
                      big_bytes=args.big_mb << 20, big2_slots=args.big2_slots, big2_bytes=args.big2_mb << 20)
    d = cfg["spec"]["F"].shape[0]
    b = np.atleast_2d(cfg["spec"]["R"]).shape[0]
    n = g["n_per_axis"]
    states, meas = trajectories(cfg, runs)
    kf = cfg["steps"]
    dev = torch.device("cuda", local)
    peak_fp64 = rl.measure_fp64_peak(torch, dev)
    peak_fp64_sustained = rl.measure_fp64_sustained(torch, dev)
    bank = FilterBank(cfg["spec"], bcfg, B)
    stats = {"flops": 0.0, "flops_exec": 0.0, "cycles": np.zeros(8), "prof": np.zeros(32), "ranks": None}

    # warm-up: W filter steps per filter (one persistent launch)
    if args.warmup:
        bank.run(meas, args.warmup, cfg["x0_mean"], cfg["x0_cov"])
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    bank.timeline = []
    h2d0, d2h0 = bank.bytes_h2d, bank.bytes_d2h
    with Clocks(local) as clk:
        t0 = time.perf_counter()
        recs = bank.run(meas, args.steps, cfg["x0_mean"], cfg["x0_cov"])   # K steps, one launch
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
    if world > 1:
        torch.distributed.barrier()
    dg = bank._diag()
    if args.dump:
        np.savez_compressed(args.dump, recs=recs, cycles=dg["cycles"], prof=dg["prof"])
    ok = recs["status"] == 0
    stats["completed"] = int(ok.sum())
    stats["failed"] = int((recs["status"] > 0).sum())
    stats["restarts"] = int((recs["status"] != 0).sum())
    vals, cnts = np.unique(recs["status"], return_counts=True)
    stats["status_counts"] = {str(int(v)): int(n) for v, n in zip(vals, cnts)}
    step_fl = []
    for i, s_ in zip(*np.nonzero(recs["status"] >= 0)):
        fl = sum(rl.rec_flops(recs[i, s_], d, b, n))
        stats["flops"] += fl
        stats["flops_exec"] += sum(rl.rec_flops(recs[i, s_], d, b, n, executed=True))
        step_fl.append(fl)
    step_fl = np.array(step_fl) if step_fl else np.zeros(1)
    stats["step_gflop_pcts"] = [round(float(np.percentile(step_fl, q)) / 1e9, 3) for q in (50, 90, 99, 100)]
    cyc = recs["cycles"][recs["status"] >= 0].astype(float) / 1.965e9
    stats["step_ms_pcts"] = [round(1e3 * float(np.percentile(cyc, q)), 2) for q in (50, 90, 99, 100)] if cyc.size else None
    stats["step_sm_s_total"] = float(recs["cycles"].astype(float).sum() / 1.965e9)
    stats["cycles"] = dg["cycles"].sum(axis=0).astype(float)
    stats["prof"] = dg["prof"].sum(axis=0).astype(float)
    stats["ws_peak"] = int(dg["ws_peak"].max())
    stats["big_used"] = int(dg["big_used"].sum())
    stats["big_peak"] = int(dg["big_peak"].max())
    stats["big_wait_s"] = float(dg["big_wait"].sum() / 1.965e9)
    att = recs["status"] >= 0
    stats["calls"] = {nm: float(recs["calls"][:, :, q][att].mean()) if att.any() else 0.0
                      for q, nm in enumerate(["likelihood", "kernel", "realign"])}
    stats["stage_s_per_step"] = (dg["cycles"].sum(axis=0) / 1.965e9 / max(1, int(att.sum()))).round(4).tolist()
    if ok.any():
        i0, s0 = [int(v[0]) for v in np.nonzero(ok)]
        stats["ranks"] = {nm: [int(v) for v in recs[i0, s0]["ranks"][sl][: d + 1]]
                          for sl, nm in [(3, "shifted"), (4, "kernel"), (9, "kernel_squeezed"), (5, "conv"),
                                         (6, "realign")]}
    from paper_2501_07942_b200.mc import gather_rmse, run_error_sums
    local_err = run_error_sums(recs["mean"], states, recs["k"], ok, d)
    dev_s = sum(a.elapsed_time(e) / 1e3 for _, a, e in bank.timeline)
    per_kernel = {}
    for name, a, e in bank.timeline:
        per_kernel.setdefault(name, []).append(a.elapsed_time(e) / 1e3)
    kern_total = sum(sum(v) for v in per_kernel.values())
    # max over ranks of the device time; completed steps summed
    t_max, done_all = dev_s, stats["completed"]
    wall_max = wall
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([dev_s, wall], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max, wall_max = float(tt[0]), float(tt[1])
        cc = torch.tensor([float(stats["completed"])], device=dev, dtype=torch.float64)
        dist.all_reduce(cc)
        done_all = int(cc[0])
    # RMSE statistics: one NCCL all_gather of per-run sums, no other collective
    rmse, _ = gather_rmse(local_err, device=dev if world > 1 else None)
    rmse = rmse.tolist()

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    value = done_all / t_max
    e2e = done_all / wall_max
    dom = max(per_kernel, key=lambda k: sum(per_kernel[k]))
    dom_time = sum(per_kernel[dom]) / len(per_kernel[dom])
    flops_per_launch = stats["flops"] / max(1, len(per_kernel[dom]))
    achieved = flops_per_launch / dom_time / 1e12
    achieved_exec = stats["flops_exec"] / max(1, len(per_kernel[dom])) / dom_time / 1e12
    per_step, traffic_src = dram_traffic_per_step()
    attempted = int((recs["status"] >= 0).sum())
    traffic_per_launch = per_step * attempted / max(1, len(per_kernel[dom])) if per_step else None
    hbm_peak = None
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        hbm_peak = json.load(open(pk)).get("hbm_gbs")
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.batch <= 0 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded trajectories, SeedSequence((2024, run, 0)))",
        "config": {"workload": WORKLOAD, "filters_per_gpu": B, "runs": total_runs, "parallelism": f"dp{world}",
                   "workspace_slots": args.slots, "workspace_mb_per_slot": args.ws_mb,
                   "l2": "per-filter working sets stream from HBM (batch footprint >> 126 MB L2)",
                   "completed_steps": done_all, "restarts": stats["restarts"], "failed_steps": stats["failed"],
                   "status_counts": stats["status_counts"]},
        "gpu_launches": len(bank.timeline),
        "launch_note": "one persistent ttgbf_filter_run launch runs all K steps of all filters (device geometry)",
        "roofline": {"bound": "tensor", "precision": "fp64", "kernel": dom, "achieved": achieved,
                     "peak": peak_fp64, "unit": "TFLOP/s", "frac": achieved / peak_fp64,
                     "traffic": traffic_per_launch,
                     "traffic_source": traffic_src,
                     "hbm_achieved_gbs": (traffic_per_launch / dom_time / 1e9) if traffic_per_launch and dom_time else None,
                     "hbm_peak_gbs": hbm_peak,
                     "peak_source": "cuBLAS DGEMM 8192^3 burst measured in this run (MEASURED_PEAKS.json has no FP64)",
                     "peak_sustained": peak_fp64_sustained,
                     "frac_of_sustained": achieved / peak_fp64_sustained,
                     "algorithmic_flops_per_launch": flops_per_launch, "launch_s": dom_time,
                     "flops_model": "SURVEY 8(d) formulas on the reference algorithm's shapes (products of the "
                                    "cross outputs as they come)",
                     "achieved_executed": achieved_exec, "frac_executed": achieved_exec / peak_fp64,
                     "executed_note": "same formulas on the product ranks after the engine's exact-rank squeeze "
                                      "of the likelihood/kernel cross outputs (what the kernels actually factor)"},
        "kernel_time_s": {k: sum(v) for k, v in per_kernel.items()},
        "device_busy_frac": kern_total / dev_s if dev_s > 0 else None,
        "stage_cycles_share": (stats["cycles"] / max(stats["cycles"].sum(), 1)).round(4).tolist(),
        "engine_prof_share": dict(zip(PROF_NAMES, (stats["prof"][:22] / max(stats["cycles"].sum(), 1)).round(4).tolist())),
        "lstsq_factor_share": round(float(stats["prof"][31] / max(stats["cycles"].sum(), 1)), 4),
        "squeeze_share": round(float(stats["prof"][30] / max(stats["cycles"].sum(), 1)), 4),
        "svd_rrqr_mean_rank": float(stats["prof"][22] / max(stats["prof"][23], 1)),
        "svd_detail": {"max_rank": int(dg["prof"][:, 24].max()),
                       "jacobi": round(float(stats["prof"][25] / max(stats["cycles"].sum(), 1)), 4),
                       "u_apply": round(float(stats["prof"][26] / max(stats["cycles"].sum(), 1)), 4),
                       "bt_qr_v": round(float(stats["prof"][27] / max(stats["cycles"].sum(), 1)), 4),
                       "calls_rank_gt64": int(stats["prof"][28]),
                       "share_rank_gt64": round(float(stats["prof"][29] / max(stats["cycles"].sum(), 1)), 4)},
        "completed_frac": stats["completed"] / max(1, B * args.steps),
        "ws_peak_mb": stats["ws_peak"] / 2 ** 20,
        "overflow_ws": {"slots": args.big_slots, "mb": args.big_mb, "slots2": args.big2_slots, "mb2": args.big2_mb,
                        "steps_used": stats["big_used"],
                        "peak_mb": stats["big_peak"] / 2 ** 20, "cta_seconds_waiting": stats["big_wait_s"]},
        "mean_cross_calls": stats["calls"],
        "step_gflop_p50_p90_p99_max": stats["step_gflop_pcts"],
        "step_ms_p50_p90_p99_max": stats["step_ms_pcts"],
        "cta_seconds_in_steps": stats["step_sm_s_total"],
        "stage_sm_seconds_per_attempted_step": stats["stage_s_per_step"],
        "example_ranks": stats["ranks"],
        "rmse": rmse,
        "clocks": clk.summary(),
        "e2e": {"value": e2e, "unit": "steps/s",
                "h2d_bytes_per_step": (bank.bytes_h2d - h2d0) / args.steps,
                "d2h_bytes_per_step": (bank.bytes_d2h - d2h0) / args.steps,
                "note": "FilterBank.run API: host measurement trajectories in, host step records out, wall clock"},
    }
    if world == 1 and not args.no_cpu_baseline:
        v, done, w = cpu_reference(args.config, 1, args.cpu_sample_s)
        line["cpu_baseline"] = {"value": v, "unit": "steps/s", "cores": 1, "kind": "port",
                                "sample": f"{done} oracle steps of {args.config} run 0 from the prior in {w:.1f}s "
                                          "(1 thread)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def self_launch(args) -> int:
    """--gpus N outside torchrun: re-run this command as N ranks (one per GPU)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
