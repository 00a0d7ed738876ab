#!/usr/bin/env python
"""Benchmark of the FP32 sqrt-BA hot path on B200 (BASELINE.json metric: "LM iterations/s and
QR-marginalized obs/s (FP32) at 1-8 B200; % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one Levenberg-Marquardt iteration (every SURVEY §8a row: linearize, marginalize + damp,
preconditioner, PCG with the matrix-free RCS product, back-substitution, trial cost, LM update) of
the seeded synthetic workload `--config` (default 4: venice1778-shaped, 5.0M observations; its
15.7 GB landmark-block arena is far larger than the 126 MB L2, so no flush is needed).  W warm-up
iterations run first; then the state is reset to the seeded start and K iterations are timed with
CUDA events on the solver's stream, bracketed by barrier + synchronize, max over ranks; the K
iterations run as one device-side loop (rba_lm_solve), so the timed region has a single host
synchronization.  With N > 1
(torchrun) landmarks are sharded across ranks (strong scaling, fixed problem) and the camera
vectors are all-reduced over NCCL inside librba.

`--impl reference` times the FP64 CPU oracle (the reference arm of this tier) on the full workload:
each phase of an LM iteration once, composed over the oracle's own recorded LM trajectory; rank 0
only.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2103_01843_b200 import synth  # noqa: E402

WORKLOADS = {
    1: "cfg1: tiny circle BA, 16 cams, 200 lms, ~1.1k obs",
    2: "cfg2: trafalgar257-shaped street BA, 257 cams, 65k lms, ~225k obs",
    3: "cfg3: dubrovnik356-shaped street BA, 356 cams, 226k lms, ~1.26M obs",
    4: "cfg4: venice1778-shaped street BA, 1778 cams, 993k lms, ~5.0M obs (0.5% tracks 50-400)",
    5: "cfg5: final13682-shaped street BA, 13682 cams, 4.46M lms, ~30M obs",
}
SOLVERS = {"sqrtba": 0, "sc32": 1, "sc64": 2}
METRIC = "LM iterations/s (FP32 sqrt-BA step) and QR-marginalized obs/s; % of HBM roofline"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy benchmark)"
    return 6650.0, "fallback (B200_PROFILING.md)"


MATVEC_KERNELS = re.compile(r"k_large_pipe<\d+, \d+, (0|false)>|k_small_pipe<(0|false)>|k_huge_y|k_huge_out<(0|false)>|"
                            r"k_huge_fused|k_fac_matvec|k_sc_spmv|k_rcs64_(ws|tma)<[^>]*(0|false)>|k_pcg_a")
MARG_KERNELS = re.compile(r"k_marg_(small|large)<|k_marg64")


def _round_key(f):
    """Sort key of a profiles/ capture name r<round>[<letter>]_...: (round, refresh letter); names
    that do not follow the pattern sort first."""
    m = re.search(r"/r(\d+)([a-z]?)_[^/]*$", f)
    return (int(m.group(1)), m.group(2)) if m else (-1, "")


def ncu_traffic(cfg, variant=""):
    """DRAM bytes (read + write) of ONE launch of the matvec and of the marginalization, summed over
    their per-class kernels, from the newest committed `ncu --set full` summary of this config
    (profiles/r*_cfg<cfg>_ncu_full.json, written by tools/ncu_summary.py).  None if absent."""
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_cfg{cfg}{variant}_ncu_full.json")),
                   key=_round_key)
    if not files:
        return None, None, None
    rows = json.load(open(files[-1]))

    def first_of_each(rx):
        # one launch of each matching kernel, counted from the first non-reduction match on (the
        # slice reduction of the preconditioner pass precedes the first product)
        seen, tot, on = set(), 0.0, False
        for r in rows:
            name = r["kernel"].split("(")[0].replace("void ", "")
            if not rx.search(name):
                continue
            on = on or "reduce" not in name
            if on and name not in seen:
                seen.add(name)
                tot += r["dram_read_bytes"] + r["dram_write_bytes"]
        return tot if seen else None

    return first_of_each(MATVEC_KERNELS), first_of_each(MARG_KERNELS), os.path.relpath(files[-1], ROOT)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, smax = [], []
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_phase_times(prob, cfg):
    """The FP64 oracle, as it stands, on the FULL workload (no subsample): each phase of an LM
    iteration timed once on the box's host cores -- O1-O5 (linearize, Givens QR marginalization,
    damping), a re-damp (backtracking), O6 preconditioner + b~, PCG iterations (O6 product + O7
    vector work), O8 back-substitution + O9 trial cost.  Returns (phase seconds, description)."""
    import oracle
    o = oracle.Oracle(prob)
    t = {}
    t0 = time.perf_counter()
    o.linearize()
    o.marginalize()
    o.damp(1e-4)
    t["linearize_marginalize"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    o.damp(2e-4)
    t["redamp"] = time.perf_counter() - t0
    o.damp(1e-4)
    t0 = time.perf_counter()
    o.precond_rhs()
    t["precond"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    it, _, _ = o.pcg(0.0, 2)
    t["pcg_iteration"] = (time.perf_counter() - t0) / max(it, 1)
    t0 = time.perf_counter()
    o.backsub()
    o.model_decrease()
    o.trial_cost()
    t["trial"] = time.perf_counter() - t0
    return t, oracle.num_threads()


def compose_oracle(t, iters):
    """Seconds of the oracle's LM iterations with the given (relinearized, pcg_iters) sequence."""
    return sum((t["linearize_marginalize"] if relin else t["redamp"]) + t["precond"] + n * t["pcg_iteration"] +
               t["trial"] for relin, n in iters)


def oracle_trajectory(cfg):
    """The oracle's own LM trajectory on this config (tests/oracle_data/cfg<C>_lm*.json, written by
    tools/oracle_trajectory.py, which calls only oracle/)."""
    files = sorted(glob.glob(os.path.join(ROOT, "tests", "oracle_data", f"cfg{cfg}_lm*.json")))
    if not files:
        return None
    d = json.load(open(files[-1]))
    its = d["iterations"]
    relin = [True] + [bool(r["accepted"]) for r in its[:-1]]
    return [(rl, int(r["pcg_iters"])) for rl, r in zip(relin, its)], os.path.relpath(files[-1], ROOT)


def bench_config(args, prob, world):
    """The workload description shared by both arms (ours and --impl reference)."""
    return {"workload": WORKLOADS[args.config], "cfg": args.config, "n_p": int(prob["cameras_init"].shape[0]),
            "n_l": int(prob["points_init"].shape[0]), "n_obs": int(len(prob["obs_cam"])),
            "solver": {"sqrtba": "sqrt-BA-32 (QR nullspace marginalization)", "sc32": "explicit-32 (Schur complement)",
                       "sc64": "explicit-64 (Schur complement)"}[args.solver],
            "storage": args.storage, "precision": args.precision,
            "parallelism": f"landmark-shard x{world}",
            "l2": "inputs larger than L2 (landmark-block arena >> 126 MB)" if args.config >= 3 else
            "working set L2-resident (no flush)"}


def bench_reference(args, prob, rank):
    """Reference arm: the FP64 oracle (this tier's reference) on the full workload.  Each phase of an
    LM iteration is timed once on the full problem; the K timed steps are the oracle's own first K
    LM iterations (its recorded trajectory: relinearize / re-damp sequence and PCG counts), composed
    from those measured phase times."""
    if rank != 0:
        return
    t, cores = oracle_phase_times(prob, args.config)
    traj = oracle_trajectory(args.config)
    if traj is not None and len(traj[0]) >= args.steps:
        iters, src = traj[0][:args.steps], traj[1]
    elif traj is not None and traj[0]:
        # the recorded trajectory is shorter than K: its last iterations already run PCG to its
        # 500-iteration cap; the remaining steps are taken at the cap, relinearizing
        n_rec = len(traj[0])
        iters = traj[0] + [(True, 500)] * (args.steps - n_rec)
        src = f"{traj[1]}: {n_rec} recorded iterations, the other {args.steps - n_rec} at the PCG cap of 500"
    else:  # no recorded trajectory: the GPU-independent lower bound of one PCG iteration per step
        iters, src = [(True, 1)] * args.steps, "none (1 PCG iteration per step assumed)"
    sec = compose_oracle(t, iters)
    val = args.steps / sec
    sample = (f"oracle phases on the full cfg{args.config} ({len(prob['obs_cam'])} obs), each timed once: "
              + ", ".join(f"{k} {v:.3f} s" for k, v in t.items())
              + f"; composed over the oracle's own first {args.steps} LM iterations ({src}: "
              f"{sum(n for _, n in iters)} PCG iterations, {sum(r for r, _ in iters)} linearizations)")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "LM iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, prob, args.gpus),
            "cpu_baseline": {"kind": "oracle", "cores": cores, "sample": sample, "value": val,
                             "unit": "LM iterations/s", "phase_s": t},
            "e2e": {"value": val, "unit": "LM iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--marg-reps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the factored / FP64 / explicit-SC context lines")
    ap.add_argument("--storage", default="dense", choices=["dense", "factored"],
                    help="landmark-block storage: the paper's dense blocks (default) or the factored "
                         "form (SURVEY §8f f4, beyond the paper)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="sqrt-BA-32 (default, the paper's headline) or sqrt-BA-64 (SURVEY §8f f2)")
    ap.add_argument("--solver", default="sqrtba", choices=list(SOLVERS),
                    help="landmark elimination: sqrt-BA (the paper's method, default) or the explicit "
                         "Schur-complement baselines explicit-32 / explicit-64 (SURVEY §8f f3)")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise-reproducible camera-space sums (rba_options.deterministic)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    prob = synth.make_problem(args.config)
    if args.impl == "reference":
        bench_reference(args, prob, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2103_01843_b200 import rba
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [rba.rba_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    n_p, n_l, n_obs = prob["cameras_init"].shape[0], prob["points_init"].shape[0], len(prob["obs_cam"])
    s = rba.Solver(prob, device=local, world=world, rank=rank, nccl_id=nccl_id, solver=SOLVERS[args.solver],
                   storage=1 if args.storage == "factored" else 0, precision=1 if args.precision == "fp64" else 0,
                   deterministic=1 if args.deterministic else 0)
    stream = s.stream

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up, then reset to the seeded start
    s.lm_solve(args.warmup, 0.0)
    s.set_state(prob["cameras_init"], prob["points_init"])
    s.reset_lm()
    barrier()
    # ---- timed: K LM iterations as ONE device-side loop (rba_lm_solve: a CUDA graph `while` node
    # around the iteration; ftol = 0, so exactly K attempts), CUDA events on the solver's stream
    clocks = ClockSampler(local)
    clocks.start()
    l0 = s.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    reps = s.lm_solve(args.steps, 0.0)
    ev1.record(stream)
    barrier()
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = s.launches() - l0
    clk = clocks.stop()
    assert len(reps) == args.steps, len(reps)
    marg_b, mv_b = rba.rba_plan_bytes(s.h)

    # ---- QR-marginalized observations/s: linearize + marginalize (+ fused damping) at lambda0,
    # CUDA events around the step-by-step calls; K2 alone from the library's per-launch events
    barrier()
    rba.rba_profile(s.h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mts = []
    for _ in range(args.marg_reps):
        s.set_state(prob["cameras_init"], prob["points_init"])
        barrier()
        e0.record(stream)
        s.linearize()
        s.marginalize(1e-4)
        e1.record(stream)
        barrier()
        mts.append(max_over_ranks(e0.elapsed_time(e1)))
    mprof = rba.rba_profile_get(s.h, "marginalize")
    rba.rba_profile(s.h, False)
    t_marg = statistics.median(mts)
    s.reset_lm()

    # ---- end to end through the public API with host buffers: per step upload the state
    # (pinned host -> device), one LM iteration, download the state.
    e2e = None
    if not args.no_e2e:
        cams = torch.from_numpy(prob["cameras_init"]).pin_memory().numpy()
        pts = torch.from_numpy(prob["points_init"]).pin_memory().numpy()
        s.set_state(cams, pts)
        s.reset_lm()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.set_state(cams, pts)
            s.lm_step()
            s.state(out=(cams, pts))
        barrier()
        t_e2e = max_over_ranks(time.perf_counter() - t0)
        nb = (9 * n_p + 3 * n_l) * 8  # FP64 state (host and device)
        e2e = {"value": args.steps / t_e2e, "unit": "LM iterations/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb,
               "note": "per step: rba_set_state(host FP64 state) + rba_lm_step + rba_get_state(host); "
                       "same LM trajectory as the device-resident run (each step relinearizes at the uploaded state)"}

    peak, peak_src = peaks()
    phases = {k: sum(r[f"t_{k}_ms"] for r in reps) for k in ("linearize", "marginalize", "precond", "pcg", "trial")}
    tot = sum(r["t_total_ms"] for r in reps)
    phases["control"] = max(tot - sum(phases.values()), 0.0)
    n_pcg = sum(r["pcg_iters"] for r in reps)
    variant = "" if (args.storage == "dense" and args.solver == "sqrtba" and args.precision == "fp32") else \
        ("_factored" if args.storage == "factored" else ("_fp64" if args.precision == "fp64" else f"_{args.solver}"))
    tr_mv, tr_mg, tr_src = ncu_traffic(args.config, variant)
    roof_mv = None
    if n_pcg > 0 and phases["pcg"] > 0:
        avg = phases["pcg"] / n_pcg
        ach = mv_b / (avg * 1e-3) / 1e9
        roof_mv = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": tr_mv,
                   "traffic_source": tr_src, "peak_source": peak_src, "launches": n_pcg, "avg_ms": avg,
                   "bytes_per_launch": mv_b,
                   "timer": "device %globaltimer stamps at the PCG loop's ends inside the timed graph; per PCG "
                            "iteration = product + the 3 update kernels (conservative for the product)",
                   "kernel": {
                       "": "matvec (K5: k_small_pipe + k_large_pipe<NS> + k_huge_*, slices summed in k_pcg_a), algorithmic 72k^2 B/landmark",
                       "_factored": "factored matvec (k_fac_matvec<G>), algorithmic 176+112k B/landmark",
                       "_fp64": "sqrt-BA-64 product (k_rcs64_ws<G> + k_rcs64_tma<NT>), algorithmic 8 x 2k(9k+1) B/landmark",
                   }.get(variant, "explicit-SC SpMV (k_sc_spmv), algorithmic 81 x sizeof(T) B per 9x9 block")}
    roof_mg = None
    if mprof[1] > 0 and mprof[0] > 0:
        ach = mprof[2] / mprof[1] / (mprof[0] / mprof[1] * 1e-3) / 1e9
        roof_mg = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": tr_mg,
                   "traffic_source": tr_src, "peak_source": peak_src, "launches": mprof[1],
                   "avg_ms": mprof[0] / mprof[1], "bytes_per_launch": mprof[2] / mprof[1],
                   "timer": "CUDA events on the solver stream around each K2 launch set",
                   "kernel": "marginalize (K2: k_marg_small<G> + k_marg_large<NT>), algorithmic (2k+3)(9k+4)*4+48+20k B/landmark"
                   if variant == "" else "K2 of the variant"}
    dom = max(phases, key=phases.get)
    line = {
        "metric": METRIC, "value": args.steps / (t_ms * 1e-3), "unit": "LM iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if (args.solver == "sc64" or args.precision == "fp64") else "f32", "data": "synthetic",
        "config": bench_config(args, prob, world),
        "qr_marginalized_obs_per_s": n_obs / (t_marg * 1e-3),
        "marginalize_ms": t_marg,
        "pcg_iters": [r["pcg_iters"] for r in reps],
        "pcg_iters_total": n_pcg,
        "costs": [r["cost_after"] for r in reps],
        "accepted": [r["accepted"] for r in reps],
        "gpu_launches": launches,
        "host_syncs_in_timed_region": 1,
        "dominant_phase": dom,
        "phase_ms_share": {k: (v / tot if tot else 0.0) for k, v in phases.items()},
        "roofline": roof_mv if (dom == "pcg" and roof_mv) or roof_mg is None else roof_mg,
        "roofline_matvec": roof_mv,
        "roofline_marginalize": roof_mg,
        "device_bytes": reps[0]["device_bytes"],
        "clocks": clk,
        "e2e": e2e,
    }
    # the same workload through the other landmark eliminations / storages of this library (NEXT
    # rows f2-f4), timed the same way: context for the headline, which stays dense sqrt-BA-32
    if not args.no_variants and args.solver == "sqrtba" and args.storage == "dense" and args.precision == "fp32" \
            and world == 1 and not args.deterministic:
        s.close()
        variants = {}
        for vname, kw in (("sqrtba32_factored", dict(storage=1)), ("sqrtba64", dict(precision=1)),
                          ("explicit32", dict(solver=1)), ("explicit64", dict(solver=2)),
                          ("sqrtba32_deterministic", dict(deterministic=1))):
            if vname == "sqrtba64" and int(np.bincount(prob["obs_pt"]).max()) > 1024:
                continue  # sqrt-BA-64 supports tracks up to 1024
            if vname.startswith("explicit") and args.config >= 5:
                continue  # covisibility H~ too large / slow to form for the final13682 shape
            try:
                sv = rba.Solver(prob, device=local, world=world, rank=rank, nccl_id=nccl_id, **kw)
            except rba.RBAError as e:
                variants[vname] = {"unavailable": str(e)}
                continue
            sv.lm_solve(args.warmup, 0.0)
            sv.set_state(prob["cameras_init"], prob["points_init"])
            sv.reset_lm()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(sv.stream)
            vr = sv.lm_solve(args.steps, 0.0)
            a1.record(sv.stream)
            barrier()
            vt = max_over_ranks(a0.elapsed_time(a1))
            variants[vname] = {"value": args.steps / (vt * 1e-3), "unit": "LM iterations/s",
                               "ms_per_step": vt / args.steps, "costs": [r["cost_after"] for r in vr],
                               "pcg_iters": [r["pcg_iters"] for r in vr],
                               "indefinite": sum(r["pcg_reason"] == 2 for r in vr),
                               "storage_bytes": sv.arena_bytes()[0]}
            sv.close()
        line["variants"] = variants
    if rank == 0 and world == 1 and not args.no_cpu and args.config <= 4:
        # the oracle on the full workload: phases timed once, composed with the GPU run's own
        # per-iteration sequence (relinearize / re-damp, PCG count) -- same iteration counts
        t, cores = oracle_phase_times(prob, args.config)
        iters = [(bool(r["relinearized"]), int(r["pcg_iters"])) for r in reps]
        val = args.steps / compose_oracle(t, iters)
        line["cpu_baseline"] = {
            "kind": "oracle", "cores": cores, "value": val, "unit": "LM iterations/s", "phase_s": t,
            "sample": (f"oracle phases on the full cfg{args.config} ({n_obs} obs, no subsample), each timed once: "
                       + ", ".join(f"{k} {v:.3f} s" for k, v in t.items())
                       + f"; composed with this run's {args.steps} LM iterations ({n_pcg} PCG iterations, "
                       f"{sum(r for r, _ in iters)} linearizations)")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if s.h:
        s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
