#!/usr/bin/env python
"""Benchmark of the FP32 sqrt-BA hot path on B200 (BASELINE.json metric: "LM iterations/s and
QR-marginalized obs/s (FP32) at 1-8 B200; % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one Levenberg-Marquardt iteration (every SURVEY §8a row: linearize, marginalize + damp,
preconditioner, PCG with the matrix-free RCS product, back-substitution, trial cost, LM update) of
the seeded synthetic workload `--config` (default 4: venice1778-shaped, 5.0M observations; its
15.7 GB landmark-block arena is far larger than the 126 MB L2, so no flush is needed).  W warm-up
iterations run first; then the state is reset to the seeded start and K iterations are timed with
CUDA events on the solver's stream, bracketed by barrier + synchronize, max over ranks.  With N > 1
(torchrun) landmarks are sharded across ranks (strong scaling, fixed problem) and the camera
vectors are all-reduced over NCCL inside librba.

`--impl reference` times the FP64 CPU oracle (the reference arm of this tier) on a bounded
landmark subsample of the same workload, on rank 0 only.
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


def ncu_traffic(cfg, variant=""):
    """DRAM bytes (read + write) of ONE launch of the matvec and of the marginalization, summed over
    their per-class kernels, from the newest committed `ncu --set full` summary of this config
    (profiles/r*_cfg<cfg>_ncu_full.json, written by tools/ncu_summary.py).  None if absent."""
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_cfg{cfg}{variant}_ncu_full.json")),
                   key=lambda f: int(re.search(r"/r(\d+)_", f).group(1)))
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


def cpu_sample(prob, every):
    sub = synth.subsample_landmarks(prob, every)
    kf = np.bincount(prob["obs_pt"]).astype(np.float64)
    ks = np.bincount(sub["obs_pt"]).astype(np.float64)
    work_full = float(((2 * kf + 3) * (9 * kf + 4)).sum())
    work_sub = float(((2 * ks + 3) * (9 * ks + 4)).sum())
    return sub, work_full / work_sub


def run_oracle(prob, cfg, steps, warmup, every, budget_s=None):
    """Time the FP64 oracle (as it stands) on a landmark subsample; returns (it/s scaled to the full
    workload, dict)."""
    import oracle
    sub, scale = cpu_sample(prob, every)
    o = oracle.Oracle(sub)
    for _ in range(warmup):
        o.lm_step()
    o.set_state(sub["cameras_init"], sub["points_init"])
    o.set_lm(1e-4, 2.0)
    t0 = time.perf_counter()
    n = 0
    pcg = 0
    for _ in range(steps):
        r = o.lm_step()
        pcg += r["pcg_iters"]
        n += 1
        if budget_s and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    rate = n / dt
    return rate / scale, {
        "kind": "oracle", "cores": oracle.num_threads(),
        "sample": (f"every {every}th landmark of cfg{cfg} ({sub['points_init'].shape[0]} lms, "
                   f"{len(sub['obs_cam'])} obs), {n} LM iterations from the seeded start in {dt:.2f} s "
                   f"({pcg} PCG iterations); scaled to the full workload by block bytes x{scale:.1f}"),
        "sample_it_per_s": rate,
    }


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
    if rank != 0:
        return
    every = args.cpu_every or {1: 1, 2: 4, 3: 16, 4: 64, 5: 512}[args.config]
    val, cb = run_oracle(prob, args.config, args.steps, args.warmup, every, budget_s=240)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "LM iterations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, prob, args.gpus),
            "cpu_baseline": dict(cb, value=val, unit="LM iterations/s"),
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
    ap.add_argument("--cpu-every", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the factored / explicit-SC context lines")
    ap.add_argument("--storage", default="dense", choices=["dense", "factored"],
                    help="landmark-block storage: the paper's dense blocks (default) or the factored "
                         "form (SURVEY §8f f4, beyond the paper)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"],
                    help="sqrt-BA-32 (default, the paper's headline) or sqrt-BA-64 (SURVEY §8f f2)")
    ap.add_argument("--solver", default="sqrtba", choices=list(SOLVERS),
                    help="landmark elimination: sqrt-BA (the paper's method, default) or the explicit "
                         "Schur-complement baselines explicit-32 / explicit-64 (SURVEY §8f f3)")
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
                   storage=1 if args.storage == "factored" else 0, precision=1 if args.precision == "fp64" else 0)
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
    for _ in range(args.warmup):
        s.lm_step()
    s.set_state(prob["cameras_init"], prob["points_init"])
    s.reset_lm()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    rba.rba_profile(s.h, True)
    l0 = s.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    reps = []
    for _ in range(args.steps):
        reps.append(s.lm_step())
    ev1.record(stream)
    barrier()
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = s.launches() - l0
    prof = {k: rba.rba_profile_get(s.h, k) for k in rba.KERNELS}
    rba.rba_profile(s.h, False)
    clk = clocks.stop()

    # ---- QR-marginalized observations/s: linearize + marginalize (+ fused damping) at lambda0
    barrier()
    rba.rba_profile(s.h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mts = []
    for _ in range(args.marg_reps):
        s.set_state(prob["cameras_init"], prob["points_init"])
        s.reset_lm()
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

    # ---- end to end through the public API with host buffers: per step upload the state
    # (pinned host -> device), one LM iteration, download the state.
    e2e = None
    if not args.no_e2e:
        # pinned host buffers (torch pinned storage viewed as numpy); the state round-trips in place
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
                       "same LM trajectory as the device-resident run"}

    peak, peak_src = peaks()
    # dominant kernel by share of the timed step
    shares = {k: v[0] for k, v in prof.items()}
    dom = max(shares, key=shares.get)

    def roof(ms, n, by):
        if n == 0 or ms <= 0:
            return None
        ach = by / n / (ms / n * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "peak_source": peak_src, "launches": n, "avg_ms": ms / n,
                "bytes_per_launch": by / n}

    variant = "" if (args.storage == "dense" and args.solver == "sqrtba" and args.precision == "fp32") else \
        ("_factored" if args.storage == "factored" else ("_fp64" if args.precision == "fp64" else f"_{args.solver}"))
    tr_mv, tr_mg, tr_src = ncu_traffic(args.config, variant)
    roof_mv = roof(*prof["matvec"])
    if roof_mv:
        roof_mv["traffic"] = tr_mv
        roof_mv["traffic_source"] = tr_src
        roof_mv["kernel"] = {
            "": "matvec (K5: k_small_pipe + k_large_pipe<NS> + k_huge_*, slices summed in k_pcg_a), algorithmic 72k^2 B/landmark",
            "_factored": "factored matvec (k_fac_matvec<G>, slices summed in k_pcg_a), algorithmic 176+112k B/landmark",
            "_fp64": "sqrt-BA-64 product (k_rcs64_ws<G> + k_rcs64_tma<NT>), algorithmic 8 x 2k(9k+1) B/landmark",
        }.get(variant, "explicit-SC SpMV (k_sc_spmv), algorithmic 81 x sizeof(T) B per 9x9 block")
    roof_mg = roof(*mprof)
    if roof_mg:
        roof_mg["traffic"] = tr_mg
        roof_mg["traffic_source"] = tr_src
        roof_mg["kernel"] = {
            "": "marginalize (K2: k_marg_small<G> + k_marg_large<NT>), algorithmic (2k+3)(9k+4)*4+48+20k B/landmark",
            "_factored": "factored marginalize (K2 writing factors), algorithmic 176+132k B/landmark",
            "_fp64": "sqrt-BA-64 marginalize (k_marg64), algorithmic 8 (2k+3)(9k+4) + 96 + 40k B/landmark",
        }.get(variant, "explicit-SC build (k_sc_build), algorithmic 81 x sizeof(T) B per block + 48 B/obs")
    total_prof = sum(shares.values())
    line = {
        "metric": METRIC, "value": args.steps / (t_ms * 1e-3), "unit": "LM iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if (args.solver == "sc64" or args.precision == "fp64") else "f32", "data": "synthetic",
        "config": bench_config(args, prob, world),
        "qr_marginalized_obs_per_s": n_obs / (t_marg * 1e-3),
        "marginalize_ms": t_marg,
        "pcg_iters": [r["pcg_iters"] for r in reps],
        "costs": [r["cost_after"] for r in reps],
        "accepted": [r["accepted"] for r in reps],
        "gpu_launches": launches,
        "dominant_kernel": dom,
        "kernel_ms_share": {k: (v / total_prof if total_prof else 0.0) for k, v in shares.items()},
        "roofline": roof_mv if dom == "matvec" or roof_mg is None else roof_mg,
        "roofline_matvec": roof_mv,
        "roofline_marginalize": roof_mg,
        "clocks": clk,
        "e2e": e2e,
    }
    # the same workload through the other landmark eliminations / storages of this library (NEXT
    # rows f3, f4), timed the same way (W warm-up, reset, K steps, CUDA events): context for the
    # headline, which stays the paper's dense sqrt-BA-32
    # (single GPU only: a second NCCL communicator would need its own unique id)
    if not args.no_variants and args.solver == "sqrtba" and args.storage == "dense" and args.precision == "fp32" \
            and world == 1:
        s.close()
        variants = {}
        for vname, kw in (("sqrtba32_factored", dict(storage=1)), ("sqrtba64", dict(precision=1)),
                          ("explicit32", dict(solver=1)), ("explicit64", dict(solver=2))):
            if vname == "sqrtba64" and int(np.bincount(prob["obs_pt"]).max()) > 1024:
                continue  # sqrt-BA-64 supports tracks up to 1024
            if vname.startswith("explicit") and args.config >= 5:
                continue  # covisibility H~ too large / slow to form for the final13682 shape
            sv = rba.Solver(prob, device=local, world=world, rank=rank, nccl_id=nccl_id, **kw)
            for _ in range(args.warmup):
                sv.lm_step()
            sv.set_state(prob["cameras_init"], prob["points_init"])
            sv.reset_lm()
            barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(sv.stream)
            vr = [sv.lm_step() for _ in range(args.steps)]
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
    if rank == 0 and world == 1 and not args.no_cpu:
        every = args.cpu_every or {1: 1, 2: 4, 3: 16, 4: 64, 5: 512}[args.config]
        val, cb = run_oracle(prob, args.config, 2, 0, every, budget_s=30)
        line["cpu_baseline"] = dict(cb, value=val, unit="LM iterations/s")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if s.h:
        s.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
