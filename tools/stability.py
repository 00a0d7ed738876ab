"""Numerical-stability comparison of the landmark eliminations (the paper's claim P:500-502:
"explicit-32" loses definiteness where sqrt-BA-32 does not): N LM iterations of sqrt-BA-32,
explicit-32 and explicit-64 from the same seeded start; prints one JSON line per solver with the
cost trajectory, accepted steps, indefinite PCG solves (p^T H p <= 0) and wall time.
Usage: python tools/stability.py [--config 3] [--iters 10]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_01843_b200 import rba, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
p = synth.make_problem(a.config)
for name, solver in (("sqrt-BA-32", rba.RBA_SOLVER_SQRTBA), ("explicit-32", rba.RBA_SOLVER_EXPLICIT_SC32),
                     ("explicit-64", rba.RBA_SOLVER_EXPLICIT_SC64)):
    s = rba.Solver(p, solver=solver)
    t0 = time.perf_counter()
    reps = [s.lm_step() for _ in range(a.iters)]
    dt = time.perf_counter() - t0
    print(json.dumps({"cfg": a.config, "solver": name, "iters": a.iters, "seconds": dt,
                      "costs": [r["cost_after"] for r in reps], "accepted": sum(r["accepted"] for r in reps),
                      "indefinite": sum(r["pcg_reason"] == 2 for r in reps),
                      "pcg_iters": [r["pcg_iters"] for r in reps]}), flush=True)
    s.close()
