"""Small driver for ncu: one linearize + marginalize + `--matvecs` PCG iterations of config `--config`
through the C ABI (no timing; ncu measures).  Usage under gpurun:
    python tools/prof_step.py --config 4 && ncu ... python tools/prof_step.py --config 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2103_01843_b200 import rba, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--matvecs", type=int, default=2)
ap.add_argument("--storage", type=int, default=0)
ap.add_argument("--solver", type=int, default=0)
ap.add_argument("--precision", type=int, default=0)
args = ap.parse_args()
p = synth.make_problem(args.config)
s = rba.Solver(p, pcg_max_iters=args.matvecs, pcg_rel_tol=0.0, storage=args.storage, solver=args.solver,
               precision=args.precision)
s.linearize()
s.marginalize(1e-4)
st = s.pcg()
s.backsub()
print("ok", st, s.cost(True))
