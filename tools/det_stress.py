"""Deterministic-mode stress: N fresh contexts of one config (interleaved with other configs'
contexts, as in the test session), each lm_solve(iters); reports every trajectory that differs from
the first.  python tools/det_stress.py config runs iters [interleave-config ...]"""
import sys
import time
import numpy as np

sys.path.insert(0, ".")
from paper_2103_01843_b200 import synth  # noqa: E402
from paper_2103_01843_b200.rba import Solver  # noqa: E402


def problem(cfg):
    if cfg == 0:
        rng = np.random.default_rng(41)
        ks = [2, 3, 4, 5, 8, 9, 16, 17, 33, 65, 129, 257, 600] + list(rng.integers(2, 12, 400))
        return synth.make_tracks(41, ks, n_p=700)
    return synth.make_problem(cfg)


cfg, runs, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
others = [problem(int(a)) for a in sys.argv[4:]]
p = problem(cfg)
ref = None
bad = 0
t0 = time.time()
for n in range(runs):
    for q in others:
        s = Solver(q, deterministic=1)
        s.lm_solve(2, 0.0)
        s.close()
    s = Solver(p, deterministic=1)
    reps = s.lm_solve(iters, 0.0)
    traj = [(r["cost_after"], r["pcg_iters"], r["rho"]) for r in reps]
    cams, pts = s.state()
    s.close()
    if ref is None:
        ref = (traj, cams, pts)
        continue
    if traj != ref[0] or not np.array_equal(cams, ref[1]) or not np.array_equal(pts, ref[2]):
        bad += 1
        first = next((i for i, (a, b) in enumerate(zip(traj, ref[0])) if a != b), None)
        print(f"run {n}: DIFF at iteration {first}: {traj[first] if first is not None else ''} vs "
              f"{ref[0][first] if first is not None else ''}", flush=True)
print(f"config {cfg}: {bad} of {runs - 1} runs differ from the first ({time.time() - t0:.0f} s)")
