"""Deterministic-mode diagnosis: repeat each phase from one state (same context and a fresh
context) and report which outputs differ bitwise.  python tools/det_probe.py [config] [iters]"""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2103_01843_b200 import synth  # noqa: E402
from paper_2103_01843_b200.rba import Solver  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = synth.make_problem(cfg)


def phases(s, st, lam, v):
    out = {}
    s.set_state(*st)
    s.linearize()
    out["cost"] = np.array([s.cost()])
    out["scaling"] = np.concatenate([np.asarray(x).ravel() for x in s.scaling()])
    s.marginalize(lam)
    out["matvec"] = s.matvec(v).cpu().numpy()
    s.set_pcg_limits(0.0, 0)
    s.pcg()
    out["precond"] = s.precond_sums().ravel()
    out["rhs"] = s.rhs()
    s.set_pcg_limits(1e-2, 500)
    r = s.pcg()
    out["pcg_iters"] = np.array([r["iters"]])
    s.backsub()
    dp, dl = s.step()
    out["dp"], out["dl"] = dp, dl
    out["trial_cost"] = np.array([s.cost(at_trial=True)])
    return out


A = Solver(p, deterministic=1)
for i in range(iters):
    A.lm_step()
st = A.state()
lam, nu, _ = A.get_lm()
print("state after", iters, "iterations; lambda", lam)
v = torch.tensor(np.random.default_rng(1).normal(size=9 * p["cameras_init"].shape[0]), dtype=torch.float32,
                 device="cuda")
ref = phases(A, st, lam, v)
for tag in ("same ctx #2", "same ctx #3"):
    o = phases(A, st, lam, v)
    print(tag, {k: ("ok" if np.array_equal(ref[k], o[k]) else f"DIFF max {np.max(np.abs(ref[k] - o[k])):.3e}")
                for k in ref})
A.set_state(p["cameras_init"], p["points_init"])
A.reset_lm()
A.close()
B = Solver(p, deterministic=1)
o = phases(B, st, lam, v)
print("fresh ctx", {k: ("ok" if np.array_equal(ref[k], o[k]) else f"DIFF max {np.max(np.abs(ref[k] - o[k])):.3e}")
                    for k in ref})
# whole trajectories, same context
B.set_state(p["cameras_init"], p["points_init"])
B.reset_lm()
t1 = [(r["cost_after"], r["pcg_iters"]) for r in B.lm_solve(4, 0.0)]
B.set_state(p["cameras_init"], p["points_init"])
B.reset_lm()
t2 = [(r["cost_after"], r["pcg_iters"]) for r in B.lm_solve(4, 0.0)]
print("trajectory same ctx", t1 == t2, t1, t2)
B.close()
