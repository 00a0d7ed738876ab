"""Per-kernel-family CUDA-event times on config `--config` (step-by-step API, library profiler):
K2 marginalize (linearize + marginalize at lambda0), K4 block-Jacobi + b~, K5 product (rba_matvec,
standalone).  Algorithmic bytes per launch from the planner."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_01843_b200 import rba, synth
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--det", type=int, default=0)
a = ap.parse_args()
p = synth.make_problem(a.config)
s = rba.Solver(p, deterministic=a.det)
s.linearize(); s.marginalize(1e-4); s.pcg()
v = torch.randn(9 * s.n_p, device="cuda")
for _ in range(2): s.matvec(v)
torch.cuda.synchronize()
rba.rba_profile(s.h, True)
for _ in range(a.reps):
    s.set_state(p["cameras_init"], p["points_init"]); s.linearize(); s.marginalize(1e-4)
    s.set_pcg_limits(0.0, 0); s.pcg(); s.backsub()
    s.matvec(v)
out = {"config": a.config, "det": a.det}
for k in ("marginalize", "precond", "matvec", "backsub"):
    ms, n, by = rba.rba_profile_get(s.h, k)
    out[k] = {"ms": ms / n, "GBs": by / n / (ms / n * 1e-3) / 1e9, "bytes": by / n}
print(json.dumps(out))
