"""Time the RCS matvec kernels alone (CUDA events, L2-cold since R2 >> L2) for config `--config`."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_01843_b200 import rba, synth
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=4); ap.add_argument("--reps", type=int, default=10); ap.add_argument("--precision", type=int, default=0)
a = ap.parse_args()
p = synth.make_problem(a.config)
s = rba.Solver(p, precision=a.precision)
s.linearize(); s.marginalize(1e-4)
v = torch.randn(9 * s.n_p, device="cuda")
for _ in range(3): s.matvec(v)
torch.cuda.synchronize()
rba.rba_profile(s.h, True)
for _ in range(a.reps): s.matvec(v)
ms, n, by = rba.rba_profile_get(s.h, "matvec")
print(f"cfg{a.config} matvec {ms/n:.3f} ms  {by/n/(ms/n*1e-3)/1e9:.0f} GB/s  precision={a.precision}")
