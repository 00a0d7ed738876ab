"""Huge-track product (k > 512, `k_huge_fused`) alone: a synthetic problem whose tracks follow config
5's k > 512 tail, standalone product timed with CUDA events (library profiler),
algorithmic bytes 72 k^2 per landmark.  `--ncu`: one product only (for an ncu capture)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_01843_b200 import rba, synth
ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--ncu", action="store_true")
a = ap.parse_args()
ks = [640] * 100 + [900] * 35 + [1200] * 18 + [1600] * 8
p = synth.make_tracks(5, ks, n_p=2000)
s = rba.Solver(p)
s.linearize(); s.marginalize(1e-4)
v = torch.randn(9 * s.n_p, device="cuda")
if a.ncu:
    s.matvec(v); torch.cuda.synchronize(); print("ok"); sys.exit(0)
for _ in range(3): s.matvec(v)
torch.cuda.synchronize()
rba.rba_profile(s.h, True)
for _ in range(a.reps): s.matvec(v)
ms, n, by = rba.rba_profile_get(s.h, "matvec")
print(f"huge product {ms / n:.3f} ms  {by / n / 1e9:.2f} GB  {by / n / (ms / n * 1e-3) / 1e9:.0f} GB/s")
