"""PCG alone (graph or host loop per RBA_NO_GRAPH) on config `--config`: per-iteration time of the
product + update kernels from the library profiler, next to the standalone product (tools/time_matvec.py)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_01843_b200 import rba, synth
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=4); ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--iters", type=int, default=60)
a = ap.parse_args()
p = synth.make_problem(a.config)
s = rba.Solver(p, pcg_rel_tol=0.0, pcg_max_iters=a.iters)
s.linearize(); s.marginalize(1e-4); s.pcg()
torch.cuda.synchronize()
rba.rba_profile(s.h, True)
for _ in range(a.reps):
    s.pcg()
ms, n, by = rba.rba_profile_get(s.h, "matvec")
ms2, n2, _ = rba.rba_profile_get(s.h, "pcg")
print(f"cfg{a.config} pcg: {ms / n:.3f} ms per effective product ({n} products, {by / n / (ms / n * 1e-3) / 1e9:.0f} GB/s) "
      f"+ update {ms2 / max(n2, 1):.3f} ms x {n2}; graph={'no' if os.environ.get('RBA_NO_GRAPH') else 'yes'}")
