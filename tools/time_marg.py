"""Time linearize + marginalize (K1 + K2 at lambda0) alone for config `--config` (CUDA events via the
library's profiler; the arena is >> L2 for configs 3-5)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2103_01843_b200 import rba, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--storage", type=int, default=0)
a = ap.parse_args()
p = synth.make_problem(a.config)
s = rba.Solver(p, storage=a.storage)
s.linearize()
s.marginalize(1e-4)
torch.cuda.synchronize()
rba.rba_profile(s.h, True)
for _ in range(a.reps):
    s.set_state(p["cameras_init"], p["points_init"])
    s.linearize()
    s.marginalize(1e-4)
ms, n, by = rba.rba_profile_get(s.h, "marginalize")
ms1, n1, _ = rba.rba_profile_get(s.h, "linearize")
print(f"cfg{a.config} linearize {ms1 / max(n1, 1):.3f} ms; linearize + marginalize {ms1 / max(n1, 1) + ms / n:.3f} ms")
print(f"cfg{a.config} marginalize {ms / n:.3f} ms  {by / n / (ms / n * 1e-3) / 1e9:.0f} GB/s  "
      f"item_floats={os.environ.get('RBA_MARG_ITEM_FLOATS', 'default')}")
