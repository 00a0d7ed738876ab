"""Small driver that launches every kernel class of librba once or twice, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):
    python tools/sanitize_run.py && compute-sanitizer --tool memcheck python tools/sanitize_run.py
Problems: config 1, and a tracks problem with every kernel bucket (packs k <= 16, tiles 17..512, a
huge k > 512 track); paths: LM graph and eager (RBA_NO_GRAPH), step-by-step calls with re-damping,
deterministic mode, factored storage, sqrt-BA-64, explicit-32 / explicit-64."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2103_01843_b200 import rba, synth  # noqa: E402

rng = np.random.default_rng(5)
ks = [2, 3, 4, 5, 8, 9, 16, 17, 33, 65, 129, 257, 600] + list(rng.integers(2, 12, 120))
probs = {"cfg1": synth.make_problem(1), "tracks": synth.make_tracks(5, ks, n_p=640)}
variants = [dict(), dict(deterministic=1), dict(storage=1), dict(precision=1), dict(solver=1), dict(solver=2)]
for name, p in probs.items():
    for kw in variants:
        if kw.get("precision") == 1 and max(ks) > 1024:
            pass
        s = rba.Solver(p, **kw)
        s.lm_step()
        s.lm_step()
        s.linearize()
        s.marginalize(1e-3)
        s.marginalize(0.5)  # re-damp
        st = s.pcg()
        s.backsub()
        s.cost(True)
        v = torch.randn(9 * s.n_p, device="cuda")
        s.matvec(v)
        torch.cuda.synchronize()
        print(name, kw, st, s.info(), flush=True)
        s.close()
os.environ["RBA_NO_GRAPH"] = "1"
s = rba.Solver(probs["tracks"])
s.lm_solve(2, 0.0)
s.close()
print("SANITIZE_RUN_OK")
