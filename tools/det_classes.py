"""Deterministic-mode check per kernel class: problems whose tracks all fall in one k bucket; the
block-Jacobi sums (K4) and one product (K5) of repeated passes in one context must be bitwise
equal.  python tools/det_classes.py [reps] [case ...]"""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2103_01843_b200 import synth  # noqa: E402
from paper_2103_01843_b200.rba import Solver  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cases = {"k300": [300] * 60, "k200": [200] * 80, "k150": [150] * 100, "k256": [256] * 60, "k129": [129] * 100,
         "k100": [100] * 150, "k50": [50] * 300, "k24": [24] * 600, "k12": [12] * 1500, "k700": [700] * 12,
         "k200x1": [200]}
sel = sys.argv[2:] or list(cases)
for name in sel:
    ks = cases[name]
    p = synth.make_tracks(7, ks, n_p=800)
    s = Solver(p, deterministic=1)
    s.linearize()
    s.marginalize(1e-4)
    v = torch.tensor(np.random.default_rng(1).normal(size=9 * 800), dtype=torch.float32, device="cuda")
    outs = []
    for rep in range(reps):
        s.set_pcg_limits(0.0, 0)
        s.pcg()
        outs.append((s.precond_sums().copy(), s.matvec(v).cpu().numpy()))
    k4 = [np.array_equal(outs[0][0], o[0]) for o in outs[1:]]
    k5 = [np.array_equal(outs[0][1], o[1]) for o in outs[1:]]
    detail = ""
    for o in outs[1:]:
        if not np.array_equal(outs[0][0], o[0]):
            dif = outs[0][0] != o[0]
            cams = np.nonzero(dif.any(1))[0]
            detail = f" first diff: {dif.sum()} entries in cameras {cams[:8].tolist()} max {np.abs(outs[0][0] - o[0]).max():.3e}"
            break
    print(f"{name}: K4 {sum(k4)}/{reps - 1}  K5 {sum(k5)}/{reps - 1}{detail}", flush=True)
    s.close()
