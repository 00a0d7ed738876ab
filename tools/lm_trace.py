"""LM trace (accept, cost, trial cost, gain ratio, lambda, PCG iterations) of config argv[1] (default 5)."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2103_01843_b200 import rba, synth
p = synth.make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
s = rba.Solver(p)
for i in range(10):
    r = s.lm_step()
    print(i, r["accepted"], "%.6e %.6e rho=%.3g lam=%.3g pcg=%d" % (r["cost"], r["cost_trial"], r["rho"], r["lambda_"], r["pcg_iters"]), flush=True)
