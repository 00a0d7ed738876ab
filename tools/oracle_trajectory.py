"""The FP64 oracle's own LM trajectory on a full BASELINE config (test / measurement infrastructure:
calls only oracle/ and the seeded generator).  Writes, after every iteration, the oracle's report
(cost after the decision, PCG iterations and reason, accept, lambda) to
tests/oracle_data/cfg<C>_lm<N>.json.  The full-size GPU parity test replays these iterations at the
oracle's PCG counts and compares the costs (tests/test_gpu_fullsize.py), and bench.py's reference
arm composes the oracle's per-phase times measured on the full workload with these iteration
counts.

    OMP_NUM_THREADS=6 nice -n 19 python tools/oracle_trajectory.py --config 4 --iters 20
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2103_01843_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
out = os.path.join(ROOT, "tests", "oracle_data", f"cfg{a.config}_lm{a.iters}.json")
p = synth.make_problem(a.config)
o = oracle.Oracle(p)
rec = {"config": a.config, "digest": synth.digest(p), "lambda0": 1e-4, "pcg_tol": 1e-2, "pcg_max": 500,
       "threads": oracle.num_threads(), "iterations": []}
for i in range(a.iters):
    t0 = time.time()
    r = o.lm_step(1e-2, 500)
    r["wall_s"] = time.time() - t0
    rec["iterations"].append(r)
    with open(out + ".tmp", "w") as f:
        json.dump(rec, f, indent=1)
    os.replace(out + ".tmp", out)
    print(i, r["pcg_iters"], r["cost_after"], r["accepted"], f"{r['wall_s']:.1f}s", flush=True)
