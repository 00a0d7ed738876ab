"""Find allocations whose initial content changes a deterministic-mode LM trajectory: every
allocation (then ranges, recursively) filled with a poison byte through RBA_POISON_ALLOC.
python tools/poison_bisect.py [config] [iters]"""
import os
import sys

sys.path.insert(0, ".")
from paper_2103_01843_b200 import synth  # noqa: E402
from paper_2103_01843_b200.rba import Solver  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = synth.make_problem(cfg)


def run(spec):
    if spec is None:
        os.environ.pop("RBA_POISON_ALLOC", None)
    else:
        os.environ["RBA_POISON_ALLOC"] = spec
    s = Solver(p, deterministic=1)
    t = [(r["cost_after"], r["pcg_iters"], r["rho"]) for r in s.lm_solve(iters, 0.0)]
    st = s.state()
    s.close()
    return t, st[0].tobytes() + st[1].tobytes()


ref = run("255")
print("0xff-filled:", ref[0], flush=True)
for spec in ("255", "127", "65", "0"):
    r = run(spec)
    print(f"fill {spec}:", "same" if r == ref else f"DIFF {r[0]}", flush=True)
hits = []


def search(lo, hi, byte=0):
    r = run(f"{byte}:{lo}:{hi}:255")
    if r == ref:
        return
    if hi - lo == 1:
        hits.append(lo)
        print("allocation", lo, "matters:", r[0], flush=True)
        return
    mid = (lo + hi) // 2
    search(lo, mid, byte)
    search(mid, hi, byte)


for byte in (0, 65):
    hits = []
    search(0, 128, byte)
    print(f"fill {byte} vs 0xff: allocations read before written:", hits, flush=True)
os.environ["RBA_POISON_ALLOC"] = "0"
os.environ["RBA_ALLOC_TRACE"] = "1"
Solver(p, deterministic=1).close()
