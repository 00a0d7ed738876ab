"""Run-to-run and stale-memory check: the same LM iterations in fresh contexts, then in contexts whose
device memory (torch caching allocator) was just filled with NaN; any difference beyond FP64
summation-order noise, or a NaN, points at a read of unwritten memory.  Usage: python tools/stale_mem_check.py"""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2103_01843_b200 import rba, synth
p = synth.make_problem(2)


def run(tag, kw, poison=False):
    if poison:
        x = torch.full((6 << 30,), float("nan"), device="cuda", dtype=torch.float32)  # 24 GB of NaN
        del x
    s = rba.Solver(p, **kw)
    out = [s.lm_step()["cost_after"] for _ in range(3)]
    s.close()
    print(tag, kw, " ".join("%.10f" % c for c in out), flush=True)


for kw in (dict(), dict(storage=1), dict(precision=1), dict(solver=1), dict(huber_delta=1.0, precision=1)):
    for i in range(2):
        run("plain   ", kw)
    for i in range(2):
        run("poisoned", kw, True)
