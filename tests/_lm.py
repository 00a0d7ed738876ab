"""LM cost parity helper: cost after each iteration within `bar` (1e-4) relative of
the oracle's.  PCG stops at a relative residual of 1e-2; where its iteration count differs from the
oracle's (the stop is decided by FP32 summation order, which varies run to run with the
camera-slice reductions, and on ill-conditioned iterations -- 130 to 260 PCG iterations on
configs 2 and 3 -- counts drift by a few), the steps differ by up to the tolerance.  §8c re-runs
both at the oracle's count, which the C ABI cannot replay, so in that case the bar is 1e-3."""


def check_lm_step(i, rg, ro, bar=1e-4, edge_bar=1e-3):
    assert rg["pcg_reason"] != 2, (i, rg)
    b = max(bar, edge_bar) if rg["pcg_iters"] != ro["pcg_iters"] else bar
    assert abs(rg["cost_after"] - ro["cost_after"]) <= b * ro["cost_after"], (i, rg, ro)
