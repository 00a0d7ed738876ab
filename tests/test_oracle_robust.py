"""Pins for the oracle's robust loss (f1: Huber with IRLS): golden values of the Huber norm
and its IRLS weight (hand-computed from the definition, tests/golden/huber.txt), the IRLS
gradient identity grad E = 2 J~^T r~ against central finite differences of E = sum rho(|r|^2), and
the weighted linear step against a brute-force dense solve (P:148-155 with J~, r~)."""
import os

import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import synth

from _dense import brute_force_step, relf, stacked

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_huber_golden():
    for line in open(os.path.join(GOLD, "huber.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        s, delta, rho, w = (float(x) for x in line.split())
        assert abs(oracle.huber_rho(s, delta) - rho) <= 1e-14 * max(1.0, rho)
        assert abs(oracle.huber_weight(s, delta) - w) <= 1e-15
    # continuity of rho and rho' at s = delta^2
    for d in (0.5, 1.0, 3.0):
        s = d * d
        assert abs(oracle.huber_rho(s * (1 + 1e-12), d) - oracle.huber_rho(s, d)) < 1e-10
        assert abs(oracle.huber_weight(s * (1 + 1e-12), d) - 1.0) < 1e-10


def _robust_problem(seed):
    # pixel noise N(0,1) with delta = 1: ~60% of the residuals are outside the quadratic region
    return synth.make_random_small(seed, n_p=5, n_l=25, kmin=2, kmax=5)


@pytest.mark.parametrize("seed", [50, 51])
def test_irls_gradient_is_cost_gradient(seed):
    """E(x) = sum rho(|r(x)|^2); IRLS weights w = sqrt(rho') give grad E = 2 sum (w J)^T (w r) =
    2 J~^T r~.  Checked against central differences of the oracle's E on every state coordinate."""
    p = _robust_problem(seed)
    o = oracle.Oracle(p, cams=p["cameras_true"], pts=p["points_true"])  # residuals ~ N(0,1) px
    o.set_huber(1.0)
    o.linearize()
    r, Jc, Jl = o.linearization()
    s = (r ** 2).sum(1)
    assert 0.2 < np.mean(s > 1.0) < 0.95  # both regimes present
    g_cam = np.zeros(9 * o.n_p)
    g_pt = np.zeros(3 * o.n_l)
    lm = np.repeat(np.arange(o.n_l), np.diff(o.lm_ptr))
    np.add.at(g_cam, (9 * o.csr_cam[:, None] + np.arange(9)).ravel(), 2 * np.einsum("nij,ni->nj", Jc, r).ravel())
    np.add.at(g_pt, (3 * lm[:, None] + np.arange(3)).ravel(), 2 * np.einsum("nij,ni->nj", Jl, r).ravel())
    cams, pts = o.state()
    h = 1e-6
    fd_cam, fd_pt = np.zeros_like(g_cam), np.zeros_like(g_pt)
    for i in range(9 * o.n_p):
        c1, c2 = cams.copy(), cams.copy()
        c1.flat[i] += h * max(1.0, abs(cams.flat[i]))
        c2.flat[i] -= h * max(1.0, abs(cams.flat[i]))
        o.set_state(c1, pts)
        e1 = o.cost()
        o.set_state(c2, pts)
        e2 = o.cost()
        fd_cam[i] = (e1 - e2) / (2 * h * max(1.0, abs(cams.flat[i])))
    for i in range(3 * o.n_l):
        p1, p2 = pts.copy(), pts.copy()
        p1.flat[i] += h
        p2.flat[i] -= h
        o.set_state(cams, p1)
        e1 = o.cost()
        o.set_state(cams, p2)
        e2 = o.cost()
        fd_pt[i] = (e1 - e2) / (2 * h)
    assert relf(g_cam, fd_cam) < 1e-6, relf(g_cam, fd_cam)
    assert relf(g_pt, fd_pt) < 1e-6, relf(g_pt, fd_pt)


def test_huber_large_delta_is_squared_loss():
    p = _robust_problem(52)
    a, b = oracle.Oracle(p), oracle.Oracle(p)
    b.set_huber(1e9)
    a.linearize()
    b.linearize()
    assert a.cost() == b.cost()
    for x, y in zip(a.linearization(), b.linearization()):
        np.testing.assert_array_equal(x, y)


def test_irls_step_is_weighted_least_squares():
    """With Huber on, the oracle's (dp, dl) at PCG tol 1e-12 is the brute-force minimizer of the
    damped weighted linear problem |r~ + J~ dx|^2 + lam |D dx|^2 (Eq. linearized_residual with the
    IRLS-corrected residuals, as Ceres does)."""
    p = _robust_problem(53)
    o = oracle.Oracle(p)
    o.set_huber(1.0)
    o.linearize()
    o.marginalize()
    o.damp(1e-3)
    assert o.precond_rhs() == 0
    it, reason, _ = o.pcg(tol=1e-12, max_iters=2000)
    assert reason == 0
    o.backsub()
    J, r, D2 = stacked(o)
    dx = brute_force_step(J, r, D2, 1e-3)
    assert relf(o.dp(), dx[:9 * o.n_p]) < 1e-8
    assert relf(o.dl(), dx[9 * o.n_p:]) < 1e-8
