"""GPU parity of sqrt-BA-64 (the paper's double-precision variant) against
the FP64 oracle.  Jacobians, column scaling, blocks, QR, damping, reduced system, PCG vectors and
back-substitution are all FP64, so the bars are FP64 rounding levels (the rba_matvec test hook
returns FP32 vectors: columns of H~ read through it are bounded by FP32 output rounding)."""
import numpy as np
import pytest

import oracle
from paper_2103_01843_b200 import synth
from paper_2103_01843_b200.rba import RBA_PRECISION_FP32, RBA_PRECISION_FP64

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _solver(p, precision=RBA_PRECISION_FP64, **kw):
    from paper_2103_01843_b200.rba import Solver
    return Solver(p, precision=precision, **kw)


def _oracle(p, lam):
    o = oracle.Oracle(p)
    o.linearize()
    o.marginalize()
    o.damp(lam)
    return o


def _mv(s, v):
    return s.matvec(torch.tensor(v, dtype=torch.float32, device="cuda")).double().cpu().numpy()


@pytest.mark.parametrize("lam", [1e-4, 1.0])
def test_sqrtba64_reduced_system_and_blocks(lam):
    p = synth.make_problem(1)
    s = _solver(p)
    s.linearize()
    s.marginalize(lam)
    o = _oracle(p, lam)
    H, b = o.reduced_dense()
    N = 9 * o.n_p
    Hg = np.stack([_mv(s, np.eye(N)[i]) for i in range(N)], 1)
    assert relf(Hg, H) <= 1e-7
    for j in range(0, 200, 13):
        k = o.track_length(j)
        Bg, Bo = s.block(j), o.block(j)
        assert np.all(Bg[3:, 9 * k:9 * k + 3] == 0.0)
        assert relf(Bg.T @ Bg, Bo.T @ Bo) <= 1e-12  # rotation invariant (reading C16)
    s.pcg()
    assert relf(s.rhs(), b) <= 1e-11


def test_sqrtba64_redamp_and_long_tracks():
    ks = [2, 3, 5, 9, 17, 33, 129, 400, 1000]
    p = synth.make_tracks(41, ks, n_p=1100)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-3)
    s.marginalize(0.4)  # re-damp in place
    o = _oracle(p, 0.4)
    rng = np.random.default_rng(3)
    for _ in range(3):
        v = rng.normal(size=9 * o.n_p)
        assert relf(_mv(s, v), o.matvec(v)) <= 1e-6
    for j, k in enumerate(ks[:7]):
        Bg, Bo = s.block(j), o.block(j)
        assert relf(Bg.T @ Bg, Bo.T @ Bo) <= 1e-11


@pytest.mark.parametrize("cfg", [1, 2])
def test_sqrtba64_pcg_backsub_lm(cfg):
    p = synth.make_problem(cfg)
    s = _solver(p)
    s.linearize()
    s.marginalize(1e-4)
    o = _oracle(p, 1e-4)
    st = s.pcg()
    assert o.precond_rhs() == 0
    it, reason, _ = o.pcg(1e-2, 500)
    assert st["iters"] == it and reason == st["reason"] == 0
    s.backsub()
    o.backsub()
    dp, dl = s.step()
    assert relf(dp, o.dp()) <= 1e-8
    assert relf(dl, o.dl()) <= 1e-7  # dl is exported through the shared FP32 buffer
    s.close()
    s = _solver(p)
    o = oracle.Oracle(p)
    for i in range(5):
        rg, ro = s.lm_step(), o.lm_step()
        # 1e-6: different FP64 summation orders (camera-space atomics) can change the PCG iteration
        # count at tol 1e-2 on ill-conditioned iterations (seen: 138 vs 133 at cfg 2 iteration 3,
        # costs 7e-7 apart); still 100x inside the sqrt-BA-32 bar of SURVEY §8c
        assert abs(rg["cost_after"] - ro["cost_after"]) <= 1e-6 * ro["cost_after"], (i, rg, ro)


def test_sqrtba64_more_accurate_than_32():
    p = synth.make_problem(2)
    o = _oracle(p, 1e-4)
    rng = np.random.default_rng(9)
    V = rng.normal(size=(3, 9 * o.n_p))
    ref = np.stack([o.matvec(v) for v in V])
    err = {}
    for prec in (RBA_PRECISION_FP32, RBA_PRECISION_FP64):
        s = _solver(p, prec)
        s.linearize()
        s.marginalize(1e-4)
        err[prec] = relf(np.stack([_mv(s, v) for v in V]), ref)
        s.close()
    assert err[RBA_PRECISION_FP64] < err[RBA_PRECISION_FP32], err
